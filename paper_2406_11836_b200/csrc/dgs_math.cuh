// Exact-order float arithmetic shared by the sm_100a kernels and the host-side
// camera setup.  Every function here reproduces the reference's IEEE op
// sequence (as evaluated through Eigen's fixed-size expression rules, see
// oracle/eigen_shim/Eigen/Core) with no FMA contraction, because the
// quantities that define indices — tile bins, the per-ray order key t, the
// 3σ / D_i gates, plane tests — must be bit-exact.
#pragma once

#include <stdint.h>
#include <math.h>

#if defined(__CUDACC__)
#define DGS_HD __host__ __device__ __forceinline__
#else
#define DGS_HD inline
#endif

namespace dgs_b200 {

#if defined(__CUDA_ARCH__)
DGS_HD float fadd(float a, float b) { return __fadd_rn(a, b); }
DGS_HD float fsub(float a, float b) { return __fsub_rn(a, b); }
DGS_HD float fmul(float a, float b) { return __fmul_rn(a, b); }
DGS_HD float fdiv(float a, float b) { return __fdiv_rn(a, b); }
DGS_HD float fsqrt(float a) { return __fsqrt_rn(a); }
DGS_HD double dfma(double a, double b, double c) { return __fma_rn(a, b, c); }
DGS_HD uint64_t d2u(double d) { return (uint64_t)__double_as_longlong(d); }
DGS_HD double u2d(uint64_t u) { return __longlong_as_double((long long)u); }
DGS_HD uint32_t f2u(float f) { return __float_as_uint(f); }
DGS_HD float u2f(uint32_t u) { return __uint_as_float(u); }
#else
// Host side: the translation unit is compiled with -ffp-contract=off.
DGS_HD float fadd(float a, float b) { return a + b; }
DGS_HD float fsub(float a, float b) { return a - b; }
DGS_HD float fmul(float a, float b) { return a * b; }
DGS_HD float fdiv(float a, float b) { return a / b; }
DGS_HD float fsqrt(float a) { return sqrtf(a); }
DGS_HD double dfma(double a, double b, double c) { return fma(a, b, c); }
DGS_HD uint64_t d2u(double d) { union { double d; uint64_t u; } x; x.d = d; return x.u; }
DGS_HD double u2d(uint64_t u) { union { double d; uint64_t u; } x; x.u = u; return x.d; }
DGS_HD uint32_t f2u(float f) { union { float f; uint32_t u; } x; x.f = f; return x.u; }
DGS_HD float u2f(uint32_t u) { union { float f; uint32_t u; } x; x.u = u; return x.f; }
#endif

// Eigen redux orders (oracle/eigen_shim/Eigen/Core header).
DGS_HD float sum3(float a0, float a1, float a2) { return fadd(a0, fadd(a1, a2)); }
DGS_HD float dot3(float a0, float a1, float a2, float b0, float b1, float b2) {
    return sum3(fmul(a0, b0), fmul(a1, b1), fmul(a2, b2));
}
// Contiguous 4-float reduction: Eigen/SSE packet order (a0+a2)+(a1+a3).
DGS_HD float dot4(const float* a, const float* b) {
    return fadd(fadd(fmul(a[0], b[0]), fmul(a[2], b[2])), fadd(fmul(a[1], b[1]), fmul(a[3], b[3])));
}

// ---------------------------------------------------------------------------
// glibc 2.39 expf (sysdeps/ieee754/flt-32/e_expf.c, x86-64 FMA ifunc variant,
// the one libm dispatches to on every FMA-capable host).  Restated from the
// published algorithm: x*N/ln2 = k + r, exp(x) = 2^(k/N) * poly(r), N = 32,
// table T[i] = bits(2^(i/N)) - (i << 52)/N.  Verified bit-exact against the
// host libm on all 2.24e9 floats with |x| < 88 (tests/test_oracle_cpu.py).
// The reference calls expf in Splat::scales()/max_scale() (splat.hpp:36-37)
// and sigmoid (math.hpp:21-24); scales feed the tile bins and D_i, so they
// must be bit-exact.
// ---------------------------------------------------------------------------
#if defined(__CUDA_ARCH__)
// global (L1-cached through __ldg), not __constant__: the lanes of a warp
// index it divergently, which the constant cache serialises
__device__ static const uint64_t kExp2fTab[32] = {
#else
static const uint64_t kExp2fTab[32] = {
#endif
    0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull,
    0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull,
    0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull,
    0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull,
    0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull,
    0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull,
    0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull,
    0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull,
};

/// glibc_expf's evaluation without its special cases: bit-identical to
/// glibc_expf for |x| < 88 (top12(x) < 0x42b), the range of the blends'
/// eval_2d argument -m^2/2 whenever truncation_radius < 13.
DGS_HD float glibc_expf_core(float x, const uint64_t* tab = nullptr) {
    const double N = 32.0;
    const double InvLn2N = 0x1.71547652b82fep+0 * N;
    const double SHIFT = 0x1.8p+52;
    const double C0 = 0x1.c6af84b912394p-5 / N / N / N;
    const double C1 = 0x1.ebfce50fac4f3p-3 / N / N;
    const double C2 = 0x1.62e42ff0c52d6p-1 / N;
    const double xd = (double)x;
    double kd = dfma(InvLn2N, xd, SHIFT);
    const uint64_t ki = d2u(kd);
    kd = kd - SHIFT;
    const double r = dfma(InvLn2N, xd, -kd);
#if defined(__CUDA_ARCH__)
    // tab: a shared-memory copy of kExp2fTab (the blends' hot loops), else the global table
    uint64_t t = tab != nullptr ? tab[ki % 32] : __ldg(&kExp2fTab[ki % 32]);
#else
    (void)tab;
    uint64_t t = kExp2fTab[ki % 32];
#endif
    t += ki << (52 - 5);
    const double s = u2d(t);
    const double z = dfma(C0, r, C1);
    const double r2 = r * r;
    double y = dfma(C2, r, 1.0);
    y = dfma(z, r2, y);
    y = y * s;
    return (float)y;
}

DGS_HD float glibc_expf(float x, const uint64_t* tab = nullptr) {
    const uint32_t ux = f2u(x);
    const uint32_t abstop = (ux >> 20) & 0x7ff;
    if (abstop >= 0x42b) {  // top12(88.0f)
        if (ux == 0xff800000u) return 0.0f;       // -inf
        if (abstop >= 0x7f8) return x + x;       // inf or nan
        if (x > 0x1.62e42ep6f) return u2f(0x7f800000u);  // x > log(0x1p128): overflow
        if (x < -0x1.9fe368p6f) return 0.0f;            // x < log(0x1p-150): underflow
    }
    return glibc_expf_core(x, tab);
}

/// eval_2d's g = exp(-m^2/2) for 0 <= m^2 <= trunc^2: the special-case-free
/// core when the whole range stays below |x| < 88 (the flag is uniform).
DGS_HD float gauss_expf(float m2, bool core_ok, const uint64_t* tab = nullptr) {
    const float x = fmul(-0.5f, m2);
    return core_ok ? glibc_expf_core(x, tab) : glibc_expf(x);
}

#if defined(__CUDACC__)
/// kExp2fTab into a CTA's shared copy (threads 0..31); the caller syncs.
__device__ __forceinline__ void load_exp_tab(uint64_t* s_tab) {
    if (threadIdx.x < 32) s_tab[threadIdx.x] = kExp2fTab[threadIdx.x];
}
#endif

/// math.hpp:21-24: 1/(1+exp(-x)).
DGS_HD float sigmoidf_exact(float x, const uint64_t* tab = nullptr) {
    return fdiv(1.0f, fadd(1.0f, glibc_expf(-x, tab)));
}

/// math.hpp:33-45 rotation_from_quat (the quaternion norm is a contiguous
/// Vec4 reduction).  Row-major r[9].  Returns false for a zero quaternion
/// (the reference throws std::domain_error).
DGS_HD bool rotation_from_quat(const float q[4], float r[9]) {
    const float n = fsqrt(dot4(q, q));
    if (!(n > 0.0f)) return false;
    const float w = fdiv(q[0], n), x = fdiv(q[1], n), y = fdiv(q[2], n), z = fdiv(q[3], n);
    r[0] = fsub(1.0f, fmul(2.0f, fadd(fmul(y, y), fmul(z, z))));
    r[1] = fmul(2.0f, fsub(fmul(x, y), fmul(w, z)));
    r[2] = fmul(2.0f, fadd(fmul(x, z), fmul(w, y)));
    r[3] = fmul(2.0f, fadd(fmul(x, y), fmul(w, z)));
    r[4] = fsub(1.0f, fmul(2.0f, fadd(fmul(x, x), fmul(z, z))));
    r[5] = fmul(2.0f, fsub(fmul(y, z), fmul(w, x)));
    r[6] = fmul(2.0f, fsub(fmul(x, z), fmul(w, y)));
    r[7] = fmul(2.0f, fadd(fmul(y, z), fmul(w, x)));
    r[8] = fsub(1.0f, fmul(2.0f, fadd(fmul(x, x), fmul(y, y))));
    return true;
}

/// Per-view constants derived once on the host (exact order, see
/// Camera::rotation/center, splat.hpp:56-57, and pixel_ray, splat.hpp:83-90).
struct ViewParams {
    int width, height, tiles_x, tiles_y;
    float fx, fy, cx, cy;
    float R[9];        // world->camera rotation, row-major
    float t[3];        // t_wc
    float o[3];        // camera centre = ray origin = -(R^T t)
};

DGS_HD bool make_view_params(int width, int height, float fx, float fy, float cx, float cy, const float q[4],
                             const float t[3], ViewParams* vp) {
    vp->width = width;
    vp->height = height;
    vp->tiles_x = (width + 15) / 16;
    vp->tiles_y = (height + 15) / 16;
    vp->fx = fx;
    vp->fy = fy;
    vp->cx = cx;
    vp->cy = cy;
    if (!rotation_from_quat(q, vp->R)) return false;
    for (int i = 0; i < 3; ++i) {
        vp->t[i] = t[i];
        // (R^T t)_i = R(0,i) t0 + (R(1,i) t1 + R(2,i) t2), then negated.
        vp->o[i] = -dot3(vp->R[0 * 3 + i], vp->R[1 * 3 + i], vp->R[2 * 3 + i], t[0], t[1], t[2]);
    }
    return true;
}

/// splat.hpp:83-95 pixel_ray for pixel (ix, iy): direction = normalize(R^T dir_cam).
DGS_HD void pixel_ray_dir(const ViewParams& vp, int ix, int iy, float d[3]) {
    const float px = fadd((float)ix, 0.5f), py = fadd((float)iy, 0.5f);
    const float dc0 = fdiv(fsub(px, vp.cx), vp.fx);
    const float dc1 = fdiv(fsub(py, vp.cy), vp.fy);
    const float dc2 = 1.0f;
    float v[3];
    for (int i = 0; i < 3; ++i) v[i] = dot3(vp.R[0 * 3 + i], vp.R[1 * 3 + i], vp.R[2 * 3 + i], dc0, dc1, dc2);
    const float n2 = dot3(v[0], v[1], v[2], v[0], v[1], v[2]);
    if (n2 > 0.0f) {
        const float s = fsqrt(n2);
        for (int i = 0; i < 3; ++i) d[i] = fdiv(v[i], s);
    } else {
        for (int i = 0; i < 3; ++i) d[i] = v[i];
    }
}

/// C++ static_cast<int>(float) as executed by x86-64 cvttss2si: truncation,
/// and the "integer indefinite" INT_MIN for NaN or out-of-range values
/// (raster.hpp:118-121 relies on it only for pathological splats).
DGS_HD int x86_float_to_int(float v) {
    if (!(v > -2147483904.0f && v < 2147483648.0f)) return (int)0x80000000;
    return (int)v;
}

DGS_HD int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// SH basis constants (splat.hpp:141-147), rounded to float as T(kC...).
#define DGS_SH_C0 0.28209479177387814
#define DGS_SH_C1 0.4886025119029199

/// splat.hpp:150-176 sh::basis (float instantiation).
DGS_HD void sh_basis(const float d[3], int deg, float b[16]) {
    for (int i = 0; i < 16; ++i) b[i] = 0.0f;
    b[0] = (float)DGS_SH_C0;
    if (deg < 1) return;
    const float x = d[0], y = d[1], z = d[2];
    b[1] = fmul((float)-DGS_SH_C1, y);
    b[2] = fmul((float)DGS_SH_C1, z);
    b[3] = fmul((float)-DGS_SH_C1, x);
    if (deg < 2) return;
    const float xx = fmul(x, x), yy = fmul(y, y), zz = fmul(z, z);
    const float xy = fmul(x, y), yz = fmul(y, z), xz = fmul(x, z);
    b[4] = fmul((float)1.0925484305920792, xy);
    b[5] = fmul((float)-1.0925484305920792, yz);
    b[6] = fmul((float)0.31539156525252005, fsub(fsub(fmul(2.0f, zz), xx), yy));
    b[7] = fmul((float)-1.0925484305920792, xz);
    b[8] = fmul((float)0.5462742152960396, fsub(xx, yy));
    if (deg < 3) return;
    b[9] = fmul(fmul((float)-0.5900435899266435, y), fsub(fmul(3.0f, xx), yy));
    b[10] = fmul(fmul((float)2.890611442640554, xy), z);
    b[11] = fmul(fmul((float)-0.4570457994644657, y), fsub(fsub(fmul(4.0f, zz), xx), yy));
    b[12] = fmul(fmul((float)0.3731763325901154, z), fsub(fsub(fmul(2.0f, zz), fmul(3.0f, xx)), fmul(3.0f, yy)));
    b[13] = fmul(fmul((float)-0.4570457994644657, x), fsub(fsub(fmul(4.0f, zz), xx), yy));
    b[14] = fmul(fmul((float)1.445305721320277, z), fsub(xx, yy));
    b[15] = fmul(fmul((float)-0.5900435899266435, x), fsub(xx, fmul(3.0f, yy)));
}

constexpr float kShC1f = 0.4886025119029199f;

/// splat.hpp:180-204 sh::basis_jacobian, row i -> (dx, dy, dz).
DGS_HD void sh_basis_jac(const float d[3], int deg, int i, float j[3]) {
    j[0] = j[1] = j[2] = 0.0f;
    if (deg < 1 || i == 0) return;
    const float x = d[0], y = d[1], z = d[2];
    const float c2_0 = 1.0925484305920792f, c2_1 = -1.0925484305920792f, c2_2 = 0.31539156525252005f,
                c2_3 = -1.0925484305920792f, c2_4 = 0.5462742152960396f;
    const float c3_0 = -0.5900435899266435f, c3_1 = 2.890611442640554f, c3_2 = -0.4570457994644657f,
                c3_3 = 0.3731763325901154f, c3_4 = -0.4570457994644657f, c3_5 = 1.445305721320277f,
                c3_6 = -0.5900435899266435f;
    const float xx = x * x, yy = y * y, zz = z * z;
    switch (i) {
        case 1: j[1] = -kShC1f; break;
        case 2: j[2] = kShC1f; break;
        case 3: j[0] = -kShC1f; break;
        case 4: j[0] = c2_0 * y; j[1] = c2_0 * x; break;
        case 5: j[1] = c2_1 * z; j[2] = c2_1 * y; break;
        case 6: j[0] = (float)(-2 * 0.31539156525252005) * x; j[1] = (float)(-2 * 0.31539156525252005) * y;
                j[2] = (float)(4 * 0.31539156525252005) * z; (void)c2_2; break;
        case 7: j[0] = c2_3 * z; j[2] = c2_3 * x; break;
        case 8: j[0] = (float)(2 * 0.5462742152960396) * x; j[1] = (float)(-2 * 0.5462742152960396) * y;
                (void)c2_4; break;
        case 9: j[0] = (float)(6 * -0.5900435899266435) * x * y; j[1] = c3_0 * (3.0f * xx - 3.0f * yy); break;
        case 10: j[0] = c3_1 * y * z; j[1] = c3_1 * x * z; j[2] = c3_1 * x * y; break;
        case 11: j[0] = (float)(-2 * -0.4570457994644657) * x * y; j[1] = c3_2 * (4.0f * zz - xx - 3.0f * yy);
                 j[2] = (float)(8 * -0.4570457994644657) * y * z; break;
        case 12: j[0] = (float)(-6 * 0.3731763325901154) * x * z; j[1] = (float)(-6 * 0.3731763325901154) * y * z;
                 j[2] = c3_3 * (6.0f * zz - 3.0f * xx - 3.0f * yy); break;
        case 13: j[0] = c3_4 * (4.0f * zz - 3.0f * xx - yy); j[1] = (float)(-2 * -0.4570457994644657) * x * y;
                 j[2] = (float)(8 * -0.4570457994644657) * x * z; break;
        case 14: j[0] = (float)(2 * 1.445305721320277) * x * z; j[1] = (float)(-2 * 1.445305721320277) * y * z;
                 j[2] = c3_5 * (xx - yy); break;
        case 15: j[0] = c3_6 * (3.0f * xx - 3.0f * yy); j[1] = (float)(-6 * -0.5900435899266435) * x * y; break;
        default: break;
    }
}

}  // namespace dgs_b200

// ---------------------------------------------------------------------------
// sm_100a bulk-copy (TMA engine) + mbarrier helpers (PTX ISA 8.x).
// ---------------------------------------------------------------------------
#if defined(__CUDACC__)
namespace dgs_b200 {
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase), "r"(0x100000u)  // suspend-time hint (ns): sleep until the phase completes, do not spin
        : "memory");
}
/// global -> shared bulk copy completing on an mbarrier (UBLKCP).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
/// shared -> global bulk copy in the bulk-async group.
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
/// Make generic-proxy shared-memory writes visible to the async proxy (bulk stores).
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
}  // namespace dgs_b200
#endif
