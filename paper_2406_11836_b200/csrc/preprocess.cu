// K1 — per-member projection (EWA), SH colour, opacity sigmoid, support radius
// D_i, tile rectangle and range key.  One thread per member; HBM-bound
// (59 param floats in, one 64-byte record + 16 bytes of binning data out).
//
// Bit-exactness: every quantity that feeds an index or a gate is computed in
// the reference's op order with _rn intrinsics (no FMA contraction):
//   t = W mu + t_wc, mean2d, J, V = J W, Sigma = (R S)(R S)^T, cov2d = V Sigma V^T
//   (+0.3 I), det, inv_cov2d, 3*sqrt(c_ii), the cull test and the tile bins
//   (splat.hpp:245-321, raster.hpp:113-125), and D_i = 3*max(exp(log_scale))
//   with the glibc expf port (splat.hpp:36-37).
#include "kernels.h"

namespace dgs_b200 {

namespace {

/// Members are staged per CTA: one elected thread issues a bulk copy
/// (cp.async.bulk, the TMA engine) of each parameter row segment into shared
/// memory on one mbarrier, so all 11 + 3C rows of the CTA are in flight at
/// once; the per-member math then reads shared memory.
constexpr int kPreTB = 128;

template <int SHC>
__global__ void __launch_bounds__(kPreTB) k_preprocess(int n, const float* __restrict__ P, size_t ld,
                                                       const uint32_t* __restrict__ ids32, ViewParams vp,
                                                       RenderOpts ro, ViewBins vb) {
    constexpr int ROWS = kRowSh + 3 * SHC;
    constexpr int sh_coeffs = SHC;
    __shared__ __align__(128) float tile[ROWS * kPreTB];
    // two mbarriers: the 11 geometry rows, then the SH rows, so the projection
    // math starts while the SH rows (81 % of the bytes) are still in flight
    __shared__ uint64_t bar[2];
    const int tid = threadIdx.x;
    const int i0 = blockIdx.x * kPreTB;
    const int i = i0 + tid;
    const int cnt = min(kPreTB, n - i0);
    const uint32_t bytes = (uint32_t)((cnt + 3) / 4) * 16u;
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
        mbar_expect_tx(&bar[0], (uint32_t)kRowSh * bytes);
        for (int r = 0; r < kRowSh; ++r) bulk_g2s(tile + r * kPreTB, P + (size_t)r * ld + i0, bytes, &bar[0]);
        mbar_expect_tx(&bar[1], (uint32_t)(ROWS - kRowSh) * bytes);
        for (int r = kRowSh; r < ROWS; ++r) bulk_g2s(tile + r * kPreTB, P + (size_t)r * ld + i0, bytes, &bar[1]);
    }
    mbar_wait(&bar[0], 0);
    float dmax_local = 0.0f, rmin_local = __int_as_float(0x7f7fffff);
    if (i < n) {
        auto row = [&](int r) { return tile[r * kPreTB + tid]; };
        const float mu0 = row(kRowMu), mu1 = row(kRowMu + 1), mu2 = row(kRowMu + 2);
        // t = W mu + t_wc (splat.hpp:292)
        const float t0 = fadd(dot3(vp.R[0], vp.R[1], vp.R[2], mu0, mu1, mu2), vp.t[0]);
        const float t1 = fadd(dot3(vp.R[3], vp.R[4], vp.R[5], mu0, mu1, mu2), vp.t[1]);
        const float t2 = fadd(dot3(vp.R[6], vp.R[7], vp.R[8], mu0, mu1, mu2), vp.t[2]);
        bool visible = t2 > ro.near_plane;  // splat.hpp:293
        float mx = 0, my = 0, c00 = 0, c01 = 0, c10 = 0, c11 = 0;
        float q[4] = {row(kRowRot), row(kRowRot + 1), row(kRowRot + 2), row(kRowRot + 3)};
        float r[9];
        const bool qok = rotation_from_quat(q, r);
        if (visible && !qok) {  // math.hpp:36-37 throws only for projected splats
            atomicMin(vb.err_index, i);
            if (vb.abort) atomicOr(vb.abort, 1);
            visible = false;
        }
        const float s0 = glibc_expf(row(kRowLogScale)), s1 = glibc_expf(row(kRowLogScale + 1)),
                    s2 = glibc_expf(row(kRowLogScale + 2));
        if (visible) {
            mx = fadd(fdiv(fmul(vp.fx, t0), t2), vp.cx);  // splat.hpp:299
            my = fadd(fdiv(fmul(vp.fy, t1), t2), vp.cy);
            // perspective_jacobian (splat.hpp:276-282)
            const float iz = fdiv(1.0f, t2);
            const float J[6] = {fmul(vp.fx, iz), 0.0f, fmul(fmul(fmul(-vp.fx, t0), iz), iz),
                                0.0f, fmul(vp.fy, iz), fmul(fmul(fmul(-vp.fy, t1), iz), iz)};
            float V[6];  // V = J * W  (2x3)
            for (int a = 0; a < 2; ++a)
                for (int b = 0; b < 3; ++b)
                    V[a * 3 + b] = sum3(fmul(J[a * 3 + 0], vp.R[0 * 3 + b]), fmul(J[a * 3 + 1], vp.R[1 * 3 + b]),
                                        fmul(J[a * 3 + 2], vp.R[2 * 3 + b]));
            // covariance3d (splat.hpp:245-250): M = R diag(s), Sigma = M M^T
            const float sc[3] = {s0, s1, s2};
            float M[9];
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) M[a * 3 + b] = fmul(r[a * 3 + b], sc[b]);
            float S[9];
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b)
                    S[a * 3 + b] = sum3(fmul(M[a * 3 + 0], M[b * 3 + 0]), fmul(M[a * 3 + 1], M[b * 3 + 1]),
                                        fmul(M[a * 3 + 2], M[b * 3 + 2]));
            float VS[6];  // (V Sigma), evaluated before the outer product (Eigen nested-product rule)
            for (int a = 0; a < 2; ++a)
                for (int b = 0; b < 3; ++b)
                    VS[a * 3 + b] = sum3(fmul(V[a * 3 + 0], S[0 * 3 + b]), fmul(V[a * 3 + 1], S[1 * 3 + b]),
                                         fmul(V[a * 3 + 2], S[2 * 3 + b]));
            float C2[4];
            for (int a = 0; a < 2; ++a)
                for (int b = 0; b < 2; ++b)
                    C2[a * 2 + b] = sum3(fmul(VS[a * 3 + 0], V[b * 3 + 0]), fmul(VS[a * 3 + 1], V[b * 3 + 1]),
                                         fmul(VS[a * 3 + 2], V[b * 3 + 2]));
            c00 = fadd(C2[0], ro.cov_reg);
            c01 = C2[1];
            c10 = C2[2];
            c11 = fadd(C2[3], ro.cov_reg);
            const float rx = fmul(ro.trunc, fsqrt(c00)), ry = fmul(ro.trunc, fsqrt(c11));
            // splat.hpp:311-313 cull against the image rectangle
            if (fadd(mx, rx) < 0.0f || fsub(mx, rx) > (float)vp.width || fadd(my, ry) < 0.0f ||
                fsub(my, ry) > (float)vp.height)
                visible = false;
            if (visible) {
                const float det = fsub(fmul(c00, c11), fmul(c01, c10));
                SplatRec rec;
                rec.mx = mx;
                rec.my = my;
                rec.i00 = fdiv(c11, det);
                rec.i01 = fdiv(-c01, det);
                rec.i10 = fdiv(-c10, det);
                rec.i11 = fdiv(c00, det);
                {
                    // Conservative |dy| bound of the reference's computed m^2 <= trunc^2
                    // region (eval_2d, splat.hpp:326-332): every term of the float m^2
                    // carries <= 4 roundings, so m2_float <= 9 implies
                    // a' dx^2 - 2h|dx dy| + d' dy^2 <= 9 with a' = a(1-g), d' = d(1-g),
                    // h = (|b+c| + g(|b|+|c|))/2, g = 1e-6 > gamma_4.  Minimising over dx
                    // gives |dy| <= trunc * sqrt(a' / (a'd' - h^2)).
                    const double a = rec.i00, b = rec.i01, c = rec.i10, d = rec.i11, g = 1e-6;
                    const double ap = a * (1.0 - g), dp = d * (1.0 - g);
                    const double h = 0.5 * (fabs(b + c) + g * (fabs(b) + fabs(c)));
                    // (and symmetrically |dx| <= trunc * sqrt(d' / (a'd' - h^2)))
                    float ex = __int_as_float(0x7f800000), ey = ex;
                    if (a > 0.0 && d > 0.0 && ap * dp > h * h * (1.0 + 1e-9)) {
                        const double t2 = (double)fmul(ro.trunc, ro.trunc);
                        const double den = ap * dp - h * h;
                        ey = (float)(sqrt(t2 * ap / den) * (1.0 + 1e-6) + 1e-5);
                        ex = (float)(sqrt(t2 * dp / den) * (1.0 + 1e-6) + 1e-5);
                    }
                    vb.ext[i] = make_float2(ex, ey);
                }
                // tile rectangle (raster.hpp:117-121): C++ truncating int division, then clamp
                const int x0 = clampi(x86_float_to_int(floorf(fsub(mx, rx))) / kTileSize, 0, vp.tiles_x - 1);
                const int x1 = clampi(x86_float_to_int(floorf(fadd(mx, rx))) / kTileSize, 0, vp.tiles_x - 1);
                const int y0 = clampi(x86_float_to_int(floorf(fsub(my, ry))) / kTileSize, 0, vp.tiles_y - 1);
                const int y1 = clampi(x86_float_to_int(floorf(fadd(my, ry))) / kTileSize, 0, vp.tiles_y - 1);
                vb.rect[2 * (size_t)i] = (uint32_t)x0 | ((uint32_t)x1 << 16);
                vb.rect[2 * (size_t)i + 1] = (uint32_t)y0 | ((uint32_t)y1 << 16);
                vb.counts[i] = (uint32_t)((x1 - x0 + 1) * (y1 - y0 + 1));
                mbar_wait(&bar[1], 0);  // the SH rows
                // SH colour toward the camera centre (splat.hpp:315-317)
                const float v0 = fsub(mu0, vp.o[0]), v1 = fsub(mu1, vp.o[1]), v2 = fsub(mu2, vp.o[2]);
                const float n2 = dot3(v0, v1, v2, v0, v1, v2);
                float dir[3] = {v0, v1, v2};
                if (n2 > 0.0f) {
                    const float sn = fsqrt(n2);
                    dir[0] = fdiv(v0, sn);
                    dir[1] = fdiv(v1, sn);
                    dir[2] = fdiv(v2, sn);
                }
                int stored_deg = sh_coeffs == 16 ? 3 : (sh_coeffs == 9 ? 2 : (sh_coeffs == 4 ? 1 : 0));
                const int deg = ro.sh_degree < 0 ? stored_deg : (ro.sh_degree < stored_deg ? ro.sh_degree : stored_deg);
                float b[16];
                sh_basis(dir, deg, b);
                const int nb = (deg + 1) * (deg + 1);
                float col[3] = {0.5f, 0.5f, 0.5f};
#pragma unroll
                for (int k = 0; k < SHC; ++k)
                    if (k < nb)
#pragma unroll
                        for (int ch = 0; ch < 3; ++ch) col[ch] = fadd(col[ch], fmul(b[k], row(kRowSh + 3 * k + ch)));
                if (vb.shjac != nullptr) {
                    // d colour / d dir for the gradient record (tolerance-level, splat.hpp:223-239)
                    float J[9] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
                    for (int k = 1; k < SHC; ++k) {
                        if (k >= nb) break;
                        float jb[3];
                        sh_basis_jac(dir, deg, k, jb);
#pragma unroll
                        for (int ch = 0; ch < 3; ++ch) {
                            const float c = row(kRowSh + 3 * k + ch);
                            J[ch * 3 + 0] += jb[0] * c;
                            J[ch * 3 + 1] += jb[1] * c;
                            J[ch * 3 + 2] += jb[2] * c;
                        }
                    }
#pragma unroll
                    for (int q = 0; q < 9; ++q) vb.shjac[(size_t)q * ld + i] = J[q];
                    const uint32_t mask = (col[0] < 0.0f ? 1u : 0u) | (col[1] < 0.0f ? 2u : 0u) | (col[2] < 0.0f ? 4u : 0u);
                    vb.shjac[9 * ld + i] = __uint_as_float(mask);
                }
                rec.cr = col[0] < 0.0f ? 0.0f : col[0];  // cwiseMax(0) = std::max(c, 0)
                rec.cg = col[1] < 0.0f ? 0.0f : col[1];
                rec.cb = col[2] < 0.0f ? 0.0f : col[2];
                rec.alpha = sigmoidf_exact(row(kRowOpacity));
                float smax = s0;  // Vec3::maxCoeff (first maximum)
                if (s1 > smax) smax = s1;
                if (s2 > smax) smax = s2;
                const float wr = fmul(ro.trunc, smax);  // splat.hpp:319
                rec.d2 = fmul(wr, wr);
                rec.mux = mu0;
                rec.muy = mu1;
                rec.muz = mu2;
                rec.id = ids32[i];
                // the blends' ordering key: range ||mu - o|| (per-ray t order, exact via the
                // reorder ring), or the camera depth (camera_z_order, raster.hpp:162)
                rec.range = ro.zorder ? t2 : fsqrt(n2);
                vb.recs[i] = rec;
                vb.rkey[i] = f2u(rec.range);
                dmax_local = wr;
                rmin_local = rec.range;
            }
        }
        if (!visible) {
            vb.counts[i] = 0;
            // empty tile rectangle (x0 > x1): the binning derives counts from rect alone
            vb.rect[2 * (size_t)i] = 0x0000ffffu;
            vb.rect[2 * (size_t)i + 1] = 0x0000ffffu;
            vb.rkey[i] = 0xffffffffu;
        }
    }
    mbar_wait(&bar[1], 0);  // no CTA exits with its bulk copy in flight
    // block max of D and min of the range over visible members -> one atomic each per block
    // (and the max range, which sizes the binning's 16-bit range buckets)
    __shared__ float s_max[kPreTB / 32], s_min[kPreTB / 32], s_hi[kPreTB / 32];
    float m = dmax_local, lo = rmin_local, hi = dmax_local > 0.0f ? rmin_local : 0.0f;
    for (int off = 16; off > 0; off >>= 1) {
        m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, off));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, off));
    }
    if ((threadIdx.x & 31) == 0) {
        s_max[threadIdx.x >> 5] = m;
        s_min[threadIdx.x >> 5] = lo;
        s_hi[threadIdx.x >> 5] = hi;
    }
    const int nvis = __syncthreads_count(dmax_local > 0.0f);
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            m = fmaxf(m, s_max[w]);
            lo = fminf(lo, s_min[w]);
            hi = fmaxf(hi, s_hi[w]);
        }
        // one 16-byte partial per block (non-negative floats order like their bit
        // patterns); k_pre_reduce folds them instead of same-address atomics from
        // every one of the ~78k blocks, which serialise in L2
        reinterpret_cast<uint4*>(vb.blk_part)[blockIdx.x] =
            make_uint4(__float_as_uint(m), __float_as_uint(lo), (uint32_t)nvis, __float_as_uint(hi));
    }
}

/// Folds K1's per-block partials into dmax_bits (max D, min range, visible
/// count, max range): one atomic per quantity per warp here.
__global__ void __launch_bounds__(256) k_pre_reduce(const uint32_t* __restrict__ part, int nblk,
                                                    uint32_t* __restrict__ dmax_bits) {
    uint32_t m = 0, lo = 0x7f7fffffu, hi = 0, nv = 0;
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nblk; b += gridDim.x * blockDim.x) {
        const uint4 a = reinterpret_cast<const uint4*>(part)[b];
        m = max(m, a.x);
        lo = min(lo, a.y);
        nv += a.z;
        hi = max(hi, a.w);
    }
    m = __reduce_max_sync(0xffffffffu, m);
    lo = __reduce_min_sync(0xffffffffu, lo);
    nv = __reduce_add_sync(0xffffffffu, nv);
    hi = __reduce_max_sync(0xffffffffu, hi);
    if ((threadIdx.x & 31) == 0) {
        if (nv) atomicAdd(dmax_bits + 2, nv);
        if (m) atomicMax(dmax_bits, m);
        atomicMin(dmax_bits + 1, lo);
        if (hi) atomicMax(dmax_bits + 3, hi);
    }
}

}  // namespace

size_t preprocess_partials(int n) { return n > 0 ? 4 * (size_t)((n + kPreTB - 1) / kPreTB) : 1; }

void launch_preprocess(int n, const float* P, size_t ld, int sh_coeffs, const uint32_t* ids32, const ViewParams& vp,
                       const RenderOpts& ro, const ViewBins& vb, cudaStream_t s) {
    if (n <= 0) return;
    const unsigned grid = (unsigned)((n + kPreTB - 1) / kPreTB);
    switch (sh_coeffs) {
        case 1: k_preprocess<1><<<grid, kPreTB, 0, s>>>(n, P, ld, ids32, vp, ro, vb); break;
        case 4: k_preprocess<4><<<grid, kPreTB, 0, s>>>(n, P, ld, ids32, vp, ro, vb); break;
        case 9: k_preprocess<9><<<grid, kPreTB, 0, s>>>(n, P, ld, ids32, vp, ro, vb); break;
        default: k_preprocess<16><<<grid, kPreTB, 0, s>>>(n, P, ld, ids32, vp, ro, vb); break;
    }
    k_pre_reduce<<<64, 256, 0, s>>>(vb.blk_part, (int)grid, vb.dmax_bits);
}

}  // namespace dgs_b200
