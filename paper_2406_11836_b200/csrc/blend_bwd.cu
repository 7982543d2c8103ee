// K8 — backward blend of one KD subset (composite_ray_backward +
// render_maps_backward, raster.hpp:194-236 / 267-305; engine.hpp:74-88).
//
// Per pixel the reference replays the forward to get prefix transmittances
// A_i, then sweeps in reverse with suffix = sum_{j>i} c_j sigma_j A_j:
//   d_color_i += gc * sigma_i A_i
//   d_sigma_i  = gc.c_i A_i - gc.suffix_i/(1-sigma_i) - gT T_f/(1-sigma_i)
//   unless alpha g >= 0.99:  d_alpha += d_sigma g,  d_mean2d += (d_sigma alpha g) w,
//                            d_cov2d += 0.5 (d_sigma alpha g) w w^T,   w = inv_cov2d delta.
// Here the traversal is the forward's own (same range-ordered list, same
// reorder ring, same emission order, bitwise the same sigma and T sequence),
// and the suffix is formed as C_final - (running prefix colour), which needs
// no reverse pass and no T recovery by division (impossible once T
// underflows in stop=0 mode).
//
// Accumulation of the 9 pixel-space adjoints per member: emissions are
// grouped into warp-uniform sub-rounds (one list position each), reduced with
// a 5-step butterfly and added by one lane with native red.global.add.f32
// (shared-memory float atomics are CAS loops on sm_100).  Pixels skipped by
// the reference rule (gc.isZero() && gT == 0, raster.hpp:285) never emit.
// TrainConfig::deterministic (fixed-order reductions, optim.hpp:33;
// parallel.hpp:23-55): the same sub-round sums are added as fixed point
// (units of 2^-72, two 64-bit words) with integer atomics (acc_add), so every member's total is an exact
// integer independent of the atomics' order.
#include <algorithm>

#include "kernels.h"
#include "fallback_select.cuh"

namespace dgs_b200 {

namespace {

constexpr int KBUF = 8;  // must equal blend_fwd.cu (identical overflow decisions)
constexpr float kInf = __builtin_huge_valf();
#ifndef DGS_K8_DIRECT
#define DGS_K8_DIRECT 24  // sub-rounds of up to this many lanes add their adjoints directly (vector REDs)
#endif
constexpr unsigned kFull = 0xffffffffu;
// staged records (4 float4) + ring (t, id, sigma, list position)
constexpr size_t kBwdSmem = 4 * kBlendThreads * sizeof(float4) + 4 * KBUF * kBlendThreads * sizeof(float) +
                            kBlendThreads + (kBlendThreads / 32) * kBlendThreads * sizeof(uint16_t);

__device__ __forceinline__ float order_bound(float r, float dmax, float onorm) {
    const float S = 2.0f * onorm + 2.0f * r + 1.0f;
    const float dm = dmax * 1.0001f + 1e-6f * S;
    const float r2 = r * r * (1.0f - 2e-6f);
    const float dm2 = dm * dm;
    if (!(r2 > dm2)) return -kInf;
    return sqrtf(r2 - dm2) * (1.0f - 1e-6f) - 1e-6f * S;
}

struct PixelRay {
    float d[3];
    float pxf, pyf;
};

__device__ __forceinline__ bool eval_candidate(const PixelRay& pr, const ViewParams& vp, const RenderOpts& ro,
                                               const Subspace& gate, const float4& A, const float4& B,
                                               const float4& C, float zkey, float& t_out, float& sigma_out,
                                               float& g_out) {
    const float dx = fsub(pr.pxf, A.x), dy = fsub(pr.pyf, A.y);
    const float m2 = fadd(fmul(dx, fadd(fmul(B.x, dx), fmul(B.y, dy))), fmul(dy, fadd(fmul(B.z, dx), fmul(B.w, dy))));
    if (!(m2 <= fmul(ro.trunc, ro.trunc))) return false;
    const float t = dot3(pr.d[0], pr.d[1], pr.d[2], fsub(C.x, vp.o[0]), fsub(C.y, vp.o[1]), fsub(C.z, vp.o[2]));
    if (!(t > 0.0f)) return false;
    const float x0 = fadd(vp.o[0], fmul(t, pr.d[0]));
    const float x1 = fadd(vp.o[1], fmul(t, pr.d[1]));
    const float x2 = fadd(vp.o[2], fmul(t, pr.d[2]));
    const float e0 = fsub(x0, C.x), e1 = fsub(x1, C.y), e2 = fsub(x2, C.z);
    if (dot3(e0, e1, e2, e0, e1, e2) > A.w) return false;
    if (ro.indicator_enabled && !subspace_contains(gate, x0, x1, x2)) return false;
    const float g = gauss_expf(m2, ro.trunc < 13.0f);  // eval_2d std::exp in float (splat.hpp:331): sigma bit-exact
    const float ag = fmul(A.z, g);
    const float sigma = (ro.sigma_clamp < ag) ? ro.sigma_clamp : ag;
    if (!(sigma > 0.0f)) return false;
    t_out = ro.zorder ? zkey : t;  // camera_z_order: the per-view depth is the key (raster.hpp:162)
    sigma_out = sigma;
    g_out = g;
    return true;
}

__device__ __forceinline__ void load_rec(const SplatRec* __restrict__ recs, uint32_t m, float4& A, float4& B,
                                         float4& C, float4& D) {
    const float4* r4 = reinterpret_cast<const float4*>(recs + m);
    A = __ldg(r4 + 0);
    B = __ldg(r4 + 1);
    C = __ldg(r4 + 2);
    D = __ldg(r4 + 3);
}

/// Per-pixel backward state.
struct PixState {
    float T;                 // replayed transmittance (bitwise the forward's sequence)
    // gc . suffix_i, suffix_i = sum_{j>i} c_j sigma_j A_j (raster.hpp:212-224 accumulates
    // it backwards in float): only its dot with gc enters the adjoint, so one double carries
    // gc . (C - prefix), C the forward's double total, each term gc . c_j sigma_j A_j formed
    // in double (a float gc . c_j would add its rounding over the whole prefix); double
    // keeps the relative accuracy however much of C is already spent
    double q, gd0, gd1, gd2;
    float gc0, gc1, gc2, gT;
    float Tf;
    float pxf, pyf;
};

/// The suffix state from the forward's double colour total (gc set first).
__device__ __forceinline__ void init_suffix(PixState& ps, const double* __restrict__ cd) {
    ps.gd0 = ps.gc0;
    ps.gd1 = ps.gc1;
    ps.gd2 = ps.gc2;
    ps.q = ps.gd0 * cd[0] + ps.gd1 * cd[1] + ps.gd2 * cd[2];
}

/// One emitted contribution's 9 pixel-space adjoints:
/// [d_mean.x, d_mean.y, d_cov00, d_cov01(=d_cov10), d_cov11, d_col.r, d_col.g, d_col.b, d_alpha].
__device__ __forceinline__ void contribution_grad(PixState& ps, float sigma, float g, const float4& A,
                                                  const float4& B, const float4& D, float sigma_clamp,
                                                  float v[9]) {
    const float a_i = ps.T;
    const float w = fmul(sigma, a_i);
    const double wd = (double)sigma * (double)a_i;
    ps.q -= (ps.gd0 * (double)D.x + ps.gd1 * (double)D.y + ps.gd2 * (double)D.z) * wd;
    ps.T = fmul(ps.T, fsub(1.0f, sigma));
    // the rest in float, as in the reference
    const float gdc = ps.gc0 * D.x + ps.gc1 * D.y + ps.gc2 * D.z;
    const float num = (float)ps.q + ps.gT * ps.Tf;
    // 1/(1-sigma), 1-sigma in [0.01, 1]: MUFU reciprocal (1 ulp; the adjoint's tolerance
    // is 1e-3, and the value is still a deterministic function of sigma)
    float inv_om;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv_om) : "f"(1.0f - sigma));
    const float d_sigma = gdc * a_i - num * inv_om;
    v[5] = ps.gc0 * w;
    v[6] = ps.gc1 * w;
    v[7] = ps.gc2 * w;
    if (A.z * g >= sigma_clamp) {  // raster.hpp:228: the clamp freezes alpha/mean/cov
        v[0] = v[1] = v[2] = v[3] = v[4] = v[8] = 0.0f;
        return;
    }
    v[8] = d_sigma * g;
    const float d_g = d_sigma * A.z;
    const float dx = ps.pxf - A.x, dy = ps.pyf - A.y;
    const float w0 = B.x * dx + B.y * dy, w1 = B.z * dx + B.w * dy;
    const float s = d_g * g;
    v[0] = s * w0;
    v[1] = s * w1;
    const float h = s * 0.5f;
    v[2] = h * (w0 * w0);
    v[3] = h * (w0 * w1);
    v[4] = h * (w1 * w1);
}

// Accumulation modes of the backward kernels:
//   kAccFloat  float RED atomics into acc.f (TrainConfig::deterministic = 0)
//   kAccFixed  TrainConfig::deterministic = 1 ("fixed-order reductions",
//              optim.hpp:33): every value added to a member (one sub-round's
//              butterfly sum, itself a fixed-order float sum) is rounded once
//              to an integer V = round(v 2^72) and added as two words with
//              plain integer REDs: V mod 2^32 into an unsigned 64-bit word and
//              floor(V / 2^32) into a signed one.  Integer addition is
//              associative (the low word cannot overflow below 2^32 terms, the
//              high word's wrap-around cancels), so every member's total is the
//              same integer whatever order the atomics land in: bitwise
//              reproducible, one pass, |value| < 2^22 per (member, view, field),
//              resolution 2^-72.
constexpr int kAccFloat = 0, kAccFixed = 2;
constexpr int kFixedFrac = 72;
constexpr float kFixedMax = 4194304.0f;  // 2^22

/// v (|v| < 2^22) -> V = round(v 2^72) split as V = hi32 2^32 + lo32,
/// lo32 in [0, 2^32), hi32 = floor(V / 2^32).  With x = |v| 2^40 (exact),
/// H = floor(x) and L = (x - H) 2^32 are exact float operations for x >= 0
/// (the conversion of L rounds only below 2^-72); a negative v is
/// -(H 2^32 + L) = (-H - 1) 2^32 + (2^32 - L) for L > 0.
__device__ __forceinline__ void to_fixed(float v, unsigned long long& lo32, long long& hi32) {
    const float x = fabsf(v) * 0x1p40f;
    const float fl = floorf(x);
    const long long H = __float2ll_rn(fl);
    const unsigned long long L = __float2ull_rn((x - fl) * 0x1p32f);  // <= 2^32
    if (v >= 0.0f) {
        hi32 = H + (long long)(L >> 32);
        lo32 = L & 0xffffffffull;
    } else {
        hi32 = L ? -H - 1 : -H;
        lo32 = L ? (0x100000000ull - L) : 0ull;
    }
}

template <int MODE>
__device__ __forceinline__ void acc_add(const GradAcc& a, int f, uint32_t mem, float v, float) {
    if constexpr (MODE == kAccFloat) {
        if (v != 0.0f) atomicAdd(a.f + g2d_index(f, mem, a.ld), v);
    } else {
        if (v == 0.0f) return;
        if (!(fabsf(v) < kFixedMax)) {  // non-finite (or beyond the fixed-point range): reported
            atomicMin(a.bad, (int)mem);
            return;
        }
        unsigned long long lo;
        long long hi;
        to_fixed(v, lo, hi);
        unsigned long long* q = a.q + (size_t)(2 * f) * a.ld + mem;  // [f][lo | hi][ld]
        atomicAdd(q, lo);
        atomicAdd(q + a.ld, (unsigned long long)hi);
    }
}

/// One emission sub-round's accumulation: all `go` lanes hold adjoints of the
/// same member `mem`.  Up to DGS_K8_DIRECT lanes (float mode; two in
/// deterministic mode): direct atomics, for the float mode two vector REDs +
/// one scalar RED per lane, i.e. three instructions for the warp, cheaper than
/// the ~45-instruction butterfly while the same-sector REDs stay few.  Otherwise a
/// transposed butterfly (every exchange halves the values a lane still
/// carries: 4 + 2 + 1 + 1 + 1 shuffles for fields 0-7 instead of 8 x 5)
/// leaves the full sum of field (lane >> 2) & 7 in every lane; lanes 0, 4,
/// ..., 28 issue the eight reductions with one RED instruction.  Field 8
/// (d_alpha) takes a plain 5-step butterfly.  The butterfly's order is fixed
/// by the lanes, so in deterministic mode the sums it hands to acc_add are
/// reproducible too.
template <int MODE>
__device__ __forceinline__ void reduce_emit(unsigned gm, bool go, int lane, uint32_t mem, const float v[9],
                                            const GradAcc& acc, float scale) {
    const int n = __popc(gm);
    if (n <= (MODE == kAccFloat ? DGS_K8_DIRECT : 2)) {
        if (go) {
            if constexpr (MODE == kAccFloat) {
                // fields 0-7 are one 32-byte sector of g2d: two vector REDs
                float4* p = reinterpret_cast<float4*>(acc.f + 8 * (size_t)mem);
                atomicAdd(p, make_float4(v[0], v[1], v[2], v[3]));
                atomicAdd(p + 1, make_float4(v[4], v[5], v[6], v[7]));
                atomicAdd(acc.f + 8 * acc.ld + mem, v[8]);  // d_alpha row (g2d_index(8, ..))
            } else {
#pragma unroll
                for (int f = 0; f < 9; ++f) acc_add<MODE>(acc, f, mem, v[f], scale);
            }
        }
        return;
    }
    const int lead = __ffs(gm) - 1;
    const uint32_t mem_w = __shfl_sync(kFull, mem, lead);
    float a0 = v[0], a1 = v[1], a2 = v[2], a3 = v[3];
    {
        const bool hi = lane & 16;
        const float s0 = hi ? a0 : v[4], s1 = hi ? a1 : v[5], s2 = hi ? a2 : v[6], s3 = hi ? a3 : v[7];
        a0 = (hi ? v[4] : a0) + __shfl_xor_sync(kFull, s0, 16);
        a1 = (hi ? v[5] : a1) + __shfl_xor_sync(kFull, s1, 16);
        a2 = (hi ? v[6] : a2) + __shfl_xor_sync(kFull, s2, 16);
        a3 = (hi ? v[7] : a3) + __shfl_xor_sync(kFull, s3, 16);
    }
    {
        const bool hi = lane & 8;
        const float s0 = hi ? a0 : a2, s1 = hi ? a1 : a3;
        a0 = (hi ? a2 : a0) + __shfl_xor_sync(kFull, s0, 8);
        a1 = (hi ? a3 : a1) + __shfl_xor_sync(kFull, s1, 8);
    }
    {
        const bool hi = lane & 4;
        const float s0 = hi ? a0 : a1;
        a0 = (hi ? a1 : a0) + __shfl_xor_sync(kFull, s0, 4);
    }
    a0 += __shfl_xor_sync(kFull, a0, 2);
    a0 += __shfl_xor_sync(kFull, a0, 1);
    float a8 = v[8];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) a8 += __shfl_xor_sync(kFull, a8, off);
    if constexpr (MODE == kAccFloat) {
        // the 8 lanes' REDs land in one 32-byte sector (fields 0-7 of mem_w)
        if ((lane & 3) == 0) atomicAdd(acc.f + 8 * (size_t)mem_w + ((lane >> 2) & 7), a0);
    } else {
        if ((lane & 3) == 0) acc_add<MODE>(acc, (lane >> 2) & 7, mem_w, a0, scale);
    }
    if constexpr (MODE == kAccFloat) {
        if (lane == 0) atomicAdd(acc.f + 8 * acc.ld + mem_w, a8);
    } else {
        if (lane == 0) acc_add<MODE>(acc, 8, mem_w, a8, scale);
    }
}

template <bool STATS, int MODE>
__global__ void __launch_bounds__(kBlendThreads, 3) k_blend_bwd(ViewParams vp, RenderOpts ro, Subspace gate,
                                                             const SplatRec* __restrict__ recs,
                                                             const uint32_t* __restrict__ pair_val,
                                                             const uint2* __restrict__ ranges,
                                                             const float2* __restrict__ ext,
                                                             const uint32_t* __restrict__ dmax_bits, float onorm,
                                                             const float4* __restrict__ fwd_ct,
                                                             const double* __restrict__ fwd_cd,
                                                             const float4* __restrict__ grad_ct,
                                                             const uint8_t* __restrict__ ovf_flag,
                                                             const uint8_t* __restrict__ tile_replay,
                                                             GradAcc acc, BlendStats* __restrict__ stats,
                                                             const uint32_t* __restrict__ tile_order) {
    const int tile = tile_order ? (int)tile_order[blockIdx.x] : (int)blockIdx.x;
    if (tile_replay != nullptr && tile_replay[tile] == 0) return;  // handled by k_blend_bwd_rec
    extern __shared__ float4 smem4[];
    float4* sA = smem4;
    float4* sB = sA + kBlendThreads;
    float4* sC = sB + kBlendThreads;
    float4* sD = sC + kBlendThreads;
    typedef float Ring[kBlendThreads];
    typedef uint32_t URing[kBlendThreads];
    Ring* bt = reinterpret_cast<Ring*>(sD + kBlendThreads);
    URing* bid = reinterpret_cast<URing*>(bt + KBUF);
    Ring* bs = reinterpret_cast<Ring*>(bid + KBUF);
    URing* bpos = reinterpret_cast<URing*>(bs + KBUF);
    uint16_t* wlist = reinterpret_cast<uint16_t*>(bpos + KBUF) + (threadIdx.x >> 5) * kBlendThreads;
    uint8_t* smask = reinterpret_cast<uint8_t*>(reinterpret_cast<uint16_t*>(bpos + KBUF) +
                                                (kBlendThreads / 32) * kBlendThreads);

    const int tid = threadIdx.x, lane = tid & 31;
    const int tx = tile % vp.tiles_x, ty = tile / vp.tiles_x;
    int px, py;
    tile_pixel(tid, tx, ty, px, py);
    const bool inside = px < vp.width && py < vp.height;
    const size_t pix = (size_t)py * vp.width + px;
    PixelRay pr;
    pixel_ray_dir(vp, px, py, pr.d);
    pr.pxf = fadd((float)px, 0.5f);
    pr.pyf = fadd((float)py, 0.5f);
    const float dmax = __uint_as_float(dmax_bits[0]);
    // tile lists are ordered by 16-bit range bucket (binning.cu): an entry's
    // bound is the lower edge of its bucket
    const uint32_t r_lo_bits = dmax_bits[1];
    const int r_shift = range_key_shift(r_lo_bits, dmax_bits[3]);

    PixState ps;
    ps.T = 1.0f;
    ps.pxf = pr.pxf;
    ps.pyf = pr.pyf;
    bool done = !inside;
    if (inside) {
        const float4 g = grad_ct[pix];
        const float4 f = fwd_ct[pix];
        ps.gc0 = g.x;
        ps.gc1 = g.y;
        ps.gc2 = g.z;
        ps.gT = g.w;
        init_suffix(ps, fwd_cd + 3 * pix);
        ps.Tf = f.w;
        const float e = ro.grad_skip_eps;
        const bool gc_zero = fabsf(g.x) <= e && fabsf(g.y) <= e && fabsf(g.z) <= e;
        if ((gc_zero && g.w == 0.0f) || ovf_flag[pix]) done = true;
    }

    int head = 0, cnt = 0, nemit = 0;
    float head_t = kInf;
    uint32_t head_pos = 0xffffffffu;
    unsigned long long n_eval = 0, n_rounds = 0, n_small = 0;
    const uint2 rg = ranges[tile];
    uint32_t base = rg.x;
    int nb = 0;

    // Emit every ready entry (t < L) of every lane, one list position per
    // sub-round: the warp takes the smallest ready head position, the lanes
    // holding it pop and compute their adjoints, a butterfly reduces the 9
    // values and one lane issues native red.global.add.f32.
    auto emit_ready = [&](float L) {
        for (;;) {
            bool ready = !done && cnt > 0 && head_t < L;
            if (ready && ro.stop > 0.0f && ps.T < ro.stop) {  // raster.hpp:205 replay termination
                done = true;
                cnt = 0;
                head_t = kInf;
                head_pos = 0xffffffffu;
                ready = false;
            }
            if (!__any_sync(kFull, ready)) return;
            const uint32_t mine = ready ? head_pos : 0xffffffffu;
            const uint32_t pmin = __reduce_min_sync(kFull, mine);
            const bool go = ready && mine == pmin;
            float v[9];
#pragma unroll
            for (int f = 0; f < 9; ++f) v[f] = 0.0f;
            uint32_t mem = 0;
            float msc = 1.0f;
            if (go) {
                const int sl = head & (KBUF - 1);
                const float sigma = bs[sl][tid];
                mem = pair_val[pmin];
                float4 A, B, C, D;
                if (pmin >= base && pmin < base + (uint32_t)nb) {
                    const int j = (int)(pmin - base);
                    A = sA[j];
                    B = sB[j];
                    D = sD[j];
                } else {
                    load_rec(recs, mem, A, B, C, D);
                }
                // g = eval_2d at this pixel, recomputed exactly as in eval_candidate
                const float dx = fsub(pr.pxf, A.x), dy = fsub(pr.pyf, A.y);
                const float m2 = fadd(fmul(dx, fadd(fmul(B.x, dx), fmul(B.y, dy))),
                                      fmul(dy, fadd(fmul(B.z, dx), fmul(B.w, dy))));
                const float g = gauss_expf(m2, ro.trunc < 13.0f);  // eval_2d std::exp in float (splat.hpp:331): sigma bit-exact
                contribution_grad(ps, sigma, g, A, B, D, ro.sigma_clamp, v);
                if (STATS) ++nemit;
                ++head;
                --cnt;
                const int hs = head & (KBUF - 1);
                head_t = cnt ? bt[hs][tid] : kInf;
                head_pos = cnt ? bpos[hs][tid] : 0xffffffffu;
            }
            const unsigned gm = __ballot_sync(kFull, go);
            if (STATS) {
                ++n_rounds;
                if (__popc(gm) <= 2) ++n_small;
            }
            reduce_emit<MODE>(gm, go, lane, mem, v, acc, msc);
        }
    };

    for (base = rg.x; base < rg.y; base += kBlendThreads) {
        if (__syncthreads_count(!done) == 0) break;
        const uint32_t p = base + tid;
        nb = (int)min((uint32_t)kBlendThreads, rg.y - base);
        if (p < rg.y) {
            float4 A, B, C, D;
            const uint32_t m = pair_val[p];
            load_rec(recs, m, A, B, C, D);
            // bound on the ordering key of this and every later entry: the lower edge of
            // the range bucket mapped to t, or (camera_z_order, exact 32-bit sort) the depth
            if (!ro.zorder) D.w = order_bound(range_bucket_lo(D.w, r_lo_bits, r_shift), dmax, onorm);
            sA[tid] = A;
            sB[tid] = B;
            sC[tid] = C;
            sD[tid] = D;
            // which warps (8x4 pixel blocks of this tile) can see m^2 <= 9
            const uint32_t wm = warp_block_mask(__ldg(ext + m), A.x, A.y, tx, ty);
            smask[tid] = (uint8_t)wm;
        }
        __syncthreads();
        // this warp's candidates of the batch, in list order
        int nlist = 0;
        {
            const int wid = tid >> 5, lane = tid & 31;
            const int nbb = (int)min((uint32_t)kBlendThreads, rg.y - base);
            for (int c0 = 0; c0 < nbb; c0 += 32) {
                const int jj = c0 + lane;
                const bool hit = jj < nbb && ((smask[jj] >> wid) & 1u);
                const unsigned bm = __ballot_sync(0xffffffffu, hit);
                if (hit) wlist[nlist + __popc(bm & ((1u << lane) - 1u))] = (uint16_t)jj;
                nlist += __popc(bm);
            }
            __syncwarp();
        }
        for (int q = 0; q < nlist; ++q) {
            if (__all_sync(kFull, done)) break;  // warp finished: no lane can emit again
            const int j = wlist[q];
            emit_ready(sD[j].w);
            if (done) continue;
            const float4 A = sA[j], B = sB[j], C = sC[j];
            if (STATS) ++n_eval;
            float t, sigma, g;
            if (!eval_candidate(pr, vp, ro, gate, A, B, C, sD[j].w, t, sigma, g)) continue;
            const uint32_t id = __float_as_uint(C.w);
            if (cnt == KBUF) {  // cannot happen for pixels that did not overflow in the forward
                done = true;
                continue;
            }
            const uint32_t lpos = base + (uint32_t)j;
            int pos = head + cnt;
            while (pos > head) {
                const int pl = (pos - 1) & (KBUF - 1);
                const float tp = bt[pl][tid];
                const uint32_t ip = bid[pl][tid];
                if (t < tp || (t == tp && id < ip)) {
                    const int psl = pos & (KBUF - 1);
                    bt[psl][tid] = tp;
                    bid[psl][tid] = ip;
                    bs[psl][tid] = bs[pl][tid];
                    bpos[psl][tid] = bpos[pl][tid];
                    --pos;
                } else {
                    break;
                }
            }
            const int psl = pos & (KBUF - 1);
            bt[psl][tid] = t;
            bid[psl][tid] = id;
            bs[psl][tid] = sigma;
            bpos[psl][tid] = lpos;
            ++cnt;
            if (pos == head) {
                head_t = t;
                head_pos = lpos;
            }
        }
    }
    emit_ready(kInf);

    if (STATS && stats != nullptr && tid == 0) atomicAdd(&stats->tiles_work, 1ull);  // replayed tiles
    if (STATS && stats != nullptr) {
        unsigned long long e = n_eval, c = (unsigned long long)nemit;
        for (int off = 16; off > 0; off >>= 1) {
            e += __shfl_xor_sync(kFull, e, off);
            c += __shfl_xor_sync(kFull, c, off);
        }
        if (lane == 0) {
            atomicAdd(&stats->evals, e);
            atomicAdd(&stats->contribs, c);
            atomicAdd(&stats->subrounds, n_rounds);
            atomicAdd(&stats->small_rounds, n_small);
        }
    }
}

// Record walk (default path): every pixel replays exactly the contributions
// the forward composited, in composite order, from the forward's records
// (CompRecords: tile-list positions), so no candidate is re-evaluated and no
// reorder ring is needed.  Sub-rounds group the lanes whose next contribution
// is the same list position (the minimum over the warp), as in the replay
// kernel, and the adjoint of each sub-round is reduced once.  The next
// contribution's record is fetched right after an emission, so its L2 latency
// overlaps the reduction and the other lanes' sub-rounds.
template <bool STATS, int MODE>
__global__ void __launch_bounds__(kBlendThreads, 4) k_blend_bwd_rec(ViewParams vp, RenderOpts ro,
                                                                 const SplatRec* __restrict__ recs,
                                                                 const uint32_t* __restrict__ pair_val,
                                                                 const uint2* __restrict__ ranges,
                                                                 const float4* __restrict__ fwd_ct,
                                                                 const double* __restrict__ fwd_cd,
                                                                 const float4* __restrict__ grad_ct,
                                                                 const uint8_t* __restrict__ ovf_flag,
                                                                 CompRecords crec, GradAcc acc,
                                                                 BlendStats* __restrict__ stats,
                                                                 const uint32_t* __restrict__ tile_order) {
    const int tile = tile_order ? (int)tile_order[blockIdx.x] : (int)blockIdx.x;
    if (crec.tile_replay[tile]) return;  // handled by the replay kernel
    __shared__ uint64_t s_exptab[32];  // eval_2d's exp table
    load_exp_tab(s_exptab);
    __syncthreads();
    const int tid = threadIdx.x, lane = tid & 31;
    const int tx = tile % vp.tiles_x, ty = tile / vp.tiles_x;
    int px, py;
    tile_pixel(tid, tx, ty, px, py);
    const bool inside = px < vp.width && py < vp.height;
    const size_t pix = (size_t)py * vp.width + px;
    PixState ps;
    ps.T = 1.0f;
    ps.pxf = fadd((float)px, 0.5f);
    ps.pyf = fadd((float)py, 0.5f);
    int n = 0;
    if (inside) {
        const float4 g = grad_ct[pix];
        const float4 f = fwd_ct[pix];
        ps.gc0 = g.x;
        ps.gc1 = g.y;
        ps.gc2 = g.z;
        ps.gT = g.w;
        init_suffix(ps, fwd_cd + 3 * pix);
        ps.Tf = f.w;
        const float e = ro.grad_skip_eps;
        const bool gc_zero = fabsf(g.x) <= e && fabsf(g.y) <= e && fabsf(g.z) <= e;
        if (!((gc_zero && g.w == 0.0f) || ovf_flag[pix])) n = crec.cnt[pix];
    }
    const uint32_t base = ranges[tile].x;
    // records of 4 contributions per load: 4 u16 list positions in one 64-bit
    // word, consumed by shifts; the next group of 4 is loaded while the current
    // one is walked, so the DRAM latency stays off the sub-rounds
    const unsigned long long* rp =
        reinterpret_cast<const unsigned long long*>(crec.pos) + (size_t)tile * (kRecCap / 4) * kBlendThreads + tid;
    unsigned long long q4 = 0, q4n = n > 0 ? rp[0] : 0ull;
    int k = 0;
    uint32_t key = 0xffffffffu, m = 0;
    float4 A, B, D;
    auto fetch = [&]() {
        if (k < n) {
            if ((k & 3) == 0) {
                q4 = q4n;
                if (k + 4 < n) q4n = rp[((k >> 2) + 1) * kBlendThreads];
            }
            const uint32_t r = (uint32_t)(q4 & 0xffffu);
            q4 >>= 16;
            key = r;
            m = pair_val[base + r];
            const float4* r4 = reinterpret_cast<const float4*>(recs + m);
            A = __ldg(r4 + 0);
            B = __ldg(r4 + 1);
            D = __ldg(r4 + 3);
        } else {
            key = 0xffffffffu;
        }
    };
    fetch();
    unsigned long long n_rounds = 0, n_small = 0;
    for (;;) {
        const bool ready = key != 0xffffffffu;
        if (!__any_sync(kFull, ready)) break;
        const uint32_t pmin = __reduce_min_sync(kFull, key);
        const bool go = ready && key == pmin;
        float v[9];
#pragma unroll
        for (int f = 0; f < 9; ++f) v[f] = 0.0f;
        uint32_t mem = 0;
        float msc = 1.0f;
        if (go) {
            // sigma and g exactly as the forward computed them (eval_candidate)
            const float dx = fsub(ps.pxf, A.x), dy = fsub(ps.pyf, A.y);
            const float m2 = fadd(fmul(dx, fadd(fmul(B.x, dx), fmul(B.y, dy))),
                                  fmul(dy, fadd(fmul(B.z, dx), fmul(B.w, dy))));
            const float g = gauss_expf(m2, ro.trunc < 13.0f, s_exptab);  // eval_2d std::exp in float (splat.hpp:331): sigma bit-exact
            const float ag = fmul(A.z, g);
            const float sigma = (ro.sigma_clamp < ag) ? ro.sigma_clamp : ag;
            contribution_grad(ps, sigma, g, A, B, D, ro.sigma_clamp, v);
            mem = m;
            ++k;
            fetch();
        }
        const unsigned gm = __ballot_sync(kFull, go);
        if (STATS) {
            ++n_rounds;
            if (__popc(gm) <= 2) ++n_small;
        }
        reduce_emit<MODE>(gm, go, lane, mem, v, acc, msc);
    }
    if (STATS && stats != nullptr) {
        unsigned long long c = (unsigned long long)k;
        for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(kFull, c, off);
        if (lane == 0) {
            atomicAdd(&stats->contribs, c);
            atomicAdd(&stats->subrounds, n_rounds);
            atomicAdd(&stats->small_rounds, n_small);
        }
    }
}

// Exact fallback for ring-overflow pixels: one warp per pixel walks the tile
// list in (t, id) order (fallback_select.cuh), accumulating as it goes.
template <int MODE>
__global__ void __launch_bounds__(64) k_blend_bwd_fallback(ViewParams vp, RenderOpts ro, Subspace gate,
                                                           const SplatRec* __restrict__ recs,
                                                           const uint32_t* __restrict__ pair_val,
                                                           const uint2* __restrict__ ranges,
                                                           const float2* __restrict__ ext,
                                                           const uint32_t* __restrict__ dmax_bits, float onorm,
                                                           const float4* __restrict__ fwd_ct,
                                                           const double* __restrict__ fwd_cd,
                                                           const float4* __restrict__ grad_ct,
                                                           const uint32_t* __restrict__ ovf_list,
                                                           const uint32_t* __restrict__ n_ovf_dev, GradAcc acc) {
    // grid-stride over the device-side overflow count (no host round trip)
    const uint32_t n_ovf = *n_ovf_dev;
    const int lane = threadIdx.x & 31;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n_ovf; w += nw) {
        const uint32_t pix = ovf_list[w];
        const int px = pix % vp.width, py = pix / vp.width;
        const int tile = (py / kTileSize) * vp.tiles_x + px / kTileSize;
        PixelRay pr;
        pixel_ray_dir(vp, px, py, pr.d);
        pr.pxf = fadd((float)px, 0.5f);
        pr.pyf = fadd((float)py, 0.5f);
        PixState ps;
        ps.T = 1.0f;
        ps.pxf = pr.pxf;
        ps.pyf = pr.pyf;
        const float4 gg = grad_ct[pix], ff = fwd_ct[pix];
        ps.gc0 = gg.x;
        ps.gc1 = gg.y;
        ps.gc2 = gg.z;
        ps.gT = gg.w;
        init_suffix(ps, fwd_cd + 3 * (size_t)pix);
        ps.Tf = ff.w;
        const float e = ro.grad_skip_eps;
        if (fabsf(gg.x) <= e && fabsf(gg.y) <= e && fabsf(gg.z) <= e && gg.w == 0.0f) continue;
        auto eval = [&](uint32_t mem, float& t, float& sigma, float& g, uint32_t& id) {
            float4 A, B, C, D;
            load_rec(recs, mem, A, B, C, D);
            if (!eval_candidate(pr, vp, ro, gate, A, B, C, D.w, t, sigma, g)) return false;
            id = __float_as_uint(C.w);
            return true;
        };
        auto emit = [&](float, uint32_t, float sigma, float g, uint32_t mem) {
            if (ro.stop > 0.0f && ps.T < ro.stop) return false;
            float4 A, B, C, D;
            load_rec(recs, mem, A, B, C, D);
            float v[9];
            contribution_grad(ps, sigma, g, A, B, D, ro.sigma_clamp, v);
            if (lane == 0)
                for (int f = 0; f < 9; ++f) acc_add<MODE>(acc, f, mem, v[f], 1.0f);
            return true;
        };
        __shared__ FbRing rings[2];  // one per warp of the 64-thread block
        const float dmax = __uint_as_float(dmax_bits[0]);
        const uint32_t r_lo_bits = dmax_bits[1];
        const int r_shift = range_key_shift(r_lo_bits, dmax_bits[3]);
        auto bound = [&](float range) {
            return ro.zorder ? range : order_bound(range_bucket_lo(range, r_lo_bits, r_shift), dmax, onorm);
        };
        warp_ring_walk(pr.pxf, pr.pyf, ranges[tile], pair_val, recs, ext, rings[(threadIdx.x >> 5) & 1], bound, eval,
                       emit);
    }
}


template <int MODE>
void blend_bwd_impl(const ViewParams& vp, const RenderOpts& ro, const Subspace& gate, const ViewBins& vb,
                    const float4* fwd_ct, const double* fwd_cd, const float4* grad_ct, const uint8_t* ovf_flag,
                    const CompRecords& rec, const GradAcc& acc, BlendStats* stats, cudaStream_t s) {
    const int tiles = vp.tiles_x * vp.tiles_y;
    const float onorm = sqrtf(vp.o[0] * vp.o[0] + vp.o[1] * vp.o[1] + vp.o[2] * vp.o[2]);
    ensure_smem_attr((const void*)k_blend_bwd<true, MODE>, (int)kBwdSmem);
    ensure_smem_attr((const void*)k_blend_bwd<false, MODE>, (int)kBwdSmem);
    if (rec.pos != nullptr) {
        if (stats)
            k_blend_bwd_rec<true, MODE><<<tiles, kBlendThreads, 0, s>>>(vp, ro, vb.recs, vb.pair_val, vb.ranges, fwd_ct,
                                                                        fwd_cd, grad_ct, ovf_flag, rec, acc, stats,
                                                                        vb.tile_order);
        else
            k_blend_bwd_rec<false, MODE><<<tiles, kBlendThreads, 0, s>>>(vp, ro, vb.recs, vb.pair_val, vb.ranges,
                                                                         fwd_ct, fwd_cd, grad_ct, ovf_flag, rec, acc,
                                                                         stats, vb.tile_order);
    }
    // replay: flagged tiles only (every tile without records)
    if (stats)
        k_blend_bwd<true, MODE><<<tiles, kBlendThreads, kBwdSmem, s>>>(vp, ro, gate, vb.recs, vb.pair_val, vb.ranges,
                                                                       vb.ext, vb.dmax_bits, onorm, fwd_ct, fwd_cd,
                                                                       grad_ct, ovf_flag, rec.tile_replay, acc, stats,
                                                                       vb.tile_order);
    else
        k_blend_bwd<false, MODE><<<tiles, kBlendThreads, kBwdSmem, s>>>(vp, ro, gate, vb.recs, vb.pair_val, vb.ranges,
                                                                        vb.ext, vb.dmax_bits, onorm, fwd_ct, fwd_cd,
                                                                        grad_ct, ovf_flag, rec.tile_replay, acc, stats,
                                                                        vb.tile_order);
}

template <int MODE>
void blend_bwd_fallback_impl(const ViewParams& vp, const RenderOpts& ro, const Subspace& gate, const ViewBins& vb,
                             const float4* fwd_ct, const double* fwd_cd, const float4* grad_ct,
                             const uint32_t* ovf_list, const uint32_t* n_ovf_dev, const GradAcc& acc, cudaStream_t s) {
    const float onorm = sqrtf(vp.o[0] * vp.o[0] + vp.o[1] * vp.o[1] + vp.o[2] * vp.o[2]);
    k_blend_bwd_fallback<MODE><<<148 * 8, 64, 0, s>>>(vp, ro, gate, vb.recs, vb.pair_val, vb.ranges, vb.ext,
                                                      vb.dmax_bits, onorm, fwd_ct, fwd_cd, grad_ct, ovf_list,
                                                      n_ovf_dev, acc);
}

/// Deterministic mode: g2d = (hi 2^32 + lo) 2^-72 (acc.q [9][lo | hi][ld]),
/// then the accumulators are zeroed for the next backward (they stay zero
/// between uses).  One member per thread, coalesced 8-byte row reads, all
/// loads issued before any store: HBM-bound.  The training step fuses this
/// into K9 instead (k_grad_record's fixed-point input).
__global__ void __launch_bounds__(256) k_fixed_to_float(GradAcc acc, int n) {
    const size_t ld = acc.ld;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        float a[9];
        fixed_to_float9(acc.q, ld, i, a);
        float4* o = reinterpret_cast<float4*>(acc.f + 8 * (size_t)i);
        o[0] = make_float4(a[0], a[1], a[2], a[3]);
        o[1] = make_float4(a[4], a[5], a[6], a[7]);
        acc.f[8 * ld + i] = a[8];
    }
}

}  // namespace

void launch_blend_bwd(const ViewParams& vp, const RenderOpts& ro, const Subspace& gate, const ViewBins& vb,
                      const float4* fwd_ct, const double* fwd_cd, const float4* grad_ct, const uint8_t* ovf_flag,
                      const CompRecords& rec, const GradAcc& acc, const uint32_t* ovf_list,
                      const uint32_t* n_ovf_dev, BlendStats* stats, cudaStream_t s) {
    if (acc.q == nullptr) {
        blend_bwd_impl<kAccFloat>(vp, ro, gate, vb, fwd_ct, fwd_cd, grad_ct, ovf_flag, rec, acc, stats, s);
        blend_bwd_fallback_impl<kAccFloat>(vp, ro, gate, vb, fwd_ct, fwd_cd, grad_ct, ovf_list, n_ovf_dev, acc, s);
        return;
    }
    // deterministic: one pass of fixed-point sums; then launch_fixed_to_float
    blend_bwd_impl<kAccFixed>(vp, ro, gate, vb, fwd_ct, fwd_cd, grad_ct, ovf_flag, rec, acc, stats, s);
    blend_bwd_fallback_impl<kAccFixed>(vp, ro, gate, vb, fwd_ct, fwd_cd, grad_ct, ovf_list, n_ovf_dev, acc, s);
}

void launch_fixed_to_float(const GradAcc& acc, int n, cudaStream_t s) {
    if (n <= 0) return;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    k_fixed_to_float<<<std::min((n + 255) / 256, sms * 8), 256, 0, s>>>(acc, n);  // a warp per 32 members
}

}  // namespace dgs_b200
