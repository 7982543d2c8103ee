// K4 — forward alpha blend of one KD subset with the RetinaGS subspace gate.
//
// Reference semantics (raster.hpp:146-189, engine.hpp:31-52): per pixel, the
// contributions that pass  m^2 <= 9,  t = d.(mu-o) > 0,  ||o+td-mu||^2 <= D^2,
// the subspace indicator at x_i, and sigma = min(alpha g, 0.99) > 0  are
// composited front to back in (t, id) order; termination (T < stop) is tested
// before every contribution; no background.
//
// sm_100a design: one 256-thread CTA per 16x16 tile walks the tile's pair list
// (range-ordered, binning.cu) in batches of 256 records staged through shared
// memory (broadcast LDS.128 reads in the inner loop).  Because the list is
// ordered by range r and every contributor satisfies t >= sqrt(r^2 - D^2),
// each pixel keeps its accepted contributions in a small shared-memory ring
// (KBUF entries) sorted by (t, id) and composites an entry as soon as its t is
// below the lower bound L_n of every not-yet-seen candidate.  The composite
// order is therefore exactly the reference's per-pixel std::sort order.  A
// pixel whose ring would overflow is handed to an exact O(n^2/16) fallback.
#include "kernels.h"
#include "fallback_select.cuh"

namespace dgs_b200 {

namespace {

constexpr int KBUF = 8;  // ring capacity (power of two); must equal blend_bwd.cu
#ifndef DGS_EMIT_EVERY
#define DGS_EMIT_EVERY 4
#endif
constexpr int kEmitEvery = DGS_EMIT_EVERY;  // candidates between emission checks (power of two)
constexpr float kInf = __builtin_huge_valf();
// 4 staged float4 record fields + 4 ring fields per pixel (t, id, sigma, member).
constexpr size_t kFwdSmem = 4 * kBlendThreads * sizeof(float4) + 4 * KBUF * kBlendThreads * sizeof(float) +
                            kBlendThreads * sizeof(uint16_t) + (kBlendThreads / 32) * kBlendThreads * sizeof(uint16_t);

/// 16-bit mask of the 4x4 pixel sub-blocks of tile (tx, ty) that may contain a
/// pixel with m^2 <= trunc^2 (the conservative test of warp_block_mask at 4x4
/// granularity).  Bit (row * 4 + col).
__device__ __forceinline__ uint32_t subblock_mask(float2 ext, float mx, float my, int tx, int ty) {
    uint32_t cm = 0, rm = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const float xlo = fadd((float)(tx * kTileSize + b * 4), 0.5f), xhi = fadd(xlo, 3.0f);
        if (!(fsub(xlo, mx) > ext.x || fsub(mx, xhi) > ext.x)) cm |= 1u << b;
        const float ylo = fadd((float)(ty * kTileSize + b * 4), 0.5f), yhi = fadd(ylo, 3.0f);
        if (!(fsub(ylo, my) > ext.y || fsub(my, yhi) > ext.y)) rm |= 1u << b;
    }
    uint32_t m = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r)
        if ((rm >> r) & 1u) m |= cm << (4 * r);
    return m;
}
/// The 4x4 sub-block of a pixel slot (tile_pixel order).
__device__ __forceinline__ int slot_subblock(int q) {
    const int w = q >> 5, l = q & 31;
    return (w >> 1) * 4 + (w & 1) * 2 + ((l & 7) >> 2);  // row = 4-pixel row group, col = 4-pixel column group
}

/// Lower bound on t for every candidate at or after a list position whose
/// range is r (t >= sqrt(r^2 - D^2), with margins ≫ float
/// rounding of t, r and the D gate).
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

/// Evaluate one candidate for one pixel with the reference's gates
/// (raster.hpp:153-161).  Returns false when it does not contribute.
__device__ __forceinline__ bool eval_candidate(const PixelRay& pr, const ViewParams& vp, const RenderOpts& ro,
                                               const Subspace& gate, const float4& A, const float4& B,
                                               const float4& C, float zkey, float& t_out, float& sigma_out,
                                               float& g_out, const uint64_t* exp_tab = nullptr) {
    const float dx = fsub(pr.pxf, A.x), dy = fsub(pr.pyf, A.y);
    // eval_2d (splat.hpp:326-332): m2 = delta . (inv_cov2d * delta)
    const float m2 = fadd(fmul(dx, fadd(fmul(B.x, dx), fmul(B.y, dy))), fmul(dy, fadd(fmul(B.z, dx), fmul(B.w, dy))));
    if (!(m2 <= fmul(ro.trunc, ro.trunc))) return false;  // g = 0 (or NaN) -> !(g > 0)
    const float t = dot3(pr.d[0], pr.d[1], pr.d[2], fsub(C.x, vp.o[0]), fsub(C.y, vp.o[1]), fsub(C.z, vp.o[2]));
    if (!(t > 0.0f)) return false;
    const float x0 = fadd(vp.o[0], fmul(t, pr.d[0]));
    const float x1 = fadd(vp.o[1], fmul(t, pr.d[1]));
    const float x2 = fadd(vp.o[2], fmul(t, pr.d[2]));
    const float e0 = fsub(x0, C.x), e1 = fsub(x1, C.y), e2 = fsub(x2, C.z);
    if (dot3(e0, e1, e2, e0, e1, e2) > A.w) return false;
    if (ro.indicator_enabled && !subspace_contains(gate, x0, x1, x2)) return false;
    const float g = gauss_expf(m2, ro.trunc < 13.0f, exp_tab);  // eval_2d std::exp in float (splat.hpp:331): sigma bit-exact
    const float ag = fmul(A.z, g);
    const float sigma = (ro.sigma_clamp < ag) ? ro.sigma_clamp : ag;  // std::min(alpha*g, clamp)
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

/// Forward blend of one tile (CTA, 256 pixel slots).  Candidates are staged in
/// list batches of 256; every warp composites the candidates its pixels can
/// see through a per-pixel (t, id) ring.  Pixels terminate at very different
/// depths, so warps soon run at a few live lanes: at a batch boundary, once the
/// live pixels fit in fewer warps, they are re-packed (slot order kept, so a
/// warp's pixels stay close) and every warp culls candidates against the
/// bounding box of its own pixels.  Per-pixel state moves through shared
/// memory; the ring stays in place (indexed by pixel slot).
template <bool DBG, bool STATS>
__global__ void __launch_bounds__(kBlendThreads, 4) k_blend_fwd(ViewParams vp, RenderOpts ro, Subspace gate,
                                                             const SplatRec* __restrict__ recs,
                                                             const uint32_t* __restrict__ pair_val,
                                                             const uint2* __restrict__ ranges,
                                                             const float2* __restrict__ ext,
                                                             const uint32_t* __restrict__ dmax_bits, float onorm,
                                                             float4* __restrict__ out_ct, uint8_t* __restrict__ ovf_flag,
                                                             uint32_t* __restrict__ ovf_list,
                                                             uint32_t* __restrict__ ovf_count,
                                                             uint32_t* __restrict__ dbg_ids,
                                                             uint32_t* __restrict__ dbg_cnt, int dbg_cap,
                                                             BlendStats* __restrict__ stats,
                                                             double* __restrict__ out_cd, CompRecords crec,
                                                             const uint32_t* __restrict__ tile_order) {
    extern __shared__ float4 smem4[];
    float4* sA = smem4;
    float4* sB = sA + kBlendThreads;
    float4* sC = sB + kBlendThreads;
    float4* sD = sC + kBlendThreads;
    typedef float Ring[kBlendThreads];
    Ring* bt = reinterpret_cast<Ring*>(sD + kBlendThreads);
    uint32_t(*bid)[kBlendThreads] = reinterpret_cast<uint32_t(*)[kBlendThreads]>(bt + KBUF);
    Ring* bs = reinterpret_cast<Ring*>(bid + KBUF);
    // list position of each ring entry (colour from the staged batch or, for
    // entries accepted in an earlier batch, through pair_val; also recorded)
    uint32_t(*bpos)[kBlendThreads] = reinterpret_cast<uint32_t(*)[kBlendThreads]>(bs + KBUF);
    uint16_t* wlist = reinterpret_cast<uint16_t*>(bpos + KBUF) + (threadIdx.x >> 5) * kBlendThreads;
    uint16_t* smask = reinterpret_cast<uint16_t*>(bpos + KBUF) + (kBlendThreads / 32) * kBlendThreads;
    __shared__ int s_woff[kBlendThreads / 32];
    __shared__ int s_short;
    __shared__ uint64_t s_exptab[32];  // eval_2d's exp table (read before the first batch's barrier)
    load_exp_tab(s_exptab);

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int tile = tile_order ? (int)tile_order[blockIdx.x] : (int)blockIdx.x;
    const int tx = tile % vp.tiles_x, ty = tile / vp.tiles_x;
    const float dmax = __uint_as_float(dmax_bits[0]);
    // tile lists are ordered by 16-bit range bucket (binning.cu): an entry's
    // bound is the lower edge of its bucket
    const uint32_t r_lo_bits = dmax_bits[1];
    const int r_shift = range_key_shift(r_lo_bits, dmax_bits[3]);
    const uint2 rg = ranges[tile];
    const bool record = crec.pos != nullptr && rg.y - rg.x <= 65535u;

    // ---- per-slot pixel state (the slot travels with the pixel when re-packed) ----
    int q = tid;  // pixel slot: tile_pixel order
    bool valid = true;
    int px, py;
    size_t pix;
    bool inside;
    PixelRay pr;
    uint16_t* rec16;
    auto bind_slot = [&]() {
        tile_pixel(q, tx, ty, px, py);
        inside = px < vp.width && py < vp.height;
        pix = (size_t)py * vp.width + px;
        pixel_ray_dir(vp, px, py, pr.d);
        pr.pxf = fadd((float)px, 0.5f);
        pr.pyf = fadd((float)py, 0.5f);
        rec16 = record ? crec.pos + (size_t)tile * kRecCap * kBlendThreads + 4 * q : nullptr;
    };
    bind_slot();
    float T = 1.0f, C0 = 0.0f, C1 = 0.0f, C2 = 0.0f;
    double D0 = 0.0, D1 = 0.0, D2 = 0.0;  // exact-ish sum of c*sigma*A for the backward suffix
    bool done = !inside, ovf = false;
    int head = 0, cnt = 0, nemit = 0;
    float head_t = kInf;
    unsigned long long n_eval = 0, n_contrib = 0, n_ovf = 0;
    uint32_t cur_base = rg.x, cur_nb = 0;  // batch currently staged in shared memory
    if (tid == 0) s_short = 0;
    int live_warps = kBlendThreads / 32;
    // the 4x4 sub-blocks this warp's pixels lie in: a staged candidate concerns
    // the warp only if its sub-block mask meets this one
    uint32_t wsub = __reduce_or_sync(0xffffffffu, 1u << slot_subblock(q));

    auto emit_head = [&]() {
        if (ro.stop > 0.0f && T < ro.stop) {  // raster.hpp:183
            done = true;
            cnt = 0;
            head_t = kInf;
            return;
        }
        const int sl = head & (KBUF - 1);
        const float sg = bs[sl][q];
        const uint32_t lp = bpos[sl][q];
        const float4 col = (lp - cur_base < cur_nb) ? sD[lp - cur_base]
                                                    : __ldg(reinterpret_cast<const float4*>(recs + pair_val[lp]) + 3);
        if (record && nemit < kRecCap) rec16[(nemit >> 2) * (4 * kBlendThreads) + (nemit & 3)] = (uint16_t)(lp - rg.x);
        const float w = fmul(sg, T);
        C0 = fadd(C0, fmul(col.x, w));
        C1 = fadd(C1, fmul(col.y, w));
        C2 = fadd(C2, fmul(col.z, w));
        if (out_cd != nullptr) {
            const double wd = (double)sg * (double)T;
            D0 += (double)col.x * wd;
            D1 += (double)col.y * wd;
            D2 += (double)col.z * wd;
        }
        T = fmul(T, fsub(1.0f, sg));
        if (DBG && nemit < dbg_cap) dbg_ids[pix * dbg_cap + nemit] = bid[sl][q];
        ++nemit;
        ++head;
        --cnt;
        head_t = cnt ? bt[head & (KBUF - 1)][q] : kInf;
    };
    // final values of this slot's pixel (once it is done, or at the end)
    auto write_out = [&]() {
        if (!inside) return;
        if (crec.pos != nullptr) {
            if (!ovf && nemit > kRecCap) s_short = 1;  // records incomplete: the backward replays the tile
            crec.cnt[pix] = (uint16_t)min(nemit, kRecCap);
        }
        if (ovf) {
            ovf_flag[pix] = 1;
            ovf_list[atomicAdd(ovf_count, 1u)] = (uint32_t)pix;
        } else {
            ovf_flag[pix] = 0;
            out_ct[pix] = make_float4(C0, C1, C2, T);
            if (out_cd != nullptr) {
                out_cd[3 * pix] = D0;
                out_cd[3 * pix + 1] = D1;
                out_cd[3 * pix + 2] = D2;
            }
            if (DBG) dbg_cnt[pix] = (uint32_t)nemit;
        }
        if (STATS) {
            n_contrib += (unsigned long long)nemit;
            n_ovf += ovf ? 1ull : 0ull;
        }
    };

    // the member index of this thread's entry in the next batch is loaded one batch ahead
    uint32_t m_next = rg.x + tid < rg.y ? pair_val[rg.x + tid] : 0u;
    for (uint32_t base = rg.x; base < rg.y; base += kBlendThreads) {
        const int nact = __syncthreads_count(valid && !done);
        if (nact == 0) break;
        if ((nact + 31) / 32 < live_warps) {
            // ---- re-pack the live pixels into the first warps (slot order kept) ----
            if (valid && done) {
                write_out();
                valid = false;
            }
            const bool live = valid && !done;
            const unsigned bm = __ballot_sync(0xffffffffu, live);
            if (lane == 0) s_woff[wid] = __popc(bm);
            __syncthreads();
            int rank = __popc(bm & ((1u << lane) - 1u));
            for (int w = 0; w < wid; ++w) rank += s_woff[w];
            // state through the staging area (its batch is fully consumed)
            // (16 KB: 5 float rows at 0, 4 int rows at 5 KB, 3 double rows at 9 KB)
            char* st = reinterpret_cast<char*>(sA);
            float* fs = reinterpret_cast<float*>(st);
            int* is = reinterpret_cast<int*>(st + 5 * kBlendThreads * sizeof(float));
            double* ds = reinterpret_cast<double*>(st + 9 * kBlendThreads * sizeof(float));
            if (live) {
                fs[rank] = T;
                fs[kBlendThreads + rank] = C0;
                fs[2 * kBlendThreads + rank] = C1;
                fs[3 * kBlendThreads + rank] = C2;
                fs[4 * kBlendThreads + rank] = head_t;
                ds[rank] = D0;
                ds[kBlendThreads + rank] = D1;
                ds[2 * kBlendThreads + rank] = D2;
                is[rank] = q;
                is[kBlendThreads + rank] = head;
                is[2 * kBlendThreads + rank] = cnt;
                is[3 * kBlendThreads + rank] = nemit;
            }
            __syncthreads();
            valid = tid < nact;
            done = !valid;
            if (valid) {
                T = fs[tid];
                C0 = fs[kBlendThreads + tid];
                C1 = fs[2 * kBlendThreads + tid];
                C2 = fs[3 * kBlendThreads + tid];
                head_t = fs[4 * kBlendThreads + tid];
                D0 = ds[tid];
                D1 = ds[kBlendThreads + tid];
                D2 = ds[2 * kBlendThreads + tid];
                q = is[tid];
                head = is[kBlendThreads + tid];
                cnt = is[2 * kBlendThreads + tid];
                nemit = is[3 * kBlendThreads + tid];
                ovf = false;
                bind_slot();
            }
            live_warps = (nact + 31) / 32;
            wsub = __reduce_or_sync(0xffffffffu, valid ? 1u << slot_subblock(q) : 0u);
            __syncthreads();  // the staging area is free again
        }
        cur_base = base;
        cur_nb = min((uint32_t)kBlendThreads, rg.y - base);
        const uint32_t p = base + tid;
        const uint32_t m = m_next;
        if (p + kBlendThreads < rg.y) m_next = pair_val[p + kBlendThreads];
        if (p < rg.y) {
            float4 A, B, C, D;
            load_rec(recs, m, A, B, C, D);
            // bound on the ordering key of this and every later entry: the lower edge of
            // the range bucket mapped to t, or (camera_z_order, exact 32-bit sort) the depth
            if (!ro.zorder) D.w = order_bound(range_bucket_lo(D.w, r_lo_bits, r_shift), dmax, onorm);
            sA[tid] = A;
            sB[tid] = B;
            sC[tid] = C;
            sD[tid] = D;
            // which 4x4 pixel sub-blocks of this tile can see m^2 <= 9
            smask[tid] = (uint16_t)subblock_mask(__ldg(ext + m), A.x, A.y, tx, ty);
        }
        __syncthreads();
        // this warp's candidates of the batch, in list order
        int nlist = 0;
        if (wid < live_warps) {
            const int nbb = (int)min((uint32_t)kBlendThreads, rg.y - base);
            for (int c0 = 0; c0 < nbb; c0 += 32) {
                const int jj = c0 + lane;
                const bool hit = jj < nbb && (smask[jj] & wsub);
                const unsigned bm = __ballot_sync(0xffffffffu, hit);
                if (hit) wlist[nlist + __popc(bm & ((1u << lane) - 1u))] = (uint16_t)jj;
                nlist += __popc(bm);
            }
            __syncwarp();
        }
        for (int qq = 0; qq < nlist && !done; ++qq) {
            const int j = wlist[qq];
            const float4 D = sD[j];
            // Emission is deferred to every kEmitEvery-th candidate (qq is uniform over the
            // warp, so the lanes emit together instead of one divergent loop per candidate)
            // or to a (nearly) full ring.  Emitting later is exact: an entry with t below the
            // bound of a list position stays below every later bound, and nothing inserted
            // later can precede it; the sequence, its termination point and the overflow
            // decision (full ring with nothing emittable) are those of eager emission.
            if ((qq & (kEmitEvery - 1)) == 0 || cnt >= KBUF - 1)
                while (head_t < D.w && !done) emit_head();
            if (done) break;
            const float4 A = sA[j], B = sB[j], C = sC[j];
            if (STATS) ++n_eval;
            float t, sigma, g;
            if (!eval_candidate(pr, vp, ro, gate, A, B, C, D.w, t, sigma, g, s_exptab)) continue;
            const uint32_t id = __float_as_uint(C.w);
            if (cnt == KBUF) {
                while (head_t < D.w && !done) emit_head();
                if (done) break;
            }
            if (cnt == KBUF) {  // ring full and nothing safe to emit: exact fallback
                ovf = true;
                done = true;
                break;
            }
            int pos = head + cnt;
            while (pos > head) {
                const int pl = (pos - 1) & (KBUF - 1);
                const float tp = bt[pl][q];
                const uint32_t ip = bid[pl][q];
                if (t < tp || (t == tp && id < ip)) {
                    const int ps = pos & (KBUF - 1);
                    bt[ps][q] = tp;
                    bid[ps][q] = ip;
                    bs[ps][q] = bs[pl][q];
                    bpos[ps][q] = bpos[pl][q];
                    --pos;
                } else {
                    break;
                }
            }
            const int ps = pos & (KBUF - 1);
            bt[ps][q] = t;
            bid[ps][q] = id;
            bs[ps][q] = sigma;
            bpos[ps][q] = base + (uint32_t)j;
            ++cnt;
            if (pos == head) head_t = t;
        }
    }
    if (valid) {
        while (cnt > 0 && !done) emit_head();
        write_out();
    }
    if (crec.pos != nullptr) {
        __syncthreads();
        if (tid == 0) crec.tile_replay[tile] = (uint8_t)(s_short != 0 || !record);
    }
    if (STATS && stats != nullptr) {
        unsigned long long e = n_eval, c = n_contrib, o = n_ovf;
        for (int off = 16; off > 0; off >>= 1) {
            e += __shfl_xor_sync(0xffffffffu, e, off);
            c += __shfl_xor_sync(0xffffffffu, c, off);
            o += __shfl_xor_sync(0xffffffffu, o, off);
        }
        if ((tid & 31) == 0) {
            atomicAdd(&stats->evals, e);
            atomicAdd(&stats->contribs, c);
            atomicAdd(&stats->overflow, o);
        }
        if (tid == 0) atomicAdd(&stats->tiles_work, (unsigned long long)(rg.y - rg.x));
    }
}

// Exact fallback for ring-overflow pixels: one warp per pixel walks the tile
// list in (t, id) order (fallback_select.cuh) and composites as it goes.
__global__ void __launch_bounds__(64) k_blend_fwd_fallback(ViewParams vp, RenderOpts ro, Subspace gate,
                                                           const SplatRec* __restrict__ recs,
                                                           const uint32_t* __restrict__ pair_val,
                                                           const uint2* __restrict__ ranges,
                                                           const float2* __restrict__ ext,
                                                           const uint32_t* __restrict__ dmax_bits, float onorm, float4* __restrict__ out_ct,
                                                           const uint32_t* __restrict__ ovf_list,
                                                           const uint32_t* __restrict__ n_ovf_dev,
                                                           uint32_t* __restrict__ dbg_ids, uint32_t* __restrict__ dbg_cnt,
                                                           int dbg_cap, double* __restrict__ out_cd) {
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
        float T = 1.0f, C0 = 0.0f, C1 = 0.0f, C2 = 0.0f;
        double D0 = 0.0, D1 = 0.0, D2 = 0.0;
        int nemit = 0;
        auto eval = [&](uint32_t mem, float& t, float& sigma, float& g, uint32_t& id) {
            float4 A, B, C, D;
            load_rec(recs, mem, A, B, C, D);
            if (!eval_candidate(pr, vp, ro, gate, A, B, C, D.w, t, sigma, g)) return false;
            id = __float_as_uint(C.w);
            return true;
        };
        auto emit = [&](float, uint32_t id, float sigma, float, uint32_t mem) {
            if (ro.stop > 0.0f && T < ro.stop) return false;  // raster.hpp:183
            const float4 col = __ldg(reinterpret_cast<const float4*>(recs + mem) + 3);
            const float wgt = fmul(sigma, T);
            C0 = fadd(C0, fmul(col.x, wgt));
            C1 = fadd(C1, fmul(col.y, wgt));
            C2 = fadd(C2, fmul(col.z, wgt));
            const double wd = (double)sigma * (double)T;
            D0 += (double)col.x * wd;
            D1 += (double)col.y * wd;
            D2 += (double)col.z * wd;
            T = fmul(T, fsub(1.0f, sigma));
            if (lane == 0 && dbg_ids != nullptr && nemit < dbg_cap) dbg_ids[(size_t)pix * dbg_cap + nemit] = id;
            ++nemit;
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
        if (lane == 0) {
            out_ct[pix] = make_float4(C0, C1, C2, T);
            if (out_cd != nullptr) {
                out_cd[3 * (size_t)pix] = D0;
                out_cd[3 * (size_t)pix + 1] = D1;
                out_cd[3 * (size_t)pix + 2] = D2;
            }
            if (dbg_cnt != nullptr) dbg_cnt[pix] = (uint32_t)nemit;
        }
    }
}

}  // namespace

void launch_blend_fwd(const ViewParams& vp, const RenderOpts& ro, const Subspace& gate, const ViewBins& vb,
                      float4* out_ct, uint8_t* ovf_flag, uint32_t* ovf_list, uint32_t* ovf_count,
                      uint32_t* dbg_ids, uint32_t* dbg_cnt, int dbg_cap, BlendStats* stats, double* out_cd,
                      const CompRecords& rec, cudaStream_t s) {
    const int tiles = vp.tiles_x * vp.tiles_y;
    const float onorm = sqrtf(vp.o[0] * vp.o[0] + vp.o[1] * vp.o[1] + vp.o[2] * vp.o[2]);
    const size_t smem = kFwdSmem;
    ensure_smem_attr((const void*)k_blend_fwd<false, false>, (int)smem);
    ensure_smem_attr((const void*)k_blend_fwd<false, true>, (int)smem);
    ensure_smem_attr((const void*)k_blend_fwd<true, true>, (int)smem);
#define DGS_FWD(D, S)                                                                                              \
    k_blend_fwd<D, S><<<tiles, kBlendThreads, smem, s>>>(vp, ro, gate, vb.recs, vb.pair_val, vb.ranges, vb.ext, vb.dmax_bits, \
                                                         onorm, out_ct, ovf_flag, ovf_list, ovf_count, dbg_ids,       \
                                                         dbg_cnt, dbg_cap, stats, out_cd, rec, vb.tile_order)
    if (dbg_ids != nullptr && dbg_cnt != nullptr) DGS_FWD(true, true);
    else if (stats != nullptr) DGS_FWD(false, true);
    else DGS_FWD(false, false);
#undef DGS_FWD
}

void launch_blend_fwd_fallback(const ViewParams& vp, const RenderOpts& ro, const Subspace& gate, const ViewBins& vb,
                               float4* out_ct, const uint32_t* ovf_list, const uint32_t* n_ovf_dev, uint32_t* dbg_ids,
                               uint32_t* dbg_cnt, int dbg_cap, double* out_cd, cudaStream_t s) {
    // fixed grid, device-side count: launched unconditionally (exits at once when nothing overflowed)
    const float onorm = sqrtf(vp.o[0] * vp.o[0] + vp.o[1] * vp.o[1] + vp.o[2] * vp.o[2]);
    k_blend_fwd_fallback<<<148 * 8, 64, 0, s>>>(vp, ro, gate, vb.recs, vb.pair_val, vb.ranges, vb.ext, vb.dmax_bits,
                                               onorm, out_ct, ovf_list, n_ovf_dev, dbg_ids, dbg_cnt, dbg_cap, out_cd);
}

}  // namespace dgs_b200
