// Warp-cooperative exact ordering for the ring-overflow fallbacks (K4 and K8):
// one warp per overflowing pixel.  Each round, the lanes scan the tile list in
// parallel (position rg.x + lane + 32 k; entries whose m^2 <= 9 extent misses
// the pixel are skipped before the full evaluation), each keeps its FB
// smallest (t, id) contributions above the watermark, and the warp merges the
// lanes' sorted lists by repeated argmin: the next FB contributions of the
// pixel in the reference's (t, id) order (raster.hpp:162-166), handed to
// `emit` one by one on every lane.  The pixel-state arithmetic in `emit` runs
// redundantly on all lanes (identical values); side effects belong to lane 0.
#pragma once

namespace dgs_b200 {

constexpr int kFbBatch = 64;

/// Returns when `emit` returns false (the pixel terminated) or the list is exhausted.
template <class Eval, class Emit>
__device__ __forceinline__ void warp_ordered_walk(float pxf, float pyf, uint2 rg, const uint32_t* __restrict__ pair_val,
                                                  const SplatRec* __restrict__ recs, const float2* __restrict__ ext,
                                                  Eval eval, Emit emit, bool have_w = false,
                                                  float wt = -__builtin_huge_valf(), uint32_t wid = 0) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        float lt[kFbBatch], ls[kFbBatch], lg[kFbBatch];
        uint32_t li[kFbBatch], lm[kFbBatch];
        int m = 0;
        for (uint32_t p = rg.x + lane; p < rg.y; p += 32) {
            const uint32_t mem = pair_val[p];
            const float4 A0 = __ldg(reinterpret_cast<const float4*>(recs + mem));
            const float2 e = __ldg(ext + mem);
            if (fsub(pxf, A0.x) > e.x || fsub(A0.x, pxf) > e.x || fsub(pyf, A0.y) > e.y || fsub(A0.y, pyf) > e.y)
                continue;  // m^2 > 9 for this pixel (the conservative extent test of the blends)
            float t, sigma, g;
            uint32_t id;
            if (!eval(mem, t, sigma, g, id)) continue;
            if (have_w && !(t > wt || (t == wt && id > wid))) continue;
            if (m == kFbBatch && !(t < lt[kFbBatch - 1] || (t == lt[kFbBatch - 1] && id < li[kFbBatch - 1]))) continue;
            int pos = m < kFbBatch ? m : kFbBatch - 1;
            while (pos > 0 && (t < lt[pos - 1] || (t == lt[pos - 1] && id < li[pos - 1]))) {
                lt[pos] = lt[pos - 1];
                li[pos] = li[pos - 1];
                ls[pos] = ls[pos - 1];
                lg[pos] = lg[pos - 1];
                lm[pos] = lm[pos - 1];
                --pos;
            }
            lt[pos] = t;
            li[pos] = id;
            ls[pos] = sigma;
            lg[pos] = g;
            lm[pos] = mem;
            if (m < kFbBatch) ++m;
        }
        // merge: kFbBatch rounds of the warp-wide smallest head (t > 0, so its bits order like t)
        int h = 0, taken = 0;
        float last_t = 0.0f;
        uint32_t last_id = 0;
        for (int k = 0; k < kFbBatch; ++k) {
            const unsigned long long key =
                h < m ? ((unsigned long long)__float_as_uint(lt[h]) << 32) | li[h] : ~0ull;
            unsigned long long best = key;
            for (int off = 16; off > 0; off >>= 1) {
                const unsigned long long o = __shfl_xor_sync(0xffffffffu, best, off);
                best = o < best ? o : best;
            }
            if (best == ~0ull) break;  // every lane exhausted
            const int src = __ffs(__ballot_sync(0xffffffffu, key == best)) - 1;
            const float s_sig = __shfl_sync(0xffffffffu, h < m ? ls[h] : 0.0f, src);
            const float s_g = __shfl_sync(0xffffffffu, h < m ? lg[h] : 0.0f, src);
            const uint32_t s_mem = __shfl_sync(0xffffffffu, h < m ? lm[h] : 0u, src);
            if (lane == src) ++h;
            last_t = __uint_as_float((uint32_t)(best >> 32));
            last_id = (uint32_t)best;
            ++taken;
            if (!emit(last_t, last_id, s_sig, s_g, s_mem)) return;
        }
        // fewer than a full batch above the watermark: the list is exhausted
        if (taken < kFbBatch) return;
        wt = last_t;
        wid = last_id;
        have_w = true;
    }
}

/// One list pass per pixel: the lanes evaluate 32 list entries at a time and
/// the contributing ones enter a (t, id)-sorted ring of kFbRing entries in
/// this warp's shared memory, in list order; the ring head is emitted once it
/// is below the order bound of the next list entry (the blends' invariant:
/// every later entry has t >= that bound).  O(list length) instead of one pass
/// per batch.  If the ring fills, the walk continues exactly from the last
/// emitted contribution with warp_ordered_walk.
constexpr int kFbRing = 256;
struct FbRing {
    float t[kFbRing], s[kFbRing], g[kFbRing];
    uint32_t id[kFbRing], mem[kFbRing];
};

template <class Bound, class Eval, class Emit>
__device__ __forceinline__ void warp_ring_walk(float pxf, float pyf, uint2 rg, const uint32_t* __restrict__ pair_val,
                                               const SplatRec* __restrict__ recs, const float2* __restrict__ ext,
                                               FbRing& ring, Bound bound, Eval eval, Emit emit) {
    const int lane = threadIdx.x & 31;
    __syncwarp();  // the previous pixel's last pops read the ring this walk rewrites
    int head = 0, cnt = 0;  // warp-uniform
    bool have_last = false;
    float last_t = 0.0f;
    uint32_t last_id = 0;
    auto pop = [&]() -> bool {  // emit the ring head on every lane
        const int h = head & (kFbRing - 1);
        const float t = ring.t[h], s = ring.s[h], g = ring.g[h];
        const uint32_t id = ring.id[h], mem = ring.mem[h];
        ++head;
        --cnt;
        have_last = true;
        last_t = t;
        last_id = id;
        return emit(t, id, s, g, mem);
    };
    for (uint32_t c0 = rg.x; c0 < rg.y; c0 += 32) {
        const uint32_t p = c0 + lane;
        bool hit = false;
        float t = 0.0f, sg = 0.0f, g = 0.0f, bnd = 0.0f;
        uint32_t id = 0, mem = 0;
        if (p < rg.y) {
            mem = pair_val[p];
            const float4* r4 = reinterpret_cast<const float4*>(recs + mem);
            const float4 A0 = __ldg(r4), D0 = __ldg(r4 + 3);
            bnd = bound(D0.w);  // lower bound on t for this entry and every later one
            const float2 e = __ldg(ext + mem);
            if (!(fsub(pxf, A0.x) > e.x || fsub(A0.x, pxf) > e.x || fsub(pyf, A0.y) > e.y || fsub(A0.y, pyf) > e.y))
                hit = eval(mem, t, sg, g, id);
        }
        const unsigned hits = __ballot_sync(0xffffffffu, hit);
        const int nj = (int)min(32u, rg.y - c0);
        for (int j = 0; j < nj; ++j) {
            const float bj = __shfl_sync(0xffffffffu, bnd, j);
            while (cnt > 0 && ring.t[head & (kFbRing - 1)] < bj)
                if (!pop()) return;
            if (!((hits >> j) & 1u)) continue;
            const float tj = __shfl_sync(0xffffffffu, t, j), sj = __shfl_sync(0xffffffffu, sg, j);
            const float gj = __shfl_sync(0xffffffffu, g, j);
            const uint32_t idj = __shfl_sync(0xffffffffu, id, j), mj = __shfl_sync(0xffffffffu, mem, j);
            if (cnt == kFbRing) {  // full: continue exactly after the last emitted contribution
                warp_ordered_walk(pxf, pyf, rg, pair_val, recs, ext, eval, emit, have_last, last_t, last_id);
                return;
            }
            // insertion into the sorted ring (lane 0 writes; the warp reads after the sync).
            // The head test and pop() above read ring slots on every lane: order those
            // reads before lane 0's shifts (shuffles/ballots are not memory fences).
            int pos = head + cnt;
            __syncwarp();
            if (lane == 0) {
                while (pos > head) {
                    const int pl = (pos - 1) & (kFbRing - 1);
                    const float tp = ring.t[pl];
                    const uint32_t ip = ring.id[pl];
                    if (!(tj < tp || (tj == tp && idj < ip))) break;
                    const int ps = pos & (kFbRing - 1);
                    ring.t[ps] = tp;
                    ring.id[ps] = ip;
                    ring.s[ps] = ring.s[pl];
                    ring.g[ps] = ring.g[pl];
                    ring.mem[ps] = ring.mem[pl];
                    --pos;
                }
                const int ps = pos & (kFbRing - 1);
                ring.t[ps] = tj;
                ring.id[ps] = idj;
                ring.s[ps] = sj;
                ring.g[ps] = gj;
                ring.mem[ps] = mj;
            }
            __syncwarp();
            ++cnt;
        }
    }
    while (cnt > 0)
        if (!pop()) return;
}

}  // namespace dgs_b200
