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
                                                  Eval eval, Emit emit) {
    const int lane = threadIdx.x & 31;
    float wt = -__builtin_huge_valf();
    uint32_t wid = 0;
    bool have_w = false;
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

}  // namespace dgs_b200
