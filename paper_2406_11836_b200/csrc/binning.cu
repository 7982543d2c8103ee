// K2 — (splat, tile) pair emission in range order + stable tile sort + tile
// ranges.  Replaces the reference's serial per-tile vector push
// (raster.hpp:113-125).  The reference's per-tile lists are in projected
// order and re-sorted per pixel by the ray parameter t (raster.hpp:164-166);
// here each tile list is ordered by the range r = ||mu - o|| so the blend
// kernels can restore the exact (t, id) order with a small per-pixel reorder
// buffer (t_j >= sqrt(r_j^2 - D_j^2) for every contributor).
//
// Sort strategy: one 32-bit radix sort of the members by range (N keys), then
// a stable radix sort of the emitted pairs by tile id only (ceil(log2 tiles)
// bits, two 8-bit passes at 1080p) — cheaper than a 45-bit (tile, range) key
// sort over all P pairs.
#include <cub/cub.cuh>

#include "kernels.h"

namespace dgs_b200 {

namespace {

/// 16-bit sort key: the range bucket (dgs_types.cuh range_key_shift; culled
/// members take the top key and emit nothing), plus the identity values.
__global__ void k_key16(const uint32_t* __restrict__ rkey, const uint32_t* __restrict__ dmax_bits,
                        uint32_t* __restrict__ key, uint32_t* __restrict__ vals, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t b = rkey[i], lo = dmax_bits[1];
    const int sh = range_key_shift(lo, dmax_bits[3]);
    key[i] = (b == 0xffffffffu || b < lo) ? kRangeKeyMax : min((b - lo) >> sh, kRangeKeyMax);
    vals[i] = (uint32_t)i;
}

/// camera_z_order: exact 32-bit keys (positive depths order like their bits;
/// culled members take the top key).  The stable sort keeps member order on
/// equal depths; the blends break those ties by id.
__global__ void k_key32(const uint32_t* __restrict__ rkey, uint32_t* __restrict__ key, uint32_t* __restrict__ vals,
                        int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    key[i] = rkey[i];
    vals[i] = (uint32_t)i;
}

/// Members in range order: their tile rectangle and tile count (the count is
/// derived from the rectangle; culled members carry an empty one).  One random
/// 8-byte gather per member; the scan and the emission then stream.
__global__ void k_gather_sorted_rects(const uint32_t* __restrict__ sorted_idx, const uint2* __restrict__ rect,
                                      uint2* __restrict__ rect_sorted, uint32_t* __restrict__ cnt_sorted, int n) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const uint2 r = rect[sorted_idx[j]];
    const uint32_t x0 = r.x & 0xffffu, x1 = r.x >> 16, y0 = r.y & 0xffffu, y1 = r.y >> 16;
    rect_sorted[j] = r;
    cnt_sorted[j] = (x1 >= x0 && y1 >= y0) ? (x1 - x0 + 1) * (y1 - y0 + 1) : 0u;
}


/// Pair emission, warp-cooperative: the warp's 32 members (in range order)
/// own a contiguous run of output slots; lane l writes slots l, l+32, ...
/// of that run, finding its member by a search over the warp's prefix sums,
/// so every store instruction writes 32 consecutive words.
__global__ void k_emit_pairs(const uint32_t* __restrict__ sorted_idx, const uint32_t* __restrict__ offsets,
                             const uint32_t* __restrict__ cnt_sorted, const uint2* __restrict__ rect_sorted,
                             int tiles_x, int n, uint16_t* __restrict__ pair_tile, uint32_t* __restrict__ pair_val,
                             uint32_t cap, int* __restrict__ abort) {
    // cap / abort (graph-captured steps, the pair count is not read back): slots
    // beyond the capacity are dropped and the step's abort flag is raised
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    if (abort != nullptr && j == 0 && offsets[n - 1] > cap) atomicOr(abort, 2);
    uint32_t i = 0, c = 0, off = 0, x0 = 0, w = 1, y0 = 0;
    if (j < n) {
        i = sorted_idx[j];
        c = cnt_sorted[j];
        off = offsets[j];
        if (c) {
            const uint2 r = rect_sorted[j];
            x0 = r.x & 0xffff;
            w = (r.x >> 16) - x0 + 1;
            y0 = r.y & 0xffff;
        }
    }
    // inclusive prefix of counts within the warp
    uint32_t inc = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += t;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
    // offsets[] holds inclusive ends: lane 0's start is its end minus its count
    const uint32_t base = __shfl_sync(0xffffffffu, off - c, 0);
    for (uint32_t q0 = 0; q0 < total; q0 += 32) {
        const uint32_t q = q0 + lane;
        // owner lane: first lane whose inclusive prefix exceeds q
        int lo = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
            const uint32_t v = __shfl_sync(0xffffffffu, inc, lo + step - 1);
            if (v <= q) lo += step;
        }
        const uint32_t ex = __shfl_sync(0xffffffffu, inc - c, lo);
        const uint32_t mi = __shfl_sync(0xffffffffu, i, lo);
        const uint32_t mx0 = __shfl_sync(0xffffffffu, x0, lo);
        const uint32_t mw = __shfl_sync(0xffffffffu, w, lo);
        const uint32_t my0 = __shfl_sync(0xffffffffu, y0, lo);
        if (q < total && base + q < cap) {
            const uint32_t r = q - ex;
            // r / mw by a float reciprocal: (r + 0.5) / mw <= tiles_y stays >= 0.5 / mw away from
            // an integer, far beyond the float error (r, mw < 2^16)
            const uint32_t dy = (uint32_t)(((float)r + 0.5f) * __frcp_rn((float)mw));
            const uint32_t ty = my0 + dy, tx = mx0 + (r - dy * mw);
            pair_tile[base + q] = (uint16_t)(ty * (uint32_t)tiles_x + tx);
            pair_val[base + q] = mi;
        }
    }
}

__device__ __forceinline__ uint32_t lower_bound_u16(const uint16_t* __restrict__ a, uint32_t n, uint32_t key) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

/// Longest lists first: the blends take tiles in this order, so the long
/// tiles start in the first waves instead of setting the kernel's tail.  One
/// CTA: tiles are bucketed by list length on a half-octave scale (64 buckets,
/// longest first), the order within a bucket is arbitrary (scheduling only:
/// every tile's work is independent of the block order).
__global__ void __launch_bounds__(1024) k_tile_order(const uint2* __restrict__ ranges, int tiles,
                                                     uint32_t* __restrict__ order) {
    __shared__ uint32_t cnt[64], start[64];
    const int tid = threadIdx.x;
    if (tid < 64) cnt[tid] = 0;
    __syncthreads();
    auto bucket = [](uint32_t len) -> uint32_t {  // 63 = longest
        if (len == 0) return 0;
        const uint32_t lg = 31u - __clz(len);
        const uint32_t half = lg > 0 ? (len >> (lg - 1)) & 1u : 0u;
        return min(2u * lg + half + 1u, 63u);
    };
    for (int t = tid; t < tiles; t += blockDim.x) {
        const uint2 r = ranges[t];
        atomicAdd(&cnt[bucket(r.y - r.x)], 1u);
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t acc = 0;
        for (int b = 63; b >= 0; --b) {
            start[b] = acc;
            acc += cnt[b];
        }
    }
    __syncthreads();
    for (int t = tid; t < tiles; t += blockDim.x) {
        const uint2 r = ranges[t];
        order[atomicAdd(&start[bucket(r.y - r.x)], 1u)] = (uint32_t)t;
    }
}

/// Graph-captured steps sort a fixed capacity: the slots after the device-side
/// pair count get the tile key 0xffff, above every tile, so they sort last.
__global__ void k_pad_pairs(const uint32_t* __restrict__ P_dev, uint32_t cap, uint16_t* __restrict__ pair_tile) {
    const uint32_t P = min(*P_dev, cap);
    for (uint32_t q = P + blockIdx.x * blockDim.x + threadIdx.x; q < cap; q += gridDim.x * blockDim.x)
        pair_tile[q] = 0xffffu;
}

/// Per-tile [start, end) by binary search over the sorted tile keys (one thread per tile).
__global__ void k_tile_ranges(const uint16_t* __restrict__ tile, uint32_t P, int tiles, uint2* __restrict__ ranges) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= tiles) return;
    ranges[t] = make_uint2(lower_bound_u16(tile, P, (uint32_t)t), lower_bound_u16(tile, P, (uint32_t)t + 1));
}

/// Onesweep policy for the member sort, measured on B200
/// (scripts/sortbench.cu: 10M u32 keys + u32 values, 24-bit keys / 3 passes at
/// the time): 256 threads x 23 items 0.250 ms vs 0.313 ms for the library
/// default dispatch.  The keys are 16-bit range buckets now (2 passes).  The other
/// policies of the chain are the library's sm_100 ones (unused by onesweep).
struct MemberSortHub {
    using Base = cub::detail::radix::policy_hub<uint32_t, uint32_t, int>::Policy1000;
    struct Policy : cub::ChainedPolicy<1000, Policy, Policy> {
        static constexpr bool ONESWEEP = true;
        static constexpr int ONESWEEP_RADIX_BITS = 8;
        using HistogramPolicy = Base::HistogramPolicy;
        using ExclusiveSumPolicy = Base::ExclusiveSumPolicy;
        using OnesweepPolicy =
            cub::AgentRadixSortOnesweepPolicy<256, 23, uint32_t, 1, cub::RADIX_RANK_MATCH_EARLY_COUNTS_ANY,
                                              cub::BLOCK_SCAN_RAKING_MEMOIZE, cub::RADIX_SORT_STORE_DIRECT, 8>;
        using ScanPolicy = Base::ScanPolicy;
        using DownsweepPolicy = Base::DownsweepPolicy;
        using AltDownsweepPolicy = Base::AltDownsweepPolicy;
        using UpsweepPolicy = Base::UpsweepPolicy;
        using AltUpsweepPolicy = Base::AltUpsweepPolicy;
        using SingleTilePolicy = Base::SingleTilePolicy;
        using SegmentedPolicy = Base::SegmentedPolicy;
        using AltSegmentedPolicy = Base::AltSegmentedPolicy;
    };
    using MaxPolicy = Policy;
};
using MemberSort = cub::DispatchRadixSort<false, uint32_t, uint32_t, int, MemberSortHub>;


int bits_for(uint32_t v) {
    int b = 1;
    while ((1u << b) < v && b < 32) ++b;
    return b;
}

__global__ void k_zero16(uint4* __restrict__ p, size_t n16) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_uint4(0u, 0u, 0u, 0u);
}

__global__ void k_zero1(uint8_t* __restrict__ p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = 0;
}

}  // namespace

void launch_zero(void* p, size_t bytes, cudaStream_t s) {
    if (bytes == 0) return;
    const bool vec = (reinterpret_cast<uintptr_t>(p) & 15) == 0 && bytes % 16 == 0;
    const size_t n = vec ? bytes / 16 : bytes;
    const int grid = (int)std::min<size_t>((n + 255) / 256, (size_t)148 * 8);
    if (vec) k_zero16<<<grid, 256, 0, s>>>(static_cast<uint4*>(p), n);
    else k_zero1<<<grid, 256, 0, s>>>(static_cast<uint8_t*>(p), n);
}

size_t binning_temp_bytes(int n, int64_t pair_cap) {
    size_t a = 0, b = 0, c = 0;
    {
        cub::DoubleBuffer<uint32_t> k, v;
        MemberSort::Dispatch(nullptr, a, k, v, n, 0, kRangeKeyBits, true, 0);
        size_t a32 = 0;
        MemberSort::Dispatch(nullptr, a32, k, v, n, 0, 32, true, 0);
        if (a32 > a) a = a32;
    }
    cub::DoubleBuffer<uint16_t> dk;
    cub::DoubleBuffer<uint32_t> dv;
    cub::DeviceRadixSort::SortPairs(nullptr, b, dk, dv, (int)pair_cap, 0, 16);
    cub::DeviceScan::InclusiveSum(nullptr, c, (const uint32_t*)nullptr, (uint32_t*)nullptr, n);
    size_t m = a > b ? a : b;
    return (m > c ? m : c) + 256;
}

int64_t run_binning(int n, const ViewParams& vp, ViewBins& vb, int64_t cap, void* temp, size_t temp_bytes,
                    uint32_t* sort_keys_alt, uint32_t* sort_vals, uint32_t* sort_vals_alt, uint16_t* pair_tile_alt,
                    uint32_t* pair_val_alt, uint32_t* scan_buf, uint2* rect_sorted, uint32_t* pairs_host,
                    cudaStream_t s, int64_t pad_cap) {
    const int tiles = vp.tiles_x * vp.tiles_y;
    launch_zero(vb.ranges, sizeof(uint2) * tiles, s);
    vb.pairs = 0;
    // the blends' block order (tiles longest list first) is a permutation on every path
    auto tile_order = [&]() {
        if (vb.tile_order) k_tile_order<<<1, 1024, 0, s>>>(vb.ranges, tiles, vb.tile_order);
    };
    if (n <= 0) {
        tile_order();
        return 0;
    }
    const int blk = 256, grid = (n + blk - 1) / blk;
    // 1) members by range bucket: 16-bit keys (2 radix passes)
    if (vb.zorder) k_key32<<<grid, blk, 0, s>>>(vb.rkey, scan_buf, sort_vals, n);
    else k_key16<<<grid, blk, 0, s>>>(vb.rkey, vb.dmax_bits, scan_buf, sort_vals, n);
    size_t tb = temp_bytes;
    const uint32_t* sorted_idx;
    {
        cub::DoubleBuffer<uint32_t> k(scan_buf, sort_keys_alt), v(sort_vals, sort_vals_alt);
        MemberSort::Dispatch(temp, tb, k, v, n, 0, vb.zorder ? 32 : kRangeKeyBits, true, s);
        sorted_idx = v.Current();
    }
    // 2) tile counts in range order -> inclusive scan -> pair end offsets
    uint32_t* cnt_sorted = sort_keys_alt;  // the sorted keys are not needed after the sort
    k_gather_sorted_rects<<<grid, blk, 0, s>>>(sorted_idx, reinterpret_cast<const uint2*>(vb.rect), rect_sorted,
                                               cnt_sorted, n);
    tb = temp_bytes;
    cub::DeviceScan::InclusiveSum(temp, tb, cnt_sorted, scan_buf, n, s);
    if (pad_cap > 0) {
        // graph-captured step: no readback; the pair count stays on the device
        // (scan_buf[n-1]) and the tile sort runs over pad_cap slots, the tail padded
        // with key 0xffff (sorted last, never inside a tile range); a count above
        // pad_cap raises the step's abort flag (the caller re-runs the step)
        const uint32_t pc = (uint32_t)pad_cap;
        k_emit_pairs<<<grid, blk, 0, s>>>(sorted_idx, scan_buf, cnt_sorted, rect_sorted, vp.tiles_x, n, vb.pair_tile,
                                          vb.pair_val, pc, vb.abort);
        k_pad_pairs<<<148 * 4, 256, 0, s>>>(scan_buf + (n - 1), pc, vb.pair_tile);
        cub::DoubleBuffer<uint16_t> dk(vb.pair_tile, pair_tile_alt);
        cub::DoubleBuffer<uint32_t> dv(vb.pair_val, pair_val_alt);
        tb = temp_bytes;
        cub::DeviceRadixSort::SortPairs(temp, tb, dk, dv, (int)pc, 0, 16, s);
        if (dk.Current() != vb.pair_tile) {
            cudaMemcpyAsync(vb.pair_tile, dk.Current(), 2 * (size_t)pc, cudaMemcpyDeviceToDevice, s);
            cudaMemcpyAsync(vb.pair_val, dv.Current(), 4 * (size_t)pc, cudaMemcpyDeviceToDevice, s);
        }
        k_tile_ranges<<<(unsigned)((tiles + 255) / 256), 256, 0, s>>>(vb.pair_tile, pc, tiles, vb.ranges);
        tile_order();
        vb.pairs = -1;  // known after the replay (scan_buf[n-1])
        return pad_cap;
    }
    // the one host round trip of the step's forward: the pair count sizes the
    // tile sort (pinned readback; the caller's pending readbacks ride along)
    cudaMemcpyAsync(pairs_host, scan_buf + (n - 1), 4, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    const int64_t P = (int64_t)*pairs_host;
    if (P > cap) return -P;
    vb.pairs = P;
    if (P == 0) {
        tile_order();
        return 0;
    }
    // 3) emit (tile, member) pairs, range-ordered within every tile
    k_emit_pairs<<<grid, blk, 0, s>>>(sorted_idx, scan_buf, cnt_sorted, rect_sorted, vp.tiles_x, n, vb.pair_tile,
                                      vb.pair_val, 0xffffffffu, nullptr);  // scan_buf: inclusive ends
    // 4) stable LSD radix sort by tile id only
    cub::DoubleBuffer<uint16_t> dk(vb.pair_tile, pair_tile_alt);
    cub::DoubleBuffer<uint32_t> dv(vb.pair_val, pair_val_alt);
    tb = temp_bytes;
    cub::DeviceRadixSort::SortPairs(temp, tb, dk, dv, (int)P, 0, bits_for((uint32_t)tiles), s);
    if (dk.Current() != vb.pair_tile) {
        cudaMemcpyAsync(vb.pair_tile, dk.Current(), 2 * (size_t)P, cudaMemcpyDeviceToDevice, s);
        cudaMemcpyAsync(vb.pair_val, dv.Current(), 4 * (size_t)P, cudaMemcpyDeviceToDevice, s);
    }
    // 5) per-tile [start, end)
    k_tile_ranges<<<(unsigned)((tiles + 255) / 256), 256, 0, s>>>(vb.pair_tile, (uint32_t)P, tiles, vb.ranges);
    // 6) block order for the blends: tiles by decreasing list length
    tile_order();
    return P;
}

}  // namespace dgs_b200
