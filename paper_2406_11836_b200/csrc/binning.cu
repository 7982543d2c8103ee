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

__global__ void k_iota(uint32_t* v, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = (uint32_t)i;
}

__global__ void k_gather_counts(const uint32_t* __restrict__ sorted_idx, const uint32_t* __restrict__ counts,
                                uint32_t* __restrict__ out, int n) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n) out[j] = counts[sorted_idx[j]];
}

__global__ void k_emit_pairs(const uint32_t* __restrict__ sorted_idx, const uint32_t* __restrict__ offsets,
                             const uint32_t* __restrict__ counts, const uint32_t* __restrict__ rect, int tiles_x,
                             int n, uint32_t* __restrict__ pair_tile, uint32_t* __restrict__ pair_val) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const uint32_t i = sorted_idx[j];
    if (counts[i] == 0) return;
    const uint32_t rx = rect[2 * (size_t)i], ry = rect[2 * (size_t)i + 1];
    const int x0 = rx & 0xffff, x1 = rx >> 16, y0 = ry & 0xffff, y1 = ry >> 16;
    uint32_t o = offsets[j];
    for (int ty = y0; ty <= y1; ++ty)
        for (int tx = x0; tx <= x1; ++tx) {
            pair_tile[o] = (uint32_t)(ty * tiles_x + tx);
            pair_val[o] = i;
            ++o;
        }
}

__global__ void k_tile_ranges(const uint32_t* __restrict__ tile, int64_t P, uint2* __restrict__ ranges) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    const uint32_t t = tile[p];
    if (p == 0 || tile[p - 1] != t) ranges[t].x = (uint32_t)p;
    if (p == P - 1 || tile[p + 1] != t) ranges[t].y = (uint32_t)(p + 1);
}

int bits_for(uint32_t v) {
    int b = 1;
    while ((1u << b) < v && b < 32) ++b;
    return b;
}

}  // namespace

size_t binning_temp_bytes(int n, int64_t pair_cap) {
    size_t a = 0, b = 0, c = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (uint32_t*)nullptr, n);
    cub::DoubleBuffer<uint32_t> dk, dv;
    cub::DeviceRadixSort::SortPairs(nullptr, b, dk, dv, (int)pair_cap, 0, 32);
    cub::DeviceScan::ExclusiveSum(nullptr, c, (uint32_t*)nullptr, (uint32_t*)nullptr, n);
    size_t m = a > b ? a : b;
    return (m > c ? m : c) + 256;
}

int64_t run_binning(int n, const ViewParams& vp, ViewBins& vb, int64_t cap, void* temp, size_t temp_bytes,
                    uint32_t* sort_keys_alt, uint32_t* sort_vals, uint32_t* sort_vals_alt, uint32_t* pair_tile_alt,
                    uint32_t* pair_val_alt, uint32_t* scan_buf, cudaStream_t s) {
    const int tiles = vp.tiles_x * vp.tiles_y;
    cudaMemsetAsync(vb.ranges, 0, sizeof(uint2) * tiles, s);
    vb.pairs = 0;
    if (n <= 0) return 0;
    const int blk = 256, grid = (n + blk - 1) / blk;
    k_iota<<<grid, blk, 0, s>>>(sort_vals, n);
    size_t tb = temp_bytes;
    // 1) members by range (culled members carry 0xffffffff and sort last)
    cub::DeviceRadixSort::SortPairs(temp, tb, vb.rkey, sort_keys_alt, sort_vals, sort_vals_alt, n, 0, 32, s);
    // 2) tile counts in range order -> exclusive scan -> pair offsets
    k_gather_counts<<<grid, blk, 0, s>>>(sort_vals_alt, vb.counts, sort_keys_alt, n);
    tb = temp_bytes;
    cub::DeviceScan::ExclusiveSum(temp, tb, sort_keys_alt, scan_buf, n, s);
    uint32_t last_off = 0, last_cnt = 0;
    cudaMemcpyAsync(&last_off, scan_buf + (n - 1), 4, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(&last_cnt, sort_keys_alt + (n - 1), 4, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    const int64_t P = (int64_t)last_off + last_cnt;
    if (P > cap) return -P;
    vb.pairs = P;
    if (P == 0) return 0;
    // 3) emit (tile, member) pairs, range-ordered within every tile
    k_emit_pairs<<<grid, blk, 0, s>>>(sort_vals_alt, scan_buf, vb.counts, vb.rect, vp.tiles_x, n, vb.pair_tile,
                                      vb.pair_val);
    // 4) stable LSD radix sort by tile id only
    cub::DoubleBuffer<uint32_t> dk(vb.pair_tile, pair_tile_alt), dv(vb.pair_val, pair_val_alt);
    tb = temp_bytes;
    cub::DeviceRadixSort::SortPairs(temp, tb, dk, dv, (int)P, 0, bits_for((uint32_t)tiles), s);
    if (dk.Current() != vb.pair_tile) {
        cudaMemcpyAsync(vb.pair_tile, dk.Current(), 4 * (size_t)P, cudaMemcpyDeviceToDevice, s);
        cudaMemcpyAsync(vb.pair_val, dv.Current(), 4 * (size_t)P, cudaMemcpyDeviceToDevice, s);
    }
    // 5) per-tile [start, end)
    k_tile_ranges<<<(unsigned)((P + 255) / 256), 256, 0, s>>>(vb.pair_tile, P, vb.ranges);
    return P;
}

}  // namespace dgs_b200
