// Exact k-nearest-neighbour mean distance for init_from_pointcloud
// (trainer.hpp:65-80: mean distance to the 3 nearest sampled neighbours,
// brute force O(N^2) on the CPU in the reference).
//
// Uniform grid (cell ~ 2 points on average), points sorted by cell (CUB radix
// sort of the cell keys), per-cell [start, end); one thread per point visits
// Chebyshev shells of cells around its own and keeps the k smallest squared
// distances, computed exactly as the reference ((c_j - c_i).squaredNorm() in
// float, the Eigen shim's order).  It stops once every point of the next shell
// is provably farther than the current k-th best: the next shell lies at least
// r cell widths away along some axis.  The k values are therefore the
// reference's k smallest squared distances, bit for bit; their square roots
// are summed in ascending order (the reference sums them in std::nth_element's
// unspecified order, so the mean can differ by an ulp).
#include <cub/cub.cuh>

#include "kernels.h"

namespace dgs_b200 {

namespace {

struct Grid {
    float lo[3];
    float inv_h, h;
    int dim[3];
};

__device__ __forceinline__ int cell_coord(float x, float lo, float inv_h, int dim) {
    int c = (int)floorf((x - lo) * inv_h);
    return c < 0 ? 0 : (c >= dim ? dim - 1 : c);
}

__global__ void k_cell_keys(int n, const float* __restrict__ pts, Grid g, uint32_t* __restrict__ keys,
                            uint32_t* __restrict__ vals) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int cx = cell_coord(pts[3 * i], g.lo[0], g.inv_h, g.dim[0]);
    const int cy = cell_coord(pts[3 * i + 1], g.lo[1], g.inv_h, g.dim[1]);
    const int cz = cell_coord(pts[3 * i + 2], g.lo[2], g.inv_h, g.dim[2]);
    keys[i] = ((uint32_t)cz * g.dim[1] + cy) * g.dim[0] + cx;
    vals[i] = (uint32_t)i;
}

__global__ void k_cell_ranges(int n, const uint32_t* __restrict__ keys, uint32_t* __restrict__ start,
                              uint32_t* __restrict__ end) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const uint32_t c = keys[j];
    if (j == 0 || keys[j - 1] != c) start[c] = j;
    if (j == n - 1 || keys[j + 1] != c) end[c] = j + 1;
}

/// Sorted point copy (cell order) for coalesced shell scans.
__global__ void k_gather_points(int n, const float* __restrict__ pts, const uint32_t* __restrict__ order,
                                float4* __restrict__ sorted) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const uint32_t i = order[j];
    sorted[j] = make_float4(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], __uint_as_float(i));
}

template <int KNN>
__global__ void __launch_bounds__(256) k_knn_mean(int n, int k_nn, const float4* __restrict__ sorted, Grid g,
                                                  const uint32_t* __restrict__ start, const uint32_t* __restrict__ end,
                                                  float* __restrict__ out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const float4 p = sorted[j];
    const uint32_t self = __float_as_uint(p.w);
    const int cx = cell_coord(p.x, g.lo[0], g.inv_h, g.dim[0]);
    const int cy = cell_coord(p.y, g.lo[1], g.inv_h, g.dim[1]);
    const int cz = cell_coord(p.z, g.lo[2], g.inv_h, g.dim[2]);
    float best[KNN];
#pragma unroll
    for (int q = 0; q < KNN; ++q) best[q] = __int_as_float(0x7f800000);
    const int rmax = max(g.dim[0], max(g.dim[1], g.dim[2]));
    for (int r = 0; r <= rmax; ++r) {
        // every point of shell r + 1 is >= r * h away: stop once the k-th best is provably closer
        if (r > 0) {
            const float reach = (float)(r - 1) * g.h;
            if (best[k_nn - 1] < reach * reach * (1.0f - 1e-5f)) break;
        }
        for (int dz = -r; dz <= r; ++dz) {
            const int z = cz + dz;
            if (z < 0 || z >= g.dim[2]) continue;
            for (int dy = -r; dy <= r; ++dy) {
                const int y = cy + dy;
                if (y < 0 || y >= g.dim[1]) continue;
                const bool face = abs(dz) == r || abs(dy) == r;
                for (int dx = -r; dx <= r; dx += (face ? 1 : 2 * r)) {
                    const int x = cx + dx;
                    if (x >= 0 && x < g.dim[0]) {
                        const uint32_t c = ((uint32_t)z * g.dim[1] + y) * g.dim[0] + x;
                        const uint32_t e = end[c];
                        for (uint32_t q = start[c]; q < e; ++q) {
                            const float4 o = sorted[q];
                            if (__float_as_uint(o.w) == self) continue;
                            // (c_j - c_i).squaredNorm() in the shim's order: x^2 + (y^2 + z^2)
                            const float ex = fsub(o.x, p.x), ey = fsub(o.y, p.y), ez = fsub(o.z, p.z);
                            const float d2 = dot3(ex, ey, ez, ex, ey, ez);
                            if (d2 < best[KNN - 1]) {
                                int s = KNN - 1;
                                while (s > 0 && best[s - 1] > d2) {
                                    best[s] = best[s - 1];
                                    --s;
                                }
                                best[s] = d2;
                            }
                        }
                    }
                    if (r == 0) break;
                }
            }
        }
    }
    float acc = 0.0f;
    for (int q = 0; q < k_nn; ++q) acc = fadd(acc, fsqrt(best[q]));
    out[self] = fdiv(acc, (float)k_nn);
}

}  // namespace

void knn_mean_distance(int n, int k_nn, const float* d_pts, float* d_out, const float lo[3], const float hi[3],
                       cudaStream_t s) {
    if (n <= 0 || k_nn <= 0) return;
    Grid g;
    double vol = 1.0;
    float ext[3];
    for (int a = 0; a < 3; ++a) {
        ext[a] = std::max(hi[a] - lo[a], 1e-30f);
        vol *= ext[a];
    }
    // ~2 points per cell, at most ~4n cells
    double h = std::cbrt(vol * 2.0 / n);
    for (int a = 0; a < 3; ++a) h = std::max(h, (double)ext[a] / 1024.0);
    for (int it = 0; it < 64; ++it) {
        double cells = 1.0;
        for (int a = 0; a < 3; ++a) cells *= std::max(1.0, std::ceil(ext[a] / h));
        if (cells <= 4.0 * n + 64) break;
        h *= 1.25;
    }
    g.h = (float)h;
    g.inv_h = (float)(1.0 / h);
    for (int a = 0; a < 3; ++a) {
        g.lo[a] = lo[a];
        g.dim[a] = std::max(1, (int)std::ceil(ext[a] / h));
    }
    const size_t ncell = (size_t)g.dim[0] * g.dim[1] * g.dim[2];
    uint32_t *keys, *keys_alt, *vals, *vals_alt, *cs, *ce;
    float4* sorted;
    void* temp = nullptr;
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (uint32_t*)nullptr, n);
    cudaMallocAsync(&keys, 4 * (size_t)n, s);
    cudaMallocAsync(&keys_alt, 4 * (size_t)n, s);
    cudaMallocAsync(&vals, 4 * (size_t)n, s);
    cudaMallocAsync(&vals_alt, 4 * (size_t)n, s);
    cudaMallocAsync(&cs, 4 * ncell, s);
    cudaMallocAsync(&ce, 4 * ncell, s);
    cudaMallocAsync(&sorted, 16 * (size_t)n, s);
    cudaMallocAsync(&temp, tb, s);
    cudaMemsetAsync(cs, 0, 4 * ncell, s);
    cudaMemsetAsync(ce, 0, 4 * ncell, s);
    const unsigned grid = (unsigned)((n + 255) / 256);
    k_cell_keys<<<grid, 256, 0, s>>>(n, d_pts, g, keys, vals);
    int bits = 1;
    while ((1ull << bits) < ncell && bits < 32) ++bits;
    cub::DeviceRadixSort::SortPairs(temp, tb, keys, keys_alt, vals, vals_alt, n, 0, bits, s);
    k_cell_ranges<<<grid, 256, 0, s>>>(n, keys_alt, cs, ce);
    k_gather_points<<<grid, 256, 0, s>>>(n, d_pts, vals_alt, sorted);
    if (k_nn <= 3) k_knn_mean<3><<<grid, 256, 0, s>>>(n, k_nn, sorted, g, cs, ce, d_out);
    for (void* p : {(void*)keys, (void*)keys_alt, (void*)vals, (void*)vals_alt, (void*)cs, (void*)ce, (void*)sorted,
                    temp})
        cudaFreeAsync(p, s);
}

}  // namespace dgs_b200
