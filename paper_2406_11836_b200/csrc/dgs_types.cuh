// Device data model shared by the kernels and the C-ABI layer.
//
// Parameters of one KD subset live in HBM as SoA rows of N floats
// (kParamRows = 59 for SH degree 3): row r at P + r*ld.  Optimizer moments
// m, v and the multi-view gradient accumulator use the same layout.  The
// projection kernel writes one 64-byte SplatRec per member (gathered by the
// blend kernels through the sorted (tile, range) pair list).
#pragma once

#include <stdint.h>

#include "dgs_math.cuh"

namespace dgs_b200 {

// Parameter rows (splat.hpp:17-38 field order).
constexpr int kRowMu = 0;         // 3 rows
constexpr int kRowLogScale = 3;   // 3 rows
constexpr int kRowRot = 6;        // 4 rows (w, x, y, z)
constexpr int kRowOpacity = 10;   // 1 row
constexpr int kRowSh = 11;        // (deg+1)^2 * 3 rows, coefficient-major then channel
constexpr int kMaxShCoeffs = 16;
constexpr int kMaxParamRows = kRowSh + 3 * kMaxShCoeffs;  // 59

inline int param_rows(int sh_coeffs) { return kRowSh + 3 * sh_coeffs; }

constexpr int kTileSize = 16;        // raster.hpp:78
constexpr int kBlendThreads = 256;   // one thread per tile pixel
constexpr int kMaxPlanes = 8;        // per subspace (KD depth <= 8)
constexpr int kMaxSubsets = 32;

/// Per-member projected record (raster.hpp:76-127 / splat.hpp:102-113).
struct __align__(16) SplatRec {
    float mx, my, alpha, d2;     // mean2d, sigmoid(opacity_logit), world_radius^2
    float i00, i01, i10, i11;    // inv_cov2d (full 2x2: the reference's is not exactly symmetric)
    float mux, muy, muz;         // mu_world
    uint32_t id;                 // splat id (tie-break key; ids < 2^32 enforced at load)
    float cr, cg, cb;            // SH colour
    float range;                 // ||mu - o|| (sort key and order bound)
};

/// RenderOptions (splat.hpp:118-127) as float, the way the reference's
/// T(opts.x) casts evaluate them.
struct RenderOpts {
    float trunc;        // truncation_radius
    float near_plane;
    float sigma_clamp;
    float cov_reg;
    float stop;         // stop_threshold (0 disables early termination)
    int sh_degree;      // -1: stored degree
    int indicator_enabled;
    float grad_skip_eps;  // render_maps_backward skip rule: |gc|<=eps (isZero) && gT==0
    int zorder;           // camera_z_order (splat.hpp:126): order by camera depth, ties by id
};

/// One subspace's half-space list (partition.hpp:19-41).
struct Subspace {
    int n;
    float nx[kMaxPlanes], ny[kMaxPlanes], nz[kMaxPlanes], d[kMaxPlanes];
    int closed[kMaxPlanes];
};

/// Partition table (all subsets), small enough for kernel parameters.
struct Table {
    int k_count;
    Subspace sub[kMaxSubsets];
};

/// partition.hpp:25-28 HalfSpace::contains, partition.hpp:58-63 indicator.
DGS_HD bool subspace_contains(const Subspace& s, float x0, float x1, float x2) {
    for (int p = 0; p < s.n; ++p) {
        const float v = fadd(dot3(s.nx[p], s.ny[p], s.nz[p], x0, x1, x2), s.d[p]);
        if (s.closed[p] ? !(v <= 0.0f) : !(v < 0.0f)) return false;
    }
    return true;
}

/// partition.hpp:265-300 subspace_order for one ray: writes the traversal
/// order (owner subspace first, then t_enter, then k) and returns its length.
DGS_HD int subspace_order(const Table& tb, int owner, const float o[3], const float d[3], uint16_t* order) {
    const float inf = u2f(0x7f800000u);
    int cnt = 0;
    float te[kMaxSubsets];
    int ks[kMaxSubsets];
    for (int k = 0; k < tb.k_count; ++k) {
        const Subspace& s = tb.sub[k];
        float t_lo = -inf, t_hi = inf;
        bool empty = false;
        for (int p = 0; p < s.n; ++p) {
            const float a = dot3(s.nx[p], s.ny[p], s.nz[p], d[0], d[1], d[2]);
            const float b = fadd(dot3(s.nx[p], s.ny[p], s.nz[p], o[0], o[1], o[2]), s.d[p]);
            if (a == 0.0f) {
                if (b > 0.0f) {
                    empty = true;
                    break;
                }
            } else {
                const float tstar = fdiv(-b, a);
                if (a > 0.0f) t_hi = (tstar < t_hi) ? tstar : t_hi;   // std::min
                else t_lo = (t_lo < tstar) ? tstar : t_lo;            // std::max
            }
        }
        if (empty || t_lo > t_hi || !(t_hi > 0.0f)) continue;
        const float tent = (t_lo < 0.0f) ? 0.0f : t_lo;              // std::max(t_lo, 0)
        // insertion in comparator order: owner first, then (t_enter, k)
        int pos = cnt;
        while (pos > 0) {
            const int kp = ks[pos - 1];
            const bool new_owner = (k == owner), prev_owner = (kp == owner);
            bool less;
            if (new_owner != prev_owner) less = new_owner;
            else less = tent < te[pos - 1] || (tent == te[pos - 1] && k < kp);
            if (!less) break;
            te[pos] = te[pos - 1];
            ks[pos] = ks[pos - 1];
            --pos;
        }
        te[pos] = tent;
        ks[pos] = k;
        ++cnt;
    }
    for (int i = 0; i < cnt; ++i) order[i] = (uint16_t)ks[i];
    return cnt;
}

#if defined(__CUDACC__)
/// Pixel <-> thread mapping inside a 16x16 tile (all blend kernels and the
/// composite records): warp w covers the 8x4 pixel block (w & 1, w >> 1),
/// lane l the pixel (l & 7, l >> 3) inside it.
__device__ __forceinline__ void tile_pixel(int tid, int tx, int ty, int& px, int& py) {
    const int w = tid >> 5, l = tid & 31;
    px = tx * kTileSize + (w & 1) * 8 + (l & 7);
    py = ty * kTileSize + (w >> 1) * 4 + (l >> 3);
}

/// 8-bit mask of the warps of tile (tx, ty) whose 8x4 block may contain a
/// pixel with m^2 <= trunc^2 for a splat at (mx, my) with half-extents ext
/// (K1's conservative bound on the float dx, dy of eval_2d).  A block is
/// skipped only if the float dx (dy) of its nearest pixel column (row) already
/// exceeds the extent: fsub is monotone, so every other column (row) does too.
__device__ __forceinline__ uint32_t warp_block_mask(float2 ext, float mx, float my, int tx, int ty) {
    uint32_t cm = 0, rm = 0;
#pragma unroll
    for (int bx = 0; bx < 2; ++bx) {
        const float lo = fadd((float)(tx * kTileSize + bx * 8), 0.5f);
        const float hi = fadd((float)(tx * kTileSize + bx * 8 + 7), 0.5f);
        if (!(fsub(lo, mx) > ext.x || fsub(mx, hi) > ext.x)) cm |= 1u << bx;
    }
#pragma unroll
    for (int by = 0; by < 4; ++by) {
        const float lo = fadd((float)(ty * kTileSize + by * 4), 0.5f);
        const float hi = fadd((float)(ty * kTileSize + by * 4 + 3), 0.5f);
        if (!(fsub(lo, my) > ext.y || fsub(my, hi) > ext.y)) rm |= 1u << by;
    }
    uint32_t m = 0;
#pragma unroll
    for (int by = 0; by < 4; ++by)
        if ((rm >> by) & 1u) m |= cm << (2 * by);
    return m;
}
#endif

#if defined(__CUDACC__)
/// Member sort keys (binning.cu): the range's float bits above the view's
/// minimum visible range (lo), in 16-bit buckets of 2^shift ulps, shift sized
/// by the maximum visible range (hi).  Tile lists are ordered by bucket; the
/// blends bound every later entry by the lower edge of the current bucket.
#ifndef DGS_RANGE_KEY_BITS
#define DGS_RANGE_KEY_BITS 16
#endif
constexpr int kRangeKeyBits = DGS_RANGE_KEY_BITS;
constexpr uint32_t kRangeKeyMax = (1u << kRangeKeyBits) - 1u;
__device__ __forceinline__ int range_key_shift(uint32_t lo, uint32_t hi) {
    const uint32_t span = hi > lo ? hi - lo : 0u;
    return span > kRangeKeyMax ? (32 - __clz(span)) - kRangeKeyBits : 0;
}
__device__ __forceinline__ float range_bucket_lo(float r, uint32_t lo, int shift) {
    const uint32_t b = __float_as_uint(r);
    return b > lo ? __uint_as_float(lo + (((b - lo) >> shift) << shift)) : r;
}
#endif

/// partition.hpp:66-71 locate (first subspace containing x).
DGS_HD int table_locate(const Table& tb, const float x[3]) {
    for (int k = 0; k < tb.k_count; ++k)
        if (subspace_contains(tb.sub[k], x[0], x[1], x[2])) return k;
    return -1;
}

}  // namespace dgs_b200
