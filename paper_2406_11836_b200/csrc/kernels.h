// Launchers for the sm_100a kernels (internal to libdgs_b200.so).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "dgs_types.cuh"

namespace dgs_b200 {

/// Opts `func` into `bytes` of dynamic shared memory on the CURRENT device.
/// Function attributes are per device context, so this is tracked per
/// (device, function) under a mutex (several devices or host threads may
/// launch concurrently); a failure is thrown as a CUDA error.  Defined in
/// capi.cu.
void ensure_smem_attr(const void* func, int bytes);

/// Per-view, per-subset scratch produced by the projection/binning stage and
/// consumed by both blend kernels.
struct ViewBins {
    SplatRec* recs = nullptr;        // [n]
    uint32_t* rect = nullptr;        // [2n]: x0 | x1 << 16, y0 | y1 << 16
    uint32_t* counts = nullptr;      // [n] tile count per member (0 = culled)
    uint32_t* rkey = nullptr;        // [n] range bits (0xffffffff = culled)
    float2* ext = nullptr;           // [n] conservative (x, y) half-extents of the m^2 <= 9 region (warp culling)
    uint32_t* dmax_bits = nullptr;   // [4] max world_radius over visible members, min range (float bits),
                                     //     visible member count, max range (float bits)
    uint32_t* blk_part = nullptr;    // [preprocess_partials(n)] K1's per-block partials of dmax_bits
    int* err_index = nullptr;        // [1] first member with a zero quaternion (or INT_MAX)
    int* abort = nullptr;            // [1] the step's abort flag: |= 1 on a zero quaternion, |= 2 on pair overflow
    float* shjac = nullptr;          // [10][ld] (optional): d colour_ch / d dir_a (row 3 ch + a) and the
                                     //     pre-clamp sign mask (row 9, bits) for the gradient record (K9)
    uint16_t* pair_tile = nullptr;   // [cap] tile key of each (splat, tile) pair
    uint32_t* pair_val = nullptr;    // [cap] member index
    uint2* ranges = nullptr;         // [tiles] (start, end) into the sorted pair list
    uint32_t* tile_order = nullptr;  // [tiles] tiles by decreasing list length (the blends' block order)
    int64_t pairs = 0;
    int64_t visible = 0;
    // camera_z_order: rkey / SplatRec::range hold the camera depth z and the
    // member sort is exact (32-bit keys) instead of 16-bit range buckets
    int zorder = 0;
};

// K1: projection + SH colour + tile rectangles (splat.hpp:288-321, raster.hpp:113-125),
// then the fold of its per-block partials into vb.dmax_bits (2 launches).
size_t preprocess_partials(int n);
void launch_preprocess(int n, const float* P, size_t ld, int sh_coeffs, const uint32_t* ids32, const ViewParams& vp,
                       const RenderOpts& ro, const ViewBins& vb, cudaStream_t s);

/// Zero `bytes` of device memory with a kernel.  The step path uses it instead
/// of cudaMemsetAsync: a memset node of a CUDA graph (and a runtime memset)
/// runs on a copy engine and queues behind the step's host-target upload.
void launch_zero(void* p, size_t bytes, cudaStream_t s);

// K2 helpers (CUB radix sorts live in binning.cu).
size_t binning_temp_bytes(int n, int64_t pair_cap);
// Sorts members by range, emits pairs in range order, stable-sorts them by
// tile, fills vb.ranges.  Returns the pair count (host sync).  `cap` is the
// pair buffer capacity; returns -needed if it is too small.
int64_t run_binning(int n, const ViewParams& vp, ViewBins& vb, int64_t cap, void* temp, size_t temp_bytes,
                    uint32_t* sort_keys_alt, uint32_t* sort_vals, uint32_t* sort_vals_alt, uint16_t* pair_tile_alt,
                    uint32_t* pair_val_alt, uint32_t* scan_buf, uint2* rect_sorted, uint32_t* pairs_host,
                    cudaStream_t s, int64_t pad_cap = 0);

struct BlendStats {
    unsigned long long evals;      // (pixel, candidate) 2D evaluations
    unsigned long long contribs;   // emitted contributions
    unsigned long long overflow;   // pixels routed to the exact fallback
    unsigned long long tiles_work; // sum over tiles of candidates processed
    unsigned long long subrounds;  // backward: warp emission sub-rounds
    unsigned long long small_rounds; // backward: sub-rounds with <= 2 lanes
};

/// Per-pixel composite records: the forward blend writes, for every pixel, the
/// tile-list positions (u16, relative to the tile's range start) of its first
/// kRecCap contributions in composite order; the backward blend walks them
/// directly instead of re-evaluating and re-ordering the tile list.  Tiles
/// where a pixel exceeds the cap (or the list exceeds 65,535 entries) are
/// flagged and replayed by the ordered-ring backward.
constexpr int kRecCap = 256;
struct CompRecords {
    uint16_t* pos = nullptr;         // [tiles][kRecCap / 4][256][4]
    uint16_t* cnt = nullptr;         // [px] recorded contributions
    uint8_t* tile_replay = nullptr;  // [tiles] 1: replay this tile in the backward
};

// K4: forward alpha blend with the RetinaGS subspace gate, exact per-ray (t, id) order.
// `rec` (pos == nullptr: no records) receives the composite records.
void launch_blend_fwd(const ViewParams& vp, const RenderOpts& ro, const Subspace& gate, const ViewBins& vb,
                      float4* out_ct, uint8_t* ovf_flag, uint32_t* ovf_list, uint32_t* ovf_count,
                      uint32_t* dbg_ids, uint32_t* dbg_cnt, int dbg_cap, BlendStats* stats, double* out_cd,
                      const CompRecords& rec, cudaStream_t s);
void launch_blend_fwd_fallback(const ViewParams& vp, const RenderOpts& ro, const Subspace& gate, const ViewBins& vb,
                               float4* out_ct, const uint32_t* ovf_list, const uint32_t* n_ovf_dev, uint32_t* dbg_ids,
                               uint32_t* dbg_cnt, int dbg_cap, double* out_cd, cudaStream_t s);

/// Where K8 accumulates the 9 pixel-space adjoints of each member (g2d_index layout).
/// q == nullptr: float RED atomics into f (order-dependent rounding).
/// q != nullptr (TrainConfig::deterministic, "fixed-order reductions",
/// optim.hpp:33): one pass; every sub-round sum is rounded to an integer
/// V = round(v 2^72) and added as V mod 2^32 and floor(V / 2^32) into two
/// 64-bit words (q = [9][lo|hi][ld]), so the totals are exact integers
/// whatever order the atomics land in; launch_fixed_to_float converts them
/// into f and re-zeroes q.  A non-finite value (or |value| >= 2^22) sets
/// bad = min(member index).  q must be zero on the first use.
/// Layout of the 9 pixel-space adjoints per member (g2d, acc.f): fields 0-7
/// of member i are the 32-byte sector at 8 i (one vector RED / one L2 sector
/// per warp reduction), field 8 (d_alpha) is a row at 8 ld + i.  9 ld floats.
__host__ __device__ inline size_t g2d_index(int f, size_t i, size_t ld) {
    return f < 8 ? 8 * i + (size_t)f : 8 * ld + i;
}

#ifdef __CUDACC__
/// Deterministic mode's fixed-point sums (acc.q, [9][lo | hi][ld] words):
/// member i's 9 totals (hi 2^32 + lo) 2^-72 as floats; the words are zeroed
/// for the next backward (they stay zero between uses).
__device__ __forceinline__ void fixed_to_float9(unsigned long long* __restrict__ q, size_t ld, size_t i, float a[9]) {
    unsigned long long lo[9], hi[9];
#pragma unroll
    for (int f = 0; f < 9; ++f) {
        lo[f] = __ldcs(q + (2 * f) * ld + i);
        hi[f] = __ldcs(q + (2 * f + 1) * ld + i);
    }
#pragma unroll
    for (int f = 0; f < 9; ++f) {
        __stcs(q + (2 * f) * ld + i, 0ull);
        __stcs(q + (2 * f + 1) * ld + i, 0ull);
        a[f] = (float)(fma((double)(long long)hi[f], 0x1p32, (double)lo[f]) * 0x1p-72);
    }
}
#endif

struct GradAcc {
    float* f = nullptr;  // g2d_index layout
    unsigned long long* q = nullptr;  // [9][lo | hi][ld]
    int* bad = nullptr;
    size_t ld = 0;
};

// K8: backward blend (+ the exact fallback for ring-overflow pixels);
// accumulates 9 pixel-space adjoints per member into acc (g2d_index layout).
// fwd_cd: the forward's double-precision colour sums (suffix = C - prefix without cancellation loss).
// With records (rec.pos != nullptr): the record walk for unflagged tiles plus
// the ordered-ring replay for flagged tiles; without: replay everywhere.
void launch_blend_bwd(const ViewParams& vp, const RenderOpts& ro, const Subspace& gate, const ViewBins& vb,
                      const float4* fwd_ct, const double* fwd_cd, const float4* grad_ct, const uint8_t* ovf_flag,
                      const CompRecords& rec, const GradAcc& acc, const uint32_t* ovf_list,
                      const uint32_t* n_ovf_dev, BlendStats* stats, cudaStream_t s);
// Deterministic mode: the fixed-point sums converted to float (acc.q -> acc.f, 9 rows); q re-zeroed.
void launch_fixed_to_float(const GradAcc& acc, int n, cudaStream_t s);

// Row windows: an array "with base b and rows r" holds image rows [b, b + r)
// (planar arrays: plane = r * W).  partials[k] / grad_out[k] hold float4
// rows starting at prow0 / grow0.
// K3/K5: per-pixel subset order + merge (engine.hpp:108-182) for rows [row0, row1).
void launch_merge(const ViewParams& vp, const Table* tb_dev, int owner, int row0, int row1,
                  const float4* const* partials, int prow0, const float bg[3], float* out_rgb, float* out_t,
                  int out_base, int out_rows, cudaStream_t s);
void launch_pixel_orders(const ViewParams& vp, const Table* tb_dev, int owner, uint16_t* order, uint16_t* count,
                         int kstride, cudaStream_t s);

// K6: fused L1 + D-SSIM forward and gradient (loss.hpp:33-177), per channel plane,
// outputs for rows [row0, row1); x, y, grad: planar windows (in_base, in_rows)
// that must cover [row0 - 10, row1 + 10) clipped to the image.
// Partial sums per block (double[3] each).  `kernel`: 11 taps in device memory.
void launch_loss(int W, int H, int row0, int row1, int in_base, int in_rows, const float* x, const float* y,
                 float lambda, const float* kernel, float inv_batch, float* grad, double* block_sums, int* n_blocks,
                 cudaStream_t s);
void launch_reduce_sums(const double* block_sums, int n_blocks, double* out3, cudaStream_t s);

// K7: merge adjoint (engine.hpp:195-234) for rows [row0, row1); grad_rgb window (g_base, g_rows).
void launch_merge_ordered(int px, int kstride, const uint16_t* order, const uint16_t* count, const float4* partials,
                          const float bg[3], float* out_rgb, float* out_t, cudaStream_t s);
void launch_merge_bwd_ordered(int px, int kcount, int kstride, const uint16_t* order, const uint16_t* count,
                              const float4* partials, const float* grad_color, const float* grad_tt,
                              const float bg[3], float4* out, cudaStream_t s);
void launch_merge_bwd(const ViewParams& vp, const Table* tb_dev, int owner, int row0, int row1,
                      const float4* const* partials, int prow0, const float* grad_rgb, int g_base, int g_rows,
                      const float bg[3], float4* const* grad_out, int grow0, cudaStream_t s);

// Device-side repartition (repartition.cu; orchestration in capi.cu dgs_repartition).
void repart_snapshot_keys(int n, const float* P, size_t ld, const uint32_t* ids32, const Table* tb, int k,
                          uint32_t base, uint64_t* keys, uint32_t* vals, cudaStream_t s);
size_t repart_temp_bytes(int64_t n);
void repart_sort_pairs(uint64_t*& keys, uint64_t*& keys_alt, uint32_t*& vals, uint32_t*& vals_alt, int n, int bits,
                       void* temp, size_t tb, cudaStream_t s);
void repart_sort_keys(uint64_t*& keys, uint64_t*& keys_alt, int n, int bits, void* temp, size_t tb, cudaStream_t s);
void repart_first_of_run(int n, const uint64_t* keys, uint8_t* flags, cudaStream_t s);
void repart_select(int n, const uint32_t* in, const uint8_t* flags, uint32_t* out, int* count, void* temp, size_t tb,
                   cudaStream_t s);
void repart_select_iota(int n, const uint8_t* flags, uint32_t* out, int* count, void* temp, size_t tb,
                        cudaStream_t s);
void repart_select_u64(int n, const uint64_t* in, const uint8_t* flags, uint64_t* out, int* count, void* temp,
                       size_t tb, cudaStream_t s);
void repart_gather_replicas(int n, int rows, const uint32_t* winners, const uint32_t* offsets, int K,
                            const float* const* srcP, const float* const* srcM, const float* const* srcV,
                            const uint32_t* const* srcId, const size_t* lds, float* P, float* M, float* V,
                            uint32_t* ids, size_t ld, cudaStream_t s);
void repart_node_extent(int n, const float* P, size_t ld, const uint8_t* node, int nnodes, uint32_t* lo,
                        uint32_t* hi, uint32_t* cnt, cudaStream_t s);
void repart_node_keys(int n, const float* P, size_t ld, const uint8_t* node, const int* axis, uint64_t* keys,
                      cudaStream_t s);
void repart_node_split(int n, const float* P, size_t ld, uint8_t* node, const int* axis, const float* plane,
                       cudaStream_t s);
void repart_assign(int n, const float* P, size_t ld, const Table* tb, float mult, uint32_t* mask, cudaStream_t s);
void repart_flag_bit(int n, const uint32_t* mask, int k, uint8_t* flags, cudaStream_t s);
void repart_gather_members(int n, int rows, const uint32_t* idx, const float* P, const float* M, const float* V,
                           const uint32_t* ids, size_t ld_src, float* dP, float* dM, float* dV, uint32_t* dids,
                           size_t ld_dst, cudaStream_t s);

// Multi-rank repartition helpers (repartition.cu).
void repart_flag_owned(int n, const uint32_t* mask, uint32_t owned, uint8_t* flags, cudaStream_t s);
void repart_flag_range(int n, const uint32_t* v, uint32_t lo, uint32_t hi, uint8_t* flags, cudaStream_t s);
void repart_sub_const(int n, uint32_t* v, uint32_t c, cudaStream_t s);
void repart_pack(int n, int rows, const uint32_t* idx, const float* P, const float* M, const float* V,
                 const uint32_t* ids, const uint32_t* mask, size_t ld, float* out, cudaStream_t s);
void repart_unpack(int n, int rows, const float* in, float* P, float* M, float* V, uint32_t* ids, uint32_t* mask,
                   size_t ld, cudaStream_t s);

// Gradient sync of shared replicas (config.grad_sync; manager.hpp:351-379, worker.hpp:103-144).
void shared_replica_keys(int n, const uint32_t* ids32, int k, uint32_t base, uint64_t* keys, uint32_t* vals,
                         cudaStream_t s);
void shared_run_starts(int n, const uint64_t* keys, uint8_t* flags, cudaStream_t s);
void grad_sync(int nslots, int rows, const uint32_t* starts, int nrep, const uint64_t* keys, const uint32_t* reps,
               float* const* G, const size_t* lds, cudaStream_t s);

// init_from_pointcloud's neighbour term (knn.cu): out[i] = mean of the sqrt of the
// k_nn (<= 3) smallest squared distances from point i to the others (exact).
void knn_mean_distance(int n, int k_nn, const float* d_pts, float* d_out, const float lo[3], const float hi[3],
                       cudaStream_t s);

// Cross-rank shared-replica gradient sync (repartition.cu).
void shared_mark(int n, const uint64_t* keys, uint8_t* flags, cudaStream_t s);
void shared_pack(int n, int rows, const uint32_t* pos, const uint32_t* sg, uint32_t base, const uint32_t* offs, int KL,
                 float* const* G, const size_t* lds, float* out, cudaStream_t s);
void shared_sync(int S, int rows, const uint64_t* skeys, const uint32_t* src, const float* recv, const uint8_t* mine,
                 const uint32_t* sg, uint32_t base, const uint32_t* offs, int KL, float* const* G, const size_t* lds,
                 cudaStream_t s);

struct AdamParams {
    float lr[kMaxParamRows];  // per row
    float b1, b2, eps, bc1, bc2;
    float rbc1, rbc2;         // 1/bc1, 1/bc2 (fast mode)
    int exact;                // 1: reference IEEE op sequence (TrainConfig::deterministic)
};

/// What the Adam launchers take: the step's AdamParams (a kernel argument: a
/// captured step graph gets this step's values by a kernel-node parameter
/// update, adam_param_index) and an optional device abort flag: non-zero skips
/// the write-back (a step abandoned after launch, e.g. zero quaternion or pair
/// overflow in a graph replay).
struct AdamArgs {
    AdamParams ap{};
    int exact = 0;
    const int* abort = nullptr;
};
/// For a kernel node of a captured step: the argument index of its AdamParams
/// and of its parameter rows P if `func` is one of the K10 kernels, else -1.
int adam_param_index(const void* func, int* p_index);

// K10: the streaming dense Adam over the gradient record (launch_project_bwd_adam
// runs it after the last view's K9).
void launch_adam_record(int n, float* P, float* M, float* V, size_t ld, int sh_coeffs, int deg, int nviews,
                        const AdamArgs& ap, const float* rec, cudaStream_t s);

// K9 (+K10): projection backward (splat.hpp:363-437) fused with dense Adam
// (optim.hpp:104-126) when `adam` is non-null; otherwise accumulates the
// parameter gradients into G (SoA rows).
// overwrite: G = this view's gradients (every row of every member written, so G
// needs no clearing); otherwise G += them.
void launch_project_bwd(int n, const float* P, size_t ld, int sh_coeffs, const ViewParams& vp,
                        const RenderOpts& ro, const uint32_t* counts, const float* g2d, size_t ld2, float* G,
                        int* bad_index, cudaStream_t s, bool overwrite = false);
// g_rec: scratch of kGradRecordRows(nviews) rows x ld floats (the per-member gradient record:
// 11 non-SH gradient rows summed over the views, then colour adjoint + direction per view).
// shjac: the preprocess's SH colour Jacobian rows ([10][ld], ViewBins::shjac) or nullptr (read the SH rows).
// g2q: deterministic mode's fixed-point sums (GradAcc::q) not yet converted, or nullptr (read g2d):
// K9 converts and re-zeroes them and writes g2d.
// Call once per view v = 0 .. nviews-1 in order; the last call also runs the Adam stream.
void launch_project_bwd_adam(int n, float* P, float* M, float* V, size_t ld, int sh_coeffs, const ViewParams& vp,
                             const RenderOpts& ro, const uint32_t* counts, const float* shjac, float* g2d,
                             size_t ld2, unsigned long long* g2q, int view, int nviews, const AdamArgs& ap,
                             int* bad_index, float* g_rec, cudaEvent_t mid_end, cudaEvent_t mid_begin,
                             cudaStream_t s);
constexpr size_t kGradRecordRows(int nviews) { return 11 + 6 * (size_t)nviews; }
void launch_adam(int n, float* P, float* M, float* V, size_t ld, int rows, const float* G, const AdamArgs& ap,
                 cudaStream_t s);

}  // namespace dgs_b200
