/*
 * dgs_capi.h — C-ABI of libdgs_b200.so, the B200-native drop-in for the
 * RetinaGS distributed training step of the reference header library
 * (/root/reference/proj/include/dgs, namespace dgs).
 *
 * Every entry point returns DGS_OK (0) or an error code; dgs_last_error()
 * returns the thread-local message.  The codes map onto the exception types
 * the reference throws:
 *   DGS_ERR_INVALID_ARGUMENT  std::invalid_argument (shape mismatch, missing subset, bad config)
 *   DGS_ERR_RUNTIME           std::runtime_error ("non-finite gradient for splat id N", epoch mismatch)
 *   DGS_ERR_DOMAIN            std::domain_error ("zero quaternion", math.hpp:37)
 *   DGS_ERR_CUDA / DGS_ERR_NCCL  device / collective failure (no reference analogue)
 * There is no CPU fallback: without a CUDA device every compute entry point
 * fails with DGS_ERR_CUDA.
 *
 * Unless stated otherwise all array arguments are HOST pointers in the
 * reference's own layouts (Image<T>: H x W x C row-major, splat fields per
 * splat); the context keeps the parameters, optimizer moments and all
 * per-view scratch resident in HBM.  A context is stream-ordered and not
 * thread-safe.
 */
#ifndef DGS_CAPI_H
#define DGS_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DGS_CAPI_VERSION 1

#define DGS_OK 0
#define DGS_ERR_INVALID_ARGUMENT 1
#define DGS_ERR_RUNTIME 2
#define DGS_ERR_DOMAIN 3
#define DGS_ERR_CUDA 4
#define DGS_ERR_NCCL 5

typedef struct dgs_ctx dgs_ctx;

/* Camera<T> (splat.hpp:42-72): x_cam = R(q_wc) x_world + t_wc, +z forward. */
typedef struct dgs_camera {
    int32_t width, height;
    float fx, fy, cx, cy;
    float q_wc[4]; /* w, x, y, z */
    float t_wc[3];
} dgs_camera;

/* RenderOptions (splat.hpp:118-133).  grad_skip_eps is the threshold of the
 * reference's backward pixel skip `gc.isZero() && gT == 0` (raster.hpp:285):
 * Eigen's isZero() uses dummy_precision = 1e-5 for float, which is the
 * default here; 0 skips only exact zeros.  camera_z_order != 0 selects the
 * fast mode of splat.hpp:126 (per-view camera depth order, ties by id,
 * raster.hpp:162). */
typedef struct dgs_render_options {
    double truncation_radius;
    double near_plane;
    double sigma_clamp;
    double cov2d_regularization;
    double stop_threshold;
    int32_t sh_degree;
    int32_t indicator_enabled;
    int32_t camera_z_order;
    double grad_skip_eps;
} dgs_render_options;

/* TrainConfig (optim.hpp:16-43). */
typedef struct dgs_train_config {
    uint64_t iterations;
    int32_t batch_size;
    int32_t kd_depth;
    double lambda_ssim;
    double lr_position_start, lr_position_end;
    double lr_sh_dc, lr_sh_rest, lr_opacity, lr_scale, lr_rotation;
    double adam_beta1, adam_beta2, adam_eps;
    int32_t grad_sync;
    /* TrainConfig::deterministic (default 1, "fixed-order reductions"): the
     * backward sums every member's pixel-space adjoints as fixed point in
     * units of 2^-72 (order-independent integer atomics: bitwise reproducible
     * steps; |adjoint sum| < 2^22 per member and view)
     * and the optimizer uses the reference's exact IEEE op sequence
     * (bit-identical given identical gradients).  0 selects float RED
     * atomics and the fast Adam (reciprocal bias corrections, approximate
     * sqrt/divide; within 2 ulp of the exact step). */
    int32_t deterministic;
} dgs_train_config;

/* HalfSpace (partition.hpp:19-31): n.x + d <= 0 (closed) or < 0 (open). */
typedef struct dgs_plane {
    float n[3];
    float d;
    int32_t closed;
} dgs_plane;

/* Splat fields for n splats, per-splat layout: mu[n][3], log_scale[n][3],
 * rotation[n][4] (w,x,y,z), opacity_logit[n], sh[n][sh_coeffs][3]. */
typedef struct dgs_splats {
    int64_t n;
    int32_t sh_coeffs; /* (deg+1)^2: 1, 4, 9 or 16 */
    uint64_t* id;
    float* mu;
    float* log_scale;
    float* rotation;
    float* opacity_logit;
    float* sh;
} dgs_splats;

/* Manager<T>::StepResult (manager.hpp:306-310) plus device-side counters. */
typedef struct dgs_step_result {
    double loss;
    double psnr;
    uint64_t comm_bytes;      /* reference accounting: partial-map payload, both directions */
    uint64_t nccl_bytes;      /* bytes this rank actually sent over NCCL */
    uint64_t pairs;           /* (splat, tile) pairs over all local subsets and views */
    uint64_t evals_fwd, contribs_fwd, evals_bwd, contribs_bwd; /* stats mode only */
    uint64_t overflow_pixels; /* ring-overflow pixels (exact fallback kernels), every step */
    uint64_t kernel_launches; /* kernels this call launched */
    uint64_t subrounds_bwd, small_subrounds_bwd, tiles_work_fwd; /* blend work counters (stats mode) */
    uint64_t replay_tiles_bwd; /* tiles the backward replayed (records incomplete; stats mode) */
    uint64_t visible;          /* projected (visible) members over all local subsets and views */
} dgs_step_result;

const char* dgs_last_error(void);
int dgs_version(void);
void dgs_default_render_options(dgs_render_options* o);
void dgs_oracle_render_options(dgs_render_options* o); /* oracle_options(): stop = 0 */
void dgs_default_train_config(dgs_train_config* c);
/* position_lr (optim.hpp:46-53). */
double dgs_position_lr(const dgs_train_config* c, uint64_t step);

/* ---- Partition (host, bit-exact with partition.hpp) ---------------------- */
/* build_kdtree (partition.hpp:160-184): writes 2^depth subspaces, each with
 * exactly `depth` planes, to planes_out[k*depth + i] (DFS leaf order). */
int dgs_build_kdtree(const float* centers, int64_t n, int32_t depth, dgs_plane* planes_out);
/* assign_subsets (partition.hpp:234-251): member_mask[i*k_count + k] = 1 iff
 * splat i belongs to N_k.  planes[k*planes_per_subset + j]. */
int dgs_assign_subsets(const dgs_plane* planes, int32_t k_count, int32_t planes_per_subset, const float* mu,
                       const float* log_scale, int64_t n, double d_multiplier, uint8_t* member_mask);

/* ---- Synthetic inputs (io.hpp:421-543, test_helpers.hpp:70-96; libstdc++ <random>) */
/* synth_scene splat generator (targets are not rendered here). `out` arrays
 * must hold spec.count splats with (sh_degree+1)^2 coefficients. */
int dgs_synth_splats(int32_t count, int32_t clustered, int32_t sh_degree, double extent, uint64_t seed,
                     dgs_splats* out);
/* detail::ring_camera (io.hpp:447-487). */
int dgs_ring_camera(int32_t width, int32_t height, double fov_deg, double ring_radius, double extent,
                    int32_t n_views, int32_t i, dgs_camera* out);
/* ToyProblem::perturbed (test_trainer.cpp:201-211): mu += 0.02 N, logit += 0.3 N, dc += 0.1 N. */
int dgs_perturb_splats(dgs_splats* s, uint64_t seed);

/* ---- Context --------------------------------------------------------------- */
/* One context per GPU (rank).  world > 1 requires a 128-byte ncclUniqueId
 * made by dgs_nccl_unique_id on rank 0 and shared by the caller. */
int dgs_nccl_unique_id(void* out128);
/* Grouped send/recv and an all-reduce on a one-rank NCCL communicator on
 * `device`: checks the run-time NCCL binding the rank exchange uses. */
int dgs_nccl_selftest(int32_t device);
int dgs_ctx_create(int32_t device, int32_t rank, int32_t world, const void* nccl_id, dgs_ctx** out);
/* Test transport for the multi-rank step: the exchanges and the loss
 * all-reduce go through host callbacks instead of NCCL (NCCL refuses two
 * ranks on one device; tests run two processes on one GPU over
 * torch.distributed gloo).  send() must not block; flush() completes every
 * send and receive posted since the last flush.  Callbacks return 0 on
 * success. */
typedef struct dgs_host_transport {
    void* user;
    int (*send)(void* user, const void* buf, uint64_t bytes, int32_t peer);
    int (*recv)(void* user, void* buf, uint64_t bytes, int32_t peer);
    int (*flush)(void* user);
    int (*allreduce_sum_f64)(void* user, double* buf, uint64_t n);
} dgs_host_transport;
int dgs_ctx_create_host_transport(int32_t device, int32_t rank, int32_t world, const dgs_host_transport* transport,
                                  dgs_ctx** out);
int dgs_ctx_destroy(dgs_ctx* ctx);
/* The full partition table (every rank knows every subspace). */
int dgs_set_table(dgs_ctx* ctx, const dgs_plane* planes, int32_t k_count, int32_t planes_per_subset);
int dgs_set_options(dgs_ctx* ctx, const dgs_render_options* ro, const dgs_train_config* cfg);
/* MsgRepartition (worker.hpp:38-60): install subset k on this rank with its
 * parameters; m/v may be NULL (fresh moments, AdamMoments::like). */
int dgs_subset_load(dgs_ctx* ctx, int32_t k, const dgs_splats* params, const dgs_splats* m, const dgs_splats* v,
                    uint64_t adam_step, uint64_t epoch);
/* MsgSnapshot (worker.hpp:153-160): copy parameters (and moments) back. */
int dgs_subset_store(dgs_ctx* ctx, int32_t k, dgs_splats* params, dgs_splats* m, dgs_splats* v,
                     uint64_t* adam_step);
int64_t dgs_subset_size(dgs_ctx* ctx, int32_t k);
/* The manager's partition epoch (Manager::epoch_, carried by every
 * MsgRenderTask, manager.hpp:276).  Once set, dgs_train_step and
 * dgs_render_partial refuse a local subset loaded with another epoch:
 * DGS_ERR_RUNTIME "partition epoch mismatch" (worker.hpp:63).
 * dgs_repartition sets it to its new epoch. */
int dgs_set_epoch(dgs_ctx* ctx, uint64_t epoch);

/* ---- Per-subset forward (engine.hpp:44-52 partial_render) -------------------- */
/* Projection + binning + forward blend of local subset k for one view.
 * out_ct: H*W*4 floats (C_k rgb, T_k) or NULL.  With dbg_cap > 0 the
 * emitted contributor ids per pixel are recorded (debug; contributor hook
 * raster.hpp:179/186): dbg_ids[H*W*dbg_cap], dbg_cnt[H*W]. */
int dgs_render_partial(dgs_ctx* ctx, int32_t k, const dgs_camera* cam, float* out_ct, int32_t dbg_cap,
                       uint32_t* dbg_ids, uint32_t* dbg_cnt);
/* Tile bins of the last dgs_render_partial of subset k as CSR over tiles of
 * member indices (raster.hpp:113-125); order inside a tile is range order. */
int dgs_dump_bins(dgs_ctx* ctx, int32_t k, int64_t* tile_off, int32_t* entries, int64_t cap, int64_t* n_pairs);
/* Projected records of the last render (n x 16 floats: SplatRec layout, culled rows zero) and tile counts. */
int dgs_dump_records(dgs_ctx* ctx, int32_t k, float* recs, uint32_t* counts);

/* Manager::repartition (manager.hpp:421-430 -> snapshot + distribute, :389-482)
 * entirely on the device (world == 1, every subset resident): snapshot (one
 * replica per id: the holder whose subspace contains the centre, else the
 * lowest k), build_kdtree(depth) over the merged centres (bit-exact medians),
 * assign_subsets(d_multiplier) and migration of parameters and Adam moments
 * into 2^depth new subsets (epoch `epoch`, same Adam step).  expected_splats
 * >= 0: the snapshot must hold exactly that many ids ("snapshot lost
 * splats").  planes_out (optional): 2^depth * depth planes, as
 * dgs_build_kdtree. */
int dgs_repartition(dgs_ctx* ctx, int32_t depth, double d_multiplier, int64_t expected_splats, uint64_t epoch,
                    dgs_plane* planes_out);
/* init_from_pointcloud (trainer.hpp:24-91): `target` splats sampled from the
 * cloud with the reference's libstdc++ streams (std::sample without
 * replacement, or uniform picks + Gaussian jitter when oversampling), isotropic
 * log-scale from the mean distance to the 3 nearest sampled neighbours (exact
 * k-NN on the GPU, ctx's device), identity rotation, opacity logit(0.1), DC
 * colour from the point colour.  colors may be NULL (n_colors = 0). */
int dgs_init_from_pointcloud(dgs_ctx* ctx, const float* points, int64_t n_points, const float* colors,
                             int64_t n_colors, int64_t target, uint64_t seed, int32_t sh_degree, dgs_splats* out);
/* save_splats_ply (io.hpp:257-297): 3DGS property convention, float32,
 * binary_little_endian (binary != 0) or ascii; byte-identical to the reference. */
int dgs_save_splats_ply(const dgs_splats* splats, const char* path, int32_t binary);
/* load_ply's splat mode (io.hpp:85-255) for float32 checkpoints: out == NULL
 * returns only the count and the SH coefficient count; ids are 0..n-1. */
int dgs_load_splats_ply(const char* path, dgs_splats* out, int64_t* n, int32_t* sh_coeffs);
/* Splat ids of subset k (dgs_subset_size(ctx, k) entries, member order). */
int dgs_subset_ids(dgs_ctx* ctx, int32_t k, uint64_t* ids);

/* ---- Manager side (engine.hpp:108-234, loss.hpp:153-177) ------------------------ */
int dgs_pixel_orders(dgs_ctx* ctx, const dgs_camera* cam, uint16_t* order, uint16_t* count);
/* merge: partials[k] = H*W*4 (rgb, T) for every k of the table. out_rgb HWC, out_t HW. */
int dgs_merge(dgs_ctx* ctx, const dgs_camera* cam, const float* partials, const float bg[3], float* out_rgb,
              float* out_t);
/* loss(render, target, lambda) -> value + gradient (HWC), times inv_batch. sums = {sum|d|, sum ssim, sum d^2}. */
int dgs_loss(dgs_ctx* ctx, int32_t width, int32_t height, const float* render, const float* target, double lambda,
             double inv_batch, float* grad, double* value, double* sums);
/* merge_backward with grad_trans_total = 0: out_grads[k] = H*W*4 (dL/dC_k rgb, dL/dT_k). */
int dgs_merge_backward(dgs_ctx* ctx, const dgs_camera* cam, const float* partials, const float* grad_color,
                       const float bg[3], float* out_grads);

/* merge / merge_backward on caller-supplied PixelOrders (engine.hpp:97-106
 * layout: order[px][k_stride], count[px]), exactly the reference signatures
 * merge(partials, orders, background) (engine.hpp:152-182) and
 * merge_backward(partials, orders, grad_color, grad_trans_total, background)
 * (engine.hpp:195-234).  No partition table needed.  grad_trans_total may be
 * NULL (zero). */
int dgs_merge_ordered(dgs_ctx* ctx, int32_t width, int32_t height, int32_t k_count, int32_t k_stride,
                      const uint16_t* order, const uint16_t* count, const float* partials, const float bg[3],
                      float* out_rgb, float* out_t);
int dgs_merge_backward_ordered(dgs_ctx* ctx, int32_t width, int32_t height, int32_t k_count, int32_t k_stride,
                               const uint16_t* order, const uint16_t* count, const float* partials,
                               const float* grad_color, const float* grad_trans_total, const float bg[3],
                               float* out_grads);

/* ---- Per-subset backward (engine.hpp:74-88) + optimizer ------------------------ */
/* partial_render_backward: grad_ct = H*W*4 (dL/dC_k rgb, dL/dT_k).  Writes the
 * parameter gradients (GradBuffers layout, index-aligned with the members)
 * into `grads` (arrays of the dgs_splats layout; id may be NULL). */
int dgs_render_partial_backward(dgs_ctx* ctx, int32_t k, const dgs_camera* cam, const float* grad_ct,
                                dgs_splats* grads);
/* Pixel-space adjoints (Splat2DGrad, splat.hpp:341-347) of the last
 * dgs_render_partial_backward: n x 9 = d_mean2d(2), d_cov2d(00, 01, 11),
 * d_color(3), d_alpha (debug / parity). */
int dgs_dump_pixel_grads(dgs_ctx* ctx, int32_t k, float* out);
/* apply_step (worker.hpp:162-167) with the given gradients (GradBuffers
 * layout); advances the subset's Adam step. */
int dgs_adam_apply(dgs_ctx* ctx, int32_t k, const dgs_splats* grads);

/* ---- The hot path: Manager<float>::train_step (manager.hpp:313-386) ----------- */
/* One barrier-synchronised training step over a batch of B views.
 * Multi-rank (world > 1): every rank calls it with the same cameras; rank r
 * must hold exactly the subsets k with dgs_subset_owner(k, K, world) == r;
 * partial rows are exchanged with NCCL all-to-all (grouped send/recv),
 * loss sums are all-reduced.
 * targets: B x H x W x 3 floats (Image<float> layout).  targets_on_device = 0:
 * host pointer, copied in; 1: device pointer to B planar [3][H][W] images. */
int dgs_train_step(dgs_ctx* ctx, int32_t batch, const dgs_camera* cams, const float* targets,
                   int32_t targets_on_device, const float bg[3], dgs_step_result* out);
/* Multi-rank plan: rank j owns pixel rows [r0, r1) of every
 * view for merge + loss, with a 10-row SSIM halo [h0, h1); subset k lives on
 * rank dgs_subset_owner(k, K, world).  rows4 = {r0, r1, h0, h1}. */
int dgs_slice_plan(int32_t height, int32_t slices, int32_t s, int32_t* rows4);
int32_t dgs_subset_owner(int32_t k, int32_t k_count, int32_t world);
/* Single-rank test mode: run the multi-rank manager path (halo windows,
 * exchange buffers, per-slice loss sums) over `slices` virtual slices with
 * device copies in place of NCCL.  Default 1 (whole image, zero-copy). */
/* Backward blend strategy: 1 (default) = the forward records each pixel's
 * composite sequence and the backward walks it; 0 = the backward replays the
 * ordered traversal (ring) itself.  Same contributions, same order. */
int dgs_set_backward_records(dgs_ctx* ctx, int32_t enabled);
int dgs_set_virtual_slices(dgs_ctx* ctx, int32_t slices);
/* Partial map (C_k, T_k) and its gradient (dL/dC_k, dL/dT_k) of local
 * subset k for view slot v of the last dgs_train_step (debug / parity):
 * H*W*4 floats each (either may be NULL). */
int dgs_dump_grad_maps(dgs_ctx* ctx, int32_t k, int32_t view, float* partial_ct, float* grad_ct);
/* Upload B targets (HWC host) once into a device planar buffer owned by ctx;
 * returns the device pointer for dgs_train_step(targets_on_device = 1). */
int dgs_upload_targets(dgs_ctx* ctx, int32_t batch, int32_t width, int32_t height, const float* targets_hwc,
                       const float** device_ptr);
/* Render a full image (all local subsets merged, rows owned by this rank)
 * into out_rgb (HWC host) — Manager::render (manager.hpp:250-257). */
int dgs_render(dgs_ctx* ctx, const dgs_camera* cam, const float bg[3], float* out_rgb, float* out_t);

/* Per-stage device timing with CUDA events on the context's stream.  Stages:
 * 0 preprocess (K1), 1 binning (K2, incl. CUB sorts), 2 blend_fwd (K4),
 * 3 merge (K5), 4 loss (K6), 5 merge_bwd (K7), 6 blend_bwd (K8),
 * 7 project_bwd (K9, gradient record), 8 adam (K10, streaming), 9 exchange
 * (NCCL).  Accumulated over calls while enabled; dgs_stage_times returns
 * total ms and launch counts. */
#define DGS_NUM_STAGES 10
int dgs_set_profiling(dgs_ctx* ctx, int32_t enabled);
/* Blend evaluation / contribution / overflow counters in dgs_step_result
 * (off by default: they cost a few percent in the blend kernels). */
int dgs_set_collect_stats(dgs_ctx* ctx, int32_t enabled);
int dgs_stage_times(dgs_ctx* ctx, double* ms, uint64_t* counts);
/* CUDA stream the context launches on (cudaStream_t as void*), for timing. */
void* dgs_stream(dgs_ctx* ctx);
/* Device synchronise + sticky-error check. */
int dgs_sync(dgs_ctx* ctx);
/* 1: dgs_train_step runs as a CUDA graph (single rank, device or pinned host
 * targets, stage timing and counters off, grad_sync off; otherwise eager).
 * Per key (cameras, device target pointer, background; pinned host targets
 * are uploaded outside the graph, so their pointer may change between
 * replays): the first call runs eagerly,
 * the second captures the step without any host round trip (the pair counts
 * stay on the device and the tile sort covers each slot's largest count
 * + 2 %) and replays it; later calls replay.  Results are those of the eager
 * step; a replay whose pair count outgrew the capture is redone eagerly. */
int dgs_set_graph_mode(dgs_ctx* ctx, int32_t enabled);
/* Rollback point in HBM: dgs_state_save copies every local subset's
 * parameters, Adam moments and step count into a spare device buffer of the
 * subset; dgs_state_restore copies them back in place (no reallocation, so
 * captured step graphs stay valid).  Not in the reference, which checkpoints
 * through the host snapshot (manager.hpp:390-418); used to time several
 * windows from one training state.  Restore without a save is an error. */
int dgs_state_save(dgs_ctx* ctx);
int dgs_state_restore(dgs_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* DGS_CAPI_H */
