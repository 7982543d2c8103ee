/*
 * dgs_oracle.h — CPU restatement of the reference algorithm for the RetinaGS
 * training step (float).  TEST INFRASTRUCTURE ONLY: used by tests/ as the
 * checker and by bench.py's cpu_baseline leg as the "port" baseline; never by
 * the product path.  Pinned against the reference itself (oracle/_ref ->
 * tests/golden) by tests/test_oracle_cpu.py.
 *
 * Layouts follow include/dgs_capi.h: splat fields per splat (mu[n][3],
 * log_scale[n][3], rotation[n][4], opacity_logit[n], sh[n][C][3]); images
 * H x W x C row-major.
 */
#ifndef DGS_ORACLE_H
#define DGS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_camera {
    int32_t width, height;
    float fx, fy, cx, cy;
    float q[4];
    float t[3];
} orc_camera;

typedef struct orc_opts {
    float trunc, near_plane, sigma_clamp, cov_reg, stop;
    int32_t sh_degree, indicator_enabled;
    float grad_skip_eps; /* Eigen isZero() precision of the backward pixel skip */
} orc_opts;

#define ORC_MAX_PLANES 8
typedef struct orc_subspace {
    int32_t n;
    float nx[ORC_MAX_PLANES], ny[ORC_MAX_PLANES], nz[ORC_MAX_PLANES], d[ORC_MAX_PLANES];
    int32_t closed[ORC_MAX_PLANES];
} orc_subspace;

typedef struct orc_splats {
    int64_t n;
    int32_t sh_coeffs;
    const uint64_t* id;
    const float *mu, *log_scale, *rotation, *opacity_logit, *sh;
} orc_splats;

typedef struct orc_grads {
    float *d_mu, *d_log_scale, *d_rotation, *d_opacity_logit, *d_sh;
} orc_grads;

/* project_scene (raster.hpp:91-127): per member 19 floats in the ref_dump
 * proj_rec layout (zero for culled), visibility, tile bins as CSR of member
 * indices in projected order.  Returns the pair count (or -needed). */
int64_t orc_project(const orc_splats* s, const orc_camera* cam, const orc_opts* o, float* rec19, uint8_t* visible,
                    int64_t* bins_off, int32_t* bins_ent, int64_t cap);
/* partial_render (engine.hpp:44-52): out_ct H*W*4; optional contributor ids
 * per pixel (composite order, raster.hpp:179/186). */
int orc_partial_render(const orc_splats* s, const orc_subspace* sub, const orc_camera* cam, const orc_opts* o,
                       float* out_ct, int32_t dbg_cap, uint32_t* dbg_ids, uint32_t* dbg_cnt);
/* compute_pixel_orders (engine.hpp:108-131). */
int orc_pixel_orders(const orc_subspace* subs, int32_t k_count, const orc_camera* cam, uint16_t* order,
                     uint16_t* count);
/* merge (engine.hpp:152-182): partials K*H*W*4. */
int orc_merge(const float* partials, const uint16_t* order, const uint16_t* count, int32_t k_count, int32_t w,
              int32_t h, const float bg[3], float* out_rgb, float* out_t);
/* loss (loss.hpp:153-177); returns the float loss value; grad HWC (may be NULL); sums = {l1, ssim, mse} means. */
float orc_loss(const float* render, const float* target, int32_t w, int32_t h, float lambda, float* grad,
               float* means3);
/* merge_backward (engine.hpp:195-234) with grad_trans_total = 0: out K*H*W*4. */
int orc_merge_backward(const float* partials, const uint16_t* order, const uint16_t* count, int32_t k_count,
                       int32_t w, int32_t h, const float* grad_color, const float bg[3], float* out);
/* partial_render_backward (engine.hpp:74-88 -> raster.hpp:267-317): the
 * reference's 16 row chunks merged in chunk order, then the per-splat pullback. */
int orc_partial_backward(const orc_splats* s, const orc_subspace* sub, const orc_camera* cam, const orc_opts* o,
                         const float* grad_ct, orc_grads* out);
/* 1: orc_partial_backward sums the suffix and every per-splat adjoint in double
 * (the same per-contribution float values), rounding once: a probe of the
 * reference's own accumulation rounding, not the reference's arithmetic. */
void orc_set_exact_accumulation(int on);
/* Per-gradient-entry rounding-sensitivity scale B (same layout as the
 * gradients): sum over the 10 adjoint fields of |pullback Jacobian| x the
 * cancellation-free magnitude each field sums.  Two float evaluations of the
 * backward differ by O(u B) entry-wise (tests/conftest.py grad_ok). */
int orc_partial_backward_bound(const orc_splats* s, const orc_subspace* sub, const orc_camera* cam, const orc_opts* o,
                               const float* grad_ct, orc_grads* out);
/* adam_apply over every member (optim.hpp:104-126, worker.hpp:162-167); p/m/v
 * are mutable field arrays; lr as float per group. */
int orc_adam(int64_t n, int32_t sh_coeffs, float* mu, float* ls, float* rot, float* op, float* sh, float* m_all,
             float* v_all, const orc_grads* g, double lr_pos, double lr_scale, double lr_rot, double lr_op,
             double lr_dc, double lr_rest, double b1, double b2, double eps, uint64_t step);
/* build_kdtree (partition.hpp:160-184) -> planes[k*depth + i] as (n0,n1,n2,d,closed). */
int orc_kdtree(const float* centers, int64_t n, int32_t depth, float* planes5);
/* assign_subsets (partition.hpp:234-251) -> mask[i*K + k]. */
int orc_assign(const float* planes5, int32_t k_count, int32_t depth, const float* mu, const float* log_scale,
               int64_t n, float d_mult, uint8_t* mask);

#ifdef __cplusplus
}
#endif

#endif
