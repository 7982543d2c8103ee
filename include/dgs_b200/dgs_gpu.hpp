// dgs_gpu.hpp — C++ drop-in over libdgs_b200.so for code written against the
// reference header library (proj/include/dgs, namespace dgs).
//
// Include it after the reference headers; it adds namespace dgs::gpu with the
// same names, signatures and exception types as the reference's float entry
// points, implemented by the sm_100a kernels through include/dgs_capi.h:
//
//   dgs::gpu::partial_render            engine.hpp:44-52
//   dgs::gpu::partial_render_backward   engine.hpp:74-88
//   dgs::gpu::compute_pixel_orders      engine.hpp:108-131
//   dgs::gpu::merge                     engine.hpp:152-182 (caller's PixelOrders)
//   dgs::gpu::merge_backward            engine.hpp:195-234 (with grad_trans_total)
//   dgs::gpu::loss                      loss.hpp:153-177
//   dgs::gpu::build_kdtree              partition.hpp:160-184
//   dgs::gpu::assign_subsets            partition.hpp:234-251
//   dgs::gpu::Manager                   manager.hpp:212-516 (render, train_step,
//                                       snapshot, repartition)
//
// Only T = float is offered (the reference's double instantiation remains the
// CPU oracle).  Link with -ldgs_b200.
#pragma once

#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "dgs/engine.hpp"
#include "dgs/loss.hpp"
#include "dgs/optim.hpp"
#include "dgs/partition.hpp"
#include "../dgs_capi.h"

namespace dgs::gpu {

/// Status -> the reference's exception types.
inline void check(int rc) {
    if (rc == DGS_OK) return;
    const std::string msg = dgs_last_error();
    switch (rc) {
        case DGS_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case DGS_ERR_DOMAIN: throw std::domain_error(msg);
        default: throw std::runtime_error(msg);
    }
}

inline dgs_camera to_c(const Camera<float>& c) {
    dgs_camera o{};
    o.width = c.width;
    o.height = c.height;
    o.fx = c.fx;
    o.fy = c.fy;
    o.cx = c.cx;
    o.cy = c.cy;
    for (int i = 0; i < 4; ++i) o.q_wc[i] = c.q_wc[i];
    for (int i = 0; i < 3; ++i) o.t_wc[i] = c.t_wc[i];
    return o;
}

inline dgs_render_options to_c(const RenderOptions& r) {
    dgs_render_options o{};
    dgs_default_render_options(&o);
    o.truncation_radius = r.truncation_radius;
    o.near_plane = r.near_plane;
    o.sigma_clamp = r.sigma_clamp;
    o.cov2d_regularization = r.cov2d_regularization;
    o.stop_threshold = r.stop_threshold;
    o.sh_degree = r.sh_degree;
    o.indicator_enabled = r.indicator_enabled ? 1 : 0;
    o.camera_z_order = r.camera_z_order ? 1 : 0;
    return o;
}

inline dgs_train_config to_c(const TrainConfig& c) {
    dgs_train_config o{};
    dgs_default_train_config(&o);
    o.iterations = c.iterations;
    o.batch_size = c.batch_size;
    o.kd_depth = c.kd_depth;
    o.lambda_ssim = c.lambda_ssim;
    o.lr_position_start = c.lr_position_start;
    o.lr_position_end = c.lr_position_end;
    o.lr_sh_dc = c.lr_sh_dc;
    o.lr_sh_rest = c.lr_sh_rest;
    o.lr_opacity = c.lr_opacity;
    o.lr_scale = c.lr_scale;
    o.lr_rotation = c.lr_rotation;
    o.adam_beta1 = c.adam_beta1;
    o.adam_beta2 = c.adam_beta2;
    o.adam_eps = c.adam_eps;
    o.grad_sync = c.grad_sync ? 1 : 0;
    o.deterministic = c.deterministic ? 1 : 0;
    return o;
}

/// Field-layout staging of std::vector<Splat<float>> for the C-ABI.
struct SplatArrays {
    std::vector<uint64_t> id;
    std::vector<float> mu, log_scale, rotation, opacity_logit, sh;
    int sh_coeffs = 1;

    SplatArrays() = default;
    explicit SplatArrays(std::span<const Splat<float>> s) {
        const size_t n = s.size();
        sh_coeffs = n ? static_cast<int>(s[0].sh.size()) : 1;
        id.resize(n);
        mu.resize(3 * n);
        log_scale.resize(3 * n);
        rotation.resize(4 * n);
        opacity_logit.resize(n);
        sh.resize(n * sh_coeffs * 3);
        for (size_t i = 0; i < n; ++i) {
            if (static_cast<int>(s[i].sh.size()) != sh_coeffs)
                throw std::invalid_argument("dgs::gpu: all splats of a call must share the SH degree");
            id[i] = s[i].id;
            for (int a = 0; a < 3; ++a) {
                mu[3 * i + a] = s[i].mu[a];
                log_scale[3 * i + a] = s[i].log_scale[a];
            }
            for (int a = 0; a < 4; ++a) rotation[4 * i + a] = s[i].rotation[a];
            opacity_logit[i] = s[i].opacity_logit;
            for (int c = 0; c < sh_coeffs; ++c)
                for (int a = 0; a < 3; ++a) sh[(i * sh_coeffs + c) * 3 + a] = s[i].sh[c][a];
        }
    }
    static SplatArrays zeros(size_t n, int shc) {
        SplatArrays a;
        a.sh_coeffs = shc;
        a.id.assign(n, 0);
        a.mu.assign(3 * n, 0.0f);
        a.log_scale.assign(3 * n, 0.0f);
        a.rotation.assign(4 * n, 0.0f);
        a.opacity_logit.assign(n, 0.0f);
        a.sh.assign(n * shc * 3, 0.0f);
        return a;
    }
    dgs_splats view() {
        dgs_splats v{};
        v.n = static_cast<int64_t>(id.size());
        v.sh_coeffs = sh_coeffs;
        v.id = id.data();
        v.mu = mu.data();
        v.log_scale = log_scale.data();
        v.rotation = rotation.data();
        v.opacity_logit = opacity_logit.data();
        v.sh = sh.data();
        return v;
    }
    void to_splats(std::vector<Splat<float>>& out) const {
        const size_t n = id.size();
        out.resize(n);
        for (size_t i = 0; i < n; ++i) {
            out[i].id = id[i];
            out[i].mu = {mu[3 * i], mu[3 * i + 1], mu[3 * i + 2]};
            out[i].log_scale = {log_scale[3 * i], log_scale[3 * i + 1], log_scale[3 * i + 2]};
            out[i].rotation = {rotation[4 * i], rotation[4 * i + 1], rotation[4 * i + 2], rotation[4 * i + 3]};
            out[i].opacity_logit = opacity_logit[i];
            out[i].sh.assign(sh_coeffs, Vec3<float>::Zero());
            for (int c = 0; c < sh_coeffs; ++c)
                out[i].sh[c] = {sh[(i * sh_coeffs + c) * 3], sh[(i * sh_coeffs + c) * 3 + 1],
                                sh[(i * sh_coeffs + c) * 3 + 2]};
        }
    }
    GradBuffers<float> to_grads(std::span<const Splat<float>> like) const {
        GradBuffers<float> g(like);
        for (size_t i = 0; i < id.size(); ++i) {
            g.d_mu[i] = {mu[3 * i], mu[3 * i + 1], mu[3 * i + 2]};
            g.d_log_scale[i] = {log_scale[3 * i], log_scale[3 * i + 1], log_scale[3 * i + 2]};
            g.d_rotation[i] = {rotation[4 * i], rotation[4 * i + 1], rotation[4 * i + 2], rotation[4 * i + 3]};
            g.d_opacity_logit[i] = opacity_logit[i];
            for (int c = 0; c < sh_coeffs; ++c)
                g.d_sh[i][c] = {sh[(i * sh_coeffs + c) * 3], sh[(i * sh_coeffs + c) * 3 + 1],
                                sh[(i * sh_coeffs + c) * 3 + 2]};
        }
        return g;
    }
};

inline std::vector<dgs_plane> planes_of(const std::vector<Subspace<float>>& subs, int& per) {
    per = 0;
    for (const auto& s : subs) per = std::max(per, static_cast<int>(s.planes.size()));
    std::vector<dgs_plane> out(std::max<size_t>(1, subs.size() * per));
    for (size_t k = 0; k < subs.size(); ++k) {
        if (static_cast<int>(subs[k].planes.size()) != per)
            throw std::invalid_argument("dgs::gpu: every subspace needs the same plane count");
        for (int j = 0; j < per; ++j) {
            const auto& p = subs[k].planes[j];
            dgs_plane& q = out[k * per + j];
            q.n[0] = p.n[0];
            q.n[1] = p.n[1];
            q.n[2] = p.n[2];
            q.d = p.d;
            q.closed = p.closed ? 1 : 0;
        }
    }
    return out;
}

/// One device context (one GPU).  The stateless functions below use a
/// per-THREAD default context on device 0: the reference's ThreadWorkerLink
/// runs one worker thread per subset, each calling partial_render /
/// partial_render_backward concurrently (worker.hpp:70,93), and a context is
/// not thread-safe (its subset slot, view buffers and pinned scalars are
/// per-context state).
class Device {
  public:
    explicit Device(int device = 0) { check(dgs_ctx_create(device, 0, 1, nullptr, &ctx_)); }
    ~Device() {
        if (ctx_) dgs_ctx_destroy(ctx_);
    }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;
    dgs_ctx* get() const { return ctx_; }
    static Device& default_device() {
        static thread_local Device d(0);
        return d;
    }

  private:
    dgs_ctx* ctx_ = nullptr;
};

namespace detail {
inline void install_single(dgs_ctx* ctx, std::span<const Splat<float>> members, const Subspace<float>& sub,
                           const RenderOptions& opts) {
    int per = 0;
    std::vector<Subspace<float>> one{sub};
    auto planes = planes_of(one, per);
    check(dgs_set_table(ctx, planes.data(), 1, per));
    const dgs_render_options ro = to_c(opts);
    check(dgs_set_options(ctx, &ro, nullptr));
    SplatArrays a(members);
    dgs_splats v = a.view();
    check(dgs_subset_load(ctx, 0, &v, nullptr, nullptr, 0, 0));
}
}  // namespace detail

/// engine.hpp:44-52
inline PartialImage<float> partial_render(std::span<const Splat<float>> members, const Subspace<float>& sub,
                                          const Camera<float>& cam, const RenderOptions& opts = {}) {
    dgs_ctx* ctx = Device::default_device().get();
    detail::install_single(ctx, members, sub, opts);
    const dgs_camera c = to_c(cam);
    std::vector<float> ct(static_cast<size_t>(cam.width) * cam.height * 4);
    check(dgs_render_partial(ctx, 0, &c, ct.data(), 0, nullptr, nullptr));
    PartialImage<float> out;
    out.k = sub.k;
    out.color = Image<float>(cam.width, cam.height, 3);
    out.transmittance = Image<float>(cam.width, cam.height, 1, 1.0f);
    for (size_t p = 0; p < static_cast<size_t>(cam.width) * cam.height; ++p) {
        for (int ch = 0; ch < 3; ++ch) out.color.data[3 * p + ch] = ct[4 * p + ch];
        out.transmittance.data[p] = ct[4 * p + 3];
    }
    return out;
}

/// engine.hpp:74-88
inline GradBuffers<float> partial_render_backward(std::span<const Splat<float>> members, const Subspace<float>& sub,
                                                  const Camera<float>& cam, const Image<float>& grad_color,
                                                  const Image<float>& grad_trans, const RenderOptions& opts = {}) {
    if (grad_color.width != cam.width || grad_color.height != cam.height || grad_color.channels != 3 ||
        grad_trans.width != cam.width || grad_trans.height != cam.height || grad_trans.channels != 1)
        throw std::invalid_argument("partial_render_backward: gradient shape mismatch");
    dgs_ctx* ctx = Device::default_device().get();
    detail::install_single(ctx, members, sub, opts);
    const dgs_camera c = to_c(cam);
    const size_t px = static_cast<size_t>(cam.width) * cam.height;
    std::vector<float> g(px * 4);
    for (size_t p = 0; p < px; ++p) {
        for (int ch = 0; ch < 3; ++ch) g[4 * p + ch] = grad_color.data[3 * p + ch];
        g[4 * p + 3] = grad_trans.data[p];
    }
    SplatArrays out = SplatArrays::zeros(members.size(), members.empty() ? 1 : static_cast<int>(members[0].sh.size()));
    dgs_splats v = out.view();
    check(dgs_render_partial_backward(ctx, 0, &c, g.data(), &v));
    return out.to_grads(members);
}

/// engine.hpp:108-131
inline PixelOrders compute_pixel_orders(const PartitionTable<float>& table, const Camera<float>& cam) {
    dgs_ctx* ctx = Device::default_device().get();
    int per = 0;
    auto planes = planes_of(table.subspaces, per);
    check(dgs_set_table(ctx, planes.data(), table.subset_count(), per));
    PixelOrders po;
    po.width = cam.width;
    po.height = cam.height;
    po.subset_count = table.subset_count();
    po.order.assign(static_cast<size_t>(cam.width) * cam.height * po.subset_count, 0);
    po.count.assign(static_cast<size_t>(cam.width) * cam.height, 0);
    const dgs_camera c = to_c(cam);
    check(dgs_pixel_orders(ctx, &c, po.order.data(), po.count.data()));
    return po;
}

namespace detail {
inline std::vector<float> pack_partials(std::span<const PartialImage<float>> partials, const PixelOrders& orders) {
    const size_t px = static_cast<size_t>(orders.width) * orders.height;
    std::vector<float> out(px * 4 * orders.subset_count);
    std::string missing;
    for (int k = 0; k < orders.subset_count; ++k) {
        const PartialImage<float>* p = nullptr;
        for (const auto& q : partials)
            if (q.k == k) p = &q;
        if (!p) {
            missing += (missing.empty() ? "" : " ") + std::to_string(k);
            continue;
        }
        if (p->color.width != orders.width || p->color.height != orders.height)
            throw std::invalid_argument("merge: partial shape mismatch for subset " + std::to_string(k));
        for (size_t i = 0; i < px; ++i) {
            for (int ch = 0; ch < 3; ++ch) out[(k * px + i) * 4 + ch] = p->color.data[3 * i + ch];
            out[(k * px + i) * 4 + 3] = p->transmittance.data[i];
        }
    }
    if (!missing.empty()) throw std::invalid_argument("merge: missing subset partials: " + missing);
    return out;
}
}  // namespace detail

/// engine.hpp:152-182
inline RenderedImage<float> merge(std::span<const PartialImage<float>> partials, const PixelOrders& orders,
                                  const Vec3<float>& background) {
    dgs_ctx* ctx = Device::default_device().get();
    auto packed = detail::pack_partials(partials, orders);
    const float bg[3] = {background[0], background[1], background[2]};
    RenderedImage<float> out;
    out.background = background;
    out.color = Image<float>(orders.width, orders.height, 3);
    out.transmittance = Image<float>(orders.width, orders.height, 1, 1.0f);
    check(dgs_merge_ordered(ctx, orders.width, orders.height, orders.subset_count, orders.subset_count,
                            orders.order.data(), orders.count.data(), packed.data(), bg, out.color.data.data(),
                            out.transmittance.data.data()));
    return out;
}

/// engine.hpp:195-234
inline std::vector<PartialGrad<float>> merge_backward(std::span<const PartialImage<float>> partials,
                                                      const PixelOrders& orders, const Image<float>& grad_color,
                                                      const Image<float>& grad_trans_total,
                                                      const Vec3<float>& background) {
    dgs_ctx* ctx = Device::default_device().get();
    auto packed = detail::pack_partials(partials, orders);
    const float bg[3] = {background[0], background[1], background[2]};
    const size_t px = static_cast<size_t>(orders.width) * orders.height;
    if (grad_color.data.size() != 3 * px || grad_trans_total.data.size() != px)
        throw std::invalid_argument("merge_backward: gradient shape mismatch");
    std::vector<float> g(packed.size());
    check(dgs_merge_backward_ordered(ctx, orders.width, orders.height, orders.subset_count, orders.subset_count,
                                     orders.order.data(), orders.count.data(), packed.data(),
                                     grad_color.data.data(), grad_trans_total.data.data(), bg, g.data()));
    std::vector<PartialGrad<float>> out(orders.subset_count);
    for (int k = 0; k < orders.subset_count; ++k) {
        out[k].k = k;
        out[k].d_color = Image<float>(orders.width, orders.height, 3);
        out[k].d_transmittance = Image<float>(orders.width, orders.height, 1);
        for (size_t i = 0; i < px; ++i) {
            for (int ch = 0; ch < 3; ++ch) out[k].d_color.data[3 * i + ch] = g[(k * px + i) * 4 + ch];
            out[k].d_transmittance.data[i] = g[(k * px + i) * 4 + 3];
        }
    }
    return out;
}

/// loss.hpp:153-177
inline LossResult<float> loss(const Image<float>& render, const Image<float>& target, double lambda_ssim = 0.2) {
    if (!render.same_shape(target)) throw std::invalid_argument("loss: resolution mismatch");
    dgs_ctx* ctx = Device::default_device().get();
    LossResult<float> out;
    out.grad = Image<float>(render.width, render.height, render.channels);
    double value = 0.0;
    check(dgs_loss(ctx, render.width, render.height, render.data.data(), target.data.data(), lambda_ssim, 1.0,
                   out.grad.data.data(), &value, nullptr));
    out.value = static_cast<float>(value);
    return out;
}

/// partition.hpp:160-184 (host; bit-exact)
inline PartitionTable<float> table_from_planes(const std::vector<dgs_plane>& planes, int depth) {
    const int K = 1 << std::max(depth, 0);
    PartitionTable<float> t;
    t.depth = depth;
    t.kind = PartitionKind::kKdTree;
    for (int k = 0; k < K; ++k) {
        Subspace<float> s;
        s.k = k;
        for (int j = 0; j < depth; ++j) {
            const dgs_plane& p = planes[k * depth + j];
            HalfSpace<float> h;
            h.n = {p.n[0], p.n[1], p.n[2]};
            h.d = p.d;
            h.closed = p.closed != 0;
            s.planes.push_back(h);
        }
        t.subspaces.push_back(std::move(s));
    }
    t.membership.resize(K);
    return t;
}

inline PartitionTable<float> build_kdtree(std::span<const Vec3<float>> centers, int depth) {
    std::vector<float> c(3 * centers.size());
    for (size_t i = 0; i < centers.size(); ++i)
        for (int a = 0; a < 3; ++a) c[3 * i + a] = centers[i][a];
    const int K = 1 << std::max(depth, 0);
    std::vector<dgs_plane> planes(std::max(1, K * depth));
    check(dgs_build_kdtree(c.data(), static_cast<int64_t>(centers.size()), depth, planes.data()));
    return table_from_planes(planes, depth);
}

/// partition.hpp:234-251 (host; bit-exact)
inline void assign_subsets(PartitionTable<float>& table, std::span<const Splat<float>> splats,
                           double d_multiplier = 3.0) {
    int per = 0;
    auto planes = planes_of(table.subspaces, per);
    const int K = table.subset_count();
    std::vector<float> mu(3 * splats.size()), ls(3 * splats.size());
    for (size_t i = 0; i < splats.size(); ++i)
        for (int a = 0; a < 3; ++a) {
            mu[3 * i + a] = splats[i].mu[a];
            ls[3 * i + a] = splats[i].log_scale[a];
        }
    std::vector<uint8_t> mask(splats.size() * K);
    check(dgs_assign_subsets(planes.data(), K, per, mu.data(), ls.data(), static_cast<int64_t>(splats.size()),
                             d_multiplier, mask.data()));
    for (auto& m : table.membership) m.clear();
    for (size_t i = 0; i < splats.size(); ++i)
        for (int k = 0; k < K; ++k)
            if (mask[i * K + k]) table.membership[k].push_back(splats[i].id);
}

/// Manager<float> (manager.hpp:212-516) with every subset resident on one GPU.
class Manager {
  public:
    struct StepResult {
        double loss = 0;
        double psnr = 0;
        std::uint64_t comm_bytes = 0;
    };

    /// process_workers / timeout_ms are accepted for signature parity and
    /// ignored: every subset lives on `device` (one GPU per rank; see
    /// dgs_ctx_create for the NCCL multi-rank form).
    Manager(std::vector<Splat<float>> splats, TrainConfig config, RenderOptions options, bool process_workers = false,
            int timeout_ms = 120000, int device = 0)
        : config_(config), options_(options), dev_(device) {
        (void)process_workers;
        (void)timeout_ms;
        config_.validate();
        sh_coeffs_ = splats.empty() ? 1 : static_cast<int>(splats[0].sh.size());
        for (const auto& s : splats) ids_.push_back(s.id);
        std::sort(ids_.begin(), ids_.end());
        distribute(splats, {}, {}, 0, 0);
    }

    int worker_count() const { return table_.subset_count(); }
    const PartitionTable<float>& table() const { return table_; }
    std::uint64_t epoch() const { return epoch_; }
    std::uint64_t splat_count() const { return ids_.size(); }

    /// manager.hpp:250-257
    RenderedImage<float> render(const Camera<float>& cam, const Vec3<float>& background) {
        const dgs_camera c = to_c(cam);
        const float bg[3] = {background[0], background[1], background[2]};
        RenderedImage<float> out;
        out.background = background;
        out.color = Image<float>(cam.width, cam.height, 3);
        out.transmittance = Image<float>(cam.width, cam.height, 1, 1.0f);
        check(dgs_render(dev_.get(), &c, bg, out.color.data.data(), out.transmittance.data.data()));
        return out;
    }

    /// manager.hpp:313-386
    StepResult train_step(std::span<const Camera<float>> cams, std::span<const Image<float>> targets,
                          const Vec3<float>& background) {
        if (cams.size() != targets.size() || cams.empty())
            throw std::invalid_argument("train_step: need one target per camera");
        if (static_cast<int>(cams.size()) != config_.batch_size)
            throw std::invalid_argument("train_step: batch size mismatch with config");
        std::vector<dgs_camera> cc;
        std::vector<float> t;
        for (size_t v = 0; v < cams.size(); ++v) {
            cc.push_back(to_c(cams[v]));
            if (targets[v].width != cams[v].width || targets[v].height != cams[v].height)
                throw std::invalid_argument("loss: resolution mismatch");
            t.insert(t.end(), targets[v].data.begin(), targets[v].data.end());
        }
        const float bg[3] = {background[0], background[1], background[2]};
        dgs_step_result r{};
        check(dgs_train_step(dev_.get(), static_cast<int32_t>(cams.size()), cc.data(), t.data(), 0, bg, &r));
        return {r.loss, r.psnr, r.comm_bytes};
    }

    /// manager.hpp:390-418 (the replica held by the subspace containing the centre wins)
    /// A non-empty checkpoint_path sends MsgCheckpoint instead of MsgSnapshot
    /// in the reference; its worker answers both with the same snapshot and
    /// writes no file (worker.hpp:146-147), so the path is accepted and ignored.
    std::vector<SplatPack<float>> snapshot(const std::string& checkpoint_path = "") {
        (void)checkpoint_path;
        std::vector<SplatPack<float>> merged;
        std::set<SplatId> seen;
        std::vector<std::vector<SplatPack<float>>> per(table_.subset_count());
        for (int k = 0; k < table_.subset_count(); ++k) {
            const int64_t n = dgs_subset_size(dev_.get(), k);
            SplatArrays p = SplatArrays::zeros(n, sh_coeffs_), m = SplatArrays::zeros(n, sh_coeffs_),
                        v = SplatArrays::zeros(n, sh_coeffs_);
            dgs_splats pv = p.view(), mv = m.view(), vv = v.view();
            uint64_t step = 0;
            check(dgs_subset_store(dev_.get(), k, &pv, &mv, &vv, &step));
            adam_step_ = step;
            std::vector<Splat<float>> ps, ms, vs;
            p.to_splats(ps);
            m.to_splats(ms);
            v.to_splats(vs);
            for (size_t i = 0; i < ps.size(); ++i) {
                SplatPack<float> pack;
                pack.splat = ps[i];
                pack.moments = AdamMoments<float>::like(ps[i]);
                pack.moments.m.mu = ms[i].mu;
                pack.moments.m.log_scale = ms[i].log_scale;
                pack.moments.m.rotation = ms[i].rotation;
                pack.moments.m.opacity = ms[i].opacity_logit;
                pack.moments.m.sh = ms[i].sh;
                pack.moments.v.mu = vs[i].mu;
                pack.moments.v.log_scale = vs[i].log_scale;
                pack.moments.v.rotation = vs[i].rotation;
                pack.moments.v.opacity = vs[i].opacity_logit;
                pack.moments.v.sh = vs[i].sh;
                per[k].push_back(std::move(pack));
            }
        }
        for (int k = 0; k < table_.subset_count(); ++k)
            for (auto& pack : per[k])
                if (locate(table_, pack.splat.mu) == k && seen.insert(pack.splat.id).second) merged.push_back(pack);
        for (int k = 0; k < table_.subset_count(); ++k)
            for (auto& pack : per[k])
                if (!seen.count(pack.splat.id) && seen.insert(pack.splat.id).second) merged.push_back(pack);
        if (seen.size() != ids_.size()) throw std::runtime_error("snapshot lost splats");
        return merged;
    }

    /// manager.hpp:422-430, on the device (dgs_repartition): snapshot, KD build,
    /// assignment and migration never leave the GPU.  The table's membership
    /// lists come back in id order (the reference's are in snapshot order).
    void repartition() {
        const int depth = config_.kd_depth, K = 1 << std::max(depth, 0);
        std::vector<dgs_plane> planes(std::max(1, K * depth));
        check(dgs_repartition(dev_.get(), depth, options_.truncation_radius, static_cast<int64_t>(ids_.size()),
                              epoch_ + 1, planes.data()));
        epoch_ += 1;
        table_ = table_from_planes(planes, depth);
        for (int k = 0; k < K; ++k) {
            const int64_t n = dgs_subset_size(dev_.get(), k);
            std::vector<uint64_t> ids(static_cast<size_t>(std::max<int64_t>(n, 0)));
            if (n > 0) check(dgs_subset_ids(dev_.get(), k, ids.data()));
            table_.membership[k].assign(ids.begin(), ids.end());
        }
    }

    /// The host data flow of manager.hpp:422-430 (snapshot through the host, rebuild, reload).
    void repartition_host() {
        auto packs = snapshot();
        std::vector<SplatId> ids;
        for (const auto& p : packs) ids.push_back(p.splat.id);
        std::sort(ids.begin(), ids.end());
        if (ids != ids_) throw std::runtime_error("repartition checksum mismatch");
        std::vector<Splat<float>> s;
        std::vector<AdamMoments<float>> mom;
        for (auto& p : packs) {
            s.push_back(p.splat);
            mom.push_back(p.moments);
        }
        distribute(s, mom, {}, epoch_ + 1, adam_step_);
    }

  private:
    void distribute(const std::vector<Splat<float>>& splats, const std::vector<AdamMoments<float>>& mom,
                    const std::vector<int>&, std::uint64_t epoch, std::uint64_t adam_step) {
        epoch_ = epoch;
        std::vector<Vec3<float>> centers;
        for (const auto& s : splats) centers.push_back(s.mu);
        table_ = dgs::gpu::build_kdtree(centers, config_.kd_depth);
        dgs::gpu::assign_subsets(table_, splats, options_.truncation_radius);
        int per = 0;
        auto planes = planes_of(table_.subspaces, per);
        check(dgs_set_table(dev_.get(), planes.data(), table_.subset_count(), per));
        const dgs_render_options ro = to_c(options_);
        const dgs_train_config cfg = to_c(config_);
        check(dgs_set_options(dev_.get(), &ro, &cfg));
        std::map<SplatId, size_t> index;
        for (size_t i = 0; i < splats.size(); ++i) index[splats[i].id] = i;
        for (int k = 0; k < table_.subset_count(); ++k) {
            std::vector<Splat<float>> mem;
            std::vector<size_t> rows;
            for (SplatId id : table_.membership[k]) {
                rows.push_back(index.at(id));
                mem.push_back(splats[rows.back()]);
            }
            SplatArrays p(mem);
            dgs_splats pv = p.view();
            if (mom.empty()) {
                check(dgs_subset_load(dev_.get(), k, &pv, nullptr, nullptr, adam_step, epoch));
            } else {
                std::vector<Splat<float>> ms(mem), vs(mem);
                for (size_t i = 0; i < rows.size(); ++i) {
                    const auto& mm = mom[rows[i]];
                    ms[i].mu = mm.m.mu;
                    ms[i].log_scale = mm.m.log_scale;
                    ms[i].rotation = mm.m.rotation;
                    ms[i].opacity_logit = mm.m.opacity;
                    ms[i].sh = mm.m.sh;
                    vs[i].mu = mm.v.mu;
                    vs[i].log_scale = mm.v.log_scale;
                    vs[i].rotation = mm.v.rotation;
                    vs[i].opacity_logit = mm.v.opacity;
                    vs[i].sh = mm.v.sh;
                }
                SplatArrays ma(ms), va(vs);
                dgs_splats mv = ma.view(), vv = va.view();
                check(dgs_subset_load(dev_.get(), k, &pv, &mv, &vv, adam_step, epoch));
            }
        }
        check(dgs_set_epoch(dev_.get(), epoch));  // every render task carries it (manager.hpp:276)
    }

    TrainConfig config_;
    RenderOptions options_;
    Device dev_;
    PartitionTable<float> table_;
    std::vector<SplatId> ids_;
    int sh_coeffs_ = 1;
    std::uint64_t epoch_ = 0, adam_step_ = 0;
};

}  // namespace dgs::gpu
