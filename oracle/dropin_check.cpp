// dropin_check.cpp — TEST INFRASTRUCTURE ONLY.
//
// Compiles the UNMODIFIED reference headers (read in place from
// $(REF)/proj/include, against the Eigen shim) together with the C++ drop-in
// include/dgs_b200/dgs_gpu.hpp, and runs every drop-in entry point beside the
// reference function it replaces on the same inputs:
//
//   build_kdtree / assign_subsets      partition.hpp:160-251   bit-exact
//   partial_render                     engine.hpp:44-52        <= 1e-4 abs
//   compute_pixel_orders               engine.hpp:108-131      bit-exact
//   merge                              engine.hpp:152-182      bit-exact
//   loss                               loss.hpp:153-177        grad bit-exact, value 1e-4 rel
//   merge_backward (+grad_trans_total) engine.hpp:195-234      bit-exact
//   partial_render_backward            engine.hpp:74-88        <= 1e-3 of field max
//   Manager::train_step/snapshot       manager.hpp:313-418     loss 1e-4 rel, params 1e-3
//
// Prints one JSON object of error figures and exits 0 iff all are inside
// tolerance.  Built by `make -C oracle dropin` into _ref/ (needs the
// reference, so it is built here and travels prebuilt); run by
// tests/test_dropin_gpu.py on the GPU box.
#include "dgs/engine.hpp"
#include "dgs/io.hpp"
#include "dgs/loss.hpp"
#include "dgs/manager.hpp"
#include "dgs/optim.hpp"
#include "dgs/partition.hpp"
#include "dgs_b200/dgs_gpu.hpp"

#include <cstdio>
#include <random>
#include <string>
#include <thread>
#include <vector>

using namespace dgs;

namespace {

struct Report {
    std::string json = "{";
    bool ok = true;
    void add(const char* key, double v, double tol) {
        char buf[160];
        std::snprintf(buf, sizeof buf, "%s\"%s\": %.6g", json.size() > 1 ? ", " : "", key, v);
        json += buf;
        if (!(v <= tol)) {
            ok = false;
            std::fprintf(stderr, "FAIL %s = %.6g > %.3g\n", key, v, tol);
        }
    }
};

double max_abs(const std::vector<float>& a, const std::vector<float>& b) {
    if (a.size() != b.size()) return 1e30;
    double m = 0;
    for (size_t i = 0; i < a.size(); ++i) m = std::max(m, (double)std::fabs(a[i] - b[i]));
    return m;
}

template <typename V>
void flat_into(std::vector<float>& out, const V& v, int n) {
    for (int i = 0; i < n; ++i) out.push_back(v[i]);
}

// max |a-b| / max |a| per GradBuffers field, worst field
double grad_rel(const GradBuffers<float>& r, const GradBuffers<float>& g) {
    std::vector<std::vector<float>> fr(5), fg(5);
    for (size_t i = 0; i < r.size(); ++i) {
        flat_into(fr[0], r.d_mu[i], 3);
        flat_into(fg[0], g.d_mu[i], 3);
        flat_into(fr[1], r.d_log_scale[i], 3);
        flat_into(fg[1], g.d_log_scale[i], 3);
        flat_into(fr[2], r.d_rotation[i], 4);
        flat_into(fg[2], g.d_rotation[i], 4);
        fr[3].push_back(r.d_opacity_logit[i]);
        fg[3].push_back(g.d_opacity_logit[i]);
        for (size_t c = 0; c < r.d_sh[i].size(); ++c) {
            flat_into(fr[4], r.d_sh[i][c], 3);
            flat_into(fg[4], g.d_sh[i][c], 3);
        }
    }
    double worst = 0;
    for (int f = 0; f < 5; ++f) {
        double mx = 0;
        for (float x : fr[f]) mx = std::max(mx, (double)std::fabs(x));
        if (mx == 0) continue;
        worst = std::max(worst, max_abs(fr[f], fg[f]) / mx);
    }
    return worst;
}

std::vector<Splat<float>> members_of(const PartitionTable<float>& t, int k, const std::vector<Splat<float>>& all) {
    std::map<SplatId, size_t> idx;
    for (size_t i = 0; i < all.size(); ++i) idx[all[i].id] = i;
    std::vector<Splat<float>> m;
    for (SplatId id : t.membership[k]) m.push_back(all[idx.at(id)]);
    return m;
}

}  // namespace

int main() {
    Report rep;
    SynthSpec spec;
    spec.count = 1500;
    spec.n_views = 0;
    spec.width = 96;
    spec.height = 72;
    spec.sh_degree = 3;
    auto bundle = synth_scene<float>(spec, 11);
    std::vector<Splat<float>> gt = bundle.gt_splats;
    std::vector<Splat<float>> splats = gt;
    {  // tests/test_trainer.cpp:201-211 (ToyProblem::perturbed)
        std::mt19937_64 rng(5);
        std::normal_distribution<double> g;
        for (auto& s : splats) {
            s.mu += Vec3<float>{float(g(rng)), float(g(rng)), float(g(rng))} * 0.02f;
            s.opacity_logit += float(0.3 * g(rng));
            s.sh[0] += Vec3<float>{float(g(rng)), float(g(rng)), float(g(rng))} * 0.1f;
        }
    }
    SynthSpec vs = spec;
    vs.n_views = 8;
    const Camera<float> cam = detail::ring_camera<float>(vs, 1);
    const RenderOptions opts;  // default: early termination on
    const Vec3<float> bg{0.2f, 0.5f, 0.9f};

    // ---- partition -------------------------------------------------------
    std::vector<Vec3<float>> centers;
    for (const auto& s : splats) centers.push_back(s.mu);
    PartitionTable<float> tr = build_kdtree<float>(centers, 2);
    assign_subsets<float>(tr, splats, opts.truncation_radius);
    PartitionTable<float> tg = gpu::build_kdtree(centers, 2);
    gpu::assign_subsets(tg, splats, opts.truncation_radius);
    double plane_err = 0, member_err = 0;
    for (int k = 0; k < tr.subset_count(); ++k) {
        for (size_t j = 0; j < tr.subspaces[k].planes.size(); ++j) {
            const auto &a = tr.subspaces[k].planes[j], &b = tg.subspaces[k].planes[j];
            plane_err += (a.n - b.n).norm() + std::fabs(a.d - b.d) + (a.closed != b.closed);
        }
        member_err += tr.membership[k] != tg.membership[k];
    }
    rep.add("kdtree_plane_err", plane_err, 0);
    rep.add("membership_mismatch", member_err, 0);

    // ---- per-subset partial renders ---------------------------------------
    std::vector<PartialImage<float>> pr, pg;
    double render_err = 0;
    for (int k = 0; k < tr.subset_count(); ++k) {
        const auto mem = members_of(tr, k, splats);
        pr.push_back(partial_render<float>(mem, tr.subspaces[k], cam, opts));
        pg.push_back(gpu::partial_render(mem, tr.subspaces[k], cam, opts));
        render_err = std::max({render_err, max_abs(pr.back().color.data, pg.back().color.data),
                               max_abs(pr.back().transmittance.data, pg.back().transmittance.data)});
    }
    rep.add("partial_render_max_abs", render_err, 1e-4);

    // ---- orders, merge (GPU merge fed the reference's partials: bitwise) --
    const PixelOrders orr = compute_pixel_orders<float>(tr, cam);
    const PixelOrders og = gpu::compute_pixel_orders(tr, cam);
    rep.add("orders_mismatch", (orr.order != og.order) + (orr.count != og.count), 0);
    const RenderedImage<float> mr = merge<float>(pr, orr, bg);
    const RenderedImage<float> mg = gpu::merge(pr, orr, bg);
    rep.add("merge_max_abs", std::max(max_abs(mr.color.data, mg.color.data),
                                      max_abs(mr.transmittance.data, mg.transmittance.data)), 0);

    // ---- loss on the merged image against the GT render -------------------
    std::vector<PartialImage<float>> pt;
    for (int k = 0; k < tr.subset_count(); ++k) {
        std::vector<Splat<float>> gm;
        for (const auto& s : gt)
            if (indicator(s.mu, tr.subspaces[k])) gm.push_back(s);
        pt.push_back(partial_render<float>(gm, tr.subspaces[k], cam, oracle_options()));
    }
    const Image<float> target = merge<float>(pt, orr, bg).color;
    const LossResult<float> lr = loss<float>(mr.color, target, 0.2);
    const LossResult<float> lg = gpu::loss(mr.color, target, 0.2);
    // the reference accumulates the loss scalar sequentially in float
    // (loss.hpp:160-170, 3·H·W terms); the device reduces in double
    rep.add("loss_rel", std::fabs(lr.value - lg.value) / std::max(1e-12, (double)std::fabs(lr.value)), 1e-4);
    rep.add("loss_grad_max_abs", max_abs(lr.grad.data, lg.grad.data), 0);

    // ---- merge adjoint with a non-zero grad_trans_total -------------------
    Image<float> gtt(cam.width, cam.height, 1);
    std::mt19937 rng(3);
    std::uniform_real_distribution<float> u(-1e-3f, 1e-3f);
    for (auto& x : gtt.data) x = u(rng);
    const auto br = merge_backward<float>(pr, orr, lr.grad, gtt, bg);
    const auto bgp = gpu::merge_backward(pr, orr, lr.grad, gtt, bg);
    double mb_err = 0;
    for (int k = 0; k < tr.subset_count(); ++k)
        mb_err = std::max({mb_err, max_abs(br[k].d_color.data, bgp[k].d_color.data),
                           max_abs(br[k].d_transmittance.data, bgp[k].d_transmittance.data)});
    rep.add("merge_backward_max_abs", mb_err, 0);

    // ---- partial_render_backward per subset --------------------------------
    double pb_err = 0;
    for (int k = 0; k < tr.subset_count(); ++k) {
        const auto mem = members_of(tr, k, splats);
        const auto gr = partial_render_backward<float>(mem, tr.subspaces[k], cam, br[k].d_color,
                                                       br[k].d_transmittance, opts);
        const auto gg = gpu::partial_render_backward(mem, tr.subspaces[k], cam, br[k].d_color,
                                                     br[k].d_transmittance, opts);
        pb_err = std::max(pb_err, grad_rel(gr, gg));
    }
    rep.add("partial_backward_rel", pb_err, 1e-3);

    // ---- concurrency: one host thread per subset, as the reference's
    //      ThreadWorkerLink runs its workers (worker.hpp:70,93) ---------------
    // Each thread calls the stateless drop-ins (per-thread default context) at
    // the same time as the others; the results must equal the single-thread ones.
    {
        const int K = tr.subset_count();
        std::vector<PartialImage<float>> pc(K);
        std::vector<GradBuffers<float>> gc;
        std::vector<GradBuffers<float>> g1;
        for (int k = 0; k < K; ++k) {
            const auto mem = members_of(tr, k, splats);
            gc.emplace_back(std::span<const Splat<float>>(mem));
            g1.push_back(gpu::partial_render_backward(mem, tr.subspaces[k], cam, br[k].d_color, br[k].d_transmittance,
                                                      opts));
        }
        std::vector<std::string> errs(K);
        for (int round = 0; round < 3; ++round) {
            std::vector<std::thread> ts;
            for (int k = 0; k < K; ++k)
                ts.emplace_back([&, k] {
                    try {
                        const auto mem = members_of(tr, k, splats);
                        for (int rep_i = 0; rep_i < 4; ++rep_i) {
                            pc[k] = gpu::partial_render(mem, tr.subspaces[k], cam, opts);
                            gc[k] = gpu::partial_render_backward(mem, tr.subspaces[k], cam, br[k].d_color,
                                                                 br[k].d_transmittance, opts);
                        }
                    } catch (const std::exception& e) {
                        errs[k] = e.what();
                    }
                });
            for (auto& t : ts) t.join();
        }
        double thr_render = 0, thr_grad = 0, thr_fail = 0;
        for (int k = 0; k < K; ++k) {
            if (!errs[k].empty()) {
                thr_fail += 1;
                std::fprintf(stderr, "thread %d: %s\n", k, errs[k].c_str());
                continue;
            }
            thr_render = std::max({thr_render, max_abs(pc[k].color.data, pg[k].color.data),
                                   max_abs(pc[k].transmittance.data, pg[k].transmittance.data)});
            thr_grad = std::max(thr_grad, grad_rel(g1[k], gc[k]));
        }
        rep.add("threaded_failures", thr_fail, 0);
        rep.add("threaded_partial_render_max_abs", thr_render, 0);
        // float-atomic accumulation order may differ between runs
        rep.add("threaded_partial_backward_rel", thr_grad, 1e-3);
    }

    // ---- Manager: two training steps, then snapshot ------------------------
    TrainConfig cfg;
    cfg.kd_depth = 1;
    cfg.iterations = 100;
    Manager<float> m_ref(splats, cfg, opts);
    gpu::Manager m_gpu(splats, cfg, opts);
    const Camera<float> cams[1] = {cam};
    const Image<float> tgts[1] = {target};
    double step_loss_err = 0;
    for (int it = 0; it < 2; ++it) {
        const auto a = m_ref.train_step(cams, tgts, bg);
        const auto b = m_gpu.train_step(cams, tgts, bg);
        step_loss_err = std::max(step_loss_err, std::fabs(a.loss - b.loss) / std::max(1e-12, std::fabs(a.loss)));
        if (a.comm_bytes != b.comm_bytes) rep.add("comm_bytes_mismatch", 1, 0);
    }
    rep.add("train_step_loss_rel", step_loss_err, 1e-4);
    auto sr = m_ref.snapshot();
    auto sg = m_gpu.snapshot();
    std::map<SplatId, const Splat<float>*> by_id;
    for (const auto& p : sg) by_id[p.splat.id] = &p.splat;
    double mu_err = 0, op_err = 0, lost = 0;
    for (const auto& p : sr) {
        auto it = by_id.find(p.splat.id);
        if (it == by_id.end()) {
            lost += 1;
            continue;
        }
        mu_err = std::max(mu_err, (double)(p.splat.mu - it->second->mu).cwiseAbs().maxCoeff());
        op_err = std::max(op_err, (double)std::fabs(p.splat.opacity_logit - it->second->opacity_logit));
    }
    rep.add("snapshot_lost", lost + std::fabs(double(sr.size()) - double(sg.size())), 0);
    // an Adam step moves a parameter by about lr; a gradient whose sign differs
    // below the noise floor can put two steps 4 lr apart
    rep.add("snapshot_mu_max_abs", mu_err, 4 * 1.6e-4);
    rep.add("snapshot_opacity_max_abs", op_err, 4 * 0.025);
    // snapshot(checkpoint_path): the worker answers MsgCheckpoint with a plain
    // snapshot (worker.hpp:147), so a path must not change the result
    rep.add("snapshot_checkpoint_size_err", std::fabs(double(m_gpu.snapshot("unused.ckpt").size()) - double(sg.size())), 0);
    m_gpu.repartition();
    rep.add("repartition_epoch_err", std::fabs(double(m_gpu.epoch()) - 1.0), 0);

    rep.json += std::string(", \"ok\": ") + (rep.ok ? "true" : "false") + "}";
    std::printf("%s\n", rep.json.c_str());
    return rep.ok ? 0 : 1;
}
