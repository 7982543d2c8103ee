// Host-side C++ of the drop-in: KD partition (partition.hpp:93-251),
// synthetic inputs (io.hpp:421-543 with libstdc++ <random>, so streams are
// bit-identical to the reference's), configuration defaults.  Compiled with
// -ffp-contract=off; the float op order follows the Eigen evaluation rules of
// oracle/eigen_shim/Eigen/Core (dgs_math.cuh helpers).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <sstream>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/dgs_capi.h"
#include "capi_internal.h"
#include "dgs_math.cuh"

using namespace dgs_b200;

namespace {

struct Region {
    std::vector<dgs_plane> planes;
    float aabb_min[3], aabb_max[3];
};

struct Pt {
    float v[3];
};

/// partition.hpp:93-153 kd_split.
void kd_split(std::vector<Pt>& pts, size_t begin, size_t end, int depth, int target, Region region,
              std::vector<Region>& leaves) {
    if (depth == target) {
        leaves.push_back(std::move(region));
        return;
    }
    int axis = 0;
    float plane = 0.0f;
    if (begin < end) {
        float lo[3], hi[3];
        for (int a = 0; a < 3; ++a) lo[a] = hi[a] = pts[begin].v[a];
        for (size_t i = begin + 1; i < end; ++i)
            for (int a = 0; a < 3; ++a) {
                lo[a] = std::min(lo[a], pts[i].v[a]);
                hi[a] = std::max(hi[a], pts[i].v[a]);
            }
        float ext[3];
        for (int a = 0; a < 3; ++a) ext[a] = hi[a] - lo[a];
        float m = ext[0];  // maxCoeff(&axis): first maximum
        for (int a = 1; a < 3; ++a)
            if (ext[a] > m) {
                m = ext[a];
                axis = a;
            }
        std::vector<float> coords(end - begin);
        for (size_t i = begin; i < end; ++i) coords[i - begin] = pts[i].v[axis];
        const size_t n = coords.size();
        if (n % 2 == 0) {
            std::nth_element(coords.begin(), coords.begin() + n / 2, coords.end());
            const float upper = coords[n / 2];
            const float lower = *std::max_element(coords.begin(), coords.begin() + n / 2);
            plane = (lower + upper) / 2.0f;
        } else {
            std::nth_element(coords.begin(), coords.begin() + n / 2, coords.end());
            plane = coords[n / 2];
        }
    } else {
        const float lo = region.aabb_min[axis], hi = region.aabb_max[axis];
        plane = (std::isfinite(lo) && std::isfinite(hi)) ? (lo + hi) / 2.0f
                : std::isfinite(lo)                      ? lo + 1.0f
                : std::isfinite(hi)                      ? hi - 1.0f
                                                         : 0.0f;
    }
    size_t mid = begin;
    for (size_t i = begin; i < end; ++i)
        if (pts[i].v[axis] < plane) std::swap(pts[i], pts[mid++]);
    Region left = region, right = std::move(region);
    dgs_plane lp{};
    lp.n[axis] = 1.0f;
    lp.d = -plane;
    lp.closed = 0;
    left.planes.push_back(lp);
    left.aabb_max[axis] = std::min(left.aabb_max[axis], plane);
    dgs_plane rp{};
    rp.n[axis] = -1.0f;
    rp.d = plane;
    rp.closed = 1;
    right.planes.push_back(rp);
    right.aabb_min[axis] = std::max(right.aabb_min[axis], plane);
    kd_split(pts, begin, mid, depth + 1, target, std::move(left), leaves);
    kd_split(pts, mid, end, depth + 1, target, std::move(right), leaves);
}

/// Vec4<float>::normalized() (contiguous packet order, see Eigen shim).
void normalize4(float q[4]) {
    const float n2 = dot4(q, q);
    if (n2 > 0.0f) {
        const float s = std::sqrt(n2);
        for (int a = 0; a < 4; ++a) q[a] = q[a] / s;
    }
}

void normalize3(float v[3]) {
    const float n2 = dot3(v[0], v[1], v[2], v[0], v[1], v[2]);
    if (n2 > 0.0f) {
        const float s = std::sqrt(n2);
        for (int a = 0; a < 3; ++a) v[a] = v[a] / s;
    }
}

void cross3(const float a[3], const float b[3], float o[3]) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}

}  // namespace

extern "C" {

int dgs_version(void) { return DGS_CAPI_VERSION; }

void dgs_default_render_options(dgs_render_options* o) {
    o->truncation_radius = 3.0;
    o->near_plane = 0.01;
    o->sigma_clamp = 0.99;
    o->cov2d_regularization = 0.3;
    o->stop_threshold = 1e-4;
    o->sh_degree = -1;
    o->indicator_enabled = 1;
    o->camera_z_order = 0;
    o->grad_skip_eps = 1e-5;  // Eigen NumTraits<float>::dummy_precision() (isZero default)
}

void dgs_oracle_render_options(dgs_render_options* o) {
    dgs_default_render_options(o);
    o->stop_threshold = 0.0;
}

void dgs_default_train_config(dgs_train_config* c) {
    c->iterations = 2000;
    c->batch_size = 1;
    c->kd_depth = 0;
    c->lambda_ssim = 0.2;
    c->lr_position_start = 1.6e-4;
    c->lr_position_end = 1.6e-6;
    c->lr_sh_dc = 2.5e-3;
    c->lr_sh_rest = 2.5e-3 / 20.0;
    c->lr_opacity = 0.025;
    c->lr_scale = 5e-3;
    c->lr_rotation = 1e-3;
    c->adam_beta1 = 0.9;
    c->adam_beta2 = 0.999;
    c->adam_eps = 1e-15;
    c->grad_sync = 0;
    c->deterministic = 1;
}

double dgs_position_lr(const dgs_train_config* c, uint64_t step) {
    if (c->iterations == 0 || c->lr_position_start <= 0.0) return c->lr_position_start;
    if (step == 0) return c->lr_position_start;
    if (step >= c->iterations) return c->lr_position_end;
    const double frac = double(step) / double(c->iterations);
    return c->lr_position_start * std::pow(c->lr_position_end / c->lr_position_start, frac);
}

int dgs_build_kdtree(const float* centers, int64_t n, int32_t depth, dgs_plane* planes_out) {
    return dgs_guard([&] {
        if (n <= 0) throw std::invalid_argument("build_kdtree: empty point set");
        if (depth < 0) throw std::invalid_argument("build_kdtree: negative depth");
        if (depth > 16) throw std::invalid_argument("build_kdtree: depth > 16 unsupported");
        std::vector<Pt> pts((size_t)n);
        for (int64_t i = 0; i < n; ++i)
            for (int a = 0; a < 3; ++a) pts[i].v[a] = centers[3 * i + a];
        if (depth > 0) {
            float lo[3], hi[3];
            for (int a = 0; a < 3; ++a) lo[a] = hi[a] = pts[0].v[a];
            for (const auto& p : pts)
                for (int a = 0; a < 3; ++a) {
                    lo[a] = std::min(lo[a], p.v[a]);
                    hi[a] = std::max(hi[a], p.v[a]);
                }
            float m = hi[0] - lo[0];
            for (int a = 1; a < 3; ++a) m = std::max(m, hi[a] - lo[a]);
            if (m <= 0.0f) throw std::invalid_argument("degenerate point set");
        }
        Region root;
        for (int a = 0; a < 3; ++a) {
            root.aabb_min[a] = -INFINITY;
            root.aabb_max[a] = INFINITY;
        }
        std::vector<Region> leaves;
        kd_split(pts, 0, pts.size(), 0, depth, root, leaves);
        for (size_t k = 0; k < leaves.size(); ++k)
            for (int i = 0; i < depth; ++i) planes_out[k * depth + i] = leaves[k].planes[i];
    });
}

int dgs_assign_subsets(const dgs_plane* planes, int32_t k_count, int32_t ppk, const float* mu,
                       const float* log_scale, int64_t n, double d_multiplier, uint8_t* member_mask) {
    return dgs_guard([&] {
        const float mult = (float)d_multiplier;
        for (int64_t i = 0; i < n; ++i) {
            const float s0 = glibc_expf(log_scale[3 * i]), s1 = glibc_expf(log_scale[3 * i + 1]),
                        s2 = glibc_expf(log_scale[3 * i + 2]);
            float smax = s0;
            if (s1 > smax) smax = s1;
            if (s2 > smax) smax = s2;
            const float di = mult * smax;
            for (int k = 0; k < k_count; ++k) {
                bool member = true;
                for (int j = 0; j < ppk; ++j) {
                    const dgs_plane& p = planes[k * ppk + j];
                    const float v = dot3(p.n[0], p.n[1], p.n[2], mu[3 * i], mu[3 * i + 1], mu[3 * i + 2]) + p.d;
                    if (v > di) {
                        member = false;
                        break;
                    }
                }
                member_mask[i * k_count + k] = member ? 1 : 0;
            }
        }
    });
}

int dgs_synth_splats(int32_t count, int32_t clustered, int32_t sh_degree, double extent, uint64_t seed,
                     dgs_splats* out) {
    return dgs_guard([&] {
        if (sh_degree < 0 || sh_degree > 3) throw std::invalid_argument("synth: sh_degree must be 0..3");
        const int n_coeff = (sh_degree + 1) * (sh_degree + 1);
        if (out->sh_coeffs != n_coeff || out->n < count) throw std::invalid_argument("synth: output too small");
        std::mt19937_64 rng(seed);
        std::uniform_real_distribution<double> u01(0.0, 1.0);
        std::normal_distribution<double> gauss;
        const double e = extent;
        const double spacing = 1.1 * e * std::pow(double(std::max(count, 1)), -1.0 / 3.0);
        const double kC0 = DGS_SH_C0;
        for (int i = 0; i < count; ++i) {
            if (out->id) out->id[i] = (uint64_t)i;
            float* mu = out->mu + 3 * (size_t)i;
            if (clustered && u01(rng) < 0.9) {
                const double c[3] = {-0.55 * e, -0.55 * e, -0.55 * e};
                for (int a = 0; a < 3; ++a) mu[a] = (float)std::clamp(c[a] + gauss(rng) * 0.12 * e, -e, e);
            } else {
                for (int a = 0; a < 3; ++a) mu[a] = (float)((2 * u01(rng) - 1) * e);
            }
            const double base = spacing * (0.6 + 0.9 * u01(rng));
            for (int a = 0; a < 3; ++a) out->log_scale[3 * (size_t)i + a] = (float)std::log(base * (0.7 + 0.6 * u01(rng)));
            float q[4];
            for (int a = 0; a < 4; ++a) q[a] = (float)gauss(rng);
            normalize4(q);
            for (int a = 0; a < 4; ++a) out->rotation[4 * (size_t)i + a] = q[a];
            const double alpha = 0.5 + 0.45 * u01(rng);
            out->opacity_logit[i] = (float)std::log(alpha / (1.0 - alpha));
            float* sh = out->sh + (size_t)i * n_coeff * 3;
            for (int c = 0; c < n_coeff * 3; ++c) sh[c] = 0.0f;
            for (int a = 0; a < 3; ++a) sh[a] = (float)((0.1 + 0.8 * u01(rng) - 0.5) / kC0);
        }
    });
}

int dgs_ring_camera(int32_t width, int32_t height, double fov_deg, double ring_radius, double extent,
                    int32_t n_views, int32_t i, dgs_camera* out) {
    return dgs_guard([&] {
        const double a = 2.0 * M_PI * double(i) / double(n_views);
        const double h = 0.55 * extent * ((i % 2 == 0) ? 1.0 : -1.0);
        const float pos[3] = {(float)(ring_radius * extent * std::cos(a)), (float)h,
                              (float)(ring_radius * extent * std::sin(a))};
        out->width = width;
        out->height = height;
        out->fx = out->fy = (float)(width / (2.0 * std::tan(fov_deg * M_PI / 360.0)));
        out->cx = (float)width / 2.0f;
        out->cy = (float)height / 2.0f;
        float z[3] = {-pos[0], -pos[1], -pos[2]};
        normalize3(z);
        float up[3] = {0.0f, 1.0f, 0.0f};
        if (std::abs(double(dot3(z[0], z[1], z[2], up[0], up[1], up[2]))) > 0.99) {
            up[0] = 1.0f;
            up[1] = 0.0f;
        }
        float x[3], y[3];
        cross3(z, up, x);
        normalize3(x);
        cross3(z, x, y);
        const float r[9] = {x[0], x[1], x[2], y[0], y[1], y[2], z[0], z[1], z[2]};
        auto R = [&](int rr, int cc) { return r[rr * 3 + cc]; };
        float q[4];
        const float tr = sum3(R(0, 0), R(1, 1), R(2, 2));
        if (tr > 0.0f) {
            const float s = std::sqrt(tr + 1.0f) * 2.0f;
            q[0] = s / 4.0f;
            q[1] = (R(2, 1) - R(1, 2)) / s;
            q[2] = (R(0, 2) - R(2, 0)) / s;
            q[3] = (R(1, 0) - R(0, 1)) / s;
        } else if (R(0, 0) > R(1, 1) && R(0, 0) > R(2, 2)) {
            const float s = std::sqrt(1.0f + R(0, 0) - R(1, 1) - R(2, 2)) * 2.0f;
            q[0] = (R(2, 1) - R(1, 2)) / s;
            q[1] = s / 4.0f;
            q[2] = (R(0, 1) + R(1, 0)) / s;
            q[3] = (R(0, 2) + R(2, 0)) / s;
        } else if (R(1, 1) > R(2, 2)) {
            const float s = std::sqrt(1.0f + R(1, 1) - R(0, 0) - R(2, 2)) * 2.0f;
            q[0] = (R(0, 2) - R(2, 0)) / s;
            q[1] = (R(0, 1) + R(1, 0)) / s;
            q[2] = s / 4.0f;
            q[3] = (R(1, 2) + R(2, 1)) / s;
        } else {
            const float s = std::sqrt(1.0f + R(2, 2) - R(0, 0) - R(1, 1)) * 2.0f;
            q[0] = (R(1, 0) - R(0, 1)) / s;
            q[1] = (R(0, 2) + R(2, 0)) / s;
            q[2] = (R(1, 2) + R(2, 1)) / s;
            q[3] = s / 4.0f;
        }
        normalize4(q);
        for (int k = 0; k < 4; ++k) out->q_wc[k] = q[k];
        for (int k = 0; k < 3; ++k) out->t_wc[k] = -dot3(R(k, 0), R(k, 1), R(k, 2), pos[0], pos[1], pos[2]);
    });
}

int dgs_perturb_splats(dgs_splats* s, uint64_t seed) {
    return dgs_guard([&] {
        std::mt19937_64 rng(seed);
        std::normal_distribution<double> g;
        for (int64_t i = 0; i < s->n; ++i) {
            float gm[3];
            for (int a = 0; a < 3; ++a) gm[a] = (float)g(rng);
            for (int a = 0; a < 3; ++a) s->mu[3 * i + a] = s->mu[3 * i + a] + gm[a] * 0.02f;
            s->opacity_logit[i] = s->opacity_logit[i] + (float)(0.3 * g(rng));
            float gs[3];
            for (int a = 0; a < 3; ++a) gs[a] = (float)g(rng);
            float* sh = s->sh + (size_t)i * s->sh_coeffs * 3;
            for (int a = 0; a < 3; ++a) sh[a] = sh[a] + gs[a] * 0.1f;
        }
    });
}

/* save_splats_ply (io.hpp:257-297): the 3DGS property convention, float32. */
int dgs_save_splats_ply(const dgs_splats* s, const char* path, int32_t binary) {
    return dgs_guard([&] {
        std::ofstream f(path, std::ios::binary);
        if (!f) throw std::runtime_error(std::string("save_splats_ply: cannot open ") + path);
        const int n_coeff = s->n ? s->sh_coeffs : 1;
        const int rest = 3 * (n_coeff - 1);
        f << "ply\nformat " << (binary ? "binary_little_endian" : "ascii") << " 1.0\n";
        f << "element vertex " << s->n << "\n";
        for (const char* p : {"x", "y", "z", "nx", "ny", "nz"}) f << "property float " << p << "\n";
        for (int a = 0; a < 3; ++a) f << "property float f_dc_" << a << "\n";
        for (int a = 0; a < rest; ++a) f << "property float f_rest_" << a << "\n";
        f << "property float opacity\n";
        for (int a = 0; a < 3; ++a) f << "property float scale_" << a << "\n";
        for (int a = 0; a < 4; ++a) f << "property float rot_" << a << "\n";
        f << "end_header\n";
        std::vector<float> row;
        for (int64_t i = 0; i < s->n; ++i) {
            row.clear();
            for (int a = 0; a < 3; ++a) row.push_back(s->mu[3 * i + a]);
            for (int a = 0; a < 3; ++a) row.push_back(0.0f);  // normals unused
            for (int a = 0; a < 3; ++a) row.push_back(s->sh[(i * n_coeff) * 3 + a]);
            for (int a = 0; a < 3; ++a)  // f_rest channel-major
                for (int c = 1; c < n_coeff; ++c) row.push_back(s->sh[(i * n_coeff + c) * 3 + a]);
            row.push_back(s->opacity_logit[i]);
            for (int a = 0; a < 3; ++a) row.push_back(s->log_scale[3 * i + a]);
            for (int a = 0; a < 4; ++a) row.push_back(s->rotation[4 * i + a]);
            if (binary) {
                f.write(reinterpret_cast<const char*>(row.data()), std::streamsize(row.size() * sizeof(float)));
            } else {
                for (size_t q = 0; q < row.size(); ++q) f << (q ? " " : "") << row[q];
                f << "\n";
            }
        }
        if (!f) throw std::runtime_error(std::string("save_splats_ply: write failed for ") + path);
    });
}

/* Splat checkpoints written by dgs_save_splats_ply / the reference's
 * save_splats_ply (binary_little_endian float32 or ascii, any property order
 * of the 3DGS convention; load_ply's splat mode, io.hpp:85-255).  out == NULL:
 * only *n and *sh_coeffs are returned.  Ids are 0..n-1 (io.hpp:236-238). */
int dgs_load_splats_ply(const char* path, dgs_splats* out, int64_t* n_out, int32_t* sh_coeffs_out) {
    return dgs_guard([&] {
        std::ifstream in(path, std::ios::binary);
        if (!in) throw std::runtime_error(std::string("load_ply: cannot open ") + path);
        std::string line;
        std::getline(in, line);
        if (line != "ply") throw std::runtime_error("ply: missing magic");
        bool binary = false, in_vertex = false;
        int64_t count = -1;
        std::vector<std::string> props;
        while (std::getline(in, line)) {
            std::istringstream ls(line);
            std::string w;
            ls >> w;
            if (w == "format") {
                std::string fmt;
                ls >> fmt;
                if (fmt == "binary_little_endian") binary = true;
                else if (fmt != "ascii") throw std::runtime_error("ply: unsupported format " + fmt);
            } else if (w == "element") {
                std::string name;
                ls >> name >> count;
                in_vertex = name == "vertex";
                if (!in_vertex) throw std::runtime_error("ply: only a vertex element is supported here");
            } else if (w == "property" && in_vertex) {
                std::string type, name;
                ls >> type >> name;
                if (type != "float" && type != "float32") throw std::runtime_error("ply: float32 properties only");
                props.push_back(name);
            } else if (w == "end_header") {
                break;
            }
        }
        if (count < 0) throw std::runtime_error("ply: no vertex element");
        auto index_of = [&](const std::string& nme) {
            for (size_t q = 0; q < props.size(); ++q)
                if (props[q] == nme) return int(q);
            return -1;
        };
        size_t rest = 0;
        while (index_of("f_rest_" + std::to_string(rest)) >= 0) ++rest;
        int degree = -1;
        for (int d = 0; d <= 3; ++d)
            if (rest == size_t(3 * ((d + 1) * (d + 1) - 1))) degree = d;
        if (degree < 0) throw std::runtime_error("ply: f_rest count does not match any SH degree <= 3");
        const int n_coeff = (degree + 1) * (degree + 1);
        if (n_out) *n_out = count;
        if (sh_coeffs_out) *sh_coeffs_out = n_coeff;
        if (!out) return;
        if (out->n < count || out->sh_coeffs != n_coeff) throw std::invalid_argument("load_ply: output too small");
        const int ix = index_of("x"), iy = index_of("y"), iz = index_of("z"), iop = index_of("opacity");
        int isc[3], irt[4], idc[3];
        for (int a = 0; a < 3; ++a) isc[a] = index_of("scale_" + std::to_string(a));
        for (int a = 0; a < 4; ++a) irt[a] = index_of("rot_" + std::to_string(a));
        for (int a = 0; a < 3; ++a) idc[a] = index_of("f_dc_" + std::to_string(a));
        if (ix < 0 || iy < 0 || iz < 0) throw std::runtime_error("ply: vertex element lacks x/y/z");
        if (iop < 0 || isc[2] < 0 || irt[3] < 0 || idc[2] < 0)
            throw std::runtime_error("ply: incomplete splat property set");
        std::vector<float> row(props.size());
        for (int64_t i = 0; i < count; ++i) {
            if (binary) {
                in.read(reinterpret_cast<char*>(row.data()), std::streamsize(row.size() * sizeof(float)));
            } else {
                for (auto& v : row) in >> v;
            }
            if (!in) throw std::runtime_error("ply: truncated vertex data");
            if (out->id) out->id[i] = (uint64_t)i;
            out->mu[3 * i] = row[ix];
            out->mu[3 * i + 1] = row[iy];
            out->mu[3 * i + 2] = row[iz];
            for (int a = 0; a < 3; ++a) out->log_scale[3 * i + a] = row[isc[a]];
            for (int a = 0; a < 4; ++a) out->rotation[4 * i + a] = row[irt[a]];
            out->opacity_logit[i] = row[iop];
            for (int a = 0; a < 3; ++a) out->sh[(i * n_coeff) * 3 + a] = row[idc[a]];
            for (int c = 1; c < n_coeff; ++c)
                for (int a = 0; a < 3; ++a)
                    out->sh[(i * n_coeff + c) * 3 + a] =
                        row[index_of("f_rest_" + std::to_string(size_t(a) * (n_coeff - 1) + (c - 1)))];
        }
    });
}

}  // extern "C"
