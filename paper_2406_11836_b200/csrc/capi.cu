// C-ABI of libdgs_b200.so: device context, subset state, and the training
// step orchestration (Manager<float>::train_step, manager.hpp:313-386, with
// the worker side WorkerCore::dispatch, worker.hpp:62-167).  Parameters,
// optimizer moments and every per-view buffer stay resident in HBM; the host
// only passes cameras, targets and options.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>
#include <cstring>
#include <iterator>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "../../include/dgs_capi.h"
#include "capi_internal.h"
#include "kernels.h"
#include "nccl_dyn.h"

namespace dgs_b200 {

static thread_local std::string g_last_error;
void set_last_error(const std::string& msg) { g_last_error = msg; }

void ensure_smem_attr(const void* func, int bytes) {
    // per (device, kernel): the largest size set so far; a launch asking for
    // more raises the attribute again (it is a limit, not a reservation)
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, int> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) throw CudaError(std::string("CUDA error: ") + cudaGetErrorString(e) + " (cudaGetDevice)");
    std::lock_guard<std::mutex> lock(mu);
    auto it = done.find({dev, func});
    if (it != done.end() && it->second >= bytes) return;
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess)
        throw CudaError(std::string("CUDA error: ") + cudaGetErrorString(e) + " (cudaFuncSetAttribute, " +
                        std::to_string(bytes) + " B dynamic shared memory)");
    done[{dev, func}] = bytes;
}

#define CK(call)                                                                                 \
    do {                                                                                         \
        cudaError_t e_ = (call);                                                                 \
        if (e_ != cudaSuccess)                                                                   \
            throw CudaError(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #call); \
    } while (0)
#define NK(call)                                                                                       \
    do {                                                                                               \
        ncclResult_t r_ = (call);                                                                      \
        if (r_ != ncclSuccess) throw NcclError(std::string("NCCL error: ") + nccl().GetErrorString(r_)); \
    } while (0)

const NcclApi& nccl() {
    static NcclApi api{};
    static bool loaded = false;
    if (!loaded) {
        // RTLD_NOLOAD first: reuse the NCCL torch already mapped, if any.
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) throw NcclError(std::string("cannot load libnccl.so.2: ") + dlerror());
        auto sym = [&](const char* n) {
            void* f = dlsym(h, n);
            if (!f) throw NcclError(std::string("libnccl.so.2 lacks ") + n);
            return f;
        };
        api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
        api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
        api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
        api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
        api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
        api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
        api.Send = (decltype(api.Send))sym("ncclSend");
        api.Recv = (decltype(api.Recv))sym("ncclRecv");
        api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
        loaded = true;
    }
    return api;
}

/// Bumped whenever any device buffer is (re)allocated or freed.
std::atomic<uint64_t> g_buffer_epoch{0};

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) {
            cudaFree(p);
            g_buffer_epoch.fetch_add(1);
        }
    }
    T* ensure(size_t count) {
        if (count > n || p == nullptr) {
            g_buffer_epoch.fetch_add(1);  // captured step graphs hold device pointers: they must be re-captured
            if (p) CK(cudaFree(p));
            p = nullptr;
            const size_t c = std::max<size_t>(count, 1);
            CK(cudaMalloc(&p, c * sizeof(T)));
            n = c;
        }
        return p;
    }
};

struct ViewSlot {
    DevBuf<SplatRec> recs;
    DevBuf<uint32_t> rect, counts, rkey, dmax, pair_val, pair_val_alt;
    DevBuf<uint16_t> pair_tile, pair_tile_alt;
    DevBuf<float2> ext;
    DevBuf<uint2> rect_sorted;
    DevBuf<uint32_t> sort_keys_alt, sort_vals, sort_vals_alt, scan, ovf_list, ovf_count;
    DevBuf<int> err;
    DevBuf<uint2> ranges;
    DevBuf<uint32_t> tile_order;
    DevBuf<uint8_t> temp, ovf_flag;
    DevBuf<float4> ct, grad_ct;
    DevBuf<double> cd;  // double colour sums for the backward suffix
    DevBuf<uint16_t> rec_pos;  // composite records (kernels.h CompRecords)
    DevBuf<float> shjac;       // [10][ld] SH colour Jacobian + clamp mask (ViewBins::shjac)
    DevBuf<uint16_t> rec_cnt;
    DevBuf<uint8_t> rec_replay;
    DevBuf<uint32_t> blkp;     // K1 per-block partials (ViewBins::blk_part)
    bool rec_valid = false;  // the last forward of this slot wrote records
    CompRecords crec() const {
        CompRecords r;
        r.pos = rec_pos.p;
        r.cnt = rec_cnt.p;
        r.tile_replay = rec_replay.p;
        return r;
    }
    int64_t pair_cap = 0;
    int64_t pairs_max = 0;  // largest pair count of the eager steps (sizes graph_cap)
    int64_t graph_cap = 0;  // pair slots sorted by a captured step (<= pair_cap)
    size_t temp_bytes = 0;
    ViewBins vb;
    ViewParams vp{};
};

struct SubsetState {
    int k = 0;
    int64_t n = 0;
    int sh_coeffs = 16;
    int rows = 59;
    size_t ld = 0;
    DevBuf<float> P, M, V, G, g2d, rec;
    DevBuf<float> saved;  // dgs_state_save: (P, M, V) rollback copy in HBM
    uint64_t saved_step = 0;
    DevBuf<unsigned long long> g2q;  // deterministic mode: fixed-point adjoint sums [9][lo|hi][ld], zero between uses
    DevBuf<uint32_t> ids32;
    std::vector<uint64_t> ids64;
    uint64_t adam_step = 0, epoch = 0;

    std::vector<std::unique_ptr<ViewSlot>> slots;
    ViewSlot& slot(int v) {
        while ((int)slots.size() <= v) slots.emplace_back(new ViewSlot());
        return *slots[v];
    }
};

/// Pinned host block the step's results land in (one per context, fixed
/// capacity so a captured graph's copy targets never move).
constexpr int kTailMaxBatch = 64, kTailMaxSlices = 64, kTailMaxLocal = 64;
struct StepTail {
    double sums[3 * kTailMaxBatch * kTailMaxSlices];
    size_t nsums = 0;
    BlendStats st[2];
    int bad = INT_MAX, abort = 0;
    uint32_t ovf[kTailMaxLocal * kTailMaxBatch], pairs[kTailMaxLocal * kTailMaxBatch],
        visible[kTailMaxLocal * kTailMaxBatch];
    int err[kTailMaxLocal * kTailMaxBatch];
    double px[kTailMaxBatch];
    int batch = 0, slices = 0, nlocal = 0;
    uint64_t nccl_bytes = 0, launches = 0, comm_bytes = 0;
};
/// Event pairs around every stage launch, resolved at the next sync point.
struct StageTimer {
    static constexpr int kStages = 10;
    bool on = false;
    double ms[kStages] = {};
    uint64_t count[kStages] = {};
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
    std::vector<cudaEvent_t> pool;
    cudaEvent_t get() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        return e;
    }
    void resolve() {
        for (auto& p : pending) {
            float t = 0.0f;
            CK(cudaEventSynchronize(p.second.second));
            CK(cudaEventElapsedTime(&t, p.second.first, p.second.second));
            ms[p.first] += t;
            count[p.first] += 1;
            pool.push_back(p.second.first);
            pool.push_back(p.second.second);
        }
        pending.clear();
    }
    ~StageTimer() {
        for (auto& p : pending) {
            cudaEventDestroy(p.second.first);
            cudaEventDestroy(p.second.second);
        }
        for (auto e : pool) cudaEventDestroy(e);
    }
};

/// Stage scope: records start/stop events when profiling is on; end() (or
/// the destructor) closes it.
struct Stage {
    StageTimer& t;
    int id;
    cudaStream_t s;
    cudaEvent_t a = nullptr;
    Stage(StageTimer& t_, int id_, cudaStream_t s_) : t(t_), id(id_), s(s_) {
        if (t.on) {
            a = t.get();
            CK(cudaEventRecord(a, s));
        }
    }
    void end() {
        if (a) {
            cudaEvent_t b = t.get();
            cudaEventRecord(b, s);
            t.pending.push_back({id, {a, b}});
            a = nullptr;
        }
    }
    ~Stage() { end(); }
};
enum { kStPre = 0, kStBin, kStFwd, kStMerge, kStLoss, kStMergeBwd, kStBwd, kStProjBwd, kStAdam, kStExchange };

/// Pinned host scalars read back once per forward (one stream sync).
struct HostScalars {
    int err;
    uint32_t pairs;
    uint32_t visible;
};

struct Ctx {
    int device = 0, rank = 0, world = 1;
    bool host_xfer = false;        // exchange through host callbacks instead of NCCL (tests)
    dgs_host_transport xfer_cb{};
    HostScalars* hs = nullptr;  // cudaHostAlloc'd
    StageTimer timer;
    cudaStream_t stream = nullptr;
    ncclComm_t comm = nullptr;
    Table table{};
    bool table_set = false;
    // the manager's partition epoch (MsgRenderTask::epoch, manager.hpp:276); once
    // set, every local subset must carry it (worker.hpp:63)
    uint64_t epoch = 0;
    bool epoch_set = false;
    DevBuf<Table> table_dev;
    dgs_render_options ro_in{};
    dgs_train_config cfg{};
    RenderOpts ro{};
    std::map<int, std::unique_ptr<SubsetState>> subsets;
    DevBuf<float> merged, grad_rgb, targets, staging, kern;
    DevBuf<float> tgt_stage;                  // host targets prefetched on copy_stream (HWC windows, all views)
    cudaStream_t copy_stream = nullptr;       // H2D of host targets, overlapped with the forward
    cudaEvent_t copy_done = nullptr;
    // batch > 1: view v's exchange / merge / loss / merge adjoint / exchange-back
    // chain runs on xstream while view v+1 renders on `stream`
    cudaStream_t xstream = nullptr;
    DevBuf<int> abort;                        // per step: non-zero makes K10 skip (zero quaternion, pair overflow)
    bool capturing = false;                   // the step is being recorded into a CUDA graph (no host round trips)
    StepTail* tail = nullptr;                 // pinned: the step's results (train_step_body / finish_step)
    // dgs_set_graph_mode: train steps replayed as CUDA graphs, one per (views, targets, bg) key
    bool graph_mode = false;
    uint64_t graph_version = 0;               // bumped by every call that changes what a step launches
    struct CachedStep {
        std::vector<uint8_t> key;
        cudaGraph_t graph = nullptr;  // kept: its K10 nodes get this step's AdamParams at every replay
        cudaGraphExec_t exec = nullptr;
        struct AdamNode {
            cudaGraphNode_t node;
            int subset, ap_index;
        };
        std::vector<AdamNode> adam;
    };
    std::vector<CachedStep> graphs;
    std::vector<std::vector<uint8_t>> warmed;  // keys with one eager step done (pair maxima learnt)
    static void free_step(CachedStep& g) {
        if (g.exec) cudaGraphExecDestroy(g.exec);
        if (g.graph) cudaGraphDestroy(g.graph);
        g.graph = nullptr;
        g.exec = nullptr;
    }
    void drop_graphs() {
        for (auto& g : graphs) free_step(g);
        graphs.clear();
        warmed.clear();
    }
    std::vector<cudaEvent_t> view_done;       // forward of view v finished (stream -> xstream)
    cudaEvent_t chain_done = nullptr;         // every view's chain finished (xstream -> stream)
    // pageable host targets: a helper thread copies them into this pinned
    // buffer chunk by chunk and queues each chunk's H2D, while the forward runs
    float* pin_stage = nullptr;
    size_t pin_cap = 0;
    std::thread stager;
    std::string stager_err;
    DevBuf<double> block_sums, sums;
    DevBuf<const float4*> partial_ptrs;
    DevBuf<float4*> grad_ptrs;
    DevBuf<float4> scratch_maps, scratch_grads;
    DevBuf<float4> xrecv, xgrad;   // sliced exchange buffers (K x halo rows, K x owned rows)
    DevBuf<float> targets_win;
    int virtual_slices = 1;        // single-rank sliced mode (tests the multi-rank manager path)
    bool collect_stats = false;    // blend evaluation/contribution counters (costs ~5% in the blends)
    bool records = true;           // forward composite records -> record-walk backward (else ring replay)
    // shared replicas for config.grad_sync (rebuilt after every load / repartition)
    bool shared_dirty = true;
    DevBuf<uint64_t> sh_keys;
    DevBuf<uint32_t> sh_reps, sh_starts;
    int sh_slots = 0, sh_nrep = 0;
    DevBuf<float*> gsync_G, gsync_G2;  // grad_sync: per-subset gradient rows (by subset id / by local order)
    DevBuf<size_t> gsync_ld, gsync_ld2;
    // cross-rank variant (world > 1): the globally sorted shared replicas
    DevBuf<uint64_t> xs_keys;                 // [S] id << 8 | k
    DevBuf<uint32_t> xs_g, xs_src, xs_pos;    // [S] global replica index, row in the gathered rows; my entries
    DevBuf<uint8_t> xs_mine;                  // [S] held by this rank
    DevBuf<uint32_t> xs_offs;                 // local replica offsets (ascending k)
    std::vector<uint64_t> xs_count;           // shared entries held per rank
    uint32_t xs_base = 0;
    int xs_S = 0, xs_nmine = 0;
    DevBuf<BlendStats> stats;
    DevBuf<int> bad;
    uint64_t launches = 0;
};

namespace {

RenderOpts to_render_opts(const dgs_render_options& o) {
    RenderOpts r;
    r.trunc = (float)o.truncation_radius;
    r.near_plane = (float)o.near_plane;
    r.sigma_clamp = (float)o.sigma_clamp;
    r.cov_reg = (float)o.cov2d_regularization;
    r.stop = (float)o.stop_threshold;
    r.sh_degree = o.sh_degree;
    r.indicator_enabled = o.indicator_enabled;
    r.grad_skip_eps = (float)o.grad_skip_eps;
    r.zorder = o.camera_z_order ? 1 : 0;
    return r;
}

ViewParams view_params(const dgs_camera& c) {
    // Camera::validate (splat.hpp:49-54)
    if (c.width <= 0 || c.height <= 0) throw std::invalid_argument("camera: non-positive resolution");
    if (!(c.fx > 0.0f) || !(c.fy > 0.0f)) throw std::invalid_argument("camera: focal lengths must be positive");
    if (!(c.cx > 0.0f) || !(c.cx < (float)c.width) || !(c.cy > 0.0f) || !(c.cy < (float)c.height))
        throw std::invalid_argument("camera: principal point outside image");
    ViewParams vp;
    if (!make_view_params(c.width, c.height, c.fx, c.fy, c.cx, c.cy, c.q_wc, c.t_wc, &vp))
        throw std::domain_error("zero quaternion");
    return vp;
}

Subspace gate_of(const Ctx& ctx, int k) {
    if (!ctx.table_set || k < 0 || k >= ctx.table.k_count) throw std::invalid_argument("unknown subset " + std::to_string(k));
    return ctx.table.sub[k];
}

SubsetState& subset(Ctx& ctx, int k) {
    auto it = ctx.subsets.find(k);
    if (it == ctx.subsets.end()) throw std::invalid_argument("subset " + std::to_string(k) + " is not loaded on this rank");
    return *it->second;
}

/// WorkerCore::dispatch(MsgRenderTask) (worker.hpp:63): a render task carries
/// the manager's epoch and a worker holding another partition refuses it.
void check_epoch(const Ctx& ctx, const SubsetState& S) {
    if (ctx.epoch_set && S.epoch != ctx.epoch) throw std::runtime_error("partition epoch mismatch");
}

__global__ void k_hwc_to_planar(const float* __restrict__ in, float* __restrict__ out, size_t px) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= px) return;
    out[i] = in[3 * i];
    out[px + i] = in[3 * i + 1];
    out[2 * px + i] = in[3 * i + 2];
}

__global__ void k_planar_to_hwc(const float* __restrict__ in, float* __restrict__ out, size_t px) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= px) return;
    out[3 * i] = in[i];
    out[3 * i + 1] = in[px + i];
    out[3 * i + 2] = in[2 * px + i];
}

/// Field layout (per splat) -> SoA rows on the device.
void upload_fields(Ctx& ctx, SubsetState& S, const dgs_splats& f, float* dst) {
    const int64_t n = S.n;
    std::vector<float> h((size_t)S.rows * S.ld, 0.0f);
    for (int64_t i = 0; i < n; ++i) {
        for (int a = 0; a < 3; ++a) h[(size_t)(kRowMu + a) * S.ld + i] = f.mu[3 * i + a];
        for (int a = 0; a < 3; ++a) h[(size_t)(kRowLogScale + a) * S.ld + i] = f.log_scale[3 * i + a];
        for (int a = 0; a < 4; ++a) h[(size_t)(kRowRot + a) * S.ld + i] = f.rotation[4 * i + a];
        h[(size_t)kRowOpacity * S.ld + i] = f.opacity_logit[i];
        for (int c = 0; c < 3 * S.sh_coeffs; ++c) h[(size_t)(kRowSh + c) * S.ld + i] = f.sh[(size_t)i * 3 * S.sh_coeffs + c];
    }
    CK(cudaMemcpyAsync(dst, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice, ctx.stream));
    CK(cudaStreamSynchronize(ctx.stream));
}

void download_fields(Ctx& ctx, SubsetState& S, const float* src, dgs_splats* f) {
    if (f == nullptr) return;
    if (f->n < S.n || f->sh_coeffs != S.sh_coeffs) throw std::invalid_argument("store: output arrays too small");
    std::vector<float> h((size_t)S.rows * S.ld);
    CK(cudaMemcpyAsync(h.data(), src, h.size() * sizeof(float), cudaMemcpyDeviceToHost, ctx.stream));
    CK(cudaStreamSynchronize(ctx.stream));
    for (int64_t i = 0; i < S.n; ++i) {
        if (f->id) f->id[i] = S.ids64[i];
        for (int a = 0; a < 3; ++a) f->mu[3 * i + a] = h[(size_t)(kRowMu + a) * S.ld + i];
        for (int a = 0; a < 3; ++a) f->log_scale[3 * i + a] = h[(size_t)(kRowLogScale + a) * S.ld + i];
        for (int a = 0; a < 4; ++a) f->rotation[4 * i + a] = h[(size_t)(kRowRot + a) * S.ld + i];
        f->opacity_logit[i] = h[(size_t)kRowOpacity * S.ld + i];
        for (int c = 0; c < 3 * S.sh_coeffs; ++c) f->sh[(size_t)i * 3 * S.sh_coeffs + c] = h[(size_t)(kRowSh + c) * S.ld + i];
    }
}

struct StoreWords {
    static constexpr int kMax = 240;
    uint32_t n;
    uint32_t w[kMax];
};
__global__ void k_store_words(uint32_t* __restrict__ dst, const StoreWords v) {
    for (uint32_t i = threadIdx.x; i < v.n; i += blockDim.x) dst[i] = v.w[i];
}

/// Host->device copy of a small step-time value.  Eager: straight (a pageable
/// source is staged by the runtime before the call returns).  While a step is
/// being captured the value travels as a kernel argument of k_store_words,
/// baked into the graph: a memcpy node from host memory would queue on the H2D
/// copy engine behind the step's target upload (tens of MB) and stall the
/// forward until it drains.
void h2d(Ctx& ctx, void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (!ctx.capturing) {
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
        return;
    }
    if (bytes % 4 != 0 || (reinterpret_cast<uintptr_t>(dst) & 3) != 0)
        throw std::logic_error("graph capture: h2d of a non-word value");
    const uint32_t* w = static_cast<const uint32_t*>(src);
    for (size_t o = 0, nw = bytes / 4; o < nw; o += StoreWords::kMax) {
        StoreWords v{};
        v.n = (uint32_t)std::min<size_t>(StoreWords::kMax, nw - o);
        std::memcpy(v.w, w + o, v.n * 4);
        k_store_words<<<1, 256, 0, s>>>(static_cast<uint32_t*>(dst) + o, v);
        CK(cudaGetLastError());
        ++ctx.launches;
    }
}

/// partial_render for local subset S into view slot v (engine.hpp:44-52):
/// K1 projection, K2 binning, K4 blend (+ exact fallback).
void forward_subset(Ctx& ctx, SubsetState& S, int v, const ViewParams& vp, int dbg_cap = 0,
                    uint32_t* dbg_ids = nullptr, uint32_t* dbg_cnt = nullptr, BlendStats* stats = nullptr) {
    ViewSlot& vs = S.slot(v);
    const int64_t n = S.n;
    const int tiles = vp.tiles_x * vp.tiles_y;
    const size_t px = (size_t)vp.width * vp.height;
    vs.vp = vp;
    ViewBins& vb = vs.vb;
    vb.zorder = ctx.ro.zorder;
    if (tiles > 65535) throw std::invalid_argument("render: more than 65535 16x16 tiles (16-bit tile keys)");
    vb.shjac = vs.shjac.ensure((size_t)10 * S.ld);
    vb.recs = vs.recs.ensure(n);
    vb.rect = vs.rect.ensure(2 * n);
    vb.counts = vs.counts.ensure(n);
    vb.rkey = vs.rkey.ensure(n);
    vb.ext = vs.ext.ensure(n);
    vb.dmax_bits = vs.dmax.ensure(4);
    vb.blk_part = vs.blkp.ensure(preprocess_partials((int)n));
    vb.err_index = vs.err.ensure(1);
    vb.abort = ctx.abort.ensure(1);
    vb.ranges = vs.ranges.ensure(tiles);
    vb.tile_order = vs.tile_order.ensure(tiles);
    vs.sort_keys_alt.ensure(n);
    vs.sort_vals.ensure(n);
    vs.sort_vals_alt.ensure(n);
    vs.scan.ensure(n);
    vs.ct.ensure(px);
    vs.cd.ensure(3 * px);
    vs.ovf_flag.ensure(px);
    vs.ovf_list.ensure(px);
    vs.ovf_count.ensure(1);
    if (vs.pair_cap == 0) vs.pair_cap = std::max<int64_t>(4 * n + 1024, 1 << 16);
    auto alloc_pairs = [&]() {
        vb.pair_tile = vs.pair_tile.ensure(vs.pair_cap);
        vb.pair_val = vs.pair_val.ensure(vs.pair_cap);
        vs.pair_tile_alt.ensure(vs.pair_cap);
        vs.pair_val_alt.ensure(vs.pair_cap);
        const size_t tb = binning_temp_bytes((int)n, vs.pair_cap);
        vs.temp.ensure(tb);
        vs.temp_bytes = vs.temp.n;
    };
    alloc_pairs();
    const uint32_t dmax0[4] = {0u, 0x7f7fffffu, 0u, 0u};  // (max D, min range, visible count, max range)
    h2d(ctx, vb.dmax_bits, dmax0, sizeof(dmax0), ctx.stream);
    const int int_max = INT_MAX;
    h2d(ctx, vb.err_index, &int_max, 4, ctx.stream);
    launch_zero(vs.ovf_count.p, 4, ctx.stream);
    ++ctx.launches;
    {
        Stage st(ctx.timer, kStPre, ctx.stream);
        launch_preprocess((int)n, S.P.p, S.ld, S.sh_coeffs, S.ids32.p, vp, ctx.ro, vb, ctx.stream);
    }
    ctx.launches += 2;
    const bool capture = ctx.capturing;
    if (capture && n > 0) {
        // graph capture: no host round trip.  The pair count stays on the device and
        // the tile sort runs over the slot's graph capacity (learnt from the eager
        // steps); the zero-quaternion check and the visible count are read after
        // the replay (a zero quaternion or a pair overflow raises ctx.abort, which
        // keeps K10 from applying the step)
        if (vs.graph_cap <= 0 || vs.graph_cap > vs.pair_cap) throw std::logic_error("graph capture: no pair capacity");
        Stage st_bin(ctx.timer, kStBin, ctx.stream);
        run_binning((int)n, vp, vb, vs.pair_cap, vs.temp.p, vs.temp_bytes, vs.sort_keys_alt.p, vs.sort_vals.p,
                    vs.sort_vals_alt.p, vs.pair_tile_alt.p, vs.pair_val_alt.p, vs.scan.p, vs.rect_sorted.ensure(n),
                    &ctx.hs->pairs, ctx.stream, vs.graph_cap);
        ctx.launches += 4;
    }
    // zero-quaternion flag: rides along with the binning's pair-count readback
    if (!capture) {
        CK(cudaMemcpyAsync(&ctx.hs->err, vb.err_index, 4, cudaMemcpyDeviceToHost, ctx.stream));
        CK(cudaMemcpyAsync(&ctx.hs->visible, vb.dmax_bits + 2, 4, cudaMemcpyDeviceToHost, ctx.stream));
    }
    Stage st_bin(ctx.timer, kStBin, ctx.stream);
    int64_t P = 0;
    if (!capture) {
        P = run_binning((int)n, vp, vb, vs.pair_cap, vs.temp.p, vs.temp_bytes, vs.sort_keys_alt.p, vs.sort_vals.p,
                        vs.sort_vals_alt.p, vs.pair_tile_alt.p, vs.pair_val_alt.p, vs.scan.p, vs.rect_sorted.ensure(n),
                        &ctx.hs->pairs, ctx.stream);
        ctx.launches += 4;
        // the graph capacity of this slot: the largest pair count seen, plus 2 %
        vs.pairs_max = std::max<int64_t>(vs.pairs_max, P < 0 ? -P : P);
    }
    if (P < 0) {
        vs.pair_cap = (-P) + (-P) / 4 + 1024;
        alloc_pairs();
        P = run_binning((int)n, vp, vb, vs.pair_cap, vs.temp.p, vs.temp_bytes, vs.sort_keys_alt.p, vs.sort_vals.p,
                        vs.sort_vals_alt.p, vs.pair_tile_alt.p, vs.pair_val_alt.p, vs.scan.p, vs.rect_sorted.p,
                        &ctx.hs->pairs, ctx.stream);
        ctx.launches += 4;
        if (P < 0) throw std::runtime_error("binning: pair buffer sizing failed");
    }
    st_bin.end();
    if (!capture) {
        if (n <= 0) CK(cudaStreamSynchronize(ctx.stream));  // run_binning synced otherwise
        if (ctx.hs->err != INT_MAX) throw std::domain_error("zero quaternion");
        vb.visible = n > 0 ? ctx.hs->visible : 0;
    }
    // Composite records need tiles x 256 x kRecCap x 2 bytes per (subset, view)
    // slot (1.07 GB at 1080p, 4.2 GB at 4K).  A slot whose records would take
    // more than a quarter of the free HBM falls back to the ring-replay
    // backward (same results, slower) instead of failing the allocation.
    bool use_rec = ctx.records;
    const size_t rec_need = (size_t)tiles * kRecCap * kBlendThreads;  // u16 entries
    if (use_rec && (vs.rec_pos.p == nullptr || rec_need > vs.rec_pos.n)) {
        // any (re)allocation, e.g. a 1080p slot now rendering a 4K view
        const size_t need = rec_need * sizeof(uint16_t) + px * 2 + tiles;
        size_t free_b = 0, total_b = 0;
        CK(cudaMemGetInfo(&free_b, &total_b));
        use_rec = need <= free_b / 4;
    }
    if (use_rec) {
        vs.rec_pos.ensure(rec_need);
        vs.rec_cnt.ensure(px);
        vs.rec_replay.ensure(tiles);
    }
    vs.rec_valid = use_rec;
    CompRecords crec;
    if (use_rec) crec = vs.crec();
    Stage st_fwd(ctx.timer, kStFwd, ctx.stream);
    launch_blend_fwd(vp, ctx.ro, ctx.table.sub[S.k], vb, vs.ct.p, vs.ovf_flag.p, vs.ovf_list.p, vs.ovf_count.p,
                     dbg_ids, dbg_cnt, dbg_cap, stats, vs.cd.p, crec, ctx.stream);
    st_fwd.end();
    ++ctx.launches;
    {
        Stage st(ctx.timer, kStFwd, ctx.stream);
        launch_blend_fwd_fallback(vp, ctx.ro, ctx.table.sub[S.k], vb, vs.ct.p, vs.ovf_list.p, vs.ovf_count.p,
                                  dbg_ids, dbg_cnt, dbg_cap, vs.cd.p, ctx.stream);
        ++ctx.launches;
    }
}

/// partial_render_backward for subset S, view slot v (engine.hpp:74-88) up to
/// the pixel-space adjoints g2d (K8 + fallback).
/// TrainConfig::deterministic ("fixed-order reductions", optim.hpp:33): the
/// adjoints are summed as fixed point (2^-72 units) in one pass (kernels.h GradAcc),
/// then converted; a non-finite contribution is reported through ctx.bad like
/// K9's check.
/// fuse_convert: in deterministic mode leave the fixed-point sums in S.g2q for
/// K9 to convert (launch_project_bwd_adam's g2q) instead of a separate pass.
void backward_blend(Ctx& ctx, SubsetState& S, int v, BlendStats* stats, bool fuse_convert = false) {
    ViewSlot& vs = S.slot(v);
    S.g2d.ensure(9 * S.ld);
    const bool det = ctx.cfg.deterministic != 0;
    GradAcc acc;
    acc.f = S.g2d.p;
    acc.ld = S.ld;
    if (det) {
        if (S.g2q.p == nullptr || S.g2q.n < 18 * S.ld) {
            S.g2q.ensure(18 * S.ld);  // launch_fixed_to_float re-zeroes it after every use
            launch_zero(S.g2q.p, 18 * S.ld * sizeof(unsigned long long), ctx.stream);
            ++ctx.launches;
        }
        ctx.bad.ensure(1);
        acc.q = S.g2q.p;
        acc.bad = ctx.bad.p;
    } else {
        launch_zero(S.g2d.p, 9 * S.ld * sizeof(float), ctx.stream);
        ++ctx.launches;
    }
    Stage st(ctx.timer, kStBwd, ctx.stream);
    CompRecords crec;
    if (ctx.records && vs.rec_valid) crec = vs.crec();
    launch_blend_bwd(vs.vp, ctx.ro, ctx.table.sub[S.k], vs.vb, vs.ct.p, vs.cd.p, vs.grad_ct.p, vs.ovf_flag.p, crec,
                     acc, vs.ovf_list.p, vs.ovf_count.p, stats, ctx.stream);
    ctx.launches += det ? 6 : 3;
    if (det && !fuse_convert) {
        launch_fixed_to_float(acc, (int)S.n, ctx.stream);
        ++ctx.launches;
    }
}

AdamParams adam_params(const Ctx& ctx, const SubsetState& S, uint64_t step_after) {
    // worker.hpp:163-166: lr_pos from the pre-increment step, bias correction at step+1.
    const dgs_train_config& c = ctx.cfg;
    AdamParams ap;
    const float lr_pos = (float)dgs_position_lr(&c, step_after - 1);
    for (int r = 0; r < kMaxParamRows; ++r) ap.lr[r] = 0.0f;
    for (int a = 0; a < 3; ++a) {
        ap.lr[kRowMu + a] = lr_pos;
        ap.lr[kRowLogScale + a] = (float)c.lr_scale;
    }
    for (int a = 0; a < 4; ++a) ap.lr[kRowRot + a] = (float)c.lr_rotation;
    ap.lr[kRowOpacity] = (float)c.lr_opacity;
    for (int j = 0; j < S.sh_coeffs; ++j)
        for (int a = 0; a < 3; ++a) ap.lr[kRowSh + 3 * j + a] = j == 0 ? (float)c.lr_sh_dc : (float)c.lr_sh_rest;
    ap.b1 = (float)c.adam_beta1;
    ap.b2 = (float)c.adam_beta2;
    ap.eps = (float)c.adam_eps;
    ap.bc1 = 1.0f - std::pow(ap.b1, (float)step_after);  // optim.hpp:108-109: std::pow(float, float)
    ap.bc2 = 1.0f - std::pow(ap.b2, (float)step_after);
    ap.rbc1 = (float)(1.0 / (double)ap.bc1);
    ap.rbc2 = (float)(1.0 / (double)ap.bc2);
    ap.exact = c.deterministic ? 1 : 0;
    return ap;
}

/// K10's launch arguments for subset S this step: its AdamParams and the step's abort flag.
AdamArgs adam_args(Ctx& ctx, SubsetState& S, const int* abort) {
    AdamArgs a;
    a.ap = adam_params(ctx, S, S.adam_step + 1);
    a.exact = a.ap.exact;
    a.abort = abort;
    return a;
}

void check_bad(Ctx& ctx, SubsetState& S) {
    int bad = INT_MAX;
    CK(cudaMemcpyAsync(&bad, ctx.bad.p, 4, cudaMemcpyDeviceToHost, ctx.stream));
    CK(cudaStreamSynchronize(ctx.stream));
    if (bad != INT_MAX)
        throw std::runtime_error("partial_render_backward: non-finite gradient for splat id " +
                                 std::to_string(S.ids64[(size_t)bad]));
}

void reset_bad(Ctx& ctx) {
    ctx.bad.ensure(1);
    const int int_max = INT_MAX;
    h2d(ctx, ctx.bad.p, &int_max, 4, ctx.stream);
}

const float* ensure_kernel(Ctx& ctx) {
    if (ctx.kern.p == nullptr) {
        // loss.hpp:19-30 ssim_kernel<float>: double exp, cast, float sum, divide.
        float k[11];
        float sum = 0.0f;
        for (int i = 0; i < 11; ++i) {
            const double x = i - 11 / 2;
            k[i] = (float)std::exp(-x * x / (2.0 * 1.5 * 1.5));
            sum += k[i];
        }
        for (auto& v : k) v /= sum;
        ctx.kern.ensure(11);
        CK(cudaMemcpy(ctx.kern.p, k, sizeof(k), cudaMemcpyHostToDevice));
    }
    return ctx.kern.p;
}

/// Pixel-row slice owned by slice s of S (contiguous, balanced) and its
/// SSIM halo: the loss gradient at row y reads merged rows y-10..y+10
/// (two 5-row blur stages, loss.hpp:130-140).
struct SliceRows {
    int r0, r1, h0, h1;
};
constexpr int kSsimHalo = 10;
SliceRows slice_rows(int H, int S, int s) {
    SliceRows R;
    R.r0 = (int)((int64_t)H * s / S);
    R.r1 = (int)((int64_t)H * (s + 1) / S);
    R.h0 = std::max(0, R.r0 - kSsimHalo);
    R.h1 = std::min(H, R.r1 + kSsimHalo);
    return R;
}
/// Rank that owns KD subset k (contiguous blocks of subsets per rank).
int subset_owner(int k, int K, int W) { return (int)((int64_t)k * W / K); }

/// One grouped point-to-point exchange of a multi-rank context: NCCL
/// (production; one ncclGroup) or the host callbacks of a test transport
/// (device rows staged through host memory; the callbacks must post sends
/// without blocking, flush() completes every posted send and receive).
class Xfer {
  public:
    Xfer(Ctx& ctx, cudaStream_t s) : ctx_(ctx), s_(s) {
        if (ctx_.host_xfer) CK(cudaStreamSynchronize(s_));
        else NK(nccl().GroupStart());
    }
    void send(const float* dev, size_t floats, int peer) {
        if (!ctx_.host_xfer) {
            NK(nccl().Send(dev, floats, ncclFloat, peer, ctx_.comm, s_));
            return;
        }
        stage_.emplace_back(floats);
        CK(cudaMemcpy(stage_.back().data(), dev, floats * 4, cudaMemcpyDeviceToHost));
        if (ctx_.xfer_cb.send(ctx_.xfer_cb.user, stage_.back().data(), floats * 4, peer))
            throw std::runtime_error("host transport: send failed");
    }
    void recv(float* dev, size_t floats, int peer) {
        if (!ctx_.host_xfer) {
            NK(nccl().Recv(dev, floats, ncclFloat, peer, ctx_.comm, s_));
            return;
        }
        stage_.emplace_back(floats);
        if (ctx_.xfer_cb.recv(ctx_.xfer_cb.user, stage_.back().data(), floats * 4, peer))
            throw std::runtime_error("host transport: recv failed");
        pending_.push_back({dev, stage_.size() - 1});
    }
    void finish() {
        if (!ctx_.host_xfer) {
            NK(nccl().GroupEnd());
            return;
        }
        if (ctx_.xfer_cb.flush(ctx_.xfer_cb.user)) throw std::runtime_error("host transport: flush failed");
        for (const auto& p : pending_)
            CK(cudaMemcpy(p.first, stage_[p.second].data(), stage_[p.second].size() * 4, cudaMemcpyHostToDevice));
    }

  private:
    Ctx& ctx_;
    cudaStream_t s_;
    std::vector<std::vector<float>> stage_;
    std::vector<std::pair<float*, size_t>> pending_;
};

/// Forward exchange for slice `sl`: rows [h0, h1) of every subset's partial
/// map land in ctx.xrecv[k].  Multi-rank: one NCCL group of send/recv (the
/// all-to-all of manager.hpp:280-293's gather, sliced); single rank
/// (virtual slices): device copies with the same layout.  Returns bytes sent
/// over NCCL.
uint64_t exchange_forward(Ctx& ctx, int v, const std::vector<int>& local, int Wd, int H, int S, int sl,
                          cudaStream_t s) {
    const int K = ctx.table.k_count, W = ctx.world, rank = ctx.rank;
    const SliceRows me = slice_rows(H, S, sl);
    const size_t hr = (size_t)(me.h1 - me.h0);
    uint64_t sent = 0;
    if (W > 1) {
        Xfer x(ctx, s);
        for (int k : local) {
            const float4* src = subset(ctx, k).slot(v).ct.p;
            for (int j = 0; j < W; ++j) {
                if (j == rank) continue;
                const SliceRows R = slice_rows(H, S, j);
                const size_t cnt = (size_t)(R.h1 - R.h0) * Wd * 4;
                x.send(reinterpret_cast<const float*>(src + (size_t)R.h0 * Wd), cnt, j);
                sent += cnt * 4;
            }
        }
        for (int k = 0; k < K; ++k) {
            const int o = subset_owner(k, K, W);
            if (o == rank) continue;
            x.recv(reinterpret_cast<float*>(ctx.xrecv.p + (size_t)k * hr * Wd), hr * Wd * 4, o);
        }
        x.finish();
    }
    for (int k : local)  // own subsets: local copy
        CK(cudaMemcpyAsync(ctx.xrecv.p + (size_t)k * hr * Wd, subset(ctx, k).slot(v).ct.p + (size_t)me.h0 * Wd,
                           hr * Wd * sizeof(float4), cudaMemcpyDeviceToDevice, s));
    return sent;
}

/// Backward exchange for slice `sl`: (dL/dC_k, dL/dT_k) rows [r0, r1) from
/// ctx.xgrad[k] to the rank holding subset k (manager.hpp:336-343's
/// scatter, sliced).
uint64_t exchange_backward(Ctx& ctx, int v, const std::vector<int>& local, int Wd, int H, int S, int sl,
                           cudaStream_t s) {
    const int K = ctx.table.k_count, W = ctx.world, rank = ctx.rank;
    const SliceRows me = slice_rows(H, S, sl);
    const size_t orows = (size_t)(me.r1 - me.r0);
    uint64_t sent = 0;
    if (W > 1) {
        Xfer x(ctx, s);
        for (int k = 0; k < K; ++k) {
            const int o = subset_owner(k, K, W);
            if (o == rank) continue;
            x.send(reinterpret_cast<const float*>(ctx.xgrad.p + (size_t)k * orows * Wd), orows * Wd * 4, o);
            sent += orows * Wd * 16;
        }
        for (int k : local) {
            float4* dst = subset(ctx, k).slot(v).grad_ct.p;
            for (int j = 0; j < W; ++j) {
                if (j == rank) continue;
                const SliceRows R = slice_rows(H, S, j);
                x.recv(reinterpret_cast<float*>(dst + (size_t)R.r0 * Wd), (size_t)(R.r1 - R.r0) * Wd * 4, j);
            }
        }
        x.finish();
    }
    for (int k : local)
        CK(cudaMemcpyAsync(subset(ctx, k).slot(v).grad_ct.p + (size_t)me.r0 * Wd, ctx.xgrad.p + (size_t)k * orows * Wd,
                           orows * Wd * sizeof(float4), cudaMemcpyDeviceToDevice, s));
    return sent;
}

/// build_kdtree (partition.hpp:93-184) on device-resident centres (rows 0-2
/// of C, leading dimension ldc): per level, node extents, the widest axis,
/// exact medians from radix-sorted (node, coordinate) keys and the split.
/// Deterministic: every rank that runs it on the same centres gets the same
/// planes (KD leaves in DFS order, `depth` planes each).
std::vector<dgs_plane> kd_build_device(Ctx& ctx, const float* C, size_t ldc, int N, int depth) {
    cudaStream_t s = ctx.stream;
    DevBuf<uint64_t> keys, keys_alt;
    DevBuf<uint8_t> temp;
    keys.ensure(N);
    keys_alt.ensure(N);
    const size_t tb = repart_temp_bytes(N);
    temp.ensure(tb);
    struct HostRegion {
        std::vector<dgs_plane> planes;
        float amin[3], amax[3];
    };
    std::vector<HostRegion> regions(1);
    for (int a = 0; a < 3; ++a) {
        regions[0].amin[a] = -INFINITY;
        regions[0].amax[a] = INFINITY;
    }
    DevBuf<uint8_t> node;
    node.ensure(N);
    CK(cudaMemsetAsync(node.p, 0, N, s));
    DevBuf<uint32_t> lo, hi, cnt;
    DevBuf<int> d_axis;
    DevBuf<float> d_plane;
    const int maxn = 1 << depth;
    lo.ensure(3 * maxn);
    hi.ensure(3 * maxn);
    cnt.ensure(maxn);
    d_axis.ensure(maxn);
    d_plane.ensure(maxn);
    auto from_order = [](uint32_t o) {
        const uint32_t b = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
        float f;
        std::memcpy(&f, &b, 4);
        return f;
    };
    for (int d = 0; d < depth; ++d) {
        const int nn = 1 << d;
        std::vector<uint32_t> h_lo(3 * nn, 0xffffffffu), h_hi(3 * nn, 0u), h_cnt(nn, 0u);
        CK(cudaMemcpyAsync(lo.p, h_lo.data(), 12 * nn, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(hi.p, h_hi.data(), 12 * nn, cudaMemcpyHostToDevice, s));
        CK(cudaMemsetAsync(cnt.p, 0, 4 * nn, s));
        repart_node_extent(N, C, ldc, node.p, nn, lo.p, hi.p, cnt.p, s);
        CK(cudaMemcpyAsync(h_lo.data(), lo.p, 12 * nn, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(h_hi.data(), hi.p, 12 * nn, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(h_cnt.data(), cnt.p, 4 * nn, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (d == 0) {  // build_kdtree's degenerate-set check (partition.hpp:164-171)
            float m = from_order(h_hi[0]) - from_order(h_lo[0]);
            for (int a = 1; a < 3; ++a) m = std::max(m, from_order(h_hi[a]) - from_order(h_lo[a]));
            if (m <= 0.0f) throw std::invalid_argument("degenerate point set");
        }
        std::vector<int> axis(nn, 0);
        for (int q = 0; q < nn; ++q) {
            if (!h_cnt[q]) continue;
            float ext[3];
            for (int a = 0; a < 3; ++a) ext[a] = from_order(h_hi[3 * q + a]) - from_order(h_lo[3 * q + a]);
            float m = ext[0];  // maxCoeff(&axis): first maximum
            for (int a = 1; a < 3; ++a)
                if (ext[a] > m) {
                    m = ext[a];
                    axis[q] = a;
                }
        }
        CK(cudaMemcpyAsync(d_axis.p, axis.data(), 4 * nn, cudaMemcpyHostToDevice, s));
        // exact medians: sort (node, coordinate) keys, read the two middle values of every node
        repart_node_keys(N, C, ldc, node.p, d_axis.p, keys.p, s);
        uint64_t* k1 = keys.p;
        uint64_t* k2 = keys_alt.p;
        repart_sort_keys(k1, k2, N, 32 + d + 1, temp.p, tb, s);
        std::vector<float> plane(nn, 0.0f);
        std::vector<uint64_t> mid(2);
        uint32_t start = 0;
        for (int q = 0; q < nn; ++q) {
            const uint32_t c = h_cnt[q];
            HostRegion& reg = regions[q];
            if (c > 0) {
                const uint32_t i1 = start + c / 2;
                const uint32_t i0 = c % 2 == 0 ? i1 - 1 : i1;
                CK(cudaMemcpyAsync(&mid[0], k1 + i0, 8, cudaMemcpyDeviceToHost, s));
                CK(cudaMemcpyAsync(&mid[1], k1 + i1, 8, cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
                const float lower = from_order((uint32_t)mid[0]), upper = from_order((uint32_t)mid[1]);
                plane[q] = c % 2 == 0 ? (lower + upper) / 2.0f : upper;
            } else {
                const int a = axis[q];
                const float l = reg.amin[a], h = reg.amax[a];
                plane[q] = (std::isfinite(l) && std::isfinite(h)) ? (l + h) / 2.0f
                           : std::isfinite(l)                    ? l + 1.0f
                           : std::isfinite(h)                    ? h - 1.0f
                                                                 : 0.0f;
            }
            start += c;
        }
        CK(cudaMemcpyAsync(d_plane.p, plane.data(), 4 * nn, cudaMemcpyHostToDevice, s));
        repart_node_split(N, C, ldc, node.p, d_axis.p, d_plane.p, s);
        std::vector<HostRegion> next(2 * nn);
        for (int q = 0; q < nn; ++q) {
            const int a = axis[q];
            HostRegion left = regions[q], right = regions[q];
            dgs_plane lp{};
            lp.n[a] = 1.0f;
            lp.d = -plane[q];
            lp.closed = 0;
            left.planes.push_back(lp);
            left.amax[a] = std::min(left.amax[a], plane[q]);
            dgs_plane rp{};
            rp.n[a] = -1.0f;
            rp.d = plane[q];
            rp.closed = 1;
            right.planes.push_back(rp);
            right.amin[a] = std::max(right.amin[a], plane[q]);
            next[2 * q] = std::move(left);
            next[2 * q + 1] = std::move(right);
        }
        regions = std::move(next);
        CK(cudaStreamSynchronize(s));  // host vectors used by async copies
    }
    const int K = 1 << depth;
    std::vector<dgs_plane> planes((size_t)K * depth);
    for (int k = 0; k < K; ++k)
        for (int j = 0; j < depth; ++j) planes[(size_t)k * depth + j] = regions[k].planes[j];
    return planes;
}

/// The new partition table (device copy included).
void set_table_from_planes(Ctx& ctx, const std::vector<dgs_plane>& planes, int depth) {
    const int K = 1 << depth;
    Table t{};
    t.k_count = K;
    for (int k = 0; k < K; ++k) {
        t.sub[k].n = depth;
        for (int j = 0; j < depth; ++j) {
            const dgs_plane& p = planes[(size_t)k * depth + j];
            t.sub[k].nx[j] = p.n[0];
            t.sub[k].ny[j] = p.n[1];
            t.sub[k].nz[j] = p.n[2];
            t.sub[k].d[j] = p.d;
            t.sub[k].closed[j] = p.closed;
        }
    }
    ctx.table = t;
    ctx.table_dev.ensure(1);
    CK(cudaMemcpyAsync(ctx.table_dev.p, &ctx.table, sizeof(Table), cudaMemcpyHostToDevice, ctx.stream));
    CK(cudaStreamSynchronize(ctx.stream));
}

/// One u64 per peer: send[d] to rank d, returns what every rank sent to this one.
std::vector<uint64_t> xfer_counts(Ctx& ctx, const std::vector<uint64_t>& send) {
    const int W = ctx.world, me = ctx.rank;
    DevBuf<uint64_t> ds, dr;
    ds.ensure(W);
    dr.ensure(W);
    CK(cudaMemcpy(ds.p, send.data(), 8 * W, cudaMemcpyHostToDevice));
    {
        Xfer x(ctx, ctx.stream);
        for (int d = 0; d < W; ++d)
            if (d != me) x.send(reinterpret_cast<const float*>(ds.p + d), 2, d);
        for (int r = 0; r < W; ++r)
            if (r != me) x.recv(reinterpret_cast<float*>(dr.p + r), 2, r);
        x.finish();
    }
    CK(cudaStreamSynchronize(ctx.stream));
    std::vector<uint64_t> out(W);
    CK(cudaMemcpy(out.data(), dr.p, 8 * W, cudaMemcpyDeviceToHost));
    out[me] = send[me];
    return out;
}

/// Variable-size all-to-all of float buffers (own slot excluded: the caller copies it).
void xfer_alltoallv(Ctx& ctx, const std::vector<const float*>& sp, const std::vector<size_t>& sn,
                    const std::vector<float*>& rp, const std::vector<size_t>& rn) {
    const int W = ctx.world, me = ctx.rank;
    Xfer x(ctx, ctx.stream);
    for (int d = 0; d < W; ++d)
        if (d != me && sn[d]) x.send(sp[d], sn[d], d);
    for (int r = 0; r < W; ++r)
        if (r != me && rn[r]) x.recv(rp[r], rn[r], r);
    x.finish();
    CK(cudaStreamSynchronize(ctx.stream));
}

/// Cross-rank shared-replica index (grad sync, world > 1): every rank
/// all-gathers the (id, k) keys of all replicas, sorts them and keeps the runs
/// of >= 2 replicas; for each such replica it records the holder rank and its
/// row in the per-step gathered gradient rows.
void build_shared_multi(Ctx& ctx) {
    if (!ctx.shared_dirty) return;
    cudaStream_t s = ctx.stream;
    const int W = ctx.world, me = ctx.rank;
    std::vector<int> ks;
    std::vector<uint32_t> offs(1, 0);
    for (auto& kv : ctx.subsets) {
        ks.push_back(kv.first);
        offs.push_back(offs.back() + (uint32_t)kv.second->n);
    }
    const uint32_t Rme = offs.back();
    std::vector<uint64_t> rcount = xfer_counts(ctx, std::vector<uint64_t>(W, Rme));
    uint64_t base = 0, R = 0;
    for (int r = 0; r < W; ++r) {
        if (r < me) base += rcount[r];
        R += rcount[r];
    }
    ctx.xs_base = (uint32_t)base;
    ctx.xs_offs.ensure(ks.size() + 1);
    CK(cudaMemcpy(ctx.xs_offs.p, offs.data(), 4 * offs.size(), cudaMemcpyHostToDevice));
    DevBuf<uint64_t> keys, kalt;
    DevBuf<uint32_t> vals, valt;
    DevBuf<uint8_t> flags, temp;
    DevBuf<int> count;
    keys.ensure(std::max<uint64_t>(R, 1));
    kalt.ensure(std::max<uint64_t>(R, 1));
    vals.ensure(std::max<uint64_t>(R, 1));
    valt.ensure(std::max<uint64_t>(R, 1));
    flags.ensure(std::max<uint64_t>(R, 1));
    count.ensure(1);
    const size_t tb = repart_temp_bytes((int64_t)std::max<uint64_t>(R, 1));
    temp.ensure(tb);
    for (size_t q = 0; q < ks.size(); ++q) {
        const SubsetState& S = *ctx.subsets[ks[q]];
        shared_replica_keys((int)S.n, S.ids32.p, ks[q], (uint32_t)(base + offs[q]), keys.p, vals.p, s);
        // shared_replica_keys stores k << 27 | i as the value; here the value is the global index
    }
    {
        // global indices as values
        std::vector<uint32_t> gi(Rme);
        for (uint32_t j = 0; j < Rme; ++j) gi[j] = (uint32_t)base + j;
        CK(cudaMemcpyAsync(vals.p + base, gi.data(), 4 * (size_t)Rme, cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));
    }
    std::vector<const float*> sp(W);
    std::vector<size_t> sn(W), rn(W);
    std::vector<float*> rp(W);
    uint64_t off = 0;
    for (int r = 0; r < W; ++r) {
        sp[r] = reinterpret_cast<const float*>(keys.p + base);
        sn[r] = 2 * (size_t)Rme;
        rp[r] = reinterpret_cast<float*>(keys.p + off);
        rn[r] = 2 * (size_t)rcount[r];
        off += rcount[r];
    }
    xfer_alltoallv(ctx, sp, sn, rp, rn);
    off = 0;
    for (int r = 0; r < W; ++r) {
        sp[r] = reinterpret_cast<const float*>(vals.p + base);
        sn[r] = (size_t)Rme;
        rp[r] = reinterpret_cast<float*>(vals.p + off);
        rn[r] = (size_t)rcount[r];
        off += rcount[r];
    }
    xfer_alltoallv(ctx, sp, sn, rp, rn);
    uint64_t* kp = keys.p;
    uint64_t* kap = kalt.p;
    uint32_t* vp = vals.p;
    uint32_t* vap = valt.p;
    repart_sort_pairs(kp, kap, vp, vap, (int)R, 40, temp.p, tb, s);
    shared_mark((int)R, kp, flags.p, s);
    ctx.xs_keys.ensure(std::max<uint64_t>(R, 1));
    ctx.xs_g.ensure(std::max<uint64_t>(R, 1));
    repart_select_u64((int)R, kp, flags.p, ctx.xs_keys.p, count.p, temp.p, tb, s);
    repart_select((int)R, vp, flags.p, ctx.xs_g.p, count.p, temp.p, tb, s);
    int S = 0;
    CK(cudaMemcpyAsync(&S, count.p, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    ctx.xs_S = S;
    // holder rank, row in the gathered rows, my entries (host bookkeeping, O(S))
    std::vector<uint32_t> g(S), src(S), pos;
    std::vector<uint8_t> mine(S);
    if (S) CK(cudaMemcpy(g.data(), ctx.xs_g.p, 4 * (size_t)S, cudaMemcpyDeviceToHost));
    std::vector<uint64_t> rb(W + 1, 0);
    for (int r = 0; r < W; ++r) rb[r + 1] = rb[r] + rcount[r];
    ctx.xs_count.assign(W, 0);
    std::vector<uint32_t> owner(S);
    for (int j = 0; j < S; ++j) {
        int r = 0;
        while (r + 1 < W && rb[r + 1] <= g[j]) ++r;
        owner[j] = r;
        ++ctx.xs_count[r];
    }
    std::vector<uint64_t> cb(W + 1, 0), seen(W, 0);
    for (int r = 0; r < W; ++r) cb[r + 1] = cb[r] + ctx.xs_count[r];
    for (int j = 0; j < S; ++j) {
        const int r = owner[j];
        src[j] = (uint32_t)(cb[r] + seen[r]++);
        mine[j] = r == me;
        if (r == me) pos.push_back((uint32_t)j);
    }
    ctx.xs_nmine = (int)pos.size();
    ctx.xs_src.ensure(std::max(S, 1));
    ctx.xs_mine.ensure(std::max(S, 1));
    ctx.xs_pos.ensure(std::max<size_t>(pos.size(), 1));
    if (S) {
        CK(cudaMemcpy(ctx.xs_src.p, src.data(), 4 * (size_t)S, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx.xs_mine.p, mine.data(), (size_t)S, cudaMemcpyHostToDevice));
    }
    if (!pos.empty()) CK(cudaMemcpy(ctx.xs_pos.p, pos.data(), 4 * pos.size(), cudaMemcpyHostToDevice));
    ctx.shared_dirty = false;
}

/// One step's cross-rank sync: pack my shared replicas' gradient rows, all-gather,
/// sum per id in worker order and write back (G pointers in ascending local k).
void grad_sync_multi(Ctx& ctx, int rows, float* const* dG, const size_t* dL, int KL) {
    cudaStream_t s = ctx.stream;
    const int W = ctx.world, me = ctx.rank;
    const int S = ctx.xs_S;
    DevBuf<float> sendb, recvb;
    sendb.ensure((size_t)std::max(ctx.xs_nmine, 1) * rows);
    recvb.ensure((size_t)std::max(S, 1) * rows);
    shared_pack(ctx.xs_nmine, rows, ctx.xs_pos.p, ctx.xs_g.p, ctx.xs_base, ctx.xs_offs.p, KL, dG, dL, sendb.p, s);
    std::vector<const float*> sp(W, sendb.p);
    std::vector<size_t> sn(W, (size_t)ctx.xs_nmine * rows), rn(W);
    std::vector<float*> rp(W);
    uint64_t off = 0;
    for (int r = 0; r < W; ++r) {
        rp[r] = recvb.p + off * rows;
        rn[r] = (size_t)ctx.xs_count[r] * rows;
        off += ctx.xs_count[r];
    }
    CK(cudaStreamSynchronize(s));
    xfer_alltoallv(ctx, sp, sn, rp, rn);
    if (ctx.xs_nmine)
        CK(cudaMemcpyAsync(rp[me], sendb.p, 4 * (size_t)ctx.xs_nmine * rows, cudaMemcpyDeviceToDevice, s));
    shared_sync(S, rows, ctx.xs_keys.p, ctx.xs_src.p, recvb.p, ctx.xs_mine.p, ctx.xs_g.p, ctx.xs_base, ctx.xs_offs.p,
                KL, dG, dL, s);
    CK(cudaStreamSynchronize(s));
}

/// Shared-replica index over the resident subsets (grad sync): replicas sorted
/// by (id, k); sh_starts = first sorted position of every id held >= 2 times.
void build_shared(Ctx& ctx) {
    if (!ctx.shared_dirty) return;
    cudaStream_t s = ctx.stream;
    std::vector<uint32_t> offs(1, 0);
    std::vector<int> ks;
    for (auto& kv : ctx.subsets) {
        ks.push_back(kv.first);
        offs.push_back(offs.back() + (uint32_t)kv.second->n);
    }
    const int R = (int)offs.back();
    ctx.sh_slots = 0;
    ctx.sh_nrep = R;
    if (R > 0) {
        DevBuf<uint64_t> kalt;
        DevBuf<uint32_t> valt;
        DevBuf<uint8_t> flags, temp;
        DevBuf<int> count;
        ctx.sh_keys.ensure(R);
        kalt.ensure(R);
        ctx.sh_reps.ensure(R);
        valt.ensure(R);
        flags.ensure(R);
        count.ensure(1);
        ctx.sh_starts.ensure(R);
        const size_t tb = repart_temp_bytes(R);
        temp.ensure(tb);
        for (size_t q = 0; q < ks.size(); ++q) {
            const SubsetState& S = *ctx.subsets[ks[q]];
            shared_replica_keys((int)S.n, S.ids32.p, ks[q], offs[q], ctx.sh_keys.p, ctx.sh_reps.p, s);
        }
        uint64_t* kp = ctx.sh_keys.p;
        uint64_t* kap = kalt.p;
        uint32_t* vp = ctx.sh_reps.p;
        uint32_t* vap = valt.p;
        repart_sort_pairs(kp, kap, vp, vap, R, 40, temp.p, tb, s);
        if (kp != ctx.sh_keys.p) {  // keep the sorted data in the persistent buffers
            CK(cudaMemcpyAsync(ctx.sh_keys.p, kp, 8 * (size_t)R, cudaMemcpyDeviceToDevice, s));
            CK(cudaMemcpyAsync(ctx.sh_reps.p, vp, 4 * (size_t)R, cudaMemcpyDeviceToDevice, s));
        }
        shared_run_starts(R, ctx.sh_keys.p, flags.p, s);
        repart_select_iota(R, flags.p, ctx.sh_starts.p, count.p, temp.p, tb, s);
        CK(cudaMemcpyAsync(&ctx.sh_slots, count.p, 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    ctx.shared_dirty = false;
}

void require_table(const Ctx& ctx) {
    if (!ctx.table_set) throw std::invalid_argument("partition table not set (dgs_set_table)");
}

}  // namespace
}  // namespace dgs_b200

using namespace dgs_b200;

struct dgs_ctx : dgs_b200::Ctx {};

extern "C" {

const char* dgs_last_error(void) { return dgs_b200::g_last_error.c_str(); }

int dgs_nccl_unique_id(void* out128) {
    return dgs_guard([&] {
        ncclUniqueId id;
        NK(nccl().GetUniqueId(&id));
        std::memcpy(out128, &id, sizeof(id));
    });
}

int dgs_nccl_selftest(int32_t device) {
    return dgs_guard([&] {
        // the calls the rank exchange makes (grouped send/recv, all-reduce of the
        // loss sums), on a one-rank communicator: checks the run-time NCCL binding
        CK(cudaSetDevice(device));
        ncclUniqueId id;
        NK(nccl().GetUniqueId(&id));
        ncclComm_t comm = nullptr;
        NK(nccl().CommInitRank(&comm, 1, id, 0));
        cudaStream_t s;
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        const size_t n = 4099;
        std::vector<float> h(n), back(n);
        for (size_t i = 0; i < n; ++i) h[i] = (float)i * 0.5f - 7.0f;
        DevBuf<float> a, b;
        DevBuf<double> d;
        a.ensure(n);
        b.ensure(n);
        d.ensure(3);
        const double dh[3] = {1.5, -2.0, 3.25};
        CK(cudaMemcpy(a.p, h.data(), n * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d.p, dh, sizeof(dh), cudaMemcpyHostToDevice));
        NK(nccl().GroupStart());
        NK(nccl().Send(a.p, n, ncclFloat, 0, comm, s));
        NK(nccl().Recv(b.p, n, ncclFloat, 0, comm, s));
        NK(nccl().GroupEnd());
        NK(nccl().AllReduce(d.p, d.p, 3, ncclDouble, ncclSum, comm, s));
        CK(cudaStreamSynchronize(s));
        double dr[3];
        CK(cudaMemcpy(back.data(), b.p, n * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(dr, d.p, sizeof(dr), cudaMemcpyDeviceToHost));
        nccl().CommDestroy(comm);
        cudaStreamDestroy(s);
        if (std::memcmp(back.data(), h.data(), n * 4) != 0) throw std::runtime_error("nccl selftest: send/recv mismatch");
        if (dr[0] != dh[0] || dr[1] != dh[1] || dr[2] != dh[2])
            throw std::runtime_error("nccl selftest: all-reduce mismatch");
    });
}

int dgs_ctx_create(int32_t device, int32_t rank, int32_t world, const void* nccl_id, dgs_ctx** out) {
    return dgs_guard([&] {
        int ndev = 0;
        CK(cudaGetDeviceCount(&ndev));
        if (device < 0 || device >= ndev) throw std::invalid_argument("dgs_ctx_create: bad device index");
        if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("dgs_ctx_create: bad rank/world");
        CK(cudaSetDevice(device));
        std::unique_ptr<dgs_ctx> c(new dgs_ctx());
        c->device = device;
        c->rank = rank;
        c->world = world;
        CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        CK(cudaHostAlloc(reinterpret_cast<void**>(&c->hs), sizeof(HostScalars), cudaHostAllocDefault));
        CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&c->copy_done, cudaEventDisableTiming));
        CK(cudaStreamCreateWithFlags(&c->xstream, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&c->chain_done, cudaEventDisableTiming));
        if (world > 1) {
            if (nccl_id == nullptr) throw std::invalid_argument("dgs_ctx_create: world > 1 needs an nccl id");
            ncclUniqueId id;
            std::memcpy(&id, nccl_id, sizeof(id));
            NK(nccl().CommInitRank(&c->comm, world, id, rank));
        }
        dgs_default_render_options(&c->ro_in);
        dgs_default_train_config(&c->cfg);
        c->ro = to_render_opts(c->ro_in);
        c->stats.ensure(2);  // [0] forward blend, [1] backward blend
        *out = c.release();
    });
}

int dgs_ctx_create_host_transport(int32_t device, int32_t rank, int32_t world, const dgs_host_transport* t,
                                  dgs_ctx** out) {
    return dgs_guard([&] {
        if (!t || !t->send || !t->recv || !t->flush || !t->allreduce_sum_f64)
            throw std::invalid_argument("dgs_ctx_create_host_transport: incomplete callbacks");
        if (!out) throw std::invalid_argument("dgs_ctx_create_host_transport: null output");
        *out = nullptr;
        // validate before creating anything: an error return leaves nothing live in *out
        if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("dgs_ctx_create: bad rank/world");
        dgs_ctx* c = nullptr;
        if (dgs_ctx_create(device, 0, 1, nullptr, &c) != 0) throw std::runtime_error(g_last_error);
        c->rank = rank;
        c->world = world;
        c->host_xfer = true;
        c->xfer_cb = *t;
        *out = c;
    });
}

int dgs_ctx_destroy(dgs_ctx* ctx) {
    return dgs_guard([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        if (ctx->stager.joinable()) ctx->stager.join();
        cudaStreamSynchronize(ctx->stream);
        cudaStreamSynchronize(ctx->copy_stream);
        if (ctx->pin_stage) cudaFreeHost(ctx->pin_stage);
        if (ctx->comm) nccl().CommDestroy(ctx->comm);
        ctx->subsets.clear();
        cudaStreamDestroy(ctx->stream);
        if (ctx->hs) cudaFreeHost(ctx->hs);
        ctx->drop_graphs();
        if (ctx->tail) cudaFreeHost(ctx->tail);
        if (ctx->copy_done) cudaEventDestroy(ctx->copy_done);
        if (ctx->xstream) {
            cudaStreamSynchronize(ctx->xstream);
            cudaStreamDestroy(ctx->xstream);
        }
        if (ctx->chain_done) cudaEventDestroy(ctx->chain_done);
        for (cudaEvent_t e : ctx->view_done) cudaEventDestroy(e);
        if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
        delete ctx;
    });
}

int dgs_set_profiling(dgs_ctx* ctx, int32_t enabled) {
    return dgs_guard([&] {
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->timer.resolve();
        ctx->timer.on = enabled != 0;
        for (int i = 0; i < StageTimer::kStages; ++i) {
            ctx->timer.ms[i] = 0.0;
            ctx->timer.count[i] = 0;
        }
    });
}

int dgs_stage_times(dgs_ctx* ctx, double* ms, uint64_t* counts) {
    return dgs_guard([&] {
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->timer.resolve();
        for (int i = 0; i < StageTimer::kStages; ++i) {
            if (ms) ms[i] = ctx->timer.ms[i];
            if (counts) counts[i] = ctx->timer.count[i];
        }
    });
}

void* dgs_stream(dgs_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int dgs_sync(dgs_ctx* ctx) {
    return dgs_guard([&] {
        CK(cudaStreamSynchronize(ctx->stream));
        CK(cudaGetLastError());
    });
}

int dgs_set_table(dgs_ctx* ctx, const dgs_plane* planes, int32_t k_count, int32_t ppk) {
    return dgs_guard([&] {
        if (ctx) ++ctx->graph_version;  // captured step graphs no longer match
        if (k_count < 1 || k_count > kMaxSubsets) throw std::invalid_argument("set_table: 1..32 subsets supported");
        if (ppk < 0 || ppk > kMaxPlanes) throw std::invalid_argument("set_table: at most 8 planes per subspace");
        Table t{};
        t.k_count = k_count;
        for (int k = 0; k < k_count; ++k) {
            t.sub[k].n = ppk;
            for (int j = 0; j < ppk; ++j) {
                const dgs_plane& p = planes[k * ppk + j];
                t.sub[k].nx[j] = p.n[0];
                t.sub[k].ny[j] = p.n[1];
                t.sub[k].nz[j] = p.n[2];
                t.sub[k].d[j] = p.d;
                t.sub[k].closed[j] = p.closed;
            }
        }
        ctx->table = t;
        ctx->table_set = true;
        ctx->table_dev.ensure(1);
        CK(cudaMemcpy(ctx->table_dev.p, &ctx->table, sizeof(Table), cudaMemcpyHostToDevice));
    });
}

int dgs_set_epoch(dgs_ctx* ctx, uint64_t epoch) {
    return dgs_guard([&] {
        ctx->epoch = epoch;
        ctx->epoch_set = true;
    });
}

int dgs_set_options(dgs_ctx* ctx, const dgs_render_options* ro, const dgs_train_config* cfg) {
    return dgs_guard([&] {
        if (ctx) ++ctx->graph_version;  // captured step graphs no longer match
        if (ro) {
            ctx->ro_in = *ro;
            ctx->ro = to_render_opts(*ro);
        }
        if (cfg) {
            // TrainConfig::validate (optim.hpp:30-37)
            if (cfg->lambda_ssim < 0.0 || cfg->lambda_ssim > 1.0)
                throw std::invalid_argument("config: lambda_ssim must be in [0,1]");
            if (cfg->lr_position_end > cfg->lr_position_start)
                throw std::invalid_argument("config: position LR end must not exceed start");
            if (cfg->batch_size < 1) throw std::invalid_argument("config: batch_size must be >= 1");
            ctx->cfg = *cfg;
        }
    });
}

int dgs_subset_load(dgs_ctx* ctx, int32_t k, const dgs_splats* params, const dgs_splats* m, const dgs_splats* v,
                    uint64_t adam_step, uint64_t epoch) {
    return dgs_guard([&] {
        if (ctx) ++ctx->graph_version;  // captured step graphs no longer match
        require_table(*ctx);
        if (k < 0 || k >= ctx->table.k_count) throw std::invalid_argument("subset_load: k outside the table");
        if (params->sh_coeffs != 1 && params->sh_coeffs != 4 && params->sh_coeffs != 9 && params->sh_coeffs != 16)
            throw std::invalid_argument("splat sh coefficient count must be (deg+1)^2, deg<=3");
        if (params->n > INT_MAX / 4) throw std::invalid_argument("subset_load: subset too large for one rank");
        CK(cudaSetDevice(ctx->device));
        std::unique_ptr<SubsetState> S(new SubsetState());
        S->k = k;
        S->n = params->n;
        S->sh_coeffs = params->sh_coeffs;
        S->rows = param_rows(S->sh_coeffs);
        S->ld = (size_t)((params->n + 31) / 32 * 32);
        S->adam_step = adam_step;
        S->epoch = epoch;
        S->ids64.assign(params->id, params->id + params->n);
        std::vector<uint32_t> ids32((size_t)params->n);
        for (int64_t i = 0; i < params->n; ++i) {
            if (params->id[i] > 0xffffffffull) throw std::invalid_argument("subset_load: splat ids must be < 2^32");
            ids32[i] = (uint32_t)params->id[i];
        }
        S->ids32.ensure(params->n);
        if (params->n) CK(cudaMemcpy(S->ids32.p, ids32.data(), 4 * ids32.size(), cudaMemcpyHostToDevice));
        S->P.ensure(S->rows * S->ld);
        S->M.ensure(S->rows * S->ld);
        S->V.ensure(S->rows * S->ld);
        upload_fields(*ctx, *S, *params, S->P.p);
        if (m) upload_fields(*ctx, *S, *m, S->M.p);
        else CK(cudaMemset(S->M.p, 0, S->rows * S->ld * sizeof(float)));
        if (v) upload_fields(*ctx, *S, *v, S->V.p);
        else CK(cudaMemset(S->V.p, 0, S->rows * S->ld * sizeof(float)));
        ctx->subsets[k] = std::move(S);
        ctx->shared_dirty = true;
    });
}

int dgs_repartition(dgs_ctx* ctx, int32_t depth, double d_multiplier, int64_t expected_splats, uint64_t epoch,
                    dgs_plane* planes_out) {
    return dgs_guard([&] {
        if (ctx) ++ctx->graph_version;  // captured step graphs no longer match
        require_table(*ctx);
        if (depth < 0 || depth > 5) throw std::invalid_argument("repartition: kd depth must be 0..5 (<= 32 subsets)");
        const int W = ctx->world, me = ctx->rank;
        if ((1 << depth) < W) throw std::invalid_argument("repartition: fewer KD subsets than ranks");
        CK(cudaSetDevice(ctx->device));
        cudaStream_t s = ctx->stream;
        // local subsets in ascending k (the replica numbering of this rank)
        std::vector<int> ks;
        for (auto& kv : ctx->subsets) ks.push_back(kv.first);
        if (W == 1)
            for (int k = 0; k < ctx->table.k_count; ++k) subset(*ctx, k);  // every subset resident
        if (ks.empty()) throw std::invalid_argument("repartition: no subset resident on this rank");
        const SubsetState& S0 = *ctx->subsets.begin()->second;
        const int shc = S0.sh_coeffs, rows = S0.rows;
        const uint64_t adam_step = S0.adam_step;
        std::vector<uint32_t> offs(1, 0);
        for (int k : ks) {
            const SubsetState& S = subset(*ctx, k);
            if (S.sh_coeffs != shc) throw std::invalid_argument("repartition: subsets disagree on the SH degree");
            offs.push_back(offs.back() + (uint32_t)S.n);
        }
        const int Rme = (int)offs.back();
        // ---- snapshot (manager.hpp:389-418): one replica per id, across ranks ----
        std::vector<uint64_t> rcount(W, 0);
        rcount[me] = (uint64_t)Rme;
        if (W > 1) rcount = xfer_counts(*ctx, std::vector<uint64_t>(W, (uint64_t)Rme));
        uint64_t Rtot = 0, base = 0;
        for (int r = 0; r < W; ++r) {
            if (r < me) base += rcount[r];
            Rtot += rcount[r];
        }
        if (Rtot == 0 || Rtot > 0x7fffffffull) throw std::invalid_argument("build_kdtree: empty point set");
        const int R = (int)Rtot;
        DevBuf<uint64_t> keys, keys_alt;
        DevBuf<uint32_t> vals, vals_alt, winners;
        DevBuf<uint8_t> flags, temp;
        DevBuf<int> count;
        keys.ensure(R);
        keys_alt.ensure(R);
        vals.ensure(R);
        vals_alt.ensure(R);
        winners.ensure(R);
        flags.ensure(R);
        count.ensure(1);
        size_t tb = repart_temp_bytes(R);
        temp.ensure(tb);
        for (size_t q = 0; q < ks.size(); ++q) {
            const SubsetState& S = subset(*ctx, ks[q]);
            repart_snapshot_keys((int)S.n, S.P.p, S.ld, S.ids32.p, ctx->table_dev.p, ks[q], (uint32_t)(base + offs[q]),
                                 keys.p, vals.p, s);
        }
        if (W > 1) {  // all-gather the replica keys (u64) and their global indices
            std::vector<const float*> sp(W);
            std::vector<size_t> sn(W), rn(W);
            std::vector<float*> rp(W);
            for (int r = 0; r < W; ++r) {
                uint64_t off = 0;
                for (int q = 0; q < r; ++q) off += rcount[q];
                sp[r] = reinterpret_cast<const float*>(keys.p + base);
                sn[r] = 2 * (size_t)Rme;
                rp[r] = reinterpret_cast<float*>(keys.p + off);
                rn[r] = 2 * (size_t)rcount[r];
            }
            CK(cudaStreamSynchronize(s));
            xfer_alltoallv(*ctx, sp, sn, rp, rn);
            for (int r = 0; r < W; ++r) {
                uint64_t off = 0;
                for (int q = 0; q < r; ++q) off += rcount[q];
                sp[r] = reinterpret_cast<const float*>(vals.p + base);
                sn[r] = (size_t)Rme;
                rp[r] = reinterpret_cast<float*>(vals.p + off);
                rn[r] = (size_t)rcount[r];
            }
            xfer_alltoallv(*ctx, sp, sn, rp, rn);
        }
        uint64_t* kp = keys.p;
        uint64_t* kap = keys_alt.p;
        uint32_t* vp = vals.p;
        uint32_t* vap = vals_alt.p;
        repart_sort_pairs(kp, kap, vp, vap, R, 40, temp.p, tb, s);
        repart_first_of_run(R, kp, flags.p, s);
        repart_select(R, vp, flags.p, winners.p, count.p, temp.p, tb, s);
        int Ntot = 0;
        CK(cudaMemcpyAsync(&Ntot, count.p, 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (expected_splats >= 0 && (int64_t)Ntot != expected_splats) throw std::runtime_error("snapshot lost splats");
        // this rank's winners (global replica index in [base, base + Rme)) -> local replica index
        int N = Ntot;
        uint32_t* mine = winners.p;
        DevBuf<uint32_t> mine_buf;
        if (W > 1) {
            mine_buf.ensure(std::max(Ntot, 1));
            repart_flag_range(Ntot, winners.p, (uint32_t)base, (uint32_t)(base + Rme), flags.p, s);
            repart_select(Ntot, winners.p, flags.p, mine_buf.p, count.p, temp.p, tb, s);
            CK(cudaMemcpyAsync(&N, count.p, 4, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            repart_sub_const(N, mine_buf.p, (uint32_t)base, s);
            mine = mine_buf.p;
        }
        // my winners' state, SoA
        const size_t ldm = (size_t)(std::max(N, 1) + 31) / 32 * 32;
        DevBuf<float> mP, mM, mV;
        DevBuf<uint32_t> mIds;
        mP.ensure(rows * ldm);
        mM.ensure(rows * ldm);
        mV.ensure(rows * ldm);
        mIds.ensure(ldm);
        {
            const int KL = (int)ks.size();
            std::vector<const float*> hp(KL), hm(KL), hv(KL);
            std::vector<const uint32_t*> hi(KL);
            std::vector<size_t> hl(KL);
            for (int q = 0; q < KL; ++q) {
                const SubsetState& S = subset(*ctx, ks[q]);
                hp[q] = S.P.p;
                hm[q] = S.M.p;
                hv[q] = S.V.p;
                hi[q] = S.ids32.p;
                hl[q] = S.ld;
            }
            DevBuf<const float*> dp, dm, dv;
            DevBuf<const uint32_t*> di;
            DevBuf<size_t> dl;
            DevBuf<uint32_t> doffs;
            dp.ensure(KL);
            dm.ensure(KL);
            dv.ensure(KL);
            di.ensure(KL);
            dl.ensure(KL);
            doffs.ensure(KL + 1);
            CK(cudaMemcpyAsync(dp.p, hp.data(), KL * sizeof(void*), cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(dm.p, hm.data(), KL * sizeof(void*), cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(dv.p, hv.data(), KL * sizeof(void*), cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(di.p, hi.data(), KL * sizeof(void*), cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(dl.p, hl.data(), KL * sizeof(size_t), cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(doffs.p, offs.data(), (KL + 1) * 4, cudaMemcpyHostToDevice, s));
            repart_gather_replicas(N, rows, mine, doffs.p, KL, dp.p, dm.p, dv.p, di.p, dl.p, mP.p, mM.p, mV.p, mIds.p,
                                   ldm, s);
            CK(cudaStreamSynchronize(s));
        }
        // ---- build_kdtree (partition.hpp:93-184) over every winner's centre ----
        std::vector<dgs_plane> planes;
        if (W == 1) {
            planes = kd_build_device(*ctx, mP.p, ldm, N, depth);
        } else {
            std::vector<uint64_t> ncount = xfer_counts(*ctx, std::vector<uint64_t>(W, (uint64_t)N));
            const size_t ldc = (size_t)(Ntot + 31) / 32 * 32;
            DevBuf<float> cAll, cMine, cRecv;
            cAll.ensure(3 * ldc);
            cMine.ensure(3 * (size_t)std::max(N, 1));
            size_t maxr = 1;
            for (int r = 0; r < W; ++r) maxr = std::max<size_t>(maxr, ncount[r]);
            cRecv.ensure(3 * maxr * W);
            for (int a = 0; a < 3; ++a)
                CK(cudaMemcpyAsync(cMine.p + (size_t)a * N, mP.p + (size_t)a * ldm, 4 * (size_t)N,
                                   cudaMemcpyDeviceToDevice, s));
            CK(cudaStreamSynchronize(s));
            std::vector<const float*> sp(W, cMine.p);
            std::vector<size_t> sn(W, 3 * (size_t)N), rn(W);
            std::vector<float*> rp(W);
            for (int r = 0; r < W; ++r) {
                rp[r] = cRecv.p + 3 * maxr * r;
                rn[r] = 3 * (size_t)ncount[r];
            }
            xfer_alltoallv(*ctx, sp, sn, rp, rn);
            CK(cudaMemcpyAsync(rp[me], cMine.p, 12 * (size_t)N, cudaMemcpyDeviceToDevice, s));
            uint64_t off = 0;
            for (int r = 0; r < W; ++r) {
                for (int a = 0; a < 3; ++a)
                    CK(cudaMemcpyAsync(cAll.p + (size_t)a * ldc + off, rp[r] + (size_t)a * ncount[r],
                                       4 * (size_t)ncount[r], cudaMemcpyDeviceToDevice, s));
                off += ncount[r];
            }
            CK(cudaStreamSynchronize(s));
            planes = kd_build_device(*ctx, cAll.p, ldc, Ntot, depth);
        }
        if (planes_out) std::memcpy(planes_out, planes.data(), planes.size() * sizeof(dgs_plane));
        set_table_from_planes(*ctx, planes, depth);
        const int K = 1 << depth;
        // ---- assign_subsets (partition.hpp:234-251) ----
        DevBuf<uint32_t> mask;
        mask.ensure(std::max(N, 1));
        repart_assign(N, mP.p, ldm, ctx->table_dev.p, (float)d_multiplier, mask.p, s);
        // ---- migration (manager.hpp:440-482): winners to the ranks owning their new subsets ----
        const float* srcP = mP.p;
        const float* srcM = mM.p;
        const float* srcV = mV.p;
        const uint32_t* srcIds = mIds.p;
        const uint32_t* srcMask = mask.p;
        size_t lds = ldm;
        int Nsrc = N;
        DevBuf<float> rP, rM, rV;
        DevBuf<uint32_t> rIds, rMask;
        if (W > 1) {
            const int stride = 3 * rows + 2;
            std::vector<DevBuf<float>> packs(W);
            std::vector<uint64_t> scount(W, 0);
            DevBuf<uint32_t> idx;
            idx.ensure(std::max(N, 1));
            for (int d = 0; d < W; ++d) {
                uint32_t owned = 0;
                for (int k = 0; k < K; ++k)
                    if (subset_owner(k, K, W) == d) owned |= 1u << k;
                repart_flag_owned(N, mask.p, owned, flags.p, s);
                repart_select_iota(N, flags.p, idx.p, count.p, temp.p, tb, s);
                int nd = 0;
                CK(cudaMemcpyAsync(&nd, count.p, 4, cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
                scount[d] = (uint64_t)nd;
                packs[d].ensure((size_t)std::max(nd, 1) * stride);
                repart_pack(nd, rows, idx.p, mP.p, mM.p, mV.p, mIds.p, mask.p, ldm, packs[d].p, s);
            }
            CK(cudaStreamSynchronize(s));
            std::vector<uint64_t> rcnt = xfer_counts(*ctx, scount);
            std::vector<DevBuf<float>> inbox(W);
            std::vector<const float*> sp(W);
            std::vector<size_t> sn(W), rn(W);
            std::vector<float*> rp(W);
            uint64_t total_in = 0;
            for (int r = 0; r < W; ++r) {
                sp[r] = packs[r].p;
                sn[r] = (size_t)scount[r] * stride;
                inbox[r].ensure((size_t)std::max<uint64_t>(rcnt[r], 1) * stride);
                rp[r] = inbox[r].p;
                rn[r] = (size_t)rcnt[r] * stride;
                total_in += rcnt[r];
            }
            xfer_alltoallv(*ctx, sp, sn, rp, rn);
            if (scount[me])
                CK(cudaMemcpyAsync(inbox[me].p, packs[me].p, 4 * (size_t)scount[me] * stride,
                                   cudaMemcpyDeviceToDevice, s));
            Nsrc = (int)total_in;
            lds = (size_t)(std::max(Nsrc, 1) + 31) / 32 * 32;
            rP.ensure(rows * lds);
            rM.ensure(rows * lds);
            rV.ensure(rows * lds);
            rIds.ensure(lds);
            rMask.ensure(lds);
            uint64_t off = 0;
            for (int r = 0; r < W; ++r) {  // source-rank order
                repart_unpack((int)rcnt[r], rows, inbox[r].p, rP.p + off, rM.p + off, rV.p + off, rIds.p + off,
                              rMask.p + off, lds, s);
                off += rcnt[r];
            }
            CK(cudaStreamSynchronize(s));
            srcP = rP.p;
            srcM = rM.p;
            srcV = rV.p;
            srcIds = rIds.p;
            srcMask = rMask.p;
            if ((size_t)Nsrc > flags.n) flags.ensure(Nsrc);
            tb = repart_temp_bytes(std::max<int64_t>(Nsrc, R));
            temp.ensure(tb);
        }
        DevBuf<uint32_t> idx2;
        idx2.ensure(std::max(Nsrc, 1));
        std::map<int, std::unique_ptr<SubsetState>> fresh;
        for (int k = 0; k < K; ++k) {
            if (subset_owner(k, K, W) != me) continue;
            repart_flag_bit(Nsrc, srcMask, k, flags.p, s);
            repart_select_iota(Nsrc, flags.p, idx2.p, count.p, temp.p, tb, s);
            int nk = 0;
            CK(cudaMemcpyAsync(&nk, count.p, 4, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            std::unique_ptr<SubsetState> S(new SubsetState());
            S->k = k;
            S->n = nk;
            S->sh_coeffs = shc;
            S->rows = rows;
            S->ld = (size_t)((nk + 31) / 32 * 32);
            S->adam_step = adam_step;
            S->epoch = epoch;
            S->P.ensure(rows * S->ld);
            S->M.ensure(rows * S->ld);
            S->V.ensure(rows * S->ld);
            S->ids32.ensure(nk);
            if (S->ld > (size_t)nk) {  // keep the padded tail defined (private scratch of the Adam stream)
                CK(cudaMemsetAsync(S->P.p, 0, rows * S->ld * sizeof(float), s));
                CK(cudaMemsetAsync(S->M.p, 0, rows * S->ld * sizeof(float), s));
                CK(cudaMemsetAsync(S->V.p, 0, rows * S->ld * sizeof(float), s));
            }
            repart_gather_members(nk, rows, idx2.p, srcP, srcM, srcV, srcIds, lds, S->P.p, S->M.p, S->V.p,
                                  S->ids32.p, S->ld, s);
            std::vector<uint32_t> ids32(nk);
            if (nk) CK(cudaMemcpyAsync(ids32.data(), S->ids32.p, 4 * (size_t)nk, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            S->ids64.assign(ids32.begin(), ids32.end());
            fresh[k] = std::move(S);
        }
        ctx->subsets = std::move(fresh);
        ctx->epoch = epoch;  // the manager's new epoch (manager.hpp:441)
        ctx->epoch_set = true;
        ctx->shared_dirty = true;
    });
}

int dgs_subset_store(dgs_ctx* ctx, int32_t k, dgs_splats* params, dgs_splats* m, dgs_splats* v,
                     uint64_t* adam_step) {
    return dgs_guard([&] {
        SubsetState& S = subset(*ctx, k);
        download_fields(*ctx, S, S.P.p, params);
        download_fields(*ctx, S, S.M.p, m);
        download_fields(*ctx, S, S.V.p, v);
        if (adam_step) *adam_step = S.adam_step;
    });
}

int dgs_init_from_pointcloud(dgs_ctx* ctx, const float* points, int64_t n_points, const float* colors,
                             int64_t n_colors, int64_t target, uint64_t seed, int32_t sh_degree, dgs_splats* out) {
    return dgs_guard([&] {
        if (ctx) ++ctx->graph_version;  // captured step graphs no longer match
        // trainer.hpp:24-91, host RNG in libstdc++ (bit-identical picks/jitter), neighbour term on the GPU
        if (n_points <= 0) throw std::invalid_argument("init_from_pointcloud: empty cloud");
        if (n_colors != 0 && n_colors != n_points) throw std::invalid_argument("init_from_pointcloud: color count mismatch");
        if (sh_degree < 0 || sh_degree > 3) throw std::invalid_argument("init_from_pointcloud: sh_degree must be 0..3");
        const int n_coeff = (sh_degree + 1) * (sh_degree + 1);
        if (out->n < target || out->sh_coeffs != n_coeff) throw std::invalid_argument("init_from_pointcloud: output too small");
        std::mt19937_64 rng(seed);
        std::vector<size_t> picks;
        picks.reserve((size_t)target);
        float jitter = 0.0f;
        if ((size_t)target <= (size_t)n_points) {
            std::vector<size_t> all((size_t)n_points);
            for (size_t i = 0; i < all.size(); ++i) all[i] = i;
            std::sample(all.begin(), all.end(), std::back_inserter(picks), (size_t)target, rng);
        } else {
            float lo[3], hi[3];
            for (int a = 0; a < 3; ++a) lo[a] = hi[a] = points[a];
            for (int64_t i = 0; i < n_points; ++i)
                for (int a = 0; a < 3; ++a) {
                    lo[a] = std::min(lo[a], points[3 * i + a]);
                    hi[a] = std::max(hi[a], points[3 * i + a]);
                }
            const float d0 = hi[0] - lo[0], d1 = hi[1] - lo[1], d2 = hi[2] - lo[2];
            jitter = 1e-3f * std::sqrt(dot3(d0, d1, d2, d0, d1, d2));  // T(1e-3) * (hi - lo).norm()
            std::uniform_int_distribution<size_t> pick(0, (size_t)n_points - 1);
            for (int64_t i = 0; i < target; ++i) picks.push_back(pick(rng));
        }
        std::normal_distribution<double> gauss;
        const size_t n = picks.size();
        std::vector<float> centers(3 * n);
        float lo[3], hi[3];
        for (size_t i = 0; i < n; ++i) {
            for (int a = 0; a < 3; ++a) centers[3 * i + a] = points[3 * picks[i] + a];
            if (jitter > 0.0f) {
                const float j0 = (float)gauss(rng) * jitter, j1 = (float)gauss(rng) * jitter,
                            j2 = (float)gauss(rng) * jitter;
                centers[3 * i] += j0;
                centers[3 * i + 1] += j1;
                centers[3 * i + 2] += j2;
            }
            for (int a = 0; a < 3; ++a) {
                lo[a] = i ? std::min(lo[a], centers[3 * i + a]) : centers[3 * i + a];
                hi[a] = i ? std::max(hi[a], centers[3 * i + a]) : centers[3 * i + a];
            }
        }
        std::vector<float> nn_mean(n, 1.0f);
        const int k_nn = (int)std::min<size_t>(3, n - 1);
        if (k_nn > 0) {
            CK(cudaSetDevice(ctx->device));
            DevBuf<float> dp, dm;
            dp.ensure(3 * n);
            dm.ensure(n);
            CK(cudaMemcpyAsync(dp.p, centers.data(), 12 * n, cudaMemcpyHostToDevice, ctx->stream));
            knn_mean_distance((int)n, k_nn, dp.p, dm.p, lo, hi, ctx->stream);
            CK(cudaGetLastError());
            CK(cudaMemcpyAsync(nn_mean.data(), dm.p, 4 * n, cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
        }
        const float op = std::log(0.1f / (1.0f - 0.1f));  // logit(T(0.1)), math.hpp:27-29
        const float c0 = (float)0.28209479177387814;     // T(sh::kC0)
        for (size_t i = 0; i < n; ++i) {
            if (out->id) out->id[i] = (uint64_t)i;
            const float ls = std::log(std::max(nn_mean[i], 1e-7f));
            for (int a = 0; a < 3; ++a) {
                out->mu[3 * i + a] = centers[3 * i + a];
                out->log_scale[3 * i + a] = ls;
            }
            out->rotation[4 * i] = 1.0f;
            out->rotation[4 * i + 1] = out->rotation[4 * i + 2] = out->rotation[4 * i + 3] = 0.0f;
            out->opacity_logit[i] = op;
            for (int c = 0; c < n_coeff; ++c)
                for (int a = 0; a < 3; ++a) out->sh[(i * n_coeff + c) * 3 + a] = 0.0f;
            for (int a = 0; a < 3; ++a) {
                const float col = n_colors ? colors[3 * picks[i] + a] : 0.5f;
                out->sh[(i * n_coeff) * 3 + a] = (col - 0.5f) / c0;
            }
        }
    });
}

int dgs_subset_ids(dgs_ctx* ctx, int32_t k, uint64_t* ids) {
    return dgs_guard([&] {
        const SubsetState& S = subset(*ctx, k);
        std::memcpy(ids, S.ids64.data(), S.ids64.size() * sizeof(uint64_t));
    });
}

int64_t dgs_subset_size(dgs_ctx* ctx, int32_t k) {
    auto it = ctx->subsets.find(k);
    return it == ctx->subsets.end() ? -1 : it->second->n;
}

int dgs_render_partial(dgs_ctx* ctx, int32_t k, const dgs_camera* cam, float* out_ct, int32_t dbg_cap,
                       uint32_t* dbg_ids, uint32_t* dbg_cnt) {
    return dgs_guard([&] {
        require_table(*ctx);
        SubsetState& S = subset(*ctx, k);
        check_epoch(*ctx, S);
        const ViewParams vp = view_params(*cam);
        const size_t px = (size_t)vp.width * vp.height;
        DevBuf<uint32_t> d_ids, d_cnt;
        if (dbg_cap > 0) {
            d_ids.ensure(px * dbg_cap);
            d_cnt.ensure(px);
        }
        forward_subset(*ctx, S, 0, vp, dbg_cap, d_ids.p, d_cnt.p);
        ViewSlot& vs = S.slot(0);
        if (out_ct) CK(cudaMemcpyAsync(out_ct, vs.ct.p, px * sizeof(float4), cudaMemcpyDeviceToHost, ctx->stream));
        if (dbg_cap > 0) {
            CK(cudaMemcpyAsync(dbg_ids, d_ids.p, px * dbg_cap * 4, cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaMemcpyAsync(dbg_cnt, d_cnt.p, px * 4, cudaMemcpyDeviceToHost, ctx->stream));
        }
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int dgs_dump_bins(dgs_ctx* ctx, int32_t k, int64_t* tile_off, int32_t* entries, int64_t cap, int64_t* n_pairs) {
    return dgs_guard([&] {
        SubsetState& S = subset(*ctx, k);
        ViewSlot& vs = S.slot(0);
        const int tiles = vs.vp.tiles_x * vs.vp.tiles_y;
        const int64_t P = vs.vb.pairs;
        *n_pairs = P;
        if (P > cap) throw std::invalid_argument("dump_bins: capacity too small");
        std::vector<uint2> rg(tiles);
        CK(cudaMemcpy(rg.data(), vs.vb.ranges, tiles * sizeof(uint2), cudaMemcpyDeviceToHost));
        std::vector<uint32_t> vals((size_t)P);
        if (P) CK(cudaMemcpy(vals.data(), vs.vb.pair_val, P * 4, cudaMemcpyDeviceToHost));
        int64_t o = 0;
        tile_off[0] = 0;
        for (int t = 0; t < tiles; ++t) {
            for (uint32_t p = rg[t].x; p < rg[t].y; ++p) entries[o++] = (int32_t)vals[p];
            tile_off[t + 1] = o;
        }
    });
}

int dgs_dump_records(dgs_ctx* ctx, int32_t k, float* recs, uint32_t* counts) {
    return dgs_guard([&] {
        SubsetState& S = subset(*ctx, k);
        ViewSlot& vs = S.slot(0);
        if (recs) CK(cudaMemcpy(recs, vs.vb.recs, S.n * sizeof(SplatRec), cudaMemcpyDeviceToHost));
        if (counts) CK(cudaMemcpy(counts, vs.vb.counts, S.n * 4, cudaMemcpyDeviceToHost));
    });
}

int dgs_pixel_orders(dgs_ctx* ctx, const dgs_camera* cam, uint16_t* order, uint16_t* count) {
    return dgs_guard([&] {
        require_table(*ctx);
        const ViewParams vp = view_params(*cam);
        const size_t px = (size_t)vp.width * vp.height;
        const int K = ctx->table.k_count;
        DevBuf<uint16_t> d_o, d_c;
        d_o.ensure(px * K);
        d_c.ensure(px);
        const int owner = table_locate(ctx->table, vp.o);
        launch_pixel_orders(vp, ctx->table_dev.p, owner, d_o.p, d_c.p, K, ctx->stream);
        CK(cudaMemcpyAsync(order, d_o.p, px * K * 2, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaMemcpyAsync(count, d_c.p, px * 2, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int dgs_merge(dgs_ctx* ctx, const dgs_camera* cam, const float* partials, const float bg[3], float* out_rgb,
              float* out_t) {
    return dgs_guard([&] {
        require_table(*ctx);
        const ViewParams vp = view_params(*cam);
        const size_t px = (size_t)vp.width * vp.height;
        const int K = ctx->table.k_count;
        ctx->scratch_maps.ensure(px * K);
        CK(cudaMemcpyAsync(ctx->scratch_maps.p, partials, px * K * sizeof(float4), cudaMemcpyHostToDevice, ctx->stream));
        std::vector<const float4*> ptrs(K);
        for (int k = 0; k < K; ++k) ptrs[k] = ctx->scratch_maps.p + px * k;
        ctx->partial_ptrs.ensure(K);
        CK(cudaMemcpyAsync(ctx->partial_ptrs.p, ptrs.data(), K * sizeof(void*), cudaMemcpyHostToDevice, ctx->stream));
        ctx->merged.ensure(3 * px);
        ctx->staging.ensure(4 * px);
        const int owner = table_locate(ctx->table, vp.o);
        launch_merge(vp, ctx->table_dev.p, owner, 0, vp.height, ctx->partial_ptrs.p, 0, bg, ctx->merged.p,
                     ctx->staging.p + 3 * px, 0, vp.height, ctx->stream);
        k_planar_to_hwc<<<(unsigned)((px + 255) / 256), 256, 0, ctx->stream>>>(ctx->merged.p, ctx->staging.p, px);
        CK(cudaMemcpyAsync(out_rgb, ctx->staging.p, 3 * px * 4, cudaMemcpyDeviceToHost, ctx->stream));
        if (out_t) CK(cudaMemcpyAsync(out_t, ctx->staging.p + 3 * px, px * 4, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int dgs_loss(dgs_ctx* ctx, int32_t width, int32_t height, const float* render, const float* target, double lambda,
             double inv_batch, float* grad, double* value, double* sums) {
    return dgs_guard([&] {
        if (width <= 0 || height <= 0) throw std::invalid_argument("loss: resolution mismatch");
        const size_t px = (size_t)width * height;
        ctx->staging.ensure(3 * px);
        ctx->merged.ensure(3 * px);
        ctx->grad_rgb.ensure(3 * px);
        DevBuf<float> tgt;
        tgt.ensure(3 * px);
        const unsigned g = (unsigned)((px + 255) / 256);
        CK(cudaMemcpyAsync(ctx->staging.p, render, 3 * px * 4, cudaMemcpyHostToDevice, ctx->stream));
        k_hwc_to_planar<<<g, 256, 0, ctx->stream>>>(ctx->staging.p, ctx->merged.p, px);
        CK(cudaMemcpyAsync(ctx->staging.p, target, 3 * px * 4, cudaMemcpyHostToDevice, ctx->stream));
        k_hwc_to_planar<<<g, 256, 0, ctx->stream>>>(ctx->staging.p, tgt.p, px);
        int nb = 0;
        const int max_blocks = ((width + 31) / 32) * ((height + 31) / 32) * 3;
        ctx->block_sums.ensure((size_t)max_blocks * 3);
        ctx->sums.ensure(3);
        launch_loss(width, height, 0, height, 0, height, ctx->merged.p, tgt.p, (float)lambda, ensure_kernel(*ctx),
                    (float)inv_batch, ctx->grad_rgb.p, ctx->block_sums.p, &nb, ctx->stream);
        launch_reduce_sums(ctx->block_sums.p, nb, ctx->sums.p, ctx->stream);
        k_planar_to_hwc<<<g, 256, 0, ctx->stream>>>(ctx->grad_rgb.p, ctx->staging.p, px);
        double s[3];
        CK(cudaMemcpyAsync(s, ctx->sums.p, sizeof(s), cudaMemcpyDeviceToHost, ctx->stream));
        if (grad) CK(cudaMemcpyAsync(grad, ctx->staging.p, 3 * px * 4, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        const double n = 3.0 * px;
        if (value) *value = (1.0 - lambda) * (s[0] / n) + lambda * (1.0 - s[1] / n);
        if (sums) std::memcpy(sums, s, sizeof(s));
    });
}

int dgs_merge_backward(dgs_ctx* ctx, const dgs_camera* cam, const float* partials, const float* grad_color,
                       const float bg[3], float* out_grads) {
    return dgs_guard([&] {
        require_table(*ctx);
        const ViewParams vp = view_params(*cam);
        const size_t px = (size_t)vp.width * vp.height;
        const int K = ctx->table.k_count;
        ctx->scratch_maps.ensure(px * K);
        ctx->scratch_grads.ensure(px * K);
        CK(cudaMemcpyAsync(ctx->scratch_maps.p, partials, px * K * sizeof(float4), cudaMemcpyHostToDevice, ctx->stream));
        std::vector<const float4*> ptrs(K);
        std::vector<float4*> gptrs(K);
        for (int k = 0; k < K; ++k) {
            ptrs[k] = ctx->scratch_maps.p + px * k;
            gptrs[k] = ctx->scratch_grads.p + px * k;
        }
        ctx->partial_ptrs.ensure(K);
        ctx->grad_ptrs.ensure(K);
        CK(cudaMemcpyAsync(ctx->partial_ptrs.p, ptrs.data(), K * sizeof(void*), cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(ctx->grad_ptrs.p, gptrs.data(), K * sizeof(void*), cudaMemcpyHostToDevice, ctx->stream));
        ctx->staging.ensure(3 * px);
        ctx->grad_rgb.ensure(3 * px);
        CK(cudaMemcpyAsync(ctx->staging.p, grad_color, 3 * px * 4, cudaMemcpyHostToDevice, ctx->stream));
        k_hwc_to_planar<<<(unsigned)((px + 255) / 256), 256, 0, ctx->stream>>>(ctx->staging.p, ctx->grad_rgb.p, px);
        const int owner = table_locate(ctx->table, vp.o);
        launch_merge_bwd(vp, ctx->table_dev.p, owner, 0, vp.height, ctx->partial_ptrs.p, 0, ctx->grad_rgb.p, 0,
                         vp.height, bg, ctx->grad_ptrs.p, 0, ctx->stream);
        CK(cudaMemcpyAsync(out_grads, ctx->scratch_grads.p, px * K * sizeof(float4), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

static void check_orders(int32_t width, int32_t height, int32_t k_count, int32_t k_stride, const uint16_t* order,
                         const uint16_t* count) {
    if (width <= 0 || height <= 0) throw std::invalid_argument("merge: non-positive resolution");
    if (k_count <= 0 || k_count > kMaxSubsets || k_stride < k_count)
        throw std::invalid_argument("merge: subset count out of range");
    const size_t px = (size_t)width * height;
    for (size_t p = 0; p < px; ++p) {
        if (count[p] > k_count) throw std::invalid_argument("merge: order count exceeds subset count");
        for (int i = 0; i < count[p]; ++i)
            if (order[p * k_stride + i] >= k_count) throw std::invalid_argument("merge: order names unknown subset");
    }
}

int dgs_merge_ordered(dgs_ctx* ctx, int32_t width, int32_t height, int32_t k_count, int32_t k_stride,
                      const uint16_t* order, const uint16_t* count, const float* partials, const float bg[3],
                      float* out_rgb, float* out_t) {
    return dgs_guard([&] {
        check_orders(width, height, k_count, k_stride, order, count);
        const size_t px = (size_t)width * height;
        DevBuf<uint16_t> d_o, d_c;
        d_o.ensure(px * k_stride);
        d_c.ensure(px);
        ctx->scratch_maps.ensure(px * k_count);
        ctx->staging.ensure(4 * px);
        CK(cudaMemcpyAsync(d_o.p, order, px * k_stride * 2, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(d_c.p, count, px * 2, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(ctx->scratch_maps.p, partials, px * k_count * sizeof(float4), cudaMemcpyHostToDevice,
                           ctx->stream));
        launch_merge_ordered((int)px, k_stride, d_o.p, d_c.p, ctx->scratch_maps.p, bg, ctx->staging.p,
                             ctx->staging.p + 3 * px, ctx->stream);
        CK(cudaMemcpyAsync(out_rgb, ctx->staging.p, 3 * px * 4, cudaMemcpyDeviceToHost, ctx->stream));
        if (out_t) CK(cudaMemcpyAsync(out_t, ctx->staging.p + 3 * px, px * 4, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int dgs_merge_backward_ordered(dgs_ctx* ctx, int32_t width, int32_t height, int32_t k_count, int32_t k_stride,
                               const uint16_t* order, const uint16_t* count, const float* partials,
                               const float* grad_color, const float* grad_trans_total, const float bg[3],
                               float* out_grads) {
    return dgs_guard([&] {
        check_orders(width, height, k_count, k_stride, order, count);
        const size_t px = (size_t)width * height;
        DevBuf<uint16_t> d_o, d_c;
        d_o.ensure(px * k_stride);
        d_c.ensure(px);
        ctx->scratch_maps.ensure(px * k_count);
        ctx->scratch_grads.ensure(px * k_count);
        ctx->staging.ensure(4 * px);
        CK(cudaMemcpyAsync(d_o.p, order, px * k_stride * 2, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(d_c.p, count, px * 2, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(ctx->scratch_maps.p, partials, px * k_count * sizeof(float4), cudaMemcpyHostToDevice,
                           ctx->stream));
        CK(cudaMemcpyAsync(ctx->staging.p, grad_color, 3 * px * 4, cudaMemcpyHostToDevice, ctx->stream));
        if (grad_trans_total)
            CK(cudaMemcpyAsync(ctx->staging.p + 3 * px, grad_trans_total, px * 4, cudaMemcpyHostToDevice,
                               ctx->stream));
        launch_merge_bwd_ordered((int)px, k_count, k_stride, d_o.p, d_c.p, ctx->scratch_maps.p, ctx->staging.p,
                                 grad_trans_total ? ctx->staging.p + 3 * px : nullptr, bg, ctx->scratch_grads.p,
                                 ctx->stream);
        CK(cudaMemcpyAsync(out_grads, ctx->scratch_grads.p, px * k_count * sizeof(float4), cudaMemcpyDeviceToHost,
                           ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int dgs_render_partial_backward(dgs_ctx* ctx, int32_t k, const dgs_camera* cam, const float* grad_ct,
                                dgs_splats* grads) {
    return dgs_guard([&] {
        require_table(*ctx);
        SubsetState& S = subset(*ctx, k);
        const ViewParams vp = view_params(*cam);
        const size_t px = (size_t)vp.width * vp.height;
        forward_subset(*ctx, S, 0, vp);
        ViewSlot& vs = S.slot(0);
        vs.grad_ct.ensure(px);
        CK(cudaMemcpyAsync(vs.grad_ct.p, grad_ct, px * sizeof(float4), cudaMemcpyHostToDevice, ctx->stream));
        reset_bad(*ctx);
        backward_blend(*ctx, S, 0, nullptr);
        S.G.ensure(S.rows * S.ld);
        CK(cudaMemsetAsync(S.G.p, 0, S.rows * S.ld * sizeof(float), ctx->stream));
        launch_project_bwd((int)S.n, S.P.p, S.ld, S.sh_coeffs, vp, ctx->ro, vs.vb.counts, S.g2d.p, S.ld, S.G.p,
                           ctx->bad.p, ctx->stream);
        check_bad(*ctx, S);
        download_fields(*ctx, S, S.G.p, grads);
    });
}

int dgs_dump_pixel_grads(dgs_ctx* ctx, int32_t k, float* out) {
    return dgs_guard([&] {
        SubsetState& S = subset(*ctx, k);
        if (S.g2d.p == nullptr) throw std::invalid_argument("no backward has run for this subset");
        std::vector<float> h(9 * S.ld);
        CK(cudaMemcpy(h.data(), S.g2d.p, h.size() * 4, cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < S.n; ++i)
            for (int f = 0; f < 9; ++f) out[i * 9 + f] = h[g2d_index(f, (size_t)i, S.ld)];
    });
}

int dgs_adam_apply(dgs_ctx* ctx, int32_t k, const dgs_splats* grads) {
    return dgs_guard([&] {
        SubsetState& S = subset(*ctx, k);
        S.G.ensure(S.rows * S.ld);
        upload_fields(*ctx, S, *grads, S.G.p);
        const AdamArgs aa = adam_args(*ctx, S, nullptr);
        launch_adam((int)S.n, S.P.p, S.M.p, S.V.p, S.ld, S.rows, S.G.p, aa, ctx->stream);
        ++S.adam_step;
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int dgs_upload_targets(dgs_ctx* ctx, int32_t batch, int32_t width, int32_t height, const float* targets_hwc,
                       const float** device_ptr) {
    return dgs_guard([&] {
        const size_t px = (size_t)width * height;
        ctx->targets.ensure(batch * 3 * px);
        ctx->staging.ensure(3 * px);
        for (int b = 0; b < batch; ++b) {
            CK(cudaMemcpyAsync(ctx->staging.p, targets_hwc + b * 3 * px, 3 * px * 4, cudaMemcpyHostToDevice,
                               ctx->stream));
            k_hwc_to_planar<<<(unsigned)((px + 255) / 256), 256, 0, ctx->stream>>>(ctx->staging.p,
                                                                                    ctx->targets.p + b * 3 * px, px);
        }
        CK(cudaStreamSynchronize(ctx->stream));
        *device_ptr = ctx->targets.p;
    });
}

int dgs_render(dgs_ctx* ctx, const dgs_camera* cam, const float bg[3], float* out_rgb, float* out_t) {
    return dgs_guard([&] {
        require_table(*ctx);
        if (ctx->world != 1) throw std::invalid_argument("dgs_render: multi-rank render goes through dgs_train_step");
        const ViewParams vp = view_params(*cam);
        const size_t px = (size_t)vp.width * vp.height;
        const int K = ctx->table.k_count;
        std::vector<const float4*> ptrs(K);
        for (int k = 0; k < K; ++k) {
            SubsetState& S = subset(*ctx, k);
            forward_subset(*ctx, S, 0, vp);
            ptrs[k] = S.slot(0).ct.p;
        }
        ctx->partial_ptrs.ensure(K);
        CK(cudaMemcpyAsync(ctx->partial_ptrs.p, ptrs.data(), K * sizeof(void*), cudaMemcpyHostToDevice, ctx->stream));
        ctx->merged.ensure(3 * px);
        ctx->staging.ensure(4 * px);
        const int owner = table_locate(ctx->table, vp.o);
        launch_merge(vp, ctx->table_dev.p, owner, 0, vp.height, ctx->partial_ptrs.p, 0, bg, ctx->merged.p,
                     ctx->staging.p + 3 * px, 0, vp.height, ctx->stream);
        k_planar_to_hwc<<<(unsigned)((px + 255) / 256), 256, 0, ctx->stream>>>(ctx->merged.p, ctx->staging.p, px);
        if (out_rgb) CK(cudaMemcpyAsync(out_rgb, ctx->staging.p, 3 * px * 4, cudaMemcpyDeviceToHost, ctx->stream));
        if (out_t) CK(cudaMemcpyAsync(out_t, ctx->staging.p + 3 * px, px * 4, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

StepTail& step_tail(Ctx& ctx, int batch, int S, int nlocal) {
    if (batch > kTailMaxBatch || S > kTailMaxSlices || nlocal > kTailMaxLocal)
        throw std::invalid_argument("train_step: batch, slices and local subsets are limited to 64 each");
    if (!ctx.tail) CK(cudaHostAlloc(reinterpret_cast<void**>(&ctx.tail), sizeof(StepTail), cudaHostAllocDefault));
    ctx.tail->nsums = (size_t)3 * batch * S;
    return *ctx.tail;
}
void finish_step(Ctx& ctx_, const std::vector<int>& local, dgs_step_result* out);

/// Manager::train_step (manager.hpp:313-386).  Eager: launches and finishes the
/// step (the pair counts are read back mid-step).  With ctx->capturing it only
/// enqueues the step (no host round trip) for a CUDA graph, including the
/// copies of its results into the pinned tail buffer; finish_step() turns the
/// tail into the step result after the replay.
void train_step_graph(dgs_ctx* ctx, int32_t batch, const dgs_camera* cams, const float* targets,
                      int32_t targets_on_device, const float bg[3], dgs_step_result* out);
void train_step_body(dgs_ctx* ctx, int32_t batch, const dgs_camera* cams, const float* targets,
                     int32_t targets_on_device, const float bg[3], dgs_step_result* out);

int dgs_train_step(dgs_ctx* ctx, int32_t batch, const dgs_camera* cams, const float* targets,
                   int32_t targets_on_device, const float bg[3], dgs_step_result* out) {
    return dgs_guard([&] {
        if (!ctx) throw std::invalid_argument("train_step: null context");
        bool graph = ctx->graph_mode && ctx->world == 1 && !ctx->timer.on && !ctx->collect_stats &&
                     batch >= 1 && cams != nullptr && targets != nullptr && ctx->cfg.grad_sync == 0;
        if (graph && !targets_on_device) {  // the graph copies host targets by DMA: pinned memory only
            cudaPointerAttributes at{};
            graph = cudaPointerGetAttributes(&at, targets) == cudaSuccess && at.type == cudaMemoryTypeHost;
            cudaGetLastError();
        }
        if (graph) train_step_graph(ctx, batch, cams, targets, targets_on_device, bg, out);
        else train_step_body(ctx, batch, cams, targets, targets_on_device, bg, out);
    });
}

/// Pinned host targets: every view's window [h0, h0 + tgt_win / (3 Wd0)) H2D
/// into tgt_stage on the copy stream, after the main stream's earlier work
/// (the previous step's readers of the staging); copy_done marks the end.
__global__ void k_spin_ns(unsigned long long ns) {
    const unsigned long long t0 = clock64();
    // ~ns at >= 1 GHz; only for the upload-ordering test (DGS_TEST_UPLOAD_DELAY_US)
    while ((unsigned long long)(clock64() - t0) < ns) __nanosleep(1000);
}

static void upload_pinned_targets(Ctx* ctx, int batch, const float* targets, int Wd0, int H0, int h0,
                                  size_t tgt_win) {
    CK(cudaEventRecord(ctx->copy_done, ctx->stream));
    CK(cudaStreamWaitEvent(ctx->copy_stream, ctx->copy_done, 0));
    // tests: hold the upload back so that a consumer which did not wait for it would read stale data
    static const long delay_us = getenv("DGS_TEST_UPLOAD_DELAY_US") ? atol(getenv("DGS_TEST_UPLOAD_DELAY_US")) : 0;
    if (delay_us > 0) k_spin_ns<<<1, 1, 0, ctx->copy_stream>>>((unsigned long long)delay_us * 2000ull);
    for (int v = 0; v < batch; ++v)
        CK(cudaMemcpyAsync(ctx->tgt_stage.p + (size_t)v * tgt_win,
                           targets + (size_t)v * 3 * Wd0 * H0 + (size_t)h0 * Wd0 * 3, tgt_win * 4,
                           cudaMemcpyHostToDevice, ctx->copy_stream));
    CK(cudaEventRecord(ctx->copy_done, ctx->copy_stream));
}

void train_step_body(dgs_ctx* ctx, int32_t batch, const dgs_camera* cams, const float* targets,
                     int32_t targets_on_device, const float bg[3], dgs_step_result* out) {
    {
        require_table(*ctx);
        if (batch < 1 || cams == nullptr || targets == nullptr)
            throw std::invalid_argument("train_step: need one target per camera");
        if (batch != ctx->cfg.batch_size) throw std::invalid_argument("train_step: batch size mismatch with config");
        const int K = ctx->table.k_count, W = ctx->world, rank = ctx->rank;
        std::vector<int> local;
        for (int k = 0; k < K; ++k) {
            const int o = subset_owner(k, K, W);
            const bool here = ctx->subsets.count(k) != 0;
            if (W == 1 && !here) throw std::invalid_argument("merge: missing subset partials: " + std::to_string(k));
            if (W > 1 && (o == rank) != here)
                throw std::invalid_argument("train_step: subset " + std::to_string(k) + " must live on rank " +
                                            std::to_string(o));
            if (here) local.push_back(k);
        }
        for (int k : local) check_epoch(*ctx, subset(*ctx, k));
        const uint64_t launches0 = ctx->launches;
        uint64_t nccl_bytes = 0;
        launch_zero(ctx->stats.p, 2 * sizeof(BlendStats), ctx->stream);
        launch_zero(ctx->abort.ensure(1), sizeof(int), ctx->stream);
        ctx->launches += 2;
        std::vector<ViewParams> vps(batch);
        uint64_t pairs = 0, visible = 0;
        const float lam = (float)ctx->cfg.lambda_ssim;
        const float inv_batch = 1.0f / (float)batch;  // manager.hpp:329
        const int S = W > 1 ? W : std::max(1, ctx->virtual_slices);
        const bool zero_copy = (W == 1 && S == 1);
        static const bool no_overlap = getenv("DGS_NO_VIEW_OVERLAP") != nullptr;  // A/B switch
        const bool overlap = batch > 1 && !ctx->host_xfer && !no_overlap;
        while (overlap && (int)ctx->view_done.size() < batch) {
            cudaEvent_t e;
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            ctx->view_done.push_back(e);
        }
        ctx->partial_ptrs.ensure((size_t)K);
        ctx->grad_ptrs.ensure((size_t)K);
        ctx->sums.ensure((size_t)3 * batch * S);
        for (int v = 0; v < batch; ++v) {
            vps[v] = view_params(cams[v]);
            if (v > 0 && (vps[v].width != vps[0].width || vps[v].height != vps[0].height))
                throw std::invalid_argument("train_step: all views of a batch must share a resolution");
        }
        // Host targets: the H2D copy of every view's target window runs on the
        // copy stream while the forward renders (the main stream waits for it
        // only at the first loss); pinned host memory makes it asynchronous.
        const int my_slice = W > 1 ? rank : -1;
        size_t tgt_win = 0;
        if (!targets_on_device) {
            const int Wd0 = vps[0].width, H0 = vps[0].height;
            int h0 = 0, h1 = H0;
            if (my_slice >= 0) {
                const SliceRows R = slice_rows(H0, S, my_slice);
                h0 = R.h0;
                h1 = R.h1;
            }
            tgt_win = (size_t)(h1 - h0) * Wd0 * 3;
            ctx->tgt_stage.ensure(tgt_win * batch);
            cudaPointerAttributes at{};
            const bool pinned = cudaPointerGetAttributes(&at, targets) == cudaSuccess && at.type == cudaMemoryTypeHost;
            cudaGetLastError();  // unregistered pointers may leave an error on older runtimes
            if (pinned && ctx->capturing) {
                // graph steps: the replay wrapper enqueues the upload outside the
                // graph (upload_pinned_targets); the graph waits on copy_done as an
                // external event, so the DMA overlaps the captured forward
            } else if (pinned) {
                upload_pinned_targets(ctx, batch, targets, Wd0, H0, h0, tgt_win);
            } else {
                CK(cudaEventRecord(ctx->copy_done, ctx->stream));  // staging reuse: previous step's readers are done
                CK(cudaStreamWaitEvent(ctx->copy_stream, ctx->copy_done, 0));
                // pageable: cudaMemcpyAsync would stage synchronously on this thread
                // (the GPU idles meanwhile); copy through pinned memory on a helper
                // thread instead, overlapped with the forward (the previous step's
                // H2D from pin_stage completed before its loss)
                if (ctx->pin_cap < tgt_win * batch) {
                    if (ctx->pin_stage) CK(cudaFreeHost(ctx->pin_stage));
                    ctx->pin_stage = nullptr;
                    CK(cudaHostAlloc(reinterpret_cast<void**>(&ctx->pin_stage), tgt_win * batch * 4,
                                     cudaHostAllocDefault));
                    ctx->pin_cap = tgt_win * batch;
                }
                const size_t plane_all = (size_t)3 * Wd0 * H0, row0 = (size_t)h0 * Wd0 * 3;
                Ctx* cx = ctx;
                ctx->stager_err.clear();
                ctx->stager = std::thread([cx, targets, batch, tgt_win, plane_all, row0] {
                    // host memcpy bandwidth per core is the limit: split the copy over a
                    // few threads, each queueing the H2D of its 1 MB pieces as they land
                    const unsigned hw = std::thread::hardware_concurrency();
                    const int nt = (int)std::max(1u, std::min(8u, hw ? hw / 2 : 1u));
                    const size_t total = tgt_win * (size_t)batch, per = (total + nt - 1) / nt;
                    std::vector<std::thread> ws;
                    std::vector<int> bad(nt, 0);
                    for (int w = 0; w < nt; ++w)
                        ws.emplace_back([&, w] {
                            cudaSetDevice(cx->device);
                            constexpr size_t kPiece = (size_t)1 << 18;  // floats (1 MB)
                            const size_t b = std::min(total, (size_t)w * per), e = std::min(total, b + per);
                            for (size_t o = b; o < e;) {
                                const size_t v = o / tgt_win, in_v = o - v * tgt_win;
                                const size_t len = std::min({kPiece, e - o, tgt_win - in_v});
                                std::memcpy(cx->pin_stage + o, targets + v * plane_all + row0 + in_v, len * 4);
                                if (cudaMemcpyAsync(cx->tgt_stage.p + o, cx->pin_stage + o, len * 4,
                                                    cudaMemcpyHostToDevice, cx->copy_stream) != cudaSuccess)
                                    bad[w] = 1;
                                o += len;
                            }
                        });
                    for (auto& t : ws) t.join();
                    cudaSetDevice(cx->device);
                    for (int w = 0; w < nt; ++w)
                        if (bad[w]) cx->stager_err = "train_step: target upload failed";
                    if (cudaEventRecord(cx->copy_done, cx->copy_stream) != cudaSuccess)
                        cx->stager_err = "train_step: target upload event failed";
                });
            }
        }
        // the stager (if any) is joined before the loss waits for the copy, and on every exit
        struct JoinStager {
            Ctx* c;
            ~JoinStager() {
                if (c->stager.joinable()) c->stager.join();
            }
        } join_stager{ctx};
        bool waited_copy = false;
        for (int v = 0; v < batch; ++v) {
            const ViewParams& vp = vps[v];
            const int Wd = vp.width, H = vp.height;
            const size_t px = (size_t)Wd * H;
            // ---- render_batch (manager.hpp:262-304): per-subset partials ----
            for (int k : local) {
                SubsetState& S_ = subset(*ctx, k);
                forward_subset(*ctx, S_, v, vp, 0, nullptr, nullptr, ctx->collect_stats ? ctx->stats.p : nullptr);
                pairs += (uint64_t)S_.slot(v).vb.pairs;
                visible += (uint64_t)S_.slot(v).vb.visible;
                S_.slot(v).grad_ct.ensure(px);
            }
            const int owner = table_locate(ctx->table, vp.o);
            const float* kern = ensure_kernel(*ctx);
            // the view's exchange / merge / loss / merge-adjoint chain: on xstream when
            // a later view's forward can run meanwhile (batch > 1; not with the
            // host-staged test transport, whose exchanges synchronise the stream)
            cudaStream_t cs = ctx->stream;
            if (overlap) {
                cs = ctx->xstream;
                CK(cudaEventRecord(ctx->view_done[v], ctx->stream));
                CK(cudaStreamWaitEvent(cs, ctx->view_done[v], 0));
            }
            const std::vector<int> slices = W > 1 ? std::vector<int>{rank} : [&] {
                std::vector<int> a(S);
                for (int i = 0; i < S; ++i) a[i] = i;
                return a;
            }();
            for (int sl : slices) {
                const SliceRows R = slice_rows(H, S, sl);
                const int hr = R.h1 - R.h0, orows = R.r1 - R.r0;
                // ---- forward exchange: partial rows [h0, h1) of every subset -> this slice ----
                std::vector<const float4*> ptrs(K);
                std::vector<float4*> gptrs(K);
                int prow0 = 0, grow0 = 0;
                if (zero_copy) {
                    for (int k = 0; k < K; ++k) {
                        ptrs[k] = subset(*ctx, k).slot(v).ct.p;
                        gptrs[k] = subset(*ctx, k).slot(v).grad_ct.p;
                    }
                } else {
                    ctx->xrecv.ensure((size_t)K * hr * Wd);
                    ctx->xgrad.ensure((size_t)K * orows * Wd);
                    for (int k = 0; k < K; ++k) {
                        ptrs[k] = ctx->xrecv.p + (size_t)k * hr * Wd;
                        gptrs[k] = ctx->xgrad.p + (size_t)k * orows * Wd;
                    }
                    prow0 = R.h0;
                    grow0 = R.r0;
                    Stage st(ctx->timer, kStExchange, cs);
                    nccl_bytes += exchange_forward(*ctx, v, local, Wd, H, S, sl, cs);
                }
                h2d(*ctx, ctx->partial_ptrs.p, ptrs.data(), K * sizeof(void*), cs);
                h2d(*ctx, ctx->grad_ptrs.p, gptrs.data(), K * sizeof(void*), cs);
                // ---- merge (engine.hpp:152-182) over rows [h0, h1) ----
                ctx->merged.ensure((size_t)3 * hr * Wd);
                {
                    Stage st(ctx->timer, kStMerge, cs);
                    launch_merge(vp, ctx->table_dev.p, owner, R.h0, R.h1, ctx->partial_ptrs.p, prow0, bg,
                                 ctx->merged.p, nullptr, R.h0, hr, cs);
                }
                // ---- target window ----
                ctx->targets_win.ensure((size_t)3 * hr * Wd);
                const float* tgt;
                if (targets_on_device && zero_copy) {
                    tgt = targets + (size_t)v * 3 * px;
                } else if (targets_on_device) {
                    for (int c = 0; c < 3; ++c)
                        CK(cudaMemcpyAsync(ctx->targets_win.p + (size_t)c * hr * Wd,
                                           targets + (size_t)v * 3 * px + (size_t)c * px + (size_t)R.h0 * Wd,
                                           (size_t)hr * Wd * 4, cudaMemcpyDeviceToDevice, cs));
                    tgt = ctx->targets_win.p;
                } else {
                    if (!waited_copy) {
                        if (ctx->stager.joinable()) ctx->stager.join();
                        if (!ctx->stager_err.empty()) throw std::runtime_error(ctx->stager_err);
                        CK(cudaStreamWaitEvent(cs, ctx->copy_done, ctx->capturing ? cudaEventWaitExternal : 0));
                        waited_copy = true;
                    }
                    // window rows [h0, h1) inside the prefetched window (which starts at
                    // row 0 for a single rank, at this rank's halo start otherwise)
                    const int base_row = my_slice >= 0 ? slice_rows(H, S, my_slice).h0 : 0;
                    const float* src = ctx->tgt_stage.p + (size_t)v * tgt_win + (size_t)(R.h0 - base_row) * Wd * 3;
                    k_hwc_to_planar<<<(unsigned)(((size_t)hr * Wd + 255) / 256), 256, 0, cs>>>(
                        src, ctx->targets_win.p, (size_t)hr * Wd);
                    ++ctx->launches;
                    tgt = ctx->targets_win.p;
                }
                // ---- loss (manager.hpp:331-334) on owned rows [r0, r1) ----
                ctx->grad_rgb.ensure((size_t)3 * hr * Wd);
                const int max_blocks = ((Wd + 31) / 32) * ((orows + 31) / 32) * 3;
                ctx->block_sums.ensure((size_t)max_blocks * 3);
                int nb = 0;
                {
                    Stage st(ctx->timer, kStLoss, cs);
                    launch_loss(Wd, H, R.r0, R.r1, R.h0, hr, ctx->merged.p, tgt, lam, kern, inv_batch,
                                ctx->grad_rgb.p, ctx->block_sums.p, &nb, cs);
                    launch_reduce_sums(ctx->block_sums.p, nb, ctx->sums.p + (size_t)3 * (v * S + sl), cs);
                }
                // ---- merge_backward (engine.hpp:195-234) on owned rows ----
                {
                    Stage st(ctx->timer, kStMergeBwd, cs);
                    launch_merge_bwd(vp, ctx->table_dev.p, owner, R.r0, R.r1, ctx->partial_ptrs.p, prow0,
                                     ctx->grad_rgb.p, R.h0, hr, bg, ctx->grad_ptrs.p, grow0, cs);
                }
                ctx->launches += 4;
                // ---- backward exchange: (dL/dC_k, dL/dT_k) rows [r0, r1) -> subset owners ----
                if (!zero_copy) {
                    Stage st(ctx->timer, kStExchange, cs);
                    nccl_bytes += exchange_backward(*ctx, v, local, Wd, H, S, sl, cs);
                }
            }
        }
        if (overlap) {  // every view's chain precedes the backward
            CK(cudaEventRecord(ctx->chain_done, ctx->xstream));
            CK(cudaStreamWaitEvent(ctx->stream, ctx->chain_done, 0));
        }
        // ---- MsgBackwardTask x B, then apply_step (worker.hpp:86-127, 162-167) ----
        reset_bad(*ctx);
        const bool sync = ctx->cfg.grad_sync != 0 && K > 1;
        if (sync) {
            // config.grad_sync (worker.hpp:103-144, manager.hpp:351-379): full gradients of
            // every member, shared replicas summed in worker order, then the dense Adam step
            if (W > 1) build_shared_multi(*ctx);
            else build_shared(*ctx);
            std::vector<float*> gp;
            std::vector<size_t> gl;
            for (int k : local) {
                SubsetState& S_ = subset(*ctx, k);
                S_.G.ensure(S_.rows * S_.ld);  // the first view's pullback overwrites every row
                for (int v = 0; v < batch; ++v) {
                    ViewSlot& vs = S_.slot(v);
                    backward_blend(*ctx, S_, v, ctx->collect_stats ? ctx->stats.p + 1 : nullptr);
                    Stage st(ctx->timer, kStProjBwd, ctx->stream);
                    launch_project_bwd((int)S_.n, S_.P.p, S_.ld, S_.sh_coeffs, vs.vp, ctx->ro, vs.vb.counts, S_.g2d.p,
                                       S_.ld, S_.G.p, ctx->bad.p, ctx->stream, v == 0);
                    ++ctx->launches;
                }
            }
            // G pointers indexed by subset id k (reps encode k)
            int kmax = 0;
            for (int k : local) kmax = std::max(kmax, k);
            gp.assign(kmax + 1, nullptr);
            gl.assign(kmax + 1, 0);
            for (int k : local) {
                gp[k] = subset(*ctx, k).G.p;
                gl[k] = subset(*ctx, k).ld;
            }
            // pointer tables persist in the context (stream-ordered uploads from pageable
            // vectors: the runtime stages them before returning, no sync needed)
            float** dG = ctx->gsync_G.ensure(kmax + 1);
            size_t* dL = ctx->gsync_ld.ensure(kmax + 1);
            CK(cudaMemcpyAsync(dG, gp.data(), (kmax + 1) * sizeof(float*), cudaMemcpyHostToDevice, ctx->stream));
            CK(cudaMemcpyAsync(dL, gl.data(), (kmax + 1) * sizeof(size_t), cudaMemcpyHostToDevice, ctx->stream));
            const int rows = subset(*ctx, local[0]).rows;
            if (W > 1) {
                // G pointers in ascending local k (the order of the cross-rank replica numbering)
                std::vector<float*> gl2;
                std::vector<size_t> ll2;
                for (int k : local) {
                    gl2.push_back(subset(*ctx, k).G.p);
                    ll2.push_back(subset(*ctx, k).ld);
                }
                float** dG2 = ctx->gsync_G2.ensure(gl2.size());
                size_t* dL2 = ctx->gsync_ld2.ensure(ll2.size());
                CK(cudaMemcpyAsync(dG2, gl2.data(), gl2.size() * sizeof(float*), cudaMemcpyHostToDevice, ctx->stream));
                CK(cudaMemcpyAsync(dL2, ll2.data(), ll2.size() * sizeof(size_t), cudaMemcpyHostToDevice, ctx->stream));
                grad_sync_multi(*ctx, rows, dG2, dL2, (int)local.size());
            } else {
                grad_sync(ctx->sh_slots, rows, ctx->sh_starts.p, ctx->sh_nrep, ctx->sh_keys.p, ctx->sh_reps.p, dG, dL,
                          ctx->stream);
            }
            ++ctx->launches;
            for (int k : local) {
                SubsetState& S_ = subset(*ctx, k);
                const AdamArgs aa = adam_args(*ctx, S_, ctx->abort.p);
                Stage st(ctx->timer, kStAdam, ctx->stream);
                launch_adam((int)S_.n, S_.P.p, S_.M.p, S_.V.p, S_.ld, S_.rows, S_.G.p, aa, ctx->stream);
                ++ctx->launches;
                ++S_.adam_step;
            }
        }
        for (int k : (sync ? std::vector<int>{} : local)) {
            SubsetState& S_ = subset(*ctx, k);
            const AdamArgs ap = adam_args(*ctx, S_, ctx->abort.p);
            // K9 (gradient record, one per view) + K10 (streaming Adam after the last view)
            S_.rec.ensure(kGradRecordRows(batch) * S_.ld);
            for (int v = 0; v < batch; ++v) {
                ViewSlot& vs = S_.slot(v);
                backward_blend(*ctx, S_, v, ctx->collect_stats ? ctx->stats.p + 1 : nullptr, true);
                const bool last = v + 1 == batch;
                cudaEvent_t a = nullptr, m1 = nullptr, m2 = nullptr, b = nullptr;
                if (ctx->timer.on) {
                    a = ctx->timer.get();
                    m1 = ctx->timer.get();
                    m2 = last ? ctx->timer.get() : nullptr;
                    CK(cudaEventRecord(a, ctx->stream));
                }
                launch_project_bwd_adam((int)S_.n, S_.P.p, S_.M.p, S_.V.p, S_.ld, S_.sh_coeffs, vs.vp, ctx->ro,
                                        vs.vb.counts, vs.vb.shjac, S_.g2d.p, S_.ld,
                                        ctx->cfg.deterministic ? S_.g2q.p : nullptr, v, batch, ap, ctx->bad.p,
                                        S_.rec.p, last ? m1 : nullptr, m2, ctx->stream);
                if (ctx->timer.on) {
                    if (!last) CK(cudaEventRecord(m1, ctx->stream));
                    ctx->timer.pending.push_back({kStProjBwd, {a, m1}});
                    if (last) {
                        b = ctx->timer.get();
                        CK(cudaEventRecord(b, ctx->stream));
                        ctx->timer.pending.push_back({kStAdam, {m2, b}});
                    }
                }
                ctx->launches += last ? 2 : 1;
            }
            ++S_.adam_step;
        }
        // loss sums: slices of this rank (fixed order), then across ranks
        StepTail& T = step_tail(*ctx, batch, S, (int)local.size());
        double* sums = T.sums;
        if (W > 1) {
            if (ctx->capturing) throw std::logic_error("graph capture: single rank only");
            // every rank wrote only its own slice entry; zero the others and sum across ranks
            std::vector<double> mine((size_t)3 * batch * S, 0.0);
            CK(cudaMemcpyAsync(sums, ctx->sums.p, T.nsums * 8, cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
            for (int v = 0; v < batch; ++v)
                for (int q = 0; q < 3; ++q) mine[(size_t)3 * (v * S + rank) + q] = sums[(size_t)3 * (v * S + rank) + q];
            CK(cudaMemcpyAsync(ctx->sums.p, mine.data(), mine.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
            if (ctx->host_xfer) {
                if (ctx->xfer_cb.allreduce_sum_f64(ctx->xfer_cb.user, mine.data(), mine.size()))
                    throw std::runtime_error("host transport: allreduce failed");
                CK(cudaMemcpyAsync(ctx->sums.p, mine.data(), mine.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
                CK(cudaStreamSynchronize(ctx->stream));
            } else {
                Stage st(ctx->timer, kStExchange, ctx->stream);
                NK(nccl().AllReduce(ctx->sums.p, ctx->sums.p, mine.size(), ncclDouble, ncclSum, ctx->comm, ctx->stream));
            }
        }
        CK(cudaMemcpyAsync(sums, ctx->sums.p, T.nsums * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaMemcpyAsync(T.st, ctx->stats.p, 2 * sizeof(BlendStats), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaMemcpyAsync(&T.bad, ctx->bad.p, 4, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaMemcpyAsync(&T.abort, ctx->abort.p, 4, cudaMemcpyDeviceToHost, ctx->stream));
        // ring-overflow pixels of every (subset, view): the fallback kernels' device counts
        for (size_t i = 0; i < local.size(); ++i)
            for (int v = 0; v < batch; ++v) {
                SubsetState& S_ = subset(*ctx, local[i]);
                ViewSlot& vs = S_.slot(v);
                const size_t q = i * batch + v;
                CK(cudaMemcpyAsync(&T.ovf[q], vs.ovf_count.p, 4, cudaMemcpyDeviceToHost, ctx->stream));
                if (ctx->capturing && S_.n > 0) {  // what the eager step reads back mid-step
                    CK(cudaMemcpyAsync(&T.pairs[q], vs.scan.p + (S_.n - 1), 4, cudaMemcpyDeviceToHost, ctx->stream));
                    CK(cudaMemcpyAsync(&T.visible[q], vs.vb.dmax_bits + 2, 4, cudaMemcpyDeviceToHost, ctx->stream));
                    CK(cudaMemcpyAsync(&T.err[q], vs.vb.err_index, 4, cudaMemcpyDeviceToHost, ctx->stream));
                } else {
                    T.pairs[q] = (uint32_t)std::max<int64_t>(0, vs.vb.pairs);
                    T.visible[q] = (uint32_t)vs.vb.visible;
                    T.err[q] = INT_MAX;
                }
            }
        T.nccl_bytes = nccl_bytes;
        T.launches = ctx->launches - launches0;
        T.batch = batch;
        T.slices = S;
        T.nlocal = (int)local.size();
        for (int v = 0; v < batch; ++v) T.px[v] = (double)vps[v].width * vps[v].height;
        T.comm_bytes = (uint64_t)2 * K * batch * (uint64_t)vps[0].width * vps[0].height * 4 * sizeof(float);
        if (ctx->capturing) return;  // the replay reads the tail
        CK(cudaStreamSynchronize(ctx->stream));
        CK(cudaGetLastError());
        ctx->timer.resolve();
        finish_step(*ctx, local, out);
    }
}

std::vector<int> local_subsets(Ctx& ctx) {
    std::vector<int> local;
    for (int k = 0; k < ctx.table.k_count; ++k)
        if (ctx.subsets.count(k) != 0) local.push_back(k);
    return local;
}

/// One train step through a CUDA graph (dgs_set_graph_mode): the first call for
/// a key runs eagerly (it learns every slot's pair count), the second records
/// the step into a graph and replays it, later calls only write this step's
/// AdamParams into the pinned staging read by the graph and replay.  A replay
/// whose pair counts outgrew the captured sort capacity (ctx.abort & 2: K10
/// skipped it, nothing persistent changed) is re-run eagerly and re-captured on
/// the next call; a zero quaternion (ctx.abort & 1) is raised like the eager
/// step, with the parameters untouched.
void train_step_graph(dgs_ctx* ctx, int32_t batch, const dgs_camera* cams, const float* targets,
                      int32_t targets_on_device, const float bg[3], dgs_step_result* out) {
    std::vector<uint8_t> key(sizeof(int32_t) * 2 + sizeof(dgs_camera) * batch + sizeof(void*) + 3 * sizeof(float) +
                             2 * sizeof(uint64_t));
    uint8_t* kp = key.data();
    auto put = [&](const void* src, size_t b) {
        std::memcpy(kp, src, b);
        kp += b;
    };
    const uint64_t epoch = g_buffer_epoch.load();
    put(&batch, sizeof(batch));
    put(&targets_on_device, sizeof(targets_on_device));
    put(cams, sizeof(dgs_camera) * batch);
    const float* tkey = targets_on_device ? targets : nullptr;  // pinned targets are uploaded outside the graph
    put(&tkey, sizeof(void*));
    put(bg, 3 * sizeof(float));
    put(&ctx->graph_version, sizeof(uint64_t));
    put(&epoch, sizeof(uint64_t));
    const std::vector<int> local = local_subsets(*ctx);
    Ctx::CachedStep* g = nullptr;
    for (auto& e : ctx->graphs)
        if (e.key == key) g = &e;
    if (g == nullptr) {
        if (std::find(ctx->warmed.begin(), ctx->warmed.end(), key) == ctx->warmed.end()) {
            train_step_body(ctx, batch, cams, targets, targets_on_device, bg, out);
            if (g_buffer_epoch.load() == epoch) ctx->warmed.push_back(key);  // sizes settled: capture next time
            return;
        }
        // the sort capacity of every (subset, view) slot: its largest pair count + 2 %
        for (int k : local) {
            SubsetState& S = subset(*ctx, k);
            for (int v = 0; v < batch; ++v) {
                ViewSlot& vs = S.slot(v);
                vs.graph_cap = std::min<int64_t>(vs.pair_cap, vs.pairs_max + vs.pairs_max / 50 + 4096);
                if (getenv("DGS_GRAPH_CAP_TEST")) vs.graph_cap = std::max<int64_t>(1, vs.pairs_max / 2);  // tests: overflow
            }
        }
        std::vector<uint64_t> steps;
        for (int k : local) steps.push_back(subset(*ctx, k).adam_step);
        cudaGraph_t graph = nullptr;
        ctx->capturing = true;
        CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeRelaxed));
        try {
            train_step_body(ctx, batch, cams, targets, targets_on_device, bg, nullptr);
        } catch (...) {
            cudaStreamEndCapture(ctx->stream, &graph);
            if (graph) cudaGraphDestroy(graph);
            ctx->capturing = false;
            cudaGetLastError();
            for (size_t i = 0; i < local.size(); ++i) subset(*ctx, local[i]).adam_step = steps[i];
            throw;
        }
        const cudaError_t ec = cudaStreamEndCapture(ctx->stream, &graph);
        ctx->capturing = false;
        for (size_t i = 0; i < local.size(); ++i) subset(*ctx, local[i]).adam_step = steps[i];  // the replay counts
        if (ec != cudaSuccess) throw CudaError(std::string("CUDA error: ") + cudaGetErrorString(ec) + " (graph capture)");
        Ctx::CachedStep e;
        e.key = key;
        e.graph = graph;
        // K10's kernel nodes: their AdamParams argument is replaced at every replay
        size_t nn = 0;
        CK(cudaGraphGetNodes(graph, nullptr, &nn));
        std::vector<cudaGraphNode_t> nodes(nn);
        if (nn) CK(cudaGraphGetNodes(graph, nodes.data(), &nn));
        for (cudaGraphNode_t nd : nodes) {
            cudaGraphNodeType ty;
            CK(cudaGraphNodeGetType(nd, &ty));
            if (ty != cudaGraphNodeTypeKernel) continue;
            cudaKernelNodeParams kp{};
            CK(cudaGraphKernelNodeGetParams(nd, &kp));
            int pi = -1;
            const int ai = adam_param_index(kp.func, &pi);
            if (ai < 0) continue;
            const float* Pn = *reinterpret_cast<float* const*>(kp.kernelParams[pi]);
            for (int k : local)
                if (subset(*ctx, k).P.p == Pn) e.adam.push_back({nd, k, ai});
        }
        const cudaError_t ei = cudaGraphInstantiate(&e.exec, graph, 0);
        if (ei != cudaSuccess) {
            Ctx::free_step(e);
            throw CudaError(std::string("CUDA error: ") + cudaGetErrorString(ei) + " (graph instantiate)");
        }
        if (ctx->graphs.size() >= 64) {  // bounded cache: drop the oldest
            Ctx::free_step(ctx->graphs.front());
            ctx->graphs.erase(ctx->graphs.begin());
        }
        ctx->graphs.push_back(e);
        g = &ctx->graphs.back();
    }
    // ---- replay: this step's AdamParams into the K10 nodes, launch ----
    for (int k : local) check_epoch(*ctx, subset(*ctx, k));
    for (const auto& an : g->adam) {
        cudaKernelNodeParams kp{};
        CK(cudaGraphKernelNodeGetParams(an.node, &kp));
        AdamParams ap = adam_params(*ctx, subset(*ctx, an.subset), subset(*ctx, an.subset).adam_step + 1);
        std::vector<void*> args;
        for (int a = 0; a <= an.ap_index + 1; ++a) args.push_back(kp.kernelParams[a]);
        args[an.ap_index] = &ap;
        kp.kernelParams = args.data();
        CK(cudaGraphExecKernelNodeSetParams(g->exec, an.node, &kp));
    }
    if (!targets_on_device) {  // pinned host targets (single rank: the whole image)
        const int Wd0 = cams[0].width, H0 = cams[0].height;
        const size_t tgt_win = (size_t)H0 * Wd0 * 3;
        ctx->tgt_stage.ensure(tgt_win * batch);
        upload_pinned_targets(ctx, batch, targets, Wd0, H0, 0, tgt_win);
    }
    CK(cudaGraphLaunch(g->exec, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaGetLastError());
    StepTail& T = *ctx->tail;
    if (T.abort & 2) {  // a pair count outgrew the captured sort: redo eagerly, re-capture next time
        Ctx::free_step(*g);
        ctx->graphs.erase(ctx->graphs.begin() + (g - ctx->graphs.data()));
        ctx->warmed.erase(std::remove(ctx->warmed.begin(), ctx->warmed.end(), key), ctx->warmed.end());
        train_step_body(ctx, batch, cams, targets, targets_on_device, bg, out);
        ctx->warmed.push_back(key);
        return;
    }
    for (int q = 0; q < T.nlocal * batch; ++q)
        if (T.err[q] != INT_MAX) throw std::domain_error("zero quaternion");
    for (int k : local) ++subset(*ctx, k).adam_step;
    finish_step(*ctx, local, out);
}

/// The step result from the tail buffer (eager: just synchronised; graph:
/// after the replay).  Throws the reference's non-finite-gradient error.
void finish_step(Ctx& ctx_, const std::vector<int>& local, dgs_step_result* out) {
    Ctx* ctx = &ctx_;
    StepTail& T = *ctx->tail;
    const int batch = T.batch, S = T.slices;
    const double* sums = T.sums;
    const BlendStats* st = T.st;
    {
        if (T.bad != INT_MAX) {
            throw std::runtime_error("partial_render_backward: non-finite gradient for splat id " +
                                     std::to_string(subset(*ctx, local[0]).ids64[(size_t)T.bad]));
        }
        if (out) {
            std::memset(out, 0, sizeof(*out));
            double loss = 0.0, mse = 0.0;
            const double lambda = ctx->cfg.lambda_ssim;
            for (int v = 0; v < batch; ++v) {
                double s3[3] = {0.0, 0.0, 0.0};
                for (int sl = 0; sl < S; ++sl)
                    for (int q = 0; q < 3; ++q) s3[q] += sums[(size_t)3 * (v * S + sl) + q];
                const double n = 3.0 * T.px[v];
                loss += ((1.0 - lambda) * (s3[0] / n) + lambda * (1.0 - s3[1] / n)) / batch;
                mse += (s3[2] / n) / batch;
            }
            out->loss = loss;
            out->psnr = mse == 0.0 ? INFINITY : 10.0 * std::log10(1.0 / mse);
            // reference accounting (manager.hpp:384): every partial map and its
            // gradient cross a link: 2 * K * H * W * 4 * sizeof(float) per view.
            out->comm_bytes = T.comm_bytes;
            out->nccl_bytes = T.nccl_bytes;
            out->pairs = 0;
            out->visible = 0;
            out->overflow_pixels = 0;
            for (int q = 0; q < T.nlocal * batch; ++q) {
                out->pairs += T.pairs[q];
                out->visible += T.visible[q];
                out->overflow_pixels += T.ovf[q];
            }
            out->evals_fwd = st[0].evals;
            out->contribs_fwd = st[0].contribs;
            out->evals_bwd = st[1].evals;
            out->contribs_bwd = st[1].contribs;
            out->subrounds_bwd = st[1].subrounds;
            out->small_subrounds_bwd = st[1].small_rounds;
            out->tiles_work_fwd = st[0].tiles_work;
            out->replay_tiles_bwd = st[1].tiles_work;
            out->kernel_launches = T.launches;
        }
    }
}

int dgs_dump_grad_maps(dgs_ctx* ctx, int32_t k, int32_t view, float* partial_ct, float* grad_ct) {
    return dgs_guard([&] {
        SubsetState& S = subset(*ctx, k);
        if (view < 0 || view >= (int)S.slots.size()) throw std::invalid_argument("dump_grad_maps: no such view slot");
        ViewSlot& vs = S.slot(view);
        const size_t px = (size_t)vs.vp.width * vs.vp.height;
        if (partial_ct) CK(cudaMemcpy(partial_ct, vs.ct.p, px * sizeof(float4), cudaMemcpyDeviceToHost));
        if (grad_ct) {
            if (!vs.grad_ct.p) throw std::invalid_argument("dump_grad_maps: no backward has run");
            CK(cudaMemcpy(grad_ct, vs.grad_ct.p, px * sizeof(float4), cudaMemcpyDeviceToHost));
        }
    });
}

int dgs_set_graph_mode(dgs_ctx* ctx, int32_t enabled) {
    return dgs_guard([&] {
        if (!ctx) throw std::invalid_argument("set_graph_mode: null context");
        ctx->graph_mode = enabled != 0;
        if (!ctx->graph_mode) ctx->drop_graphs();
    });
}

int dgs_state_save(dgs_ctx* ctx) {
    return dgs_guard([&] {
        if (!ctx) throw std::invalid_argument("state_save: null context");
        CK(cudaSetDevice(ctx->device));
        for (auto& kv : ctx->subsets) {
            SubsetState& S = *kv.second;
            const size_t plane = (size_t)S.rows * S.ld;
            S.saved.ensure(3 * plane);
            CK(cudaMemcpyAsync(S.saved.p, S.P.p, plane * 4, cudaMemcpyDeviceToDevice, ctx->stream));
            CK(cudaMemcpyAsync(S.saved.p + plane, S.M.p, plane * 4, cudaMemcpyDeviceToDevice, ctx->stream));
            CK(cudaMemcpyAsync(S.saved.p + 2 * plane, S.V.p, plane * 4, cudaMemcpyDeviceToDevice, ctx->stream));
            S.saved_step = S.adam_step;
        }
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int dgs_state_restore(dgs_ctx* ctx) {
    return dgs_guard([&] {
        if (!ctx) throw std::invalid_argument("state_restore: null context");
        CK(cudaSetDevice(ctx->device));
        for (auto& kv : ctx->subsets) {
            SubsetState& S = *kv.second;
            const size_t plane = (size_t)S.rows * S.ld;
            if (S.saved.p == nullptr || S.saved.n < 3 * plane)
                throw std::invalid_argument("state_restore: no saved state for subset " + std::to_string(kv.first));
            CK(cudaMemcpyAsync(S.P.p, S.saved.p, plane * 4, cudaMemcpyDeviceToDevice, ctx->stream));
            CK(cudaMemcpyAsync(S.M.p, S.saved.p + plane, plane * 4, cudaMemcpyDeviceToDevice, ctx->stream));
            CK(cudaMemcpyAsync(S.V.p, S.saved.p + 2 * plane, plane * 4, cudaMemcpyDeviceToDevice, ctx->stream));
            S.adam_step = S.saved_step;
        }
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int dgs_set_collect_stats(dgs_ctx* ctx, int32_t enabled) {
    return dgs_guard([&] { ctx->collect_stats = enabled != 0; });
}

int dgs_set_backward_records(dgs_ctx* ctx, int32_t enabled) {
    return dgs_guard([&] {
        if (ctx) ++ctx->graph_version;  // captured step graphs no longer match
        ctx->records = enabled != 0;
    });
}

int dgs_set_virtual_slices(dgs_ctx* ctx, int32_t slices) {
    return dgs_guard([&] {
        if (ctx) ++ctx->graph_version;  // captured step graphs no longer match
        if (slices < 1) throw std::invalid_argument("virtual slices must be >= 1");
        if (ctx->world > 1 && slices != 1) throw std::invalid_argument("virtual slices are a single-rank mode");
        ctx->virtual_slices = slices;
    });
}

int dgs_slice_plan(int32_t height, int32_t slices, int32_t s, int32_t* rows4) {
    return dgs_guard([&] {
        if (height < 1 || slices < 1 || s < 0 || s >= slices) throw std::invalid_argument("slice_plan: bad arguments");
        const SliceRows R = slice_rows(height, slices, s);
        rows4[0] = R.r0;
        rows4[1] = R.r1;
        rows4[2] = R.h0;
        rows4[3] = R.h1;
    });
}

int32_t dgs_subset_owner(int32_t k, int32_t k_count, int32_t world) { return subset_owner(k, k_count, world); }

}  // extern "C"
