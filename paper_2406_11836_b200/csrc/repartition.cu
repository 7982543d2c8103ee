// Device-side repartition (Manager::repartition / snapshot / distribute,
// manager.hpp:389-482; build_kdtree / assign_subsets, partition.hpp:93-251):
// the kernels; the orchestration (a few host round trips of O(2^L) scalars)
// lives in capi.cu (dgs_repartition).
//
//   snapshot   every replica (subset k, member i) gets the key
//              id << 8 | (locate(mu) == k ? 0 : 1) << 5 | k; a radix sort and a
//              first-of-run selection keep, per splat id, the replica held by
//              the subspace containing its centre, else the lowest k
//              (manager.hpp:400-414).
//   KD build   level by level over the merged centres: per-node extents
//              (order-preserving integer atomics), the widest axis (first
//              maximum), a radix sort of (node, axis coordinate) keys for the
//              exact lower/upper medians, and the < plane / >= plane split
//              (partition.hpp:100-153).  Identical float values to the
//              reference's std::sort + std::nth_element: sorting is exact.
//   assign     one thread per splat: membership bits of every subspace
//              (plane values <= 3 max(exp(log_scale)), glibc-expf port).
//   migrate    per new subset: flagged compaction, gather of the p, m, v rows.
#include <cub/cub.cuh>

#include "kernels.h"

namespace dgs_b200 {

namespace {

__device__ __forceinline__ uint32_t float_order(float f) {
    const uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__global__ void k_snapshot_keys(int n, const float* __restrict__ P, size_t ld, const uint32_t* __restrict__ ids32,
                                const Table* __restrict__ tb, int k, uint32_t base, uint64_t* __restrict__ keys,
                                uint32_t* __restrict__ vals) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float x[3] = {P[i], P[ld + i], P[2 * ld + i]};
    const int owner = table_locate(*tb, x);
    const uint64_t prio = owner == k ? 0u : 1u;
    keys[base + i] = ((uint64_t)ids32[i] << 8) | (prio << 5) | (uint64_t)k;
    vals[base + i] = base + (uint32_t)i;
}

__global__ void k_first_of_run(int n, const uint64_t* __restrict__ keys, uint8_t* __restrict__ flags) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    flags[i] = (i == 0 || (keys[i] >> 8) != (keys[i - 1] >> 8)) ? 1 : 0;
}

/// merged[r][j] = src_k[r][i] for replica (k, i) = winners[j]; K sources given
/// as device arrays of row-0 pointers, leading dimensions and replica offsets.
__global__ void k_gather_replicas(int n, int rows, const uint32_t* __restrict__ winners,
                                  const uint32_t* __restrict__ offsets, int K, const float* const* __restrict__ srcP,
                                  const float* const* __restrict__ srcM, const float* const* __restrict__ srcV,
                                  const uint32_t* const* __restrict__ srcId, const size_t* __restrict__ lds,
                                  float* __restrict__ P, float* __restrict__ M, float* __restrict__ V,
                                  uint32_t* __restrict__ ids, size_t ld) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const uint32_t r = winners[j];
    int k = 0;
    while (k + 1 < K && offsets[k + 1] <= r) ++k;
    const size_t i = r - offsets[k], sl = lds[k];
    for (int q = 0; q < rows; ++q) {
        P[(size_t)q * ld + j] = srcP[k][(size_t)q * sl + i];
        M[(size_t)q * ld + j] = srcM[k][(size_t)q * sl + i];
        V[(size_t)q * ld + j] = srcV[k][(size_t)q * sl + i];
    }
    ids[j] = srcId[k][i];
}

/// Per-node extents and counts (nodes < 256): block-local accumulation, one
/// atomic per (block, node, quantity).
__global__ void k_node_extent(int n, const float* __restrict__ P, size_t ld, const uint8_t* __restrict__ node,
                              int nnodes, uint32_t* __restrict__ lo, uint32_t* __restrict__ hi,
                              uint32_t* __restrict__ cnt) {
    __shared__ uint32_t slo[3 * 256], shi[3 * 256], scnt[256];
    for (int q = threadIdx.x; q < nnodes; q += blockDim.x) {
        scnt[q] = 0;
        for (int a = 0; a < 3; ++a) {
            slo[3 * q + a] = 0xffffffffu;
            shi[3 * q + a] = 0u;
        }
    }
    __syncthreads();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int q = node[i];
        atomicAdd(&scnt[q], 1u);
        for (int a = 0; a < 3; ++a) {
            const uint32_t o = float_order(P[(size_t)a * ld + i]);
            atomicMin(&slo[3 * q + a], o);
            atomicMax(&shi[3 * q + a], o);
        }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < nnodes; q += blockDim.x) {
        if (scnt[q] == 0) continue;
        atomicAdd(&cnt[q], scnt[q]);
        for (int a = 0; a < 3; ++a) {
            atomicMin(&lo[3 * q + a], slo[3 * q + a]);
            atomicMax(&hi[3 * q + a], shi[3 * q + a]);
        }
    }
}

__global__ void k_node_keys(int n, const float* __restrict__ P, size_t ld, const uint8_t* __restrict__ node,
                            const int* __restrict__ axis, uint64_t* __restrict__ keys) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int q = node[i];
    keys[i] = ((uint64_t)q << 32) | float_order(P[(size_t)axis[q] * ld + i]);
}

/// partition.hpp:130-131: < plane goes left (child 2q), >= plane right (2q + 1).
__global__ void k_node_split(int n, const float* __restrict__ P, size_t ld, uint8_t* __restrict__ node,
                             const int* __restrict__ axis, const float* __restrict__ plane) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int q = node[i];
    node[i] = (uint8_t)(2 * q + (P[(size_t)axis[q] * ld + i] < plane[q] ? 0 : 1));
}

/// assign_subsets (partition.hpp:234-251): bit k set iff every plane value of
/// subspace k at mu is <= d_mult * max(exp(log_scale)).
__global__ void k_assign(int n, const float* __restrict__ P, size_t ld, const Table* __restrict__ tb, float mult,
                         uint32_t* __restrict__ mask) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float mu0 = P[i], mu1 = P[ld + i], mu2 = P[2 * ld + i];
    const float s0 = glibc_expf(P[(size_t)kRowLogScale * ld + i]), s1 = glibc_expf(P[(size_t)(kRowLogScale + 1) * ld + i]),
                s2 = glibc_expf(P[(size_t)(kRowLogScale + 2) * ld + i]);
    float smax = s0;  // Vec3::maxCoeff
    if (s1 > smax) smax = s1;
    if (s2 > smax) smax = s2;
    const float di = fmul(mult, smax);
    uint32_t m = 0;
    for (int k = 0; k < tb->k_count; ++k) {
        const Subspace& s = tb->sub[k];
        bool member = true;
        for (int p = 0; p < s.n; ++p) {
            const float v = fadd(dot3(s.nx[p], s.ny[p], s.nz[p], mu0, mu1, mu2), s.d[p]);
            if (v > di) {
                member = false;
                break;
            }
        }
        if (member) m |= 1u << k;
    }
    mask[i] = m;
}

__global__ void k_flag_bit(int n, const uint32_t* __restrict__ mask, int k, uint8_t* __restrict__ flags) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flags[i] = (mask[i] >> k) & 1u;
}

__global__ void k_gather_members(int n, int rows, const uint32_t* __restrict__ idx, const float* __restrict__ P,
                                 const float* __restrict__ M, const float* __restrict__ V,
                                 const uint32_t* __restrict__ ids, size_t ld_src, float* __restrict__ dP,
                                 float* __restrict__ dM, float* __restrict__ dV, uint32_t* __restrict__ dids,
                                 size_t ld_dst) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const size_t i = idx[j];
    for (int q = 0; q < rows; ++q) {
        dP[(size_t)q * ld_dst + j] = P[(size_t)q * ld_src + i];
        dM[(size_t)q * ld_dst + j] = M[(size_t)q * ld_src + i];
        dV[(size_t)q * ld_dst + j] = V[(size_t)q * ld_src + i];
    }
    dids[j] = ids[i];
}

/// Shared-replica index (grad sync): key id << 8 | k, value k << 27 | i.
__global__ void k_replica_keys(int n, const uint32_t* __restrict__ ids32, int k, uint32_t base,
                               uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    keys[base + i] = ((uint64_t)ids32[i] << 8) | (uint64_t)k;
    vals[base + i] = ((uint32_t)k << 27) | (uint32_t)i;
}

/// flags[j] = 1 iff sorted position j starts a run of >= 2 replicas of one id.
__global__ void k_shared_run_starts(int n, const uint64_t* __restrict__ keys, uint8_t* __restrict__ flags) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const uint64_t id = keys[j] >> 8;
    const bool start = j == 0 || (keys[j - 1] >> 8) != id;
    flags[j] = (start && j + 1 < n && (keys[j + 1] >> 8) == id) ? 1 : 0;
}

/// manager.hpp:359-378: per shared id and gradient row, the sum over its
/// replicas in worker order (first replica's value, then += the next ones),
/// written back to every replica's gradient row.
__global__ void k_grad_sync(int nslots, int rows, const uint32_t* __restrict__ starts, int nrep,
                            const uint64_t* __restrict__ keys, const uint32_t* __restrict__ reps,
                            float* const* __restrict__ G, const size_t* __restrict__ lds) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nslots * rows) return;
    const int s = t / rows, r = t % rows;
    const uint32_t b = starts[s];
    const uint64_t id = keys[b] >> 8;
    uint32_t e = b + 1;
    while (e < (uint32_t)nrep && (keys[e] >> 8) == id) ++e;
    float acc = 0.0f;
    for (uint32_t j = b; j < e; ++j) {
        const uint32_t k = reps[j] >> 27, i = reps[j] & 0x7ffffffu;
        const float g = G[k][(size_t)r * lds[k] + i];
        acc = j == b ? g : fadd(acc, g);
    }
    for (uint32_t j = b; j < e; ++j) {
        const uint32_t k = reps[j] >> 27, i = reps[j] & 0x7ffffffu;
        G[k][(size_t)r * lds[k] + i] = acc;
    }
}

inline unsigned blocks(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

}  // namespace

void repart_snapshot_keys(int n, const float* P, size_t ld, const uint32_t* ids32, const Table* tb, int k,
                          uint32_t base, uint64_t* keys, uint32_t* vals, cudaStream_t s) {
    if (n > 0) k_snapshot_keys<<<blocks(n), 256, 0, s>>>(n, P, ld, ids32, tb, k, base, keys, vals);
}

size_t repart_temp_bytes(int64_t n) {
    size_t a = 0, b = 0, c = 0;
    cub::DoubleBuffer<uint64_t> dk;
    cub::DoubleBuffer<uint32_t> dv;
    cub::DeviceRadixSort::SortPairs(nullptr, a, dk, dv, (int)n, 0, 64);
    cub::DeviceRadixSort::SortKeys(nullptr, b, dk, (int)n, 0, 64);
    cub::DeviceSelect::Flagged(nullptr, c, (const uint32_t*)nullptr, (const uint8_t*)nullptr, (uint32_t*)nullptr,
                               (int*)nullptr, (int)n);
    size_t d = 0;
    cub::DeviceSelect::Flagged(nullptr, d, cub::CountingInputIterator<uint32_t>(0u), (const uint8_t*)nullptr,
                               (uint32_t*)nullptr, (int*)nullptr, (int)n);
    size_t e = 0;
    cub::DeviceSelect::Flagged(nullptr, e, (const uint64_t*)nullptr, (const uint8_t*)nullptr, (uint64_t*)nullptr,
                               (int*)nullptr, (int)n);
    return std::max(std::max(a, b), std::max(c, std::max(d, e))) + 256;
}

void repart_sort_pairs(uint64_t*& keys, uint64_t*& keys_alt, uint32_t*& vals, uint32_t*& vals_alt, int n, int bits,
                       void* temp, size_t tb, cudaStream_t s) {
    cub::DoubleBuffer<uint64_t> dk(keys, keys_alt);
    cub::DoubleBuffer<uint32_t> dv(vals, vals_alt);
    cub::DeviceRadixSort::SortPairs(temp, tb, dk, dv, n, 0, bits, s);
    if (dk.Current() != keys) {
        std::swap(keys, keys_alt);
        std::swap(vals, vals_alt);
    }
}

void repart_sort_keys(uint64_t*& keys, uint64_t*& keys_alt, int n, int bits, void* temp, size_t tb, cudaStream_t s) {
    cub::DoubleBuffer<uint64_t> dk(keys, keys_alt);
    cub::DeviceRadixSort::SortKeys(temp, tb, dk, n, 0, bits, s);
    if (dk.Current() != keys) std::swap(keys, keys_alt);
}

void repart_first_of_run(int n, const uint64_t* keys, uint8_t* flags, cudaStream_t s) {
    if (n > 0) k_first_of_run<<<blocks(n), 256, 0, s>>>(n, keys, flags);
}

void repart_select(int n, const uint32_t* in, const uint8_t* flags, uint32_t* out, int* count, void* temp, size_t tb,
                   cudaStream_t s) {
    cub::DeviceSelect::Flagged(temp, tb, in, flags, out, count, n, s);
}

void repart_select_u64(int n, const uint64_t* in, const uint8_t* flags, uint64_t* out, int* count, void* temp,
                       size_t tb, cudaStream_t s) {
    cub::DeviceSelect::Flagged(temp, tb, in, flags, out, count, n, s);
}

void repart_select_iota(int n, const uint8_t* flags, uint32_t* out, int* count, void* temp, size_t tb,
                        cudaStream_t s) {
    cub::CountingInputIterator<uint32_t> it(0u);
    cub::DeviceSelect::Flagged(temp, tb, it, flags, out, count, n, s);
}

void repart_gather_replicas(int n, int rows, const uint32_t* winners, const uint32_t* offsets, int K,
                            const float* const* srcP, const float* const* srcM, const float* const* srcV,
                            const uint32_t* const* srcId, const size_t* lds, float* P, float* M, float* V,
                            uint32_t* ids, size_t ld, cudaStream_t s) {
    if (n > 0)
        k_gather_replicas<<<blocks(n), 256, 0, s>>>(n, rows, winners, offsets, K, srcP, srcM, srcV, srcId, lds, P, M,
                                                    V, ids, ld);
}

void repart_node_extent(int n, const float* P, size_t ld, const uint8_t* node, int nnodes, uint32_t* lo,
                        uint32_t* hi, uint32_t* cnt, cudaStream_t s) {
    if (n > 0) k_node_extent<<<std::min<unsigned>(blocks(n), 148 * 4), 256, 0, s>>>(n, P, ld, node, nnodes, lo, hi,
                                                                                     cnt);
}

void repart_node_keys(int n, const float* P, size_t ld, const uint8_t* node, const int* axis, uint64_t* keys,
                      cudaStream_t s) {
    if (n > 0) k_node_keys<<<blocks(n), 256, 0, s>>>(n, P, ld, node, axis, keys);
}

void repart_node_split(int n, const float* P, size_t ld, uint8_t* node, const int* axis, const float* plane,
                       cudaStream_t s) {
    if (n > 0) k_node_split<<<blocks(n), 256, 0, s>>>(n, P, ld, node, axis, plane);
}

void repart_assign(int n, const float* P, size_t ld, const Table* tb, float mult, uint32_t* mask, cudaStream_t s) {
    if (n > 0) k_assign<<<blocks(n), 256, 0, s>>>(n, P, ld, tb, mult, mask);
}

void repart_flag_bit(int n, const uint32_t* mask, int k, uint8_t* flags, cudaStream_t s) {
    if (n > 0) k_flag_bit<<<blocks(n), 256, 0, s>>>(n, mask, k, flags);
}

void repart_gather_members(int n, int rows, const uint32_t* idx, const float* P, const float* M, const float* V,
                           const uint32_t* ids, size_t ld_src, float* dP, float* dM, float* dV, uint32_t* dids,
                           size_t ld_dst, cudaStream_t s) {
    if (n > 0)
        k_gather_members<<<blocks(n), 256, 0, s>>>(n, rows, idx, P, M, V, ids, ld_src, dP, dM, dV, dids, ld_dst);
}

void shared_replica_keys(int n, const uint32_t* ids32, int k, uint32_t base, uint64_t* keys, uint32_t* vals,
                         cudaStream_t s) {
    if (n > 0) k_replica_keys<<<blocks(n), 256, 0, s>>>(n, ids32, k, base, keys, vals);
}

void shared_run_starts(int n, const uint64_t* keys, uint8_t* flags, cudaStream_t s) {
    if (n > 0) k_shared_run_starts<<<blocks(n), 256, 0, s>>>(n, keys, flags);
}

void grad_sync(int nslots, int rows, const uint32_t* starts, int nrep, const uint64_t* keys, const uint32_t* reps,
               float* const* G, const size_t* lds, cudaStream_t s) {
    if (nslots > 0) k_grad_sync<<<blocks((int64_t)nslots * rows), 256, 0, s>>>(nslots, rows, starts, nrep, keys, reps, G,
                                                                              lds);
}

namespace {

__global__ void k_flag_owned(int n, const uint32_t* __restrict__ mask, uint32_t owned, uint8_t* __restrict__ flags) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flags[i] = (mask[i] & owned) != 0u;
}

__global__ void k_flag_range(int n, const uint32_t* __restrict__ v, uint32_t lo, uint32_t hi,
                             uint8_t* __restrict__ flags) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flags[i] = v[i] >= lo && v[i] < hi;
}

__global__ void k_sub_const(int n, uint32_t* __restrict__ v, uint32_t c) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] -= c;
}

/// AoS record per migrating splat: rows of p, then m, then v, the id and the
/// membership mask (as float bits).
__global__ void k_pack(int n, int rows, const uint32_t* __restrict__ idx, const float* __restrict__ P,
                       const float* __restrict__ M, const float* __restrict__ V, const uint32_t* __restrict__ ids,
                       const uint32_t* __restrict__ mask, size_t ld, float* __restrict__ out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const size_t i = idx[j];
    const int stride = 3 * rows + 2;
    float* o = out + (size_t)j * stride;
    for (int q = 0; q < rows; ++q) {
        o[q] = P[(size_t)q * ld + i];
        o[rows + q] = M[(size_t)q * ld + i];
        o[2 * rows + q] = V[(size_t)q * ld + i];
    }
    o[3 * rows] = __uint_as_float(ids[i]);
    o[3 * rows + 1] = __uint_as_float(mask[i]);
}

__global__ void k_unpack(int n, int rows, const float* __restrict__ in, float* __restrict__ P, float* __restrict__ M,
                         float* __restrict__ V, uint32_t* __restrict__ ids, uint32_t* __restrict__ mask, size_t ld) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const int stride = 3 * rows + 2;
    const float* r = in + (size_t)j * stride;
    for (int q = 0; q < rows; ++q) {
        P[(size_t)q * ld + j] = r[q];
        M[(size_t)q * ld + j] = r[rows + q];
        V[(size_t)q * ld + j] = r[2 * rows + q];
    }
    ids[j] = __float_as_uint(r[3 * rows]);
    mask[j] = __float_as_uint(r[3 * rows + 1]);
}

}  // namespace

void repart_flag_owned(int n, const uint32_t* mask, uint32_t owned, uint8_t* flags, cudaStream_t s) {
    if (n > 0) k_flag_owned<<<blocks(n), 256, 0, s>>>(n, mask, owned, flags);
}
void repart_flag_range(int n, const uint32_t* v, uint32_t lo, uint32_t hi, uint8_t* flags, cudaStream_t s) {
    if (n > 0) k_flag_range<<<blocks(n), 256, 0, s>>>(n, v, lo, hi, flags);
}
void repart_sub_const(int n, uint32_t* v, uint32_t c, cudaStream_t s) {
    if (n > 0) k_sub_const<<<blocks(n), 256, 0, s>>>(n, v, c);
}
void repart_pack(int n, int rows, const uint32_t* idx, const float* P, const float* M, const float* V,
                 const uint32_t* ids, const uint32_t* mask, size_t ld, float* out, cudaStream_t s) {
    if (n > 0) k_pack<<<blocks(n), 256, 0, s>>>(n, rows, idx, P, M, V, ids, mask, ld, out);
}
void repart_unpack(int n, int rows, const float* in, float* P, float* M, float* V, uint32_t* ids, uint32_t* mask,
                   size_t ld, cudaStream_t s) {
    if (n > 0) k_unpack<<<blocks(n), 256, 0, s>>>(n, rows, in, P, M, V, ids, mask, ld);
}

// ---- cross-rank shared-replica gradient sync (grad_sync with world > 1) ----
namespace {

/// flags[j] = 1 iff sorted replica j belongs to a run of >= 2 replicas of one id.
__global__ void k_mark_shared(int n, const uint64_t* __restrict__ keys, uint8_t* __restrict__ flags) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const uint64_t id = keys[j] >> 8;
    flags[j] = ((j > 0 && (keys[j - 1] >> 8) == id) || (j + 1 < n && (keys[j + 1] >> 8) == id)) ? 1 : 0;
}

/// Map a global replica index to (local subset slot q, member i) of this rank.
__device__ __forceinline__ void local_ref(uint32_t g, uint32_t base, const uint32_t* __restrict__ offs, int KL,
                                          int& q, uint32_t& i) {
    const uint32_t r = g - base;
    q = 0;
    while (q + 1 < KL && offs[q + 1] <= r) ++q;
    i = r - offs[q];
}

__global__ void k_pack_shared(int n, int rows, const uint32_t* __restrict__ pos, const uint32_t* __restrict__ sg,
                              uint32_t base, const uint32_t* __restrict__ offs, int KL, float* const* __restrict__ G,
                              const size_t* __restrict__ lds, float* __restrict__ out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * rows) return;
    const int e = t / rows, r = t % rows;
    int q;
    uint32_t i;
    local_ref(sg[pos[e]], base, offs, KL, q, i);
    out[(size_t)e * rows + r] = G[q][(size_t)r * lds[q] + i];
}

/// sums over each id's replicas in worker (k) order, then written back to
/// this rank's replicas (manager.hpp:363-371 reduction, worker.hpp:131-140 apply).
__global__ void k_sync_shared(int S, int rows, const uint64_t* __restrict__ skeys, const uint32_t* __restrict__ src,
                              const float* __restrict__ recv, const uint8_t* __restrict__ mine,
                              const uint32_t* __restrict__ sg, uint32_t base, const uint32_t* __restrict__ offs, int KL,
                              float* const* __restrict__ G, const size_t* __restrict__ lds) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= S * rows) return;
    const int j = t / rows, r = t % rows;
    const uint64_t id = skeys[j] >> 8;
    if (!mine[j]) return;
    int b = j;
    while (b > 0 && (skeys[b - 1] >> 8) == id) --b;
    float acc = 0.0f;
    for (int e = b; e < S && (skeys[e] >> 8) == id; ++e) {
        const float g = recv[(size_t)src[e] * rows + r];
        acc = e == b ? g : fadd(acc, g);
    }
    int q;
    uint32_t i;
    local_ref(sg[j], base, offs, KL, q, i);
    G[q][(size_t)r * lds[q] + i] = acc;
}

}  // namespace

void shared_mark(int n, const uint64_t* keys, uint8_t* flags, cudaStream_t s) {
    if (n > 0) k_mark_shared<<<blocks(n), 256, 0, s>>>(n, keys, flags);
}
void shared_pack(int n, int rows, const uint32_t* pos, const uint32_t* sg, uint32_t base, const uint32_t* offs, int KL,
                 float* const* G, const size_t* lds, float* out, cudaStream_t s) {
    if (n > 0) k_pack_shared<<<blocks((int64_t)n * rows), 256, 0, s>>>(n, rows, pos, sg, base, offs, KL, G, lds, out);
}
void shared_sync(int S, int rows, const uint64_t* skeys, const uint32_t* src, const float* recv, const uint8_t* mine,
                 const uint32_t* sg, uint32_t base, const uint32_t* offs, int KL, float* const* G, const size_t* lds,
                 cudaStream_t s) {
    if (S > 0)
        k_sync_shared<<<blocks((int64_t)S * rows), 256, 0, s>>>(S, rows, skeys, src, recv, mine, sg, base, offs, KL,
                                                                   G, lds);
}

}  // namespace dgs_b200
