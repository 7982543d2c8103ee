// Micro-benchmark: CUB onesweep radix sort policies for the two binning sorts
// at C3 size (10M u32 24-bit member keys + u32 values; 42.8M u16 13-bit tile
// keys + u32 values).  Build + run:  nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -std=c++17 scripts/sortbench.cu -o /tmp/sortbench && /tmp/sortbench
#include <cub/cub.cuh>
#include <cstdio>
#include <vector>

template <typename K, typename V, int THREADS, int ITEMS, int RB = 8>
struct Hub {
    using Base = typename cub::detail::radix::policy_hub<K, V, int>::Policy1000;
    struct Policy : cub::ChainedPolicy<1000, Policy, Policy> {
        static constexpr bool ONESWEEP = true;
        static constexpr int ONESWEEP_RADIX_BITS = RB;
        using HistogramPolicy = typename Base::HistogramPolicy;
        using ExclusiveSumPolicy = typename Base::ExclusiveSumPolicy;
        using DominantT = typename cub::detail::radix::policy_hub<K, V, int>::DominantT;
        using OnesweepPolicy =
            cub::AgentRadixSortOnesweepPolicy<THREADS, ITEMS, DominantT, 1, cub::RADIX_RANK_MATCH_EARLY_COUNTS_ANY,
                                              cub::BLOCK_SCAN_RAKING_MEMOIZE, cub::RADIX_SORT_STORE_DIRECT, RB>;
        using ScanPolicy = typename Base::ScanPolicy;
        using DownsweepPolicy = typename Base::DownsweepPolicy;
        using AltDownsweepPolicy = typename Base::AltDownsweepPolicy;
        using UpsweepPolicy = typename Base::UpsweepPolicy;
        using AltUpsweepPolicy = typename Base::AltUpsweepPolicy;
        using SingleTilePolicy = typename Base::SingleTilePolicy;
        using SegmentedPolicy = typename Base::SegmentedPolicy;
        using AltSegmentedPolicy = typename Base::AltSegmentedPolicy;
    };
    using MaxPolicy = Policy;
};

template <typename K, typename V, int THREADS, int ITEMS, int RB = 8>
float run(K* k0, K* k1, V* v0, V* v1, int n, int bits, void* tmp, size_t tmpb, int reps) {
    using D = cub::DispatchRadixSort<false, K, V, int, Hub<K, V, THREADS, ITEMS, RB>>;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9f;
    for (int r = 0; r < reps; ++r) {
        cub::DoubleBuffer<K> dk(k0, k1);
        cub::DoubleBuffer<V> dv(v0, v1);
        size_t tb = tmpb;
        cudaEventRecord(a);
        cudaError_t e = D::Dispatch(tmp, tb, dk, dv, n, 0, bits, true, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        if (e != cudaSuccess) {
            printf("err %s\n", cudaGetErrorString(e));
            return -1;
        }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    return best;
}

template <typename K>
float run_default(K* k0, K* k1, uint32_t* v0, uint32_t* v1, int n, int bits, void* tmp, size_t tmpb, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9f;
    for (int r = 0; r < reps; ++r) {
        cub::DoubleBuffer<K> dk(k0, k1);
        cub::DoubleBuffer<uint32_t> dv(v0, v1);
        size_t tb = tmpb;
        cudaEventRecord(a);
        cub::DeviceRadixSort::SortPairs(tmp, tb, dk, dv, n, 0, bits);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    return best;
}

#define RUN32(T, I) printf("u32 %3d x %2d : %.3f ms\n", T, I, run<uint32_t, uint32_t, T, I>(k32a, k32b, va, vb, n1, 24, tmp, tmpb, 5))
#define RUN16(T, I) printf("u16 %3d x %2d : %.3f ms\n", T, I, run<uint16_t, uint32_t, T, I>(k16a, k16b, va, vb, n2, 13, tmp, tmpb, 5))
#define RUN16B(T, I, B) printf("u16 %3d x %2d rb %d : %.3f ms\n", T, I, B, run<uint16_t, uint32_t, T, I, B>(k16a, k16b, va, vb, n2, 13, tmp, tmpb, 5))

int main() {
    const int n1 = 10000000, n2 = 42800000;
    std::vector<uint32_t> h32(n1), hv(n2);
    std::vector<uint16_t> h16(n2);
    uint64_t s = 12345;
    auto rnd = [&]() { s = s * 6364136223846793005ull + 1442695040888963407ull; return (uint32_t)(s >> 33); };
    for (int i = 0; i < n1; ++i) h32[i] = rnd() & 0xffffffu;
    for (int i = 0; i < n2; ++i) { h16[i] = (uint16_t)(rnd() % 8160); hv[i] = i; }
    uint32_t *k32a, *k32b, *va, *vb;
    uint16_t *k16a, *k16b;
    cudaMalloc(&k32a, 4ull * n1); cudaMalloc(&k32b, 4ull * n1);
    cudaMalloc(&k16a, 2ull * n2); cudaMalloc(&k16b, 2ull * n2);
    cudaMalloc(&va, 4ull * n2); cudaMalloc(&vb, 4ull * n2);
    cudaMemcpy(k32a, h32.data(), 4ull * n1, cudaMemcpyHostToDevice);
    cudaMemcpy(k16a, h16.data(), 2ull * n2, cudaMemcpyHostToDevice);
    cudaMemcpy(va, hv.data(), 4ull * n2, cudaMemcpyHostToDevice);
    size_t tmpb = 512ull << 20;
    void* tmp;
    cudaMalloc(&tmp, tmpb);
    printf("default u32: %.3f ms\n", run_default<uint32_t>(k32a, k32b, va, vb, n1, 24, tmp, tmpb, 5));
    printf("default u16: %.3f ms\n", run_default<uint16_t>(k16a, k16b, va, vb, n2, 13, tmp, tmpb, 5));
    RUN32(384, 23); RUN32(256, 23); RUN32(256, 16); RUN32(256, 12); RUN32(512, 12); RUN32(512, 16);
    RUN32(128, 16); RUN32(256, 8); RUN32(384, 12); RUN32(192, 16);
    RUN16(512, 20); RUN16(256, 20); RUN16(256, 16); RUN16(256, 12); RUN16(512, 12); RUN16(384, 16);
    RUN16(128, 16); RUN16(256, 8); RUN16(512, 8); RUN16(192, 20);
    RUN16B(256, 16, 7); RUN16B(512, 16, 7); RUN16B(384, 16, 7); RUN16B(256, 24, 7); RUN16B(256, 20, 7);
    RUN16B(512, 12, 7); RUN16B(256, 16, 6); RUN16B(512, 16, 6); RUN16B(384, 20, 7); RUN16B(256, 32, 7);
    printf("-- repeat\n");
    printf("default u16: %.3f ms\n", run_default<uint16_t>(k16a, k16b, va, vb, n2, 13, tmp, tmpb, 5));
    RUN16B(384, 20, 7); RUN16B(384, 24, 7); RUN16B(512, 20, 7); RUN16B(320, 24, 7); RUN16B(384, 18, 7);
    RUN16B(256, 28, 7); RUN16B(384, 20, 8); RUN16B(384, 24, 8); RUN16B(448, 20, 7); RUN16B(384, 28, 7);
    printf("default u16: %.3f ms\n", run_default<uint16_t>(k16a, k16b, va, vb, n2, 13, tmp, tmpb, 5));
    return 0;
}
