// Diagnostic: does a graph's memset / D2D / D2H node queue behind a large H2D
// upload running on another stream?  Prints the graph's event-timed duration
// alone and with a 25 MB pinned H2D in flight.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
__global__ void k_spin(float* p, int n) { for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = p[i] * 1.0001f + 1.f; }
int main() {
    const size_t big = 25u << 20;
    float *h, *d, *w, *hs;
    CK(cudaHostAlloc(&h, big, 0)); CK(cudaHostAlloc(&hs, 4096, 0));
    CK(cudaMalloc(&d, big)); CK(cudaMalloc(&w, 64u << 20));
    cudaStream_t s, c; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); CK(cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const char* names[] = {"kernels only", "memset node", "D2D node", "D2H node", "H2D small node"};
    for (int variant = 0; variant < 5; ++variant) {
        cudaGraph_t g; cudaGraphExec_t x;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
        for (int r = 0; r < 10; ++r) {
            if (variant == 1) CK(cudaMemsetAsync(w + r, 0, 4, s));
            if (variant == 2) CK(cudaMemcpyAsync(w + r, w + 1000 + r, 4, cudaMemcpyDeviceToDevice, s));
            if (variant == 3) CK(cudaMemcpyAsync(hs + r, w + r, 4, cudaMemcpyDeviceToHost, s));
            if (variant == 4) CK(cudaMemcpyAsync(w + r, hs + r, 4, cudaMemcpyHostToDevice, s));
            k_spin<<<148 * 4, 256, 0, s>>>(w, 16 << 20);
        }
        CK(cudaStreamEndCapture(s, &g)); CK(cudaGraphInstantiate(&x, g, 0));
        for (int with_dma = 0; with_dma < 2; ++with_dma) {
            float best = 1e9;
            for (int it = 0; it < 20; ++it) {
                CK(cudaDeviceSynchronize());
                if (with_dma) CK(cudaMemcpyAsync(d, h, big, cudaMemcpyHostToDevice, c));
                cudaEventRecord(e0, s); CK(cudaGraphLaunch(x, s)); cudaEventRecord(e1, s);
                CK(cudaDeviceSynchronize());
                float ms; cudaEventElapsedTime(&ms, e0, e1); if (it > 2 && ms < best) best = ms;
            }
            printf("%-16s dma=%d  %.3f ms\n", names[variant], with_dma, best);
        }
    }
    return 0;
}
