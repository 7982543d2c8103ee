// K3/K5/K6/K7 — per-pixel subset order, Eq.-5 merge, fused L1 + D-SSIM loss
// with its analytic gradient, and the merge adjoint.
//
// All four follow the reference op order exactly (engine.hpp:108-234,
// loss.hpp:19-177), so the merged image, the loss-gradient image and the
// partial-map gradients are bit-identical to the CPU oracle; only the loss
// scalars (reduced in double here, sequential float there) differ by
// rounding.  The merge and adjoint are HBM-streaming (16 B per subset per
// pixel in, 16 B out); the SSIM kernel keeps its 10 separable 11-tap blurs in
// shared memory (32x32 output tile, 10-pixel halo) and reads each input once.
#include "kernels.h"

namespace dgs_b200 {

namespace {

__global__ void k_merge(ViewParams vp, const Table* __restrict__ tb, int owner, int row0, int row1,
                        const float4* const* __restrict__ partials, int prow0, float bg0, float bg1, float bg2,
                        float* __restrict__ out_rgb, float* __restrict__ out_t, int out_base, int out_rows) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = row0 + blockIdx.y;
    if (x >= vp.width || y >= row1) return;
    float d[3];
    pixel_ray_dir(vp, x, y, d);
    uint16_t ord[kMaxSubsets];
    const int n = subspace_order(*tb, owner, vp.o, d, ord);
    float c0 = 0.0f, c1 = 0.0f, c2 = 0.0f, tr = 1.0f;
    const size_t prow = (size_t)(y - prow0) * vp.width + x;
    for (int i = 0; i < n; ++i) {
        const float4 p = partials[ord[i]][prow];
        c0 = fadd(c0, fmul(tr, p.x));  // engine.hpp:174
        c1 = fadd(c1, fmul(tr, p.y));
        c2 = fadd(c2, fmul(tr, p.z));
        tr = fmul(tr, p.w);
    }
    const size_t pix = (size_t)(y - out_base) * vp.width + x;
    const size_t plane = (size_t)vp.width * out_rows;
    out_rgb[pix] = fadd(c0, fmul(tr, bg0));  // engine.hpp:177
    out_rgb[plane + pix] = fadd(c1, fmul(tr, bg1));
    out_rgb[2 * plane + pix] = fadd(c2, fmul(tr, bg2));
    if (out_t) out_t[pix] = tr;
}

__global__ void k_pixel_orders(ViewParams vp, const Table* __restrict__ tb, int owner, uint16_t* __restrict__ order,
                               uint16_t* __restrict__ count, int kstride) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    if (x >= vp.width) return;
    float d[3];
    pixel_ray_dir(vp, x, y, d);
    uint16_t ord[kMaxSubsets];
    const int n = subspace_order(*tb, owner, vp.o, d, ord);
    const size_t pix = (size_t)y * vp.width + x;
    count[pix] = (uint16_t)n;
    for (int i = 0; i < kstride; ++i) order[pix * kstride + i] = i < n ? ord[i] : 0;
}

__global__ void k_merge_bwd(ViewParams vp, const Table* __restrict__ tb, int owner, int row0, int row1,
                            const float4* const* __restrict__ partials, int prow0, const float* __restrict__ grad_rgb,
                            int g_base, int g_rows, float bg0, float bg1, float bg2,
                            float4* const* __restrict__ grad_out, int grow0) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = row0 + blockIdx.y;
    if (x >= vp.width || y >= row1) return;
    float d[3];
    pixel_ray_dir(vp, x, y, d);
    uint16_t ord[kMaxSubsets];
    const int n = subspace_order(*tb, owner, vp.o, d, ord);
    const size_t pix = (size_t)(y - g_base) * vp.width + x;
    const size_t plane = (size_t)vp.width * g_rows;
    const float gc0 = grad_rgb[pix], gc1 = grad_rgb[plane + pix], gc2 = grad_rgb[2 * plane + pix];
    const float gt_eff = fadd(0.0f, dot3(gc0, gc1, gc2, bg0, bg1, bg2));  // engine.hpp:216 (grad_T_total = 0)
    const size_t prow = (size_t)(y - prow0) * vp.width + x;
    const size_t grow = (size_t)(y - grow0) * vp.width + x;
    float prefix[kMaxSubsets + 1];
    float4 pk[kMaxSubsets];
    prefix[0] = 1.0f;
    for (int i = 0; i < n; ++i) {
        pk[i] = partials[ord[i]][prow];
        prefix[i + 1] = fmul(prefix[i], pk[i].w);
    }
    // absent subsets get exact zeros
    uint32_t present = 0;
    for (int i = 0; i < n; ++i) present |= 1u << ord[i];
    for (int k = 0; k < tb->k_count; ++k)
        if (!(present & (1u << k))) grad_out[k][grow] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    float s0 = 0.0f, s1 = 0.0f, s2 = 0.0f, tail = 1.0f;
    for (int i = n - 1; i >= 0; --i) {
        const float pf = prefix[i];
        const float dT = fmul(pf, fadd(dot3(gc0, gc1, gc2, s0, s1, s2), fmul(gt_eff, tail)));
        grad_out[ord[i]][grow] = make_float4(fmul(pf, gc0), fmul(pf, gc1), fmul(pf, gc2), dT);
        const float4 p = pk[i];
        s0 = fadd(p.x, fmul(p.w, s0));
        s1 = fadd(p.y, fmul(p.w, s1));
        s2 = fadd(p.z, fmul(p.w, s2));
        tail = fmul(tail, p.w);
    }
}

/// merge with caller-supplied PixelOrders (engine.hpp:152-182 verbatim
/// contract): order [px][kstride], count [px]; partials [K][px] float4;
/// output HWC rgb + T.
__global__ void k_merge_ordered(int px, int kstride, const uint16_t* __restrict__ order,
                                const uint16_t* __restrict__ count, const float4* __restrict__ partials, float bg0,
                                float bg1, float bg2, float* __restrict__ out_rgb, float* __restrict__ out_t) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= px) return;
    const int n = count[p];
    float c0 = 0.0f, c1 = 0.0f, c2 = 0.0f, tr = 1.0f;
    for (int i = 0; i < n; ++i) {
        const float4 q = partials[(size_t)order[(size_t)p * kstride + i] * px + p];
        c0 = fadd(c0, fmul(tr, q.x));
        c1 = fadd(c1, fmul(tr, q.y));
        c2 = fadd(c2, fmul(tr, q.z));
        tr = fmul(tr, q.w);
    }
    out_rgb[3 * (size_t)p] = fadd(c0, fmul(tr, bg0));
    out_rgb[3 * (size_t)p + 1] = fadd(c1, fmul(tr, bg1));
    out_rgb[3 * (size_t)p + 2] = fadd(c2, fmul(tr, bg2));
    out_t[p] = tr;
}

/// merge_backward with caller-supplied orders and grad_trans_total
/// (engine.hpp:195-234); grad_color HWC, grad_tt [px] or null (= 0).
__global__ void k_merge_bwd_ordered(int px, int kcount, int kstride, const uint16_t* __restrict__ order,
                                    const uint16_t* __restrict__ count, const float4* __restrict__ partials,
                                    const float* __restrict__ grad_color, const float* __restrict__ grad_tt,
                                    float bg0, float bg1, float bg2, float4* __restrict__ out) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= px) return;
    const int n = count[p];
    const float gc0 = grad_color[3 * (size_t)p], gc1 = grad_color[3 * (size_t)p + 1],
                gc2 = grad_color[3 * (size_t)p + 2];
    const float gt_eff = fadd(grad_tt ? grad_tt[p] : 0.0f, dot3(gc0, gc1, gc2, bg0, bg1, bg2));
    uint16_t ord[kMaxSubsets];
    float prefix[kMaxSubsets + 1];
    float4 pk[kMaxSubsets];
    prefix[0] = 1.0f;
    uint32_t present = 0;
    for (int i = 0; i < n; ++i) {
        ord[i] = order[(size_t)p * kstride + i];
        present |= 1u << ord[i];
        pk[i] = partials[(size_t)ord[i] * px + p];
        prefix[i + 1] = fmul(prefix[i], pk[i].w);
    }
    for (int k = 0; k < kcount; ++k)
        if (!(present & (1u << k))) out[(size_t)k * px + p] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    float s0 = 0.0f, s1 = 0.0f, s2 = 0.0f, tail = 1.0f;
    for (int i = n - 1; i >= 0; --i) {
        const float pf = prefix[i];
        const float dT = fmul(pf, fadd(dot3(gc0, gc1, gc2, s0, s1, s2), fmul(gt_eff, tail)));
        out[(size_t)ord[i] * px + p] = make_float4(fmul(pf, gc0), fmul(pf, gc1), fmul(pf, gc2), dT);
        const float4 q = pk[i];
        s0 = fadd(q.x, fmul(q.w, s0));
        s1 = fadd(q.y, fmul(q.w, s1));
        s2 = fadd(q.z, fmul(q.w, s2));
        tail = fmul(tail, q.w);
    }
}

// ---------------------------------------------------------------------------
// Fused L1 + D-SSIM (loss.hpp:94-177), one channel plane per blockIdx.z.
// ---------------------------------------------------------------------------
#ifndef DGS_LOSS_THREADS
#define DGS_LOSS_THREADS 384
#endif
constexpr int kLT = DGS_LOSS_THREADS;  // threads per loss CTA
constexpr int kOT = 32;             // output tile
constexpr int kR = 5;               // blur radius
constexpr int kIn = kOT + 4 * kR;   // 52: input tile with 10-pixel halo
constexpr int kMid = kOT + 2 * kR;  // 42: first-stage maps with 5-pixel halo
constexpr size_t kLossSmem = (2 * kIn * kIn + 5 * kIn * kMid + 5 * kMid * kMid) * sizeof(float);

// Register-blocked stages: every thread produces a run of consecutive outputs
// along the blur direction, loading the run's 11 + R - 1 inputs from shared
// memory once.  Each output is still accumulated tap by tap (k = 0..10) with
// unfused _rn multiply-adds, i.e. the reference's gauss_blur op sequence, so
// the gradient is bit-identical.  Tiles whose 10-pixel halo lies inside the
// image (BORDER = false, ~90% at 1080p) skip every per-tap padding test.
constexpr int kR1 = 6;   // stage 1 run (42 = 7 x 6)
constexpr int kR2 = 7;   // stage 2 run (42 = 6 x 7)
constexpr int kR3 = 8;   // stage 3 run (32 = 4 x 8)
constexpr int kR4 = 4;   // stage 4 run (32 = 8 x 4)

template <bool BORDER>
__device__ __forceinline__ void loss_tile(int W, int H, int row0, int row1, int in_base, int in_rows,
                                          const float* __restrict__ xp, const float* __restrict__ yp, float lam,
                                          float c1, float c2, float nf, float inv_batch, const float* kern,
                                          float* __restrict__ gp, float* X, float* Y, float* Hb, float* Vb, int ox,
                                          int oy, double& s_l1, double& s_ssim, double& s_mse) {
    const int tid = threadIdx.x;
    // stage 0: inputs with zero padding outside the image / provided window;
    // all of a thread's loads are issued before any is stored (memory-level parallelism)
    {
        constexpr int NIT = (kIn * kIn + kLT - 1) / kLT;
        float xr[NIT], yr[NIT];
#pragma unroll
        for (int u = 0; u < NIT; ++u) {
            const int i = tid + u * kLT;
            xr[u] = yr[u] = 0.0f;
            if (i < kIn * kIn) {
                const int r = i / kIn, c = i % kIn;
                const int gy = oy - 2 * kR + r, gx = ox - 2 * kR + c;
                const bool in =
                    !BORDER || (gy >= 0 && gy < H && gx >= 0 && gx < W && gy >= in_base && gy < in_base + in_rows);
                if (in) {
                    xr[u] = __ldg(xp + (size_t)(gy - in_base) * W + gx);
                    yr[u] = __ldg(yp + (size_t)(gy - in_base) * W + gx);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < NIT; ++u) {
            const int i = tid + u * kLT;
            if (i < kIn * kIn) {
                X[i] = xr[u];
                Y[i] = yr[u];
            }
        }
    }
    __syncthreads();
    // stage 1: horizontal blur of x, y, x*x, y*y, x*y (rows -10..+41, cols -5..+36)
    for (int it = tid; it < kIn * (kMid / kR1); it += kLT) {
        const int r = it / (kMid / kR1), c0 = (it % (kMid / kR1)) * kR1;
        float xv[kR1 + 10], yv[kR1 + 10];
#pragma unroll
        for (int i = 0; i < kR1 + 10; ++i) {
            xv[i] = X[r * kIn + c0 + i];
            yv[i] = Y[r * kIn + c0 + i];
        }
        const int gxb = ox - 2 * kR + c0;  // image column of input i = gxb + i
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            float in[kR1 + 10];
#pragma unroll
            for (int i = 0; i < kR1 + 10; ++i)
                in[i] = q == 0 ? xv[i] : q == 1 ? yv[i] : q == 2 ? fmul(xv[i], xv[i]) : q == 3 ? fmul(yv[i], yv[i])
                                                                                           : fmul(xv[i], yv[i]);
#pragma unroll
            for (int j = 0; j < kR1; ++j) {
                float a = 0.0f;
#pragma unroll
                for (int k = 0; k < 11; ++k) {
                    if (BORDER && (gxb + j + k < 0 || gxb + j + k >= W)) continue;  // loss.hpp:44 padding
                    a = fadd(a, fmul(kern[k], in[j + k]));
                }
                Hb[q * kIn * kMid + r * kMid + c0 + j] = a;
            }
        }
    }
    __syncthreads();
    // stage 2: vertical blur -> mu_x, mu_y, E[xx], E[yy], E[xy] at tile +-5;
    // then the per-pixel SSIM partials A, B, B mu_x, C, C mu_y (zero outside the image).
    for (int it = tid; it < kMid * (kMid / kR2); it += kLT) {
        const int c = it % kMid, r0 = (it / kMid) * kR2;
        const int gx = ox - kR + c;
        const int gyb = oy - 2 * kR + r0;  // image row of input i = gyb + i
        float m[5][kR2];
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            float col[kR2 + 10];
#pragma unroll
            for (int i = 0; i < kR2 + 10; ++i) col[i] = Hb[q * kIn * kMid + (r0 + i) * kMid + c];
#pragma unroll
            for (int j = 0; j < kR2; ++j) {
                float a = 0.0f;
#pragma unroll
                for (int k = 0; k < 11; ++k) {
                    if (BORDER && (gyb + j + k < 0 || gyb + j + k >= H)) continue;
                    a = fadd(a, fmul(kern[k], col[j + k]));
                }
                m[q][j] = a;
            }
        }
#pragma unroll
        for (int j = 0; j < kR2; ++j) {
            const int r = r0 + j, gy = oy - kR + r;
            const bool in = !BORDER || (gy >= 0 && gy < H && gx >= 0 && gx < W);
            float A = 0.0f, B = 0.0f, Cc = 0.0f, Bm = 0.0f, Cm = 0.0f;
            if (in) {
                const float mx = m[0][j], my = m[1][j];
                const float sxx = fsub(m[2][j], fmul(mx, mx));
                const float syy = fsub(m[3][j], fmul(my, my));
                const float sxy = fsub(m[4][j], fmul(mx, my));
                const float n1 = fadd(fmul(fmul(2.0f, mx), my), c1), n2 = fadd(fmul(2.0f, sxy), c2);
                const float d1 = fadd(fadd(fmul(mx, mx), fmul(my, my)), c1), d2 = fadd(fadd(sxx, syy), c2);
                const float dd = fmul(d1, d2);
                const float sv = fdiv(fmul(n1, n2), dd);
                A = fsub(fdiv(fmul(fmul(2.0f, my), n2), dd), fdiv(fmul(fmul(2.0f, mx), sv), d1));
                B = fdiv(-sv, d2);
                Cc = fdiv(fmul(2.0f, n1), dd);
                Bm = fmul(B, mx);
                Cm = fmul(Cc, my);
                const bool own = r >= kR && r < kR + kOT && c >= kR && c < kR + kOT && gy < row1;
                if (own) s_ssim += (double)sv;
            }
            const int i = r * kMid + c;
            Vb[0 * kMid * kMid + i] = A;
            Vb[1 * kMid * kMid + i] = B;
            Vb[2 * kMid * kMid + i] = Bm;
            Vb[3 * kMid * kMid + i] = Cc;
            Vb[4 * kMid * kMid + i] = Cm;
        }
    }
    __syncthreads();
    // stage 3: horizontal blur of the five maps (rows -5..+36, cols 0..31)
    float* H2 = Hb;  // [5][kMid][kOT]
    for (int it = tid; it < 5 * (kOT / kR3) * kMid; it += kLT) {
        const int r = it % kMid, qc = it / kMid;
        const int q = qc / (kOT / kR3), c0 = (qc % (kOT / kR3)) * kR3;
        const int gxb = ox - kR + c0;
        float row[kR3 + 10];
#pragma unroll
        for (int i = 0; i < kR3 + 10; ++i) row[i] = Vb[q * kMid * kMid + r * kMid + c0 + i];
#pragma unroll
        for (int j = 0; j < kR3; ++j) {
            float a = 0.0f;
#pragma unroll
            for (int k = 0; k < 11; ++k) {
                if (BORDER && (gxb + j + k < 0 || gxb + j + k >= W)) continue;
                a = fadd(a, fmul(kern[k], row[j + k]));
            }
            H2[q * kMid * kOT + r * kOT + c0 + j] = a;
        }
    }
    __syncthreads();
    // stage 4: vertical blur -> gradient (loss.hpp:138-140, 160-175)
    for (int it = tid; it < kOT * (kOT / kR4); it += kLT) {
        const int c = it % kOT, r0 = (it / kOT) * kR4;
        const int gx = ox + c;
        const int gyb = oy + r0 - kR;
        float cv[5][kR4];
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            float col[kR4 + 10];
#pragma unroll
            for (int i = 0; i < kR4 + 10; ++i) col[i] = H2[q * kMid * kOT + (r0 + i) * kOT + c];
#pragma unroll
            for (int j = 0; j < kR4; ++j) {
                float a = 0.0f;
#pragma unroll
                for (int k = 0; k < 11; ++k) {
                    if (BORDER && (gyb + j + k < 0 || gyb + j + k >= H)) continue;
                    a = fadd(a, fmul(kern[k], col[j + k]));
                }
                cv[q][j] = a;
            }
        }
#pragma unroll
        for (int j = 0; j < kR4; ++j) {
            const int r = r0 + j, gy = oy + r;
            if (gy >= row1 || gy >= H || gx >= W) continue;
            const float xv = X[(r + 2 * kR) * kIn + c + 2 * kR], yv = Y[(r + 2 * kR) * kIn + c + 2 * kR];
            // dS/dx = (conv(A) + 2x conv(B) - 2 conv(B mu_x) + y conv(C) - conv(C mu_y)) / n
            const float sg = fdiv(fsub(fadd(fsub(fadd(cv[0][j], fmul(fmul(2.0f, xv), cv[1][j])), fmul(2.0f, cv[2][j])),
                                            fmul(yv, cv[3][j])),
                                       cv[4][j]),
                                  nf);
            const float d = fsub(xv, yv);
            const float sgn = d > 0.0f ? 1.0f : (d < 0.0f ? -1.0f : 0.0f);
            const float gl1 = fdiv(fmul(fsub(1.0f, lam), sgn), nf);
            const float g = fsub(gl1, fmul(lam, sg));
            gp[(size_t)(gy - in_base) * W + gx] = fmul(g, inv_batch);
            s_l1 += (double)fabsf(d);
            s_mse += (double)fmul(d, d);
        }
    }
}

__global__ void __launch_bounds__(kLT, 2) k_loss(int W, int H, int row0, int row1, int in_base, int in_rows,
                                              const float* __restrict__ xs, const float* __restrict__ ys, float lam,
                                              float c1, float c2, float nf, float inv_batch,
                                              const float* __restrict__ kern_g, float* __restrict__ grad,
                                              double* __restrict__ block_sums) {
    // x, y, grad: planar [3][in_rows][W] covering image rows [in_base, in_base + in_rows);
    // outputs for rows [row0, row1) need inputs within +-10 rows, which the caller provides.
    extern __shared__ float sm[];
    float* X = sm;                       // [kIn][kIn]
    float* Y = X + kIn * kIn;            // [kIn][kIn]
    float* Hb = Y + kIn * kIn;           // [5][kIn][kMid] horizontal stage (reused as [5][kMid][kOT])
    float* Vb = Hb + 5 * kIn * kMid;     // [5][kMid][kMid]
    __shared__ float kern[11];
    __shared__ double red[3][kLT / 32];
    const int tid = threadIdx.x;
    if (tid < 11) kern[tid] = kern_g[tid];
    const int ox = blockIdx.x * kOT, oy = row0 + blockIdx.y * kOT;
    const int ch = blockIdx.z;
    const size_t plane = (size_t)W * in_rows;
    // interior: the 10-pixel halo is inside the image and inside the provided window
    const bool interior = ox - 2 * kR >= 0 && ox + kOT + 2 * kR <= W && oy - 2 * kR >= 0 &&
                          oy + kOT + 2 * kR <= H && oy - 2 * kR >= in_base && oy + kOT + 2 * kR <= in_base + in_rows;
    double s_l1 = 0.0, s_ssim = 0.0, s_mse = 0.0;
    __syncthreads();  // kern
    if (interior)
        loss_tile<false>(W, H, row0, row1, in_base, in_rows, xs + ch * plane, ys + ch * plane, lam, c1, c2, nf,
                         inv_batch, kern, grad + ch * plane, X, Y, Hb, Vb, ox, oy, s_l1, s_ssim, s_mse);
    else
        loss_tile<true>(W, H, row0, row1, in_base, in_rows, xs + ch * plane, ys + ch * plane, lam, c1, c2, nf,
                        inv_batch, kern, grad + ch * plane, X, Y, Hb, Vb, ox, oy, s_l1, s_ssim, s_mse);
    // block sums (deterministic)
    double v[3] = {s_l1, s_ssim, s_mse};
    for (int q = 0; q < 3; ++q) {
        double x = v[q];
        for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
        if ((tid & 31) == 0) red[q][tid >> 5] = x;
    }
    __syncthreads();
    if (tid < 3) {
        double x = 0.0;
        for (int w = 0; w < kLT / 32; ++w) x += red[tid][w];
        const int b = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        block_sums[(size_t)b * 3 + tid] = x;
    }
}

__global__ void k_reduce_sums(const double* __restrict__ bs, int n, double* __restrict__ out) {
    __shared__ double red[3][32];
    double v[3] = {0.0, 0.0, 0.0};
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        for (int q = 0; q < 3; ++q) v[q] += bs[(size_t)i * 3 + q];
    for (int q = 0; q < 3; ++q) {
        double x = v[q];
        for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
        if ((threadIdx.x & 31) == 0) red[q][threadIdx.x >> 5] = x;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        double x = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) x += red[threadIdx.x][w];
        out[threadIdx.x] = x;
    }
}

}  // namespace

void launch_merge(const ViewParams& vp, const Table* tb_dev, int owner, int row0, int row1,
                  const float4* const* partials, int prow0, const float bg[3], float* out_rgb, float* out_t,
                  int out_base, int out_rows, cudaStream_t s) {
    if (row1 <= row0) return;
    dim3 grid((vp.width + 127) / 128, row1 - row0);
    k_merge<<<grid, 128, 0, s>>>(vp, tb_dev, owner, row0, row1, partials, prow0, bg[0], bg[1], bg[2], out_rgb, out_t,
                                 out_base, out_rows);
}

void launch_pixel_orders(const ViewParams& vp, const Table* tb_dev, int owner, uint16_t* order, uint16_t* count,
                         int kstride, cudaStream_t s) {
    dim3 grid((vp.width + 127) / 128, vp.height);
    k_pixel_orders<<<grid, 128, 0, s>>>(vp, tb_dev, owner, order, count, kstride);
}

void launch_merge_bwd(const ViewParams& vp, const Table* tb_dev, int owner, int row0, int row1,
                      const float4* const* partials, int prow0, const float* grad_rgb, int g_base, int g_rows,
                      const float bg[3], float4* const* grad_out, int grow0, cudaStream_t s) {
    if (row1 <= row0) return;
    dim3 grid((vp.width + 127) / 128, row1 - row0);
    k_merge_bwd<<<grid, 128, 0, s>>>(vp, tb_dev, owner, row0, row1, partials, prow0, grad_rgb, g_base, g_rows, bg[0],
                                     bg[1], bg[2], grad_out, grow0);
}

void launch_merge_ordered(int px, int kstride, const uint16_t* order, const uint16_t* count, const float4* partials,
                          const float bg[3], float* out_rgb, float* out_t, cudaStream_t s) {
    if (px <= 0) return;
    k_merge_ordered<<<(unsigned)((px + 255) / 256), 256, 0, s>>>(px, kstride, order, count, partials, bg[0], bg[1],
                                                                  bg[2], out_rgb, out_t);
}

void launch_merge_bwd_ordered(int px, int kcount, int kstride, const uint16_t* order, const uint16_t* count,
                              const float4* partials, const float* grad_color, const float* grad_tt,
                              const float bg[3], float4* out, cudaStream_t s) {
    if (px <= 0) return;
    k_merge_bwd_ordered<<<(unsigned)((px + 255) / 256), 256, 0, s>>>(px, kcount, kstride, order, count, partials,
                                                                      grad_color, grad_tt, bg[0], bg[1], bg[2], out);
}

void launch_loss(int W, int H, int row0, int row1, int in_base, int in_rows, const float* x, const float* y,
                 float lambda, const float* kernel, float inv_batch, float* grad, double* block_sums, int* n_blocks,
                 cudaStream_t s) {
    ensure_smem_attr((const void*)k_loss, (int)kLossSmem);
    dim3 grid((W + kOT - 1) / kOT, (row1 - row0 + kOT - 1) / kOT, 3);
    *n_blocks = (int)(grid.x * grid.y * grid.z);
    // loss.hpp:16-17: C1 = (0.01)^2, C2 = (0.03)^2 evaluated in double, then T(.)
    const float c1 = (float)(0.01 * 0.01), c2 = (float)(0.03 * 0.03);
    const float nf = (float)((size_t)W * H * 3);
    k_loss<<<grid, kLT, kLossSmem, s>>>(W, H, row0, row1, in_base, in_rows, x, y, lambda, c1, c2, nf, inv_batch,
                                        kernel, grad, block_sums);
}

void launch_reduce_sums(const double* block_sums, int n_blocks, double* out3, cudaStream_t s) {
    k_reduce_sums<<<1, 256, 0, s>>>(block_sums, n_blocks, out3);
}

}  // namespace dgs_b200
