// Training step (Stage-II / joint chain of conditioned_training_loop,
// trainer.cpp:410-466) for a batch of receivers sharing one transmitter:
//
//   forward   conditioning + FLE reduction (k_cond.cu), compositing with an
//             f32 field epilogue (k_composite.cu);
//   loss      spectrum L1 (composite_loss, trainer.cpp:80-145, lambda_ssim =
//             lambda_fft = 0) fused with aggregate_modality_backward
//             (sphraster.cpp:435-445)                       -> k_loss_spectrum
//   render    d signal of every walked list entry = tw^T * dField per tile
//   adjoint   (the d_signals part of backward_render, sphraster.cpp:541-579),
//             then a fixed-order per-Gaussian reduction        -> k_composite_T,
//                                                                 k_reduce_ds
//   cond      condition_backward (conditioning.cpp:472-587) fused with the
//   adjoint   signal adjoint (backward_render :619-646): local MLP backward per
//             (Gaussian, receiver) row with deterministic per-CTA weight
//             gradients; d_base; the global branch reduced over Gaussians
//             and back-propagated in FP64                       -> k_cond_bwd,
//                                                                 k_dbase,
//                                                                 k_global_red,
//                                                                 k_global_bwd
//   update    Adam with bias correction (diffengine.cpp:10-34), per-element
//             learning-rate scale for FLE degree >= 1 (trainer.cpp:213-229)
//                                                               -> k_adam
// Every reduction runs in a fixed order (no floating-point atomics), so a
// step is bitwise reproducible, as the reference requires.

#include <cuda.h>

#include "cond_common.cuh"
#include "f32x2.cuh"
#include "rxgs_internal.cuh"
#include "tc_util.cuh"

namespace rxgs_b200 {
namespace {

using namespace cond_dev;

constexpr int kBwdThreads = 128;  // rows per tile in k_cond_bwd

__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }

// ------------------------------------------------------------------ base -> B * base
__global__ void k_refresh_gb(int K, int L, int C, const int* __restrict__ culled, const double* __restrict__ basis64,
                             const double* __restrict__ base64, float2* __restrict__ gb32) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= static_cast<long long>(K) * L * C) return;
    const int k = static_cast<int>(i / (L * C));
    const int l = static_cast<int>((i / C) % L);
    if (culled[k]) {
        gb32[i] = make_float2(0.f, 0.f);
        return;
    }
    const double br = basis64[(static_cast<size_t>(k) * L + l) * 2], bi = basis64[(static_cast<size_t>(k) * L + l) * 2 + 1];
    const double a = base64[i * 2], b = base64[i * 2 + 1];
    gb32[i] = make_float2(static_cast<float>(a * br - b * bi), static_cast<float>(a * bi + b * br));
}

// ------------------------------------------------------------------ loss + aggregate adjoint
// Spectrum L1: loss_j = lw/P sum|amp - gt|, d_amp = lw/P sign(amp - gt);
// d_re = d_amp re/amp, d_im = d_amp im/amp.  G layout: [j][cell] complex.
__global__ void k_loss_spectrum(int n_rx, int P, const float* __restrict__ field, const float* __restrict__ target,
                                double l_weight, float2* __restrict__ G, double* __restrict__ loss_part) {
    __shared__ double red[256];
    const int j = blockIdx.y;
    double acc = 0.0;
    const float* re_p = field + static_cast<size_t>(j) * 2 * P;
    const float* im_p = re_p + P;
    const float w = static_cast<float>(l_weight / P);
    for (int cell = blockIdx.x * blockDim.x + threadIdx.x; cell < P; cell += gridDim.x * blockDim.x) {
        const float re = re_p[cell], im = im_p[cell];
        const float amp = sqrtf(re * re + im * im + static_cast<float>(kAmpEps));
        const float d = amp - target[static_cast<size_t>(j) * P + cell];
        acc += fabs(static_cast<double>(d));
        const float s = d > 0.f ? w : (d < 0.f ? -w : 0.f);
        G[static_cast<size_t>(j) * P + cell] = make_float2(s * re / amp, s * im / amp);
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int st = blockDim.x / 2; st > 0; st >>= 1) {
        if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
        __syncthreads();
    }
    if (threadIdx.x == 0) loss_part[static_cast<size_t>(j) * gridDim.x + blockIdx.x] = red[0] * l_weight / P;
}

__global__ void k_loss_finalize(int n_rx, int nb, const double* __restrict__ part, double* __restrict__ loss) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n_rx) return;
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += part[static_cast<size_t>(j) * nb + b];
    loss[j] = s;
}

// ------------------------------------------------------------------ full spectrum loss
// composite_loss (trainer.cpp:80-145) with SSIM and DFT terms, FP64 from the
// f32 field:
//   L = l_w * mean|x - y| + lambda_ssim (1 - SSIM(x, y)) + lambda_fft sum|F x - F y|^2
// x = amplitude sqrt(re^2 + im^2 + 1e-8), y = target.  The orthonormal,
// zero-padded 2-D DFT is unitary, so sum|F x - F y|^2 = sum (x - y)^2
// (Parseval) and its adjoint is 2 (x - y) -- the collapse the reference uses
// for the gradient (trainer.cpp:131-138); the value is taken the same way.
// SSIM (metrics.cpp:55-112): 11x11 Gaussian window (sigma 1.5), mean over
// every fully contained window; the 2-D window is the outer product of the
// normalised 1-D window, so both the window statistics and the adjoint
//   d SSIM / d x_p = 1/n sum_{windows w containing p} k(p - w) (A_w + B_w y_p + G_w x_p),
//   A = 2 my (a2 - a1)/(b1 b2) - 2 s mx (1/b1 - 1/b2), B = 2 a1/(b1 b2), G = -2 s/b2
// (the reference's ds expanded per window) are separable passes.
constexpr int kSsimWin = 11;
__constant__ double c_ssim_g[kSsimWin];  // normalised 1-D Gaussian window

__global__ void k_loss_amp(int n_rx, int P, const float* __restrict__ field, const float* __restrict__ target,
                           double* __restrict__ amp, double* __restrict__ part) {
    __shared__ double red[2][256];
    const int j = blockIdx.y;
    const float* re_p = field + static_cast<size_t>(j) * 2 * P;
    const float* im_p = re_p + P;
    double l1 = 0.0, sq = 0.0;
    for (int cell = blockIdx.x * blockDim.x + threadIdx.x; cell < P; cell += gridDim.x * blockDim.x) {
        const double re = re_p[cell], im = im_p[cell];
        const double x = sqrt(re * re + im * im + kAmpEps);
        const double d = x - static_cast<double>(target[static_cast<size_t>(j) * P + cell]);
        amp[static_cast<size_t>(j) * P + cell] = x;
        l1 += fabs(d);
        sq += d * d;
    }
    red[0][threadIdx.x] = l1;
    red[1][threadIdx.x] = sq;
    __syncthreads();
    for (int st = blockDim.x / 2; st > 0; st >>= 1) {
        if (threadIdx.x < st) {
            red[0][threadIdx.x] += red[0][threadIdx.x + st];
            red[1][threadIdx.x] += red[1][threadIdx.x + st];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[(static_cast<size_t>(j) * gridDim.x + blockIdx.x) * 2] = red[0][0];
        part[(static_cast<size_t>(j) * gridDim.x + blockIdx.x) * 2 + 1] = red[1][0];
    }
}

// horizontal window sums of x, y, x^2, y^2, xy: H[j][q][r][c], c < cols
__global__ void k_ssim_h(int n_rx, int h, int w, const double* __restrict__ amp, const float* __restrict__ target,
                         double* __restrict__ H) {
    const int cols = w - kSsimWin + 1;
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int r = blockIdx.y, j = blockIdx.z;
    if (c >= cols) return;
    const double* x = amp + (static_cast<size_t>(j) * h + r) * w + c;
    const float* y = target + (static_cast<size_t>(j) * h + r) * w + c;
    double s[5] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int t = 0; t < kSsimWin; ++t) {
        const double g = c_ssim_g[t], xv = x[t], yv = y[t];
        s[0] += g * xv;
        s[1] += g * yv;
        s[2] += g * xv * xv;
        s[3] += g * yv * yv;
        s[4] += g * xv * yv;
    }
    const size_t plane = static_cast<size_t>(h) * cols;
#pragma unroll
    for (int q = 0; q < 5; ++q) H[(static_cast<size_t>(j) * 5 + q) * plane + static_cast<size_t>(r) * cols + c] = s[q];
}

// per window: statistics -> SSIM s and the adjoint coefficients A, B, G
__global__ void k_ssim_v(int n_rx, int h, int w, double c1, double c2, const double* __restrict__ H,
                         double* __restrict__ S, double* __restrict__ coef) {
    const int cols = w - kSsimWin + 1, rows = h - kSsimWin + 1;
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int r = blockIdx.y, j = blockIdx.z;
    if (c >= cols) return;
    const size_t hplane = static_cast<size_t>(h) * cols;
    double m[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) {
        const double* hq = H + (static_cast<size_t>(j) * 5 + q) * hplane + static_cast<size_t>(r) * cols + c;
        double a = 0.0;
#pragma unroll
        for (int t = 0; t < kSsimWin; ++t) a += c_ssim_g[t] * hq[static_cast<size_t>(t) * cols];
        m[q] = a;
    }
    const double mx = m[0], my = m[1];
    const double vx = m[2] - mx * mx, vy = m[3] - my * my, cov = m[4] - mx * my;
    const double a1 = 2.0 * mx * my + c1, b1 = mx * mx + my * my + c1;
    const double a2 = 2.0 * cov + c2, b2 = vx + vy + c2;
    const double sv = (a1 * a2) / (b1 * b2);
    const size_t wplane = static_cast<size_t>(rows) * cols, wi = static_cast<size_t>(r) * cols + c;
    S[static_cast<size_t>(j) * wplane + wi] = sv;
    coef[(static_cast<size_t>(j) * 3 + 0) * wplane + wi] =
        2.0 * my * (a2 - a1) / (b1 * b2) - 2.0 * sv * mx * (1.0 / b1 - 1.0 / b2);
    coef[(static_cast<size_t>(j) * 3 + 1) * wplane + wi] = 2.0 * a1 / (b1 * b2);
    coef[(static_cast<size_t>(j) * 3 + 2) * wplane + wi] = -2.0 * sv / b2;
}

// fixed-order per-receiver mean of the window SSIMs
__global__ void k_ssim_mean(int rows, int cols, const double* __restrict__ S, double* __restrict__ ssim) {
    __shared__ double red[256];
    const int j = blockIdx.x;
    const size_t n = static_cast<size_t>(rows) * cols;
    double a = 0.0;
    for (size_t i = threadIdx.x; i < n; i += blockDim.x) a += S[static_cast<size_t>(j) * n + i];
    red[threadIdx.x] = a;
    __syncthreads();
    for (int st = blockDim.x / 2; st > 0; st >>= 1) {
        if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
        __syncthreads();
    }
    if (threadIdx.x == 0) ssim[j] = red[0] / static_cast<double>(n);
}

// adjoint, vertical pass: V[j][q][pr][c] = sum_t g_t coef_q[pr - t][c]
__global__ void k_ssim_bv(int n_rx, int h, int w, const double* __restrict__ coef, double* __restrict__ V) {
    const int cols = w - kSsimWin + 1, rows = h - kSsimWin + 1;
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int pr = blockIdx.y, j = blockIdx.z;
    if (c >= cols) return;
    const size_t wplane = static_cast<size_t>(rows) * cols, vplane = static_cast<size_t>(h) * cols;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const double* cq = coef + (static_cast<size_t>(j) * 3 + q) * wplane;
        double a = 0.0;
#pragma unroll
        for (int t = 0; t < kSsimWin; ++t) {
            const int r = pr - t;
            if (r >= 0 && r < rows) a += c_ssim_g[t] * cq[static_cast<size_t>(r) * cols + c];
        }
        V[(static_cast<size_t>(j) * 3 + q) * vplane + static_cast<size_t>(pr) * cols + c] = a;
    }
}

// adjoint, horizontal pass + the whole d loss / d amplitude + chain to the field:
// G = dL/dx * (re, im) / x
__global__ void k_loss_grad(int n_rx, int h, int w, double l_w, double lambda_ssim, double lambda_fft,
                            const float* __restrict__ field, const float* __restrict__ target,
                            const double* __restrict__ amp, const double* __restrict__ V, float2* __restrict__ G) {
    const int P = h * w;
    const int cell = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    if (cell >= P) return;
    const double x = amp[static_cast<size_t>(j) * P + cell];
    const double y = target[static_cast<size_t>(j) * P + cell];
    const double d = x - y;
    double g = l_w * (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0)) / P + lambda_fft * 2.0 * d;
    if (lambda_ssim > 0.0) {
        const int cols = w - kSsimWin + 1, rows = h - kSsimWin + 1;
        const int pr = cell / w, pc = cell % w;
        const size_t vplane = static_cast<size_t>(h) * cols;
        double k3[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const double* vq = V + (static_cast<size_t>(j) * 3 + q) * vplane + static_cast<size_t>(pr) * cols;
            double a = 0.0;
#pragma unroll
            for (int t = 0; t < kSsimWin; ++t) {
                const int c = pc - t;
                if (c >= 0 && c < cols) a += c_ssim_g[t] * vq[c];
            }
            k3[q] = a;
        }
        const double dssim = (k3[0] + y * k3[1] + x * k3[2]) / (static_cast<double>(rows) * cols);
        g -= lambda_ssim * dssim;
    }
    const float* re_p = field + static_cast<size_t>(j) * 2 * P;
    const double re = re_p[cell], im = re_p[P + cell];
    G[static_cast<size_t>(j) * P + cell] = make_float2(static_cast<float>(g * re / x), static_cast<float>(g * im / x));
}

__global__ void k_loss_total(int n_rx, int nb, int P, double l_w, double lambda_ssim, double lambda_fft,
                             const double* __restrict__ part, const double* __restrict__ ssim, double* __restrict__ loss) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n_rx) return;
    double l1 = 0.0, sq = 0.0;
    for (int b = 0; b < nb; ++b) {
        l1 += part[(static_cast<size_t>(j) * nb + b) * 2];
        sq += part[(static_cast<size_t>(j) * nb + b) * 2 + 1];
    }
    double v = l_w * l1 / P;
    if (lambda_ssim > 0.0) v += lambda_ssim * (1.0 - ssim[j]);
    if (lambda_fft > 0.0) v += lambda_fft * sq;
    loss[j] = v;
}

// ------------------------------------------------------------------ composite transpose
// d_entry[e][j] = sum_cells tw[e][cell] * G_j[cell] for the first W rows of a tile.
// One thread per walked list position: its weight row (ncell floats) is
// read once as float4s and multiplied against every receiver's cell adjoint
// (shared memory, warp-broadcast reads), JB receivers per pass held as
// complex accumulators (FFMA2 on (re, im)).  Per (pos, j) the sum runs over
// the cells in ascending order, exactly as a scalar fmaf chain.
constexpr int kCTJ = 16;  // receivers per pass
__global__ void __launch_bounds__(128) k_composite_T(DevGrid g, const int64_t* __restrict__ tile_offsets,
                                                     const float* __restrict__ tw, const int* __restrict__ walk_len,
                                                     const float2* __restrict__ G, int n_rx,
                                                     float2* __restrict__ d_entry) {
    extern __shared__ float2 sG[];  // [cell_blocks*64][n_rx]
    const int tile = blockIdx.x;
    const int tt = tile / g.tiles_p, tp = tile % g.tiles_p;
    const int ncell = g.cell_blocks * kMaxCellsPerBlock;
    const size_t plane = static_cast<size_t>(g.nt) * g.np;
    for (int i = threadIdx.x; i < ncell * n_rx; i += blockDim.x) {
        const int j = i / ncell, lc = i % ncell;  // coalesced over cells of one receiver plane
        const int row = tt * g.ts + lc / g.ts, col = tp * g.ts + lc % g.ts;
        const bool valid = lc < g.cpt && row < g.nt && col < g.np;
        sG[lc * n_rx + j] = valid ? G[static_cast<size_t>(j) * plane + static_cast<size_t>(row) * g.np + col]
                                  : make_float2(0.f, 0.f);
    }
    __syncthreads();
    int W = 0;
    for (int b = 0; b < g.cell_blocks; ++b) W = max(W, walk_len[tile * g.cell_blocks + b]);
    const int64_t begin = tile_offsets[tile];
    const size_t stride = static_cast<size_t>(ncell);
    for (int pos = threadIdx.x; pos < W; pos += blockDim.x) {
        const float4* t4 = reinterpret_cast<const float4*>(tw + static_cast<size_t>(begin + pos) * stride);
        float2* out = d_entry + static_cast<size_t>(begin + pos) * n_rx;
        for (int j0 = 0; j0 < n_rx; j0 += kCTJ) {
            const int nj = n_rx - j0 < kCTJ ? n_rx - j0 : kCTJ;
            float2 acc[kCTJ];
#pragma unroll
            for (int q = 0; q < kCTJ; ++q) acc[q] = make_float2(0.f, 0.f);
            for (int c4 = 0; c4 < ncell / 4; ++c4) {
                const float4 w4 = t4[c4];
                const float wv[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float2* gr = sG + (4 * c4 + u) * n_rx + j0;
                    if (nj == kCTJ) {
#pragma unroll
                        for (int q = 0; q < kCTJ; ++q) acc[q] = x2::fma(x2::bc(wv[u]), gr[q], acc[q]);
                    } else {
#pragma unroll
                        for (int q = 0; q < kCTJ; ++q)
                            if (q < nj) acc[q] = x2::fma(x2::bc(wv[u]), gr[q], acc[q]);
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < kCTJ; ++q)
                if (q < nj) out[j0 + q] = acc[q];
        }
    }
}

// keys for the per-Gaussian regrouping of walked entries (others -> K)
__global__ void k_entry_keys(DevGrid g, int K, const int64_t* __restrict__ tile_offsets, const int* __restrict__ list,
                             const int* __restrict__ walk_len, int* __restrict__ keys, int* __restrict__ vals) {
    const int tile = blockIdx.x;
    int W = 0;
    for (int b = 0; b < g.cell_blocks; ++b) W = max(W, walk_len[tile * g.cell_blocks + b]);
    const int64_t begin = tile_offsets[tile], n = tile_offsets[tile + 1] - begin;
    for (int p = threadIdx.x; p < n; p += blockDim.x) {
        keys[begin + p] = p < W ? list[begin + p] : K;
        vals[begin + p] = static_cast<int>(begin + p);
    }
}

// entries per Gaussian; the unwalked entries' sentinel key K is not counted
// (the exclusive scan of hist[0..K] never reads hist[K], and those entries
// would otherwise serialise on one counter)
__global__ void k_key_hist(int64_t n, int K, const int* __restrict__ keys, int* __restrict__ hist) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) {
        const int k = keys[i];
        if (k < K) atomicAdd(hist + k, 1);
    }
}

// d_s[k][j] = sum of the k's walked entries, in tile order.
__global__ void k_reduce_ds(const int* __restrict__ n_rows, const int* __restrict__ rows, const int* __restrict__ goff,
                            const int* __restrict__ gent, const float2* __restrict__ d_entry, int n_rx,
                            float2* __restrict__ d_s) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= static_cast<long long>(*n_rows) * n_rx) return;
    const int k = rows[i / n_rx], j = static_cast<int>(i % n_rx);
    float2 acc = make_float2(0.f, 0.f);
    for (int e = goff[k]; e < goff[k + 1]; ++e) acc = cadd(acc, d_entry[static_cast<size_t>(gent[e]) * n_rx + j]);
    d_s[static_cast<size_t>(k) * n_rx + j] = acc;
}

// ------------------------------------------------------------------ conditioning adjoint
// Local-parameter partial layout per CTA (floats): w1 H*6 | b1 H | w2 H*H | b2 H | w3 4H | b3 4
__host__ __device__ constexpr int local_grad_count(int H) { return H * 6 + H + H * H + H + 4 * H + 4; }

// One row = (needed Gaussian k, receiver j), C == 1, hidden H == 64.
// Per row, the MLP forward recompute and backward run out of registers (h1,
// dh1: 64 each; the weights are shared-memory broadcasts); h1, h2, dh1, dh2
// then go to shared memory with a padded row stride (65 floats: conflict-free
// both for one-row-per-thread writes and for the per-weight reads of the
// gradient phase), where each thread owns fixed weight-gradient entries and
// sums the tile's 128 rows in row order (deterministic).
// smem per CTA: W2 (H*H) | h1 | h2 | dh2 | dh1 (4 x 128 x 65) | x (128 x 6) | dy (128 x 4)
// even row pitch: 8-byte aligned float2 rows; 33 float2 per row keeps the
// per-thread row accesses bank-conflict free
constexpr int kBwdPad = 66;
template <int ST, int RT>
__global__ void __launch_bounds__(kBwdThreads) k_cond_bwd(CondDev c, const int* __restrict__ n_rows,
                                                          const int* __restrict__ rows, const float4* __restrict__ pos32,
                                                          const double* __restrict__ rx, int n_rx,
                                                          const float2* __restrict__ Bm, const float2* __restrict__ GB,
                                                          const float* __restrict__ ag, const float2* __restrict__ d_s,
                                                          float2* __restrict__ u_out, float* __restrict__ part) {
    constexpr int H = 64;
    extern __shared__ __align__(16) float sm[];
    float* sW2 = sm;
    float2* sW2T2 = reinterpret_cast<float2*>(sW2 + H * H);  // [i][o/2] = (W2[o][i], W2[o+1][i])
    float* sH1 = sW2 + 2 * H * H;
    float* sH2 = sH1 + kBwdThreads * kBwdPad;
    float* sDH2 = sH2 + kBwdThreads * kBwdPad;
    float* sDH1 = sDH2 + kBwdThreads * kBwdPad;
    float* sX = sDH1 + kBwdThreads * kBwdPad;
    float* sDY = sX + kBwdThreads * 6;
    const float* p = c.p32;
    for (int i = threadIdx.x; i < H * H; i += blockDim.x) sW2[i] = p[c.o_lw2 + i];
    for (int i = threadIdx.x; i < H * H / 2; i += blockDim.x) {
        const int ii = i / (H / 2), op = i % (H / 2);
        sW2T2[i] = make_float2(p[c.o_lw2 + (2 * op) * H + ii], p[c.o_lw2 + (2 * op + 1) * H + ii]);
    }
    __syncthreads();
    const int t = threadIdx.x;
    // per-thread ownership of the weight-gradient accumulators; the 64x64
    // loops run on FFMA2 (two lanes per instruction, each exactly fmaf, in
    // the same order as the scalar code: bit-identical results)
    float2 gw2[16];  // dW2[o = t/2][i = (t%2)*32 .. +32), pairs
    for (int q = 0; q < 16; ++q) gw2[q] = make_float2(0.f, 0.f);
    float gw1[3] = {0.f, 0.f, 0.f};  // dW1 entries t*3 .. t*3+2 (of 384)
    float gw3[2] = {0.f, 0.f};        // dW3 entries t*2, t*2+1 (of 256)
    float gb1 = 0.f, gb2 = 0.f, gb3 = 0.f;  // b1[t], b2[t] (t < 64), b3[t] (t < 4)
    const long long rows_total = static_cast<long long>(*n_rows) * n_rx;
    const int L = c.L;
    for (long long base_row = static_cast<long long>(blockIdx.x) * kBwdThreads; base_row < rows_total;
         base_row += static_cast<long long>(gridDim.x) * kBwdThreads) {
        const long long row = base_row + t;
        const bool active = row < rows_total;
        float* h2s = sH2 + t * kBwdPad;
        float* dh2s = sDH2 + t * kBwdPad;
        float x[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        float dy[4] = {0.f, 0.f, 0.f, 0.f};
        if (c.use_local) {  // warp-uniform: every lane takes part in the probe's vote
            const int kk = active ? rows[row / n_rx] : 0, jj = active ? static_cast<int>(row % n_rx) : 0;
            cube_features<ST, RT>(c, active, active ? pos32[kk] : make_float4(0.f, 0.f, 0.f, 0.f),
                                 static_cast<float>(rx[3 * jj]), static_cast<float>(rx[3 * jj + 1]),
                                 static_cast<float>(rx[3 * jj + 2]), x);
        }
        float h1[H];
        float2 dh1[H / 2];
#pragma unroll
        for (int o = 0; o < H; ++o) h1[o] = 0.f;
#pragma unroll
        for (int o = 0; o < H / 2; ++o) dh1[o] = make_float2(0.f, 0.f);
        if (active && !c.use_local) {  // global-only mode: no local branch, u = d_s
            const int k = rows[row / n_rx], j = static_cast<int>(row % n_rx);
            u_out[static_cast<size_t>(k) * n_rx + j] = d_s[static_cast<size_t>(k) * n_rx + j];
            for (int o = 0; o < H; ++o) h2s[o] = dh2s[o] = 0.f;
        } else if (active) {
            const int k = rows[row / n_rx], j = static_cast<int>(row % n_rx);
            // forward (same arithmetic as the SIMT forward kernel)
#pragma unroll
            for (int o = 0; o < H; ++o) {
                float a = p[c.o_lb1 + o];
#pragma unroll
                for (int i = 0; i < 6; ++i) a = fmaf(p[c.o_lw1 + o * 6 + i], x[i], a);
                h1[o] = fmaxf(a, 0.f);
            }
            float y[4] = {p[c.o_lb3], p[c.o_lb3 + 1], p[c.o_lb3 + 2], p[c.o_lb3 + 3]};
            // four output pairs per pass: independent FFMA2 chains (the 64-long
            // dot products are latency-bound at one warp per SM sub-partition)
#pragma unroll 1
            for (int op0 = 0; op0 < H / 2; op0 += 4) {  // outputs o = 2 op0 .. 2 op0 + 7
                float2 a[4];
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    a[u] = make_float2(p[c.o_lb2 + 2 * (op0 + u)], p[c.o_lb2 + 2 * (op0 + u) + 1]);
#pragma unroll
                for (int i = 0; i < H; ++i) {
                    const float4* wq = reinterpret_cast<const float4*>(sW2T2 + i * (H / 2) + op0);
                    const float4 w01 = wq[0], w23 = wq[1];
                    a[0] = x2::fma(make_float2(w01.x, w01.y), x2::bc(h1[i]), a[0]);
                    a[1] = x2::fma(make_float2(w01.z, w01.w), x2::bc(h1[i]), a[1]);
                    a[2] = x2::fma(make_float2(w23.x, w23.y), x2::bc(h1[i]), a[2]);
                    a[3] = x2::fma(make_float2(w23.z, w23.w), x2::bc(h1[i]), a[3]);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int o = 2 * (op0 + u);
                    const float hv0 = fmaxf(a[u].x, 0.f), hv1 = fmaxf(a[u].y, 0.f);
                    h2s[o] = hv0;
                    h2s[o + 1] = hv1;
#pragma unroll
                    for (int q = 0; q < 4; ++q) y[q] = fmaf(p[c.o_lw3 + q * H + o], hv0, y[q]);
#pragma unroll
                    for (int q = 0; q < 4; ++q) y[q] = fmaf(p[c.o_lw3 + q * H + o + 1], hv1, y[q]);
                }
            }
            // signal pieces M = sum_l mid_l B_l, Bs = sum_l B_l (k_cond signal math)
            float2 M = make_float2(0.f, 0.f), Bs = make_float2(0.f, 0.f);
            const float4* a4 = reinterpret_cast<const float4*>(ag) + static_cast<size_t>(j) * L;
            for (int l = 0; l < L; ++l) {
                const float2 b = Bm[static_cast<size_t>(k) * L + l];
                const float2 gb = GB[static_cast<size_t>(k) * L + l];
                const float4 a = a4[l];
                const float2 t0 = cmul(make_float2(1.f + a.x, a.y), gb), t1 = cmul(make_float2(a.z, a.w), b);
                M = cadd(M, cadd(t0, t1));
                Bs = cadd(Bs, b);
            }
            const float ar = c.additive ? 0.f : y[0], ai = c.additive ? 0.f : y[1];
            const float2 ds = d_s[static_cast<size_t>(k) * n_rx + j];
            // d alpha_L = ds conj(M), d beta_L = ds conj(Bs), u = conj(1 + alpha_L) ds
            const float2 da = cmul(ds, cconj(M)), db = cmul(ds, cconj(Bs));
            dy[0] = c.additive ? 0.f : da.x;
            dy[1] = c.additive ? 0.f : da.y;
            dy[2] = db.x;
            dy[3] = db.y;
            u_out[static_cast<size_t>(k) * n_rx + j] = cmul(make_float2(1.f + ar, -ai), ds);
            // backward through layer 3 and the layer-2 ReLU, then through W2
#pragma unroll 1
            for (int o = 0; o < H; ++o) {
                float a = 0.f;
#pragma unroll
                for (int q = 0; q < 4; ++q) a = fmaf(p[c.o_lw3 + q * H + o], dy[q], a);
                const float g = h2s[o] > 0.f ? a : 0.f;
                dh2s[o] = g;
                if (g == 0.f) continue;
                const float2* wr = reinterpret_cast<const float2*>(sW2 + o * H);
#pragma unroll
                for (int i = 0; i < H / 2; ++i) dh1[i] = x2::fma(wr[i], x2::bc(g), dh1[i]);
            }
#pragma unroll
            for (int i = 0; i < H / 2; ++i)
                dh1[i] = make_float2(h1[2 * i] > 0.f ? dh1[i].x : 0.f, h1[2 * i + 1] > 0.f ? dh1[i].y : 0.f);
        } else {
            for (int o = 0; o < H; ++o) h2s[o] = dh2s[o] = 0.f;
        }
#pragma unroll
        for (int i = 0; i < H / 2; ++i) {
            reinterpret_cast<float2*>(sH1 + t * kBwdPad)[i] = make_float2(h1[2 * i], h1[2 * i + 1]);
            reinterpret_cast<float2*>(sDH1 + t * kBwdPad)[i] = dh1[i];
        }
        for (int i = 0; i < 6; ++i) sX[t * 6 + i] = x[i];
        for (int q = 0; q < 4; ++q) sDY[t * 4 + q] = dy[q];
        __syncthreads();
        // ---- weight gradients over the 128 rows of this tile, fixed row order
        {
            const int o = t >> 1, i0 = (t & 1) * 32;
            for (int r = 0; r < kBwdThreads; ++r) {
                const float g = sDH2[r * kBwdPad + o];
                if (g == 0.f) continue;
                const float2* hr = reinterpret_cast<const float2*>(sH1 + r * kBwdPad + i0);
#pragma unroll
                for (int q = 0; q < 16; ++q) gw2[q] = x2::fma(x2::bc(g), hr[q], gw2[q]);
            }
            for (int e = 0; e < 3; ++e) {
                const int idx = t * 3 + e, oi = idx / 6, fi = idx % 6;
                float a = gw1[e];
                for (int r = 0; r < kBwdThreads; ++r) a = fmaf(sDH1[r * kBwdPad + oi], sX[r * 6 + fi], a);
                gw1[e] = a;
            }
            for (int e = 0; e < 2; ++e) {
                const int idx = t * 2 + e, q = idx / H, oo = idx % H;
                float a = gw3[e];
                for (int r = 0; r < kBwdThreads; ++r) a = fmaf(sDY[r * 4 + q], sH2[r * kBwdPad + oo], a);
                gw3[e] = a;
            }
            if (t < H) {
                float a1 = gb1, a2 = gb2;
                for (int r = 0; r < kBwdThreads; ++r) {
                    a1 += sDH1[r * kBwdPad + t];
                    a2 += sDH2[r * kBwdPad + t];
                }
                gb1 = a1;
                gb2 = a2;
            }
            if (t < 4) {
                float a = gb3;
                for (int r = 0; r < kBwdThreads; ++r) a += sDY[r * 4 + t];
                gb3 = a;
            }
        }
        __syncthreads();
    }
    // ---- per-CTA partials
    constexpr int NG = local_grad_count(H);
    float* out = part + static_cast<size_t>(blockIdx.x) * NG;
    const int o_w1 = 0, o_b1 = H * 6, o_w2 = o_b1 + H, o_b2 = o_w2 + H * H, o_w3 = o_b2 + H, o_b3 = o_w3 + 4 * H;
    for (int q = 0; q < 16; ++q) {
        out[o_w2 + (t >> 1) * H + (t & 1) * 32 + 2 * q] = gw2[q].x;
        out[o_w2 + (t >> 1) * H + (t & 1) * 32 + 2 * q + 1] = gw2[q].y;
    }
    for (int e = 0; e < 3; ++e) out[o_w1 + t * 3 + e] = gw1[e];
    for (int e = 0; e < 2; ++e) out[o_w3 + t * 2 + e] = gw3[e];
    if (t < H) {
        out[o_b1 + t] = gb1;
        out[o_b2 + t] = gb2;
    }
    if (t < 4) out[o_b3 + t] = gb3;
}

// ---- RXGS_BWD_SPLIT: the same backward in two kernels.  k_cond_bwd_rows
// runs the per-row recompute + adjoint at three 4-warp CTAs per SM (no
// per-row activation tiles in shared memory) and writes the activations
// feature-major, act[f][row] (h1 64 | h2 64 | dh1 64 | dh2 64 | x 6 | dy 4);
// k_cond_bwd_grads forms the weight gradients from them as fixed-order
// per-CTA partial sums over contiguous row ranges (dW2 = dH2^T H1 on a 4x4
// register tile per thread), in the k_cond_bwd partial layout.
#ifndef RXGS_BWD_SPLIT
#define RXGS_BWD_SPLIT 1
#endif
#ifndef RXGS_BWD_GRAD_CTAS
#define RXGS_BWD_GRAD_CTAS 4
#endif
template <int ST, int RT>
__global__ void __launch_bounds__(128, 3) k_cond_bwd_rows(CondDev c, const int* __restrict__ n_rows,
                                                          const int* __restrict__ rows, const float4* __restrict__ pos32,
                                                          const double* __restrict__ rx, int n_rx,
                                                          const float2* __restrict__ Bm, const float2* __restrict__ GB,
                                                          const float* __restrict__ ag, const float2* __restrict__ d_s,
                                                          float2* __restrict__ u_out, ActOut act) {
    constexpr int H = 64;
    extern __shared__ __align__(16) float sm[];
    float* sW2 = sm;
    float2* sW2T2 = reinterpret_cast<float2*>(sW2 + H * H);
    const float* p = c.p32;
    for (int i = threadIdx.x; i < H * H; i += blockDim.x) sW2[i] = p[c.o_lw2 + i];
    for (int i = threadIdx.x; i < H * H / 2; i += blockDim.x) {
        const int ii = i / (H / 2), op = i % (H / 2);
        sW2T2[i] = make_float2(p[c.o_lw2 + (2 * op) * H + ii], p[c.o_lw2 + (2 * op + 1) * H + ii]);
    }
    __syncthreads();
    const long long rows_total = static_cast<long long>(*n_rows) * n_rx;
    const int L = c.L;
    if (blockIdx.x == 0) {  // zero the last 64-row chunk's tail: k_cond_grads_tc reads whole chunks
        const long long tail_end = (rows_total + kActRowAlign - 1) / kActRowAlign * kActRowAlign;
        for (long long e = threadIdx.x; e < (tail_end - rows_total) * 2 * kActF; e += blockDim.x)
            act.p[static_cast<size_t>(e / (tail_end - rows_total)) * act.rpad + rows_total +
                  e % (tail_end - rows_total)] = 0;
    }
    for (long long base_row = static_cast<long long>(blockIdx.x) * blockDim.x; base_row < rows_total;
         base_row += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long row = base_row + threadIdx.x;
        const bool active = row < rows_total;
        float x[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        const int kk = active ? rows[row / n_rx] : 0, jj = active ? static_cast<int>(row % n_rx) : 0;
        if (c.use_local)  // warp-uniform: every lane takes part in the probe's vote
            cube_features<ST, RT>(c, active, active ? pos32[kk] : make_float4(0.f, 0.f, 0.f, 0.f),
                                  static_cast<float>(rx[3 * jj]), static_cast<float>(rx[3 * jj + 1]),
                                  static_cast<float>(rx[3 * jj + 2]), x);
        if (!active) continue;
        const int k = kk, j = jj;
        if (!c.use_local) {  // global-only mode: no local branch, u = d_s
            u_out[static_cast<size_t>(k) * n_rx + j] = d_s[static_cast<size_t>(k) * n_rx + j];
            continue;
        }
        float h1[H];
#pragma unroll
        for (int o = 0; o < H; ++o) {
            float acc = p[c.o_lb1 + o];
#pragma unroll
            for (int i = 0; i < 6; ++i) acc = fmaf(p[c.o_lw1 + o * 6 + i], x[i], acc);
            h1[o] = fmaxf(acc, 0.f);
            act.put(row, kAh1 + o, h1[o]);
        }
        float y[4] = {p[c.o_lb3], p[c.o_lb3 + 1], p[c.o_lb3 + 2], p[c.o_lb3 + 3]};
        uint32_t pos_lo = 0u, pos_hi = 0u;  // h2 > 0 mask (the ReLU of layer 2)
#pragma unroll 1
        for (int op0 = 0; op0 < H / 2; op0 += 4) {
            float2 ac[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                ac[u] = make_float2(p[c.o_lb2 + 2 * (op0 + u)], p[c.o_lb2 + 2 * (op0 + u) + 1]);
#pragma unroll
            for (int i = 0; i < H; ++i) {
                const float4* wq = reinterpret_cast<const float4*>(sW2T2 + i * (H / 2) + op0);
                const float4 w01 = wq[0], w23 = wq[1];
                ac[0] = x2::fma(make_float2(w01.x, w01.y), x2::bc(h1[i]), ac[0]);
                ac[1] = x2::fma(make_float2(w01.z, w01.w), x2::bc(h1[i]), ac[1]);
                ac[2] = x2::fma(make_float2(w23.x, w23.y), x2::bc(h1[i]), ac[2]);
                ac[3] = x2::fma(make_float2(w23.z, w23.w), x2::bc(h1[i]), ac[3]);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int o = 2 * (op0 + u);
                const float hv0 = fmaxf(ac[u].x, 0.f), hv1 = fmaxf(ac[u].y, 0.f);
                act.put(row, kAh2 + o, hv0);
                act.put(row, kAh2 + o + 1, hv1);
                const uint32_t bits = (hv0 > 0.f ? 1u : 0u) | (hv1 > 0.f ? 2u : 0u);
                if (o < 32) pos_lo |= bits << o; else pos_hi |= bits << (o - 32);
#pragma unroll
                for (int q = 0; q < 4; ++q) y[q] = fmaf(p[c.o_lw3 + q * H + o], hv0, y[q]);
#pragma unroll
                for (int q = 0; q < 4; ++q) y[q] = fmaf(p[c.o_lw3 + q * H + o + 1], hv1, y[q]);
            }
        }
        float2 M = make_float2(0.f, 0.f), Bs = make_float2(0.f, 0.f);
        const float4* a4 = reinterpret_cast<const float4*>(ag) + static_cast<size_t>(j) * L;
        for (int l = 0; l < L; ++l) {
            const float2 b = Bm[static_cast<size_t>(k) * L + l];
            const float2 gb = GB[static_cast<size_t>(k) * L + l];
            const float4 av = a4[l];
            const float2 t0 = cmul(make_float2(1.f + av.x, av.y), gb), t1 = cmul(make_float2(av.z, av.w), b);
            M = cadd(M, cadd(t0, t1));
            Bs = cadd(Bs, b);
        }
        const float ar = c.additive ? 0.f : y[0], ai = c.additive ? 0.f : y[1];
        const float2 ds = d_s[static_cast<size_t>(k) * n_rx + j];
        const float2 da = cmul(ds, cconj(M)), db = cmul(ds, cconj(Bs));
        float dy[4];
        dy[0] = c.additive ? 0.f : da.x;
        dy[1] = c.additive ? 0.f : da.y;
        dy[2] = db.x;
        dy[3] = db.y;
        u_out[static_cast<size_t>(k) * n_rx + j] = cmul(make_float2(1.f + ar, -ai), ds);
#pragma unroll
        for (int f = 0; f < 6; ++f) act.put(row, kAx + f, x[f]);
#pragma unroll
        for (int q = 0; q < 4; ++q) act.put(row, kAdy + q, dy[q]);
        float2 dh1[H / 2];
#pragma unroll
        for (int i = 0; i < H / 2; ++i) dh1[i] = make_float2(0.f, 0.f);
#pragma unroll 1
        for (int o = 0; o < H; ++o) {
            float gs = 0.f;
#pragma unroll
            for (int q = 0; q < 4; ++q) gs = fmaf(p[c.o_lw3 + q * H + o], dy[q], gs);
            const bool on = ((o < 32 ? pos_lo >> o : pos_hi >> (o - 32)) & 1u) != 0u;
            const float g = on ? gs : 0.f;
            act.put(row, kAdh2 + o, g);
            if (g == 0.f) continue;
            const float2* wr = reinterpret_cast<const float2*>(sW2 + o * H);
#pragma unroll
            for (int i = 0; i < H / 2; ++i) dh1[i] = x2::fma(wr[i], x2::bc(g), dh1[i]);
        }
#pragma unroll
        for (int i = 0; i < H / 2; ++i) {
            act.put(row, kAdh1 + 2 * i, h1[2 * i] > 0.f ? dh1[i].x : 0.f);
            act.put(row, kAdh1 + 2 * i + 1, h1[2 * i + 1] > 0.f ? dh1[i].y : 0.f);
        }
    }
}

// Weight gradients of the local MLP as two GEMMs over rows on tcgen05
// (conditioning.cpp:472-587, mlp_backward: g.w += dy x h summed over the
// batch), K = rows, fed by the TMA engine from the bf16 hi/lo feature planes:
//   GEMM 1: D1[128 x 80] += A1 B1^T,  A1 = [dh2 | dh1] (M 128),
//           B1 = [h1 | x | 1 | 0..] (N 80)  ->  dW2 | db2 (rows 0-63),
//                                              dW1 | db1 (rows 64-127);
//   GEMM 2: D2[128 x 16] += A2 B2^T,  A2 = [h2 | 1 ..] (M 128),
//           B2 = [dy | 0..] (N 16)       ->  dW3^T (rows 0-63), db3 (row 64).
// bf16x3 (Ahi Bhi + Ahi Blo + Alo Bhi, ~2^-17), f32 accumulation in TMEM over
// a contiguous row range per CTA, partials in CTA order (k_reduce_parts):
// deterministic.  Operand tiles are K-major, 128-byte swizzled (64 rows =
// one 128 B line per feature); the constant rows (the bias "1" features and
// the zero padding) are written once per stage buffer and never by the TMA.
// Per 64-row chunk: 8 tiled TMA loads (68 KB), 24 MMAs; 2-stage ring.
constexpr int kGradK = 64;                              // rows per chunk (one SW128 line)
constexpr int kG1N = 80, kG2N = 16;
constexpr int kGA1 = 128 * 128, kGB1 = kG1N * 128, kGA2 = 128 * 128, kGB2 = kG2N * 128;  // bytes per plane
constexpr int kGOffA1 = 0, kGOffB1 = 2 * kGA1, kGOffA2 = kGOffB1 + 2 * kGB1, kGOffB2 = kGOffA2 + 2 * kGA2;
constexpr int kGStage = kGOffB2 + 2 * kGB2;             // 90112 B
constexpr int kGStages = 2;
constexpr uint32_t kGTx = 2u * (128 + 70 + 64 + 4) * 128;  // bytes the TMA brings per chunk
constexpr uint32_t kGIdesc1 = tc::idesc_bf16_f32(128, kG1N), kGIdesc2 = tc::idesc_bf16_f32(128, kG2N);

__device__ __forceinline__ uint64_t sdesc_k_sw128(uint32_t saddr) {  // K-major, 128 B swizzle, 8-row groups 1 KB
    return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (1ull << 16) | (static_cast<uint64_t>(1024 >> 4) << 32) |
           (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void g_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void g_tma_2d(uint32_t dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(tc::smem_u32(bar))
        : "memory");
}

__global__ void __launch_bounds__(128, 1) k_cond_grads_tc(const __grid_constant__ CUtensorMap tm_a1,
                                                          const __grid_constant__ CUtensorMap tm_b1,
                                                          const __grid_constant__ CUtensorMap tm_a2,
                                                          const __grid_constant__ CUtensorMap tm_b2,
                                                          const int* __restrict__ n_rows, int n_rx,
                                                          float* __restrict__ part) {
    constexpr int H = 64;
    extern __shared__ uint8_t g_smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(g_smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[kGStages], empty[kGStages], done;
    __shared__ uint32_t tbase_s;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const long long rows_total = static_cast<long long>(*n_rows) * n_rx;
    const long long chunks = (rows_total + kGradK - 1) / kGradK;
    const long long per = (chunks + gridDim.x - 1) / gridDim.x;
    const long long c_begin = static_cast<long long>(blockIdx.x) * per;
    const long long c_end = c_begin + per < chunks ? c_begin + per : chunks;
    const int n_chunks = c_begin < c_end ? static_cast<int>(c_end - c_begin) : 0;

    // constant rows of every stage: B1 row 70 = 1 (hi) / 0 (lo), rows 71-79 =
    // 0; A2 rows 64-127 = 1 (hi) / 0 (lo); B2 rows 4-15 = 0.  Each row is one
    // 128 B line of a swizzle atom; uniform rows are swizzle-invariant.
    for (int i = tid; i < kGStages * 2 * 10 * 32; i += blockDim.x) {  // B1 rows 70..79
        const int st = i / (2 * 10 * 32), pl = (i / (10 * 32)) % 2, row = 70 + (i / 32) % 10, w = i % 32;
        reinterpret_cast<uint32_t*>(smem + st * kGStage + kGOffB1 + pl * kGB1 + row * 128)[w] =
            (row == 70 && pl == 0) ? 0x3F803F80u : 0u;
    }
    for (int i = tid; i < kGStages * 2 * 64 * 32; i += blockDim.x) {  // A2 rows 64..127
        const int st = i / (2 * 64 * 32), pl = (i / (64 * 32)) % 2, row = 64 + (i / 32) % 64, w = i % 32;
        reinterpret_cast<uint32_t*>(smem + st * kGStage + kGOffA2 + pl * kGA2 + row * 128)[w] =
            pl == 0 ? 0x3F803F80u : 0u;
    }
    for (int i = tid; i < kGStages * 2 * 12 * 32; i += blockDim.x) {  // B2 rows 4..15
        const int st = i / (2 * 12 * 32), pl = (i / (12 * 32)) % 2, row = 4 + (i / 32) % 12, w = i % 32;
        reinterpret_cast<uint32_t*>(smem + st * kGStage + kGOffB2 + pl * kGB2 + row * 128)[w] = 0u;
    }
    if (warp == 0) {
        tc::tmem_alloc(&tbase_s, 128);
        tc::tmem_relinquish();
    }
    if (tid == 0) {
        for (int q = 0; q < kGStages; ++q) {
            tc::mbar_init(&full[q], 1);
            tc::mbar_init(&empty[q], 1);
        }
        tc::mbar_init(&done, 1);
        tc::fence_mbar_init();
    }
    tc::fence_proxy_async_smem();  // the constant rows -> the MMA's async-proxy reads
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm_d1 = tbase_s, tm_d2 = tbase_s + 96;
    const uint32_t sbase = tc::smem_u32(smem);

    if (warp == 0 && lane == 0) {  // TMA producer
        for (int i = 0; i < n_chunks; ++i) {
            const int s = i % kGStages;
            if (i >= kGStages) tc::mbar_wait(&empty[s], ((i / kGStages) - 1) & 1);
            const int x = static_cast<int>((c_begin + i) * kGradK);
            const uint32_t st = sbase + s * kGStage;
            g_expect_tx(&full[s], kGTx);
#pragma unroll
            for (int pl = 0; pl < 2; ++pl) {  // feature planes hi, lo
                g_tma_2d(st + kGOffA1 + pl * kGA1, &tm_a1, x, pl * kActF + kAdh2, &full[s]);
                g_tma_2d(st + kGOffB1 + pl * kGB1, &tm_b1, x, pl * kActF + kAh1, &full[s]);
                g_tma_2d(st + kGOffA2 + pl * kGA2, &tm_a2, x, pl * kActF + kAh2, &full[s]);
                g_tma_2d(st + kGOffB2 + pl * kGB2, &tm_b2, x, pl * kActF + kAdy, &full[s]);
            }
        }
    } else if (warp == 1 && lane == 0) {  // MMA issuer
        for (int i = 0; i < n_chunks; ++i) {
            const int s = i % kGStages;
            tc::mbar_wait(&full[s], (i / kGStages) & 1);
            tc::fence_after_sync();
            const uint32_t st = sbase + s * kGStage;
#pragma unroll
            for (int ks = 0; ks < kGradK / 16; ++ks) {
                const uint32_t ko = 32 * ks;  // 16 K elements within the swizzled 128 B line
                const uint32_t acc0 = (i > 0 || ks > 0) ? 1u : 0u;
                const uint64_t a1h = sdesc_k_sw128(st + kGOffA1 + ko), a1l = sdesc_k_sw128(st + kGOffA1 + kGA1 + ko);
                const uint64_t b1h = sdesc_k_sw128(st + kGOffB1 + ko), b1l = sdesc_k_sw128(st + kGOffB1 + kGB1 + ko);
                tc::mma_ss(tm_d1, a1h, b1h, kGIdesc1, acc0);
                tc::mma_ss(tm_d1, a1h, b1l, kGIdesc1, 1u);
                tc::mma_ss(tm_d1, a1l, b1h, kGIdesc1, 1u);
                const uint64_t a2h = sdesc_k_sw128(st + kGOffA2 + ko), a2l = sdesc_k_sw128(st + kGOffA2 + kGA2 + ko);
                const uint64_t b2h = sdesc_k_sw128(st + kGOffB2 + ko), b2l = sdesc_k_sw128(st + kGOffB2 + kGB2 + ko);
                tc::mma_ss(tm_d2, a2h, b2h, kGIdesc2, acc0);
                tc::mma_ss(tm_d2, a2h, b2l, kGIdesc2, 1u);
                tc::mma_ss(tm_d2, a2l, b2h, kGIdesc2, 1u);
            }
            tc::mma_commit(&empty[s]);
        }
        tc::mma_commit(&done);
    }
    __syncwarp();
    if (n_chunks > 0) tc::mbar_wait_backoff(&done, 0);
    tc::fence_after_sync();
    // ---- epilogue: TMEM lane m = 32 warp + lane = row m of D1 / D2
    constexpr int NG = local_grad_count(H);
    constexpr int o_w1 = 0, o_b1 = H * 6, o_w2 = o_b1 + H, o_b2 = o_w2 + H * H, o_w3 = o_b2 + H, o_b3 = o_w3 + 4 * H;
    float* out = part + static_cast<size_t>(blockIdx.x) * NG;
    const int m = 32 * warp + lane;
    const uint32_t lo = static_cast<uint32_t>(32 * warp) << 16;
    uint32_t r[16];
#pragma unroll
    for (int cb = 0; cb < 5; ++cb) {  // D1 columns 16 cb ..
        if (n_chunks > 0) {
            tc::tmem_ld16(tm_d1 + lo + 16 * cb, r);
            tc::wait_ld();
        } else {
#pragma unroll
            for (int q = 0; q < 16; ++q) r[q] = 0u;
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const int col = 16 * cb + q;
            const float v = __uint_as_float(r[q]);
            if (m < H) {  // dh2 row o = m
                if (col < H) out[o_w2 + m * H + col] = v;
                else if (col == 70) out[o_b2 + m] = v;
            } else {      // dh1 row o = m - 64
                if (col >= 64 && col < 70) out[o_w1 + (m - H) * 6 + (col - 64)] = v;
                else if (col == 70) out[o_b1 + (m - H)] = v;
            }
        }
    }
    if (n_chunks > 0) {
        tc::tmem_ld16(tm_d2 + lo, r);
        tc::wait_ld();
    } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) r[q] = 0u;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const float v = __uint_as_float(r[q]);
        if (m < H) out[o_w3 + q * H + m] = v;  // dW3[q][o] from row o = h2 feature
        else if (m == H) out[o_b3 + q] = v;    // the "1" row: sum of dy
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tbase_s, 128);
}

// sum CTA partials in CTA order into the f64 gradient vector
__global__ void k_reduce_parts(int n_parts, int n, const float* __restrict__ part, double* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;
    for (int b = 0; b < n_parts; ++b) s += part[static_cast<size_t>(b) * n + i];
    out[i] += s;
}

// d_base[k][l] = conj(B_kl) * sum_j conj(1 + aG_jl) u_kj   (C == 1)
__global__ void k_dbase(const int* __restrict__ n_rows, const int* __restrict__ rows, int L, int n_rx,
                        const float2* __restrict__ Bm, const float* __restrict__ ag, int use_global, int additive,
                        const float2* __restrict__ u, double* __restrict__ d_base) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= static_cast<long long>(*n_rows) * L) return;
    const int k = rows[i / L], l = static_cast<int>(i % L);
    double sr = 0.0, si = 0.0;
    for (int j = 0; j < n_rx; ++j) {
        const float2 uv = u[static_cast<size_t>(k) * n_rx + j];
        const float* a = ag + (static_cast<size_t>(j) * L + l) * 4;
        const double ar = (use_global && !additive) ? a[0] : 0.0, ai = (use_global && !additive) ? a[1] : 0.0;
        // conj(1 + a) * u
        sr += (1.0 + ar) * uv.x + ai * uv.y;
        si += (1.0 + ar) * uv.y - ai * uv.x;
    }
    const float2 b = Bm[static_cast<size_t>(k) * L + l];
    // conj(B) * s
    d_base[(static_cast<size_t>(k) * L + l) * 2] += b.x * sr + b.y * si;
    d_base[(static_cast<size_t>(k) * L + l) * 2 + 1] += b.x * si - b.y * sr;
}

// partial sums over Gaussians for the global branch:
// daG_jl = sum_k u_kj conj(GB_kl), dbG_jl = sum_k u_kj conj(B_kl)
__global__ void k_global_red(const int* __restrict__ n_rows, const int* __restrict__ rows, int L, int n_rx,
                             const float2* __restrict__ Bm, const float2* __restrict__ GB,
                             const float2* __restrict__ u, double* __restrict__ part) {
    const int npair = n_rx * L;
    const int nk = *n_rows;
    const int per = (nk + gridDim.x - 1) / gridDim.x;
    const int k0 = blockIdx.x * per, k1 = min(nk, k0 + per);
    for (int pr = threadIdx.x; pr < npair; pr += blockDim.x) {
        const int j = pr / L, l = pr % L;
        double ar = 0, ai = 0, br = 0, bi = 0;
        for (int r = k0; r < k1; ++r) {
            const int k = rows[r];
            const float2 uv = u[static_cast<size_t>(k) * n_rx + j];
            const float2 g = GB[static_cast<size_t>(k) * L + l], b = Bm[static_cast<size_t>(k) * L + l];
            ar += static_cast<double>(uv.x) * g.x + static_cast<double>(uv.y) * g.y;
            ai += static_cast<double>(uv.y) * g.x - static_cast<double>(uv.x) * g.y;
            br += static_cast<double>(uv.x) * b.x + static_cast<double>(uv.y) * b.y;
            bi += static_cast<double>(uv.y) * b.x - static_cast<double>(uv.x) * b.y;
        }
        double* o = part + (static_cast<size_t>(blockIdx.x) * npair + pr) * 4;
        o[0] = ar;
        o[1] = ai;
        o[2] = br;
        o[3] = bi;
    }
}

// Global branch adjoint for one (receiver, l) row in FP64 (mlp_backward
// conditioning.cpp:33-70 with d_input, :530-583).  Writes the row's partial
// gradient over [freqs | global w1 b1 w2 b2 w3 b3 | embed] (packed order).
__global__ void k_global_bwd(CondDev c, int n_rx, const double* __restrict__ rx, const double* __restrict__ red_part,
                             int n_red, double* __restrict__ row_part, int n_gpar) {
    extern __shared__ double gs[];
    const int H = c.H, gin = c.gin, L = c.L, F = c.F;
    double* in = gs;
    double* h1 = in + gin;
    double* h2 = h1 + H;
    double* dh2 = h2 + H;
    double* dh1 = dh2 + H;
    double* din = dh1 + H;
    double* dy = din + gin;
    const int row = blockIdx.x;
    const int j = row / L, comp = row % L;
    const double* p = c.p64;
    double* out = row_part + static_cast<size_t>(row) * n_gpar;
    for (int i = threadIdx.x; i < n_gpar; i += blockDim.x) out[i] = 0.0;
    int l = 0;
    while ((l + 1) * (l + 1) <= comp) ++l;
    const int m = comp - l * l - l;
    int l_max = 0;
    while ((l_max + 1) * (l_max + 1) < L) ++l_max;
    const double den = l_max > 0 ? static_cast<double>(l_max) : 1.0;
    for (int i = threadIdx.x; i < gin; i += blockDim.x) {
        double v;
        if (i < 6 * F) {
            const int a = i / (2 * F), band = (i % (2 * F)) / 2;
            const double arg = p[c.o_freq + band * 3 + a] * rx[3 * j + a];
            v = (i % 2) ? cos(arg) : sin(arg);
        } else if (i == 6 * F) {
            v = l / den;
        } else if (i == 6 * F + 1) {
            v = m / den;
        } else {
            v = p[c.o_emb + comp * c.dc + (i - 6 * F - 2)];
        }
        in[i] = v;
    }
    {  // dy[q] = sum of the n_red k_global_red partials: warp q, lane l sums
       // b = l, l + 32, ... in order, then a fixed shuffle tree (deterministic)
        const int q = threadIdx.x >> 5, ln = threadIdx.x & 31;
        if (q < 4) {
            double s = 0.0;
            for (int b = ln; b < n_red; b += 32) s += red_part[(static_cast<size_t>(b) * n_rx * L + row) * 4 + q];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
            if (ln == 0) dy[q] = (c.additive && q < 2) ? 0.0 : s;
        }
    }
    __syncthreads();
    for (int o = threadIdx.x; o < H; o += blockDim.x) {
        double a = p[c.o_gb1 + o];
        for (int i = 0; i < gin; ++i) a += p[c.o_gw1 + static_cast<size_t>(o) * gin + i] * in[i];
        h1[o] = a > 0.0 ? a : 0.0;
    }
    __syncthreads();
    for (int o = threadIdx.x; o < H; o += blockDim.x) {
        double a = p[c.o_gb2 + o];
        for (int i = 0; i < H; ++i) a += p[c.o_gw2 + static_cast<size_t>(o) * H + i] * h1[i];
        h2[o] = a > 0.0 ? a : 0.0;
    }
    __syncthreads();
    // offsets inside the packed global slice [freqs | w1 b1 w2 b2 w3 b3 | embed]
    const int g_w1 = F * 3, g_b1 = g_w1 + H * gin, g_w2 = g_b1 + H, g_b2 = g_w2 + H * H, g_w3 = g_b2 + H,
              g_b3 = g_w3 + 4 * H, g_emb = g_b3 + 4;
    for (int o = threadIdx.x; o < H; o += blockDim.x) {
        double a = 0.0;
        for (int q = 0; q < 4; ++q) a += p[c.o_gw3 + q * H + o] * dy[q];
        dh2[o] = h2[o] > 0.0 ? a : 0.0;
        for (int q = 0; q < 4; ++q) out[g_w3 + q * H + o] = dy[q] * h2[o];
    }
    if (threadIdx.x < 4) out[g_b3 + threadIdx.x] = dy[threadIdx.x];
    __syncthreads();
    for (int i = threadIdx.x; i < H; i += blockDim.x) {
        double a = 0.0;
        for (int o = 0; o < H; ++o) a += p[c.o_gw2 + static_cast<size_t>(o) * H + i] * dh2[o];
        dh1[i] = h1[i] > 0.0 ? a : 0.0;
    }
    for (int e = threadIdx.x; e < H * H; e += blockDim.x) out[g_w2 + e] = dh2[e / H] * h1[e % H];
    for (int o = threadIdx.x; o < H; o += blockDim.x) out[g_b2 + o] = dh2[o];
    __syncthreads();
    for (int e = threadIdx.x; e < H * gin; e += blockDim.x) out[g_w1 + e] = dh1[e / gin] * in[e % gin];
    for (int o = threadIdx.x; o < H; o += blockDim.x) out[g_b1 + o] = dh1[o];
    for (int i = threadIdx.x; i < gin; i += blockDim.x) {
        double a = 0.0;
        for (int o = 0; o < H; ++o) a += p[c.o_gw1 + static_cast<size_t>(o) * gin + i] * dh1[o];
        din[i] = a;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < c.dc; e += blockDim.x) out[g_emb + comp * c.dc + e] = din[6 * F + 2 + e];
    for (int i = threadIdx.x; i < 3 * F; i += blockDim.x) {  // fourier adjoint (conditioning.cpp:573-583)
        const int a = i / F, band = i % F;
        const double freq = p[c.o_freq + band * 3 + a];
        const double arg = freq * rx[3 * j + a];
        const double ds = din[(a * F + band) * 2], dc = din[(a * F + band) * 2 + 1];
        out[band * 3 + a] = ds * rx[3 * j + a] * cos(arg) - dc * rx[3 * j + a] * sin(arg);
    }
}

__global__ void k_reduce_rows64(int n_rows, int n, const double* __restrict__ part, double* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;
    for (int r = 0; r < n_rows; ++r) s += part[static_cast<size_t>(r) * n + i];
    out[i] += s;
}

// scatter of the packed-global slice into the full packed parameter order
__global__ void k_scatter_global(int n_freq, int n_mlp, int n_emb, size_t o_gw1, size_t o_emb,
                                 const double* __restrict__ g, double* __restrict__ grad) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n_freq) grad[i] += g[i];
    else if (i < n_freq + n_mlp) grad[o_gw1 + (i - n_freq)] += g[i];
    else if (i < n_freq + n_mlp + n_emb) grad[o_emb + (i - n_freq - n_mlp)] += g[i];
}

__global__ void k_check_finite64(int64_t n, const double* __restrict__ v, int* __restrict__ bad) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n && !isfinite(v[i])) atomicMin(bad, 0);
}

// Adam with bias correction (diffengine.cpp:10-34) on f64 masters; lr_scale
// for FLE degree >= 1 coefficients; f32 mirror refreshed in the same pass.
__global__ void k_adam(int64_t n, double* __restrict__ w, const double* __restrict__ g, double* __restrict__ m,
                       double* __restrict__ v, double lr, double bc1, double bc2, double b1, double b2, double eps,
                       int lr_scale_L, int per_comp, double rest_ratio, float* __restrict__ w32) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const double gi = g[i];
    const double mi = b1 * m[i] + (1.0 - b1) * gi;
    const double vi = b2 * v[i] + (1.0 - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    double rate = lr;
    if (lr_scale_L > 0) {
        const int comp = static_cast<int>((i / per_comp) % lr_scale_L);
        if (comp > 0) rate = lr * rest_ratio;  // degree 0 <=> comp 0
    }
    const double wn = w[i] - rate * (mi / bc1) / (sqrt(vi / bc2) + eps);
    w[i] = wn;
    if (w32) w32[i] = static_cast<float>(wn);
}

}  // namespace

int train_regroup(rxgs_ctx ctx, rxgs_txstate_s& st, cudaStream_t s) {
    const int64_t E = st.entries;
    const int K = st.k;
    RXGS_CUDA(st.gauss_off.ensure(sizeof(int) * (K + 2)));
    RXGS_CUDA(st.gauss_ent.ensure(sizeof(int) * (E + 1)));
    auto al = [](size_t x) { return (x + 255) & ~static_cast<size_t>(255); };
    const int En = static_cast<int>(E);
    const size_t o_vals = al(sizeof(int) * (E + 1)), o_ks = o_vals + al(sizeof(int) * (E + 1)),
                 o_hist = o_ks + al(sizeof(int) * (E + 1)), o_work = o_hist + al(sizeof(int) * (K + 2)),
                 o_bsum = o_work + al(sizeof(int) * radix_sort_work_ints(En));
    RXGS_CUDA(ctx->scratch_b.ensure(o_bsum + al(sizeof(int64_t) * scan_bsum_count(K + 1))));
    char* pb = ctx->scratch_b.as<char>();
    uint32_t* keys = reinterpret_cast<uint32_t*>(pb);
    int* vals = reinterpret_cast<int*>(pb + o_vals);
    uint32_t* ks = reinterpret_cast<uint32_t*>(pb + o_ks);
    int* hist = reinterpret_cast<int*>(pb + o_hist);
    int* work = reinterpret_cast<int*>(pb + o_work);
    int64_t* bsum = reinterpret_cast<int64_t*>(pb + o_bsum);
    RXGS_CUDA(cudaMemsetAsync(hist, 0, sizeof(int) * (K + 2), s));
    if (E > 0) {
        // entries (key = Gaussian, value = entry index) straight into gauss_ent;
        // the stable radix sort leaves them grouped by Gaussian in entry order
        k_entry_keys<<<st.grid.n_tiles, 128, 0, s>>>(st.grid, K, st.tile_offsets.as<int64_t>(), st.list.as<int>(),
                                                      st.walk_len.as<int>(), reinterpret_cast<int*>(keys),
                                                      st.gauss_ent.as<int>());
        k_key_hist<<<static_cast<unsigned>((E + 255) / 256), 256, 0, s>>>(E, K, reinterpret_cast<int*>(keys), hist);
        int bits = 1;
        while ((1 << bits) <= K) ++bits;
        RXGS_CUDA(cudaMemsetAsync(work, 0, sizeof(int) * radix_sort_work_ints(En), s));
        RXGS_CUDA(radix_sort_pairs(En, bits, keys, st.gauss_ent.as<int>(), ks, vals, work, false, s));
    }
    RXGS_CUDA(scan_i32(K + 1, hist, st.gauss_off.as<int>(), bsum, s));
    st.regrouped = true;
    ctx->launches += 5;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? RXGS_OK : cuda_fail(e, "train_regroup");
}

cudaError_t launch_refresh_gb(const rxgs_scene_s& sc, rxgs_txstate_s& st, cudaStream_t s) {
    st.version = next_version();  // basis*base changes: cached row data is stale
    const long long n = static_cast<long long>(sc.k) * sc.L * sc.channels;
    if (n == 0) return cudaSuccess;
    k_refresh_gb<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(sc.k, sc.L, sc.channels, st.culled.as<int>(),
                                                                         st.basis64.as<double>(),
                                                                         sc.d_coeffs64.as<double>(), st.gb32.as<float2>());
    return cudaGetLastError();
}

cudaError_t launch_loss_spectrum(int n_rx, int P, const float* field, const float* target, double l_weight,
                                 float2* G, double* loss_part, double* loss, cudaStream_t s) {
    const int nb = 16;
    k_loss_spectrum<<<dim3(nb, n_rx), 256, 0, s>>>(n_rx, P, field, target, l_weight, G, loss_part);
    k_loss_finalize<<<(n_rx + 127) / 128, 128, 0, s>>>(n_rx, nb, loss_part, loss);
    return cudaGetLastError();
}

size_t loss_full_ws_bytes(int n_rx, int h, int w) {
    const size_t P = static_cast<size_t>(h) * w, cols = w >= kSsimWin ? w - kSsimWin + 1 : 0,
                 rows = h >= kSsimWin ? h - kSsimWin + 1 : 0;
    return sizeof(double) * n_rx * (P + 5 * h * cols + 4 * rows * cols + 3 * h * cols + 2 * 16 + 1);
}

cudaError_t launch_loss_full(int n_rx, int h, int w, const float* field, const float* target, double l_w,
                             double lambda_ssim, double lambda_fft, double dyn_range, float2* G, void* ws, double* loss,
                             cudaStream_t s) {
    const int P = h * w, nb = 16;
    const int cols = w - kSsimWin + 1, rows = h - kSsimWin + 1;
    double* amp = static_cast<double*>(ws);
    double* H = amp + static_cast<size_t>(n_rx) * P;
    double* S = H + static_cast<size_t>(n_rx) * 5 * h * (cols > 0 ? cols : 0);
    double* coef = S + static_cast<size_t>(n_rx) * (rows > 0 ? rows : 0) * (cols > 0 ? cols : 0);
    double* V = coef + static_cast<size_t>(n_rx) * 3 * (rows > 0 ? rows : 0) * (cols > 0 ? cols : 0);
    double* part = V + static_cast<size_t>(n_rx) * 3 * h * (cols > 0 ? cols : 0);
    double* ssim = part + static_cast<size_t>(n_rx) * 2 * nb;
    k_loss_amp<<<dim3(nb, n_rx), 256, 0, s>>>(n_rx, P, field, target, amp, part);
    if (lambda_ssim > 0.0) {
        double g[kSsimWin], sum = 0.0;  // gaussian_window (metrics.cpp:38-51), 1-D factor
        for (int t = 0; t < kSsimWin; ++t) {
            const double d = t - kSsimWin / 2;
            g[t] = std::exp(-(d * d) / (2.0 * 1.5 * 1.5));
            sum += g[t];
        }
        for (double& v : g) v /= sum;
        cudaError_t e = cudaMemcpyToSymbolAsync(c_ssim_g, g, sizeof(g), 0, cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return e;
        const double c1 = 0.01 * dyn_range * 0.01 * dyn_range, c2 = 0.03 * dyn_range * 0.03 * dyn_range;
        const int tb = 128;
        k_ssim_h<<<dim3((cols + tb - 1) / tb, h, n_rx), tb, 0, s>>>(n_rx, h, w, amp, target, H);
        k_ssim_v<<<dim3((cols + tb - 1) / tb, rows, n_rx), tb, 0, s>>>(n_rx, h, w, c1, c2, H, S, coef);
        k_ssim_mean<<<n_rx, 256, 0, s>>>(rows, cols, S, ssim);
        k_ssim_bv<<<dim3((cols + tb - 1) / tb, h, n_rx), tb, 0, s>>>(n_rx, h, w, coef, V);
    }
    k_loss_grad<<<dim3((P + 255) / 256, n_rx), 256, 0, s>>>(n_rx, h, w, l_w, lambda_ssim, lambda_fft, field, target,
                                                          amp, V, G);
    k_loss_total<<<(n_rx + 127) / 128, 128, 0, s>>>(n_rx, nb, P, l_w, lambda_ssim, lambda_fft, part, ssim, loss);
    return cudaGetLastError();
}

cudaError_t launch_render_adjoint(const rxgs_txstate_s& st, const float2* G, int n_rx, float2* d_entry, float2* d_s,
                                  cudaStream_t s) {
    const DevGrid& g = st.grid;
    const size_t smem = sizeof(float2) * g.cell_blocks * kMaxCellsPerBlock * n_rx;
    if (st.entries > 0) {
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(k_composite_T, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        k_composite_T<<<g.n_tiles, 128, smem, s>>>(g, st.tile_offsets.as<int64_t>(), st.tw.as<float>(),
                                                   st.walk_len.as<int>(), G, n_rx, d_entry);
    }
    const long long rows = static_cast<long long>(st.visible) * n_rx;
    if (rows > 0)
        k_reduce_ds<<<static_cast<unsigned>((rows + 255) / 256), 256, 0, s>>>(
            st.needed_count.as<int>(), st.needed_order.as<int>(), st.gauss_off.as<int>(), st.gauss_ent.as<int>(),
            d_entry, n_rx, d_s);
    return cudaGetLastError();
}

size_t cond_bwd_smem() { return sizeof(float) * (2 * 64 * 64 + 4 * kBwdThreads * kBwdPad + kBwdThreads * 10); }
// partial-sum CTAs: the split backward's gradient kernel needs many CTAs in
// flight to cover its staged loads
int cond_bwd_parts(int sms) { return RXGS_BWD_SPLIT ? sms : sms * 2; }  // split: one k_cond_grads_tc CTA per SM
int local_grad_n() { return local_grad_count(64); }

size_t cond_bwd_act_bytes(long long rows) {
    return RXGS_BWD_SPLIT ? 2 * sizeof(uint16_t) * kActF *
                                static_cast<size_t>((rows + kActRowAlign - 1) / kActRowAlign * kActRowAlign)
                          : 0;
}

namespace {
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiled encode_tiled() {
    static EncodeTiled fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<EncodeTiled>(p);
    }();
    return fn;
}
// the activation planes as a 2D bf16 tensor {rows (inner), 2 kActF features},
// box {64 rows, box_f features}, 128-byte swizzle; rows past `rows` read as 0
cudaError_t make_act_map(CUtensorMap* m, const void* base, uint64_t rows, long long rpad, uint32_t box_f) {
    EncodeTiled enc = encode_tiled();
    if (!enc) return cudaErrorNotSupported;
    const cuuint64_t dims[2] = {rows, static_cast<cuuint64_t>(2 * kActF)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(rpad) * 2};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(kGradK), box_f};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}
}  // namespace

cudaError_t launch_cond_bwd(const rxgs_cond_s& cs, const rxgs_scene_s& sc, const rxgs_txstate_s& st,
                            const double* d_rx, int n_rx, const float* d_ag, const float2* d_s, float2* u,
                            float* part, int n_parts, cudaStream_t s, float* act, bool tc_rows) {
    const CondDev d = make_dev(cs);
    if (RXGS_BWD_SPLIT && act) {
        const long long rows_bound = static_cast<long long>(st.visible) * n_rx;
        const long long rpad = (rows_bound + kActRowAlign - 1) / kActRowAlign * kActRowAlign;
        const size_t smem_r = sizeof(float) * 2 * 64 * 64;
        auto kr = (d.S == 16 && d.R == 32) ? k_cond_bwd_rows<16, 32> : k_cond_bwd_rows<0, 0>;
        cudaError_t e = cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_r));
        if (e != cudaSuccess) return e;
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        ActOut ao{reinterpret_cast<uint16_t*>(act), rpad};
        if (tc_rows && d.use_local) {
            if ((e = launch_cond_bwd_tc(cs, sc, st, d_rx, n_rx, d_ag, d_s, u, ao.p, rpad, s)) != cudaSuccess) return e;
        } else {
            kr<<<sms * 3, 128, smem_r, s>>>(d, st.needed_count.as<int>(), st.needed_order.as<int>(),
                                            sc.d_pos32.as<float4>(), d_rx, n_rx, st.basis32.as<float2>(),
                                            st.gb32.as<float2>(), d_ag, d_s, u, ao);
            if ((e = cudaGetLastError()) != cudaSuccess) return e;
        }
        if (!d.use_local) return cudaSuccess;
        // the row extent of the tensor maps is the host bound (rows past the
        // needed ones are never read: each CTA stops at needed x n_rx)
        CUtensorMap ma1, mb1, ma2, mb2;
        const uint64_t rows = static_cast<uint64_t>(rows_bound > 0 ? rows_bound : 1);
        if ((e = make_act_map(&ma1, act, rows, rpad, 128)) != cudaSuccess) return e;
        if ((e = make_act_map(&mb1, act, rows, rpad, 70)) != cudaSuccess) return e;
        if ((e = make_act_map(&ma2, act, rows, rpad, 64)) != cudaSuccess) return e;
        if ((e = make_act_map(&mb2, act, rows, rpad, 4)) != cudaSuccess) return e;
        const size_t smem_g = static_cast<size_t>(kGStages) * kGStage + 1024;
        if ((e = cudaFuncSetAttribute(k_cond_grads_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem_g))) != cudaSuccess)
            return e;
        k_cond_grads_tc<<<n_parts, 128, smem_g, s>>>(ma1, mb1, ma2, mb2, st.needed_count.as<int>(), n_rx, part);
        return cudaGetLastError();
    }
    const size_t smem = cond_bwd_smem();
    auto kern = (d.S == 16 && d.R == 32) ? k_cond_bwd<16, 32> : k_cond_bwd<0, 0>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    kern<<<n_parts, kBwdThreads, smem, s>>>(d, st.needed_count.as<int>(), st.needed_order.as<int>(),
                                                  sc.d_pos32.as<float4>(), d_rx, n_rx, st.basis32.as<float2>(),
                                                  st.gb32.as<float2>(), d_ag, d_s, u, part);
    return cudaGetLastError();
}

cudaError_t launch_reduce_parts(int n_parts, int n, const float* part, double* out, cudaStream_t s) {
    k_reduce_parts<<<(n + 255) / 256, 256, 0, s>>>(n_parts, n, part, out);
    return cudaGetLastError();
}

cudaError_t launch_dbase(const rxgs_cond_s* cs, const rxgs_scene_s& sc, const rxgs_txstate_s& st, int n_rx,
                         const float* d_ag, const float2* u, double* d_base, cudaStream_t s) {
    const long long n = static_cast<long long>(st.visible) * sc.L;
    if (n == 0) return cudaSuccess;
    k_dbase<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(
        st.needed_count.as<int>(), st.needed_order.as<int>(), sc.L, n_rx, st.basis32.as<float2>(), d_ag,
        cs && cs->use_global() ? 1 : 0, cs && cs->additive() ? 1 : 0, u, d_base);
    return cudaGetLastError();
}

cudaError_t launch_global_bwd(const rxgs_cond_s& cs, const rxgs_scene_s& sc, const rxgs_txstate_s& st, int n_rx,
                              const double* d_rx, const float2* u, double* red_part, int n_red, double* row_part,
                              double* gslice, double* grad, cudaStream_t s) {
    const CondDev d = make_dev(cs);
    const int npair = n_rx * cs.L;
    // one pass over the pairs per thread (a 128-thread block ran 144 pairs as two passes)
    const int red_threads = std::min(1024, (npair + 31) / 32 * 32);
    k_global_red<<<n_red, red_threads, 0, s>>>(st.needed_count.as<int>(), st.needed_order.as<int>(), cs.L, n_rx,
                                       st.basis32.as<float2>(), st.gb32.as<float2>(), u, red_part);
    const int n_gpar = static_cast<int>(cs.F * 3 + (cs.o_emb - cs.o_gw1) + cs.L * cs.dc);
    const size_t smem = sizeof(double) * (2 * cs.gin + 4 * cs.hidden + 4);
    k_global_bwd<<<npair, 128, smem, s>>>(d, n_rx, d_rx, red_part, n_red, row_part, n_gpar);
    cudaMemsetAsync(gslice, 0, sizeof(double) * n_gpar, s);
    k_reduce_rows64<<<(n_gpar + 255) / 256, 256, 0, s>>>(npair, n_gpar, row_part, gslice);
    const int n_freq = cs.F * 3, n_mlp = static_cast<int>(cs.o_emb - cs.o_gw1), n_emb = cs.L * cs.dc;
    k_scatter_global<<<(n_gpar + 255) / 256, 256, 0, s>>>(n_freq, n_mlp, n_emb, cs.o_gw1, cs.o_emb, gslice, grad);
    return cudaGetLastError();
}

cudaError_t launch_check_finite64(int64_t n, const double* v, int* bad, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_check_finite64<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(n, v, bad);
    return cudaGetLastError();
}

cudaError_t launch_adam(int64_t n, double* w, const double* g, double* m, double* v, double lr, int64_t step,
                        double b1, double b2, double eps, int lr_scale_L, int per_comp, double rest_ratio, float* w32,
                        cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const double bc1 = 1.0 - pow(b1, static_cast<double>(step)), bc2 = 1.0 - pow(b2, static_cast<double>(step));
    k_adam<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(n, w, g, m, v, lr, bc1, bc2, b1, b2, eps,
                                                                  lr_scale_L, per_comp, rest_ratio, w32);
    return cudaGetLastError();
}


// ---------------------------------------------------------------- joint step
// (trainer.cpp:440-463 with train_geometry: backward_render's geometry
// gradients, FLE degree mask, Adam on the geometry groups, quaternion
// renormalisation)
namespace {

// field adjoint G[j][cell] (complex f32) -> d_values[j][c=0][re/im][cell] f64
__global__ void k_dv_from_G(int64_t n, int P, const float2* __restrict__ G, double* __restrict__ dv) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const int64_t j = i / P, cell = i % P;
    const float2 g = G[i];
    dv[(2 * j) * P + cell] = g.x;
    dv[(2 * j + 1) * P + cell] = g.y;
}

// apply_degree_mask (trainer.cpp:233-248): zero the gradient of every
// component of degree > active; component_degree(comp) = floor(sqrt(comp))
__global__ void k_degree_mask(int64_t n, int L, int per_comp, int active, double* __restrict__ g) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const int comp = static_cast<int>((i / per_comp) % L);
    int deg = 0;
    while ((deg + 1) * (deg + 1) <= comp) ++deg;
    if (deg > active) g[i] = 0.0;
}

__global__ void k_add64(int64_t n, const double* __restrict__ a, double* __restrict__ out) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) out[i] += a[i];
}

// per-segment non-finite flags over one flat buffer (segments in buffer order)
__global__ void k_check_groups(int64_t n, GroupBounds b, const double* __restrict__ g, int* __restrict__ bad) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n || isfinite(g[i])) return;
    int seg = 0;
    while (seg + 1 < b.n && i >= b.start[seg + 1]) ++seg;
    bad[seg] = 1;
}

// renormalize_quaternions (scene.cpp:281-288) + the f32 position mirrors
// (index order and the scene's Morton order) read by the conditioning kernels
__global__ void k_geo_post(int K, double* __restrict__ q, const double* __restrict__ pos,
                           const int* __restrict__ morton, float4* __restrict__ pos32, float4* __restrict__ mpos32) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    double* qk = q + 4 * static_cast<size_t>(k);
    double n2 = 0.0;
    for (int a = 0; a < 4; ++a) n2 += qk[a] * qk[a];
    const double inv = 1.0 / sqrt(n2);
    for (int a = 0; a < 4; ++a) qk[a] *= inv;
    pos32[k] = make_float4(static_cast<float>(pos[3 * k]), static_cast<float>(pos[3 * k + 1]),
                           static_cast<float>(pos[3 * k + 2]), 0.f);
    const int src = morton[k];
    mpos32[k] = make_float4(static_cast<float>(pos[3 * src]), static_cast<float>(pos[3 * src + 1]),
                            static_cast<float>(pos[3 * src + 2]), 0.f);
}

unsigned blocks_for(int64_t n) { return static_cast<unsigned>((n + 255) / 256); }

}  // namespace

cudaError_t launch_dv_from_G(int n_rx, int P, const float2* G, double* dv, cudaStream_t s) {
    const int64_t n = static_cast<int64_t>(n_rx) * P;
    if (n == 0) return cudaSuccess;
    k_dv_from_G<<<blocks_for(n), 256, 0, s>>>(n, P, G, dv);
    return cudaGetLastError();
}

cudaError_t launch_degree_mask(int64_t n, int L, int per_comp, int active, double* g, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_degree_mask<<<blocks_for(n), 256, 0, s>>>(n, L, per_comp, active, g);
    return cudaGetLastError();
}

cudaError_t launch_add64(int64_t n, const double* a, double* out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_add64<<<blocks_for(n), 256, 0, s>>>(n, a, out);
    return cudaGetLastError();
}

cudaError_t launch_check_groups(int64_t n, const GroupBounds& b, const double* g, int* bad, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_check_groups<<<blocks_for(n), 256, 0, s>>>(n, b, g, bad);
    return cudaGetLastError();
}

cudaError_t launch_geo_post(rxgs_scene_s& sc, cudaStream_t s) {
    if (sc.k == 0) return cudaSuccess;
    k_geo_post<<<(sc.k + 255) / 256, 256, 0, s>>>(sc.k, sc.d_q.as<double>(), sc.d_pos.as<double>(),
                                                  sc.d_morton.as<int>(), sc.d_pos32.as<float4>(),
                                                  sc.d_mpos32.as<float4>());
    return cudaGetLastError();
}


// ---------------------------------------------------------------- metrics
// met::mae / mse / psnr / ssim (metrics.cpp:11-112) for a batch of images:
// fixed-order per-image sums, SSIM through the same separable window passes
// as the loss (any window size up to kMetMaxWin, the 1-D factor of
// gaussian_window normalised so its outer product sums to 1).
constexpr int kMetMaxWin = 64, kMetParts = 16;
__constant__ double c_met_g[kMetMaxWin];

namespace {

template <typename TP>
__global__ void k_met_sums(int P, const TP* __restrict__ pred, const double* __restrict__ gt, double* __restrict__ part) {
    __shared__ double red[2][256];
    const int j = blockIdx.y;
    double l1 = 0.0, sq = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P; i += gridDim.x * blockDim.x) {
        const double d = static_cast<double>(pred[static_cast<size_t>(j) * P + i]) - gt[static_cast<size_t>(j) * P + i];
        l1 += fabs(d);
        sq += d * d;
    }
    red[0][threadIdx.x] = l1;
    red[1][threadIdx.x] = sq;
    __syncthreads();
    for (int st = blockDim.x / 2; st > 0; st >>= 1) {
        if (threadIdx.x < st) {
            red[0][threadIdx.x] += red[0][threadIdx.x + st];
            red[1][threadIdx.x] += red[1][threadIdx.x + st];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[(static_cast<size_t>(j) * gridDim.x + blockIdx.x) * 2] = red[0][0];
        part[(static_cast<size_t>(j) * gridDim.x + blockIdx.x) * 2 + 1] = red[1][0];
    }
}

template <typename TP>
__global__ void k_met_ssim_h(int h, int w, int win, const TP* __restrict__ pred, const double* __restrict__ gt,
                             double* __restrict__ H) {
    const int cols = w - win + 1;
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int r = blockIdx.y, j = blockIdx.z;
    if (c >= cols) return;
    const TP* x = pred + (static_cast<size_t>(j) * h + r) * w + c;
    const double* y = gt + (static_cast<size_t>(j) * h + r) * w + c;
    double s[5] = {0, 0, 0, 0, 0};
    for (int t = 0; t < win; ++t) {
        const double g = c_met_g[t], xv = static_cast<double>(x[t]), yv = y[t];
        s[0] += g * xv;
        s[1] += g * yv;
        s[2] += g * xv * xv;
        s[3] += g * yv * yv;
        s[4] += g * xv * yv;
    }
    const size_t plane = static_cast<size_t>(h) * cols;
#pragma unroll
    for (int q = 0; q < 5; ++q) H[(static_cast<size_t>(j) * 5 + q) * plane + static_cast<size_t>(r) * cols + c] = s[q];
}

__global__ void k_met_ssim_v(int h, int w, int win, double c1, double c2, const double* __restrict__ H,
                             double* __restrict__ S) {
    const int cols = w - win + 1, rows = h - win + 1;
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int r = blockIdx.y, j = blockIdx.z;
    if (c >= cols) return;
    const size_t hplane = static_cast<size_t>(h) * cols;
    double m[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) {
        const double* hq = H + (static_cast<size_t>(j) * 5 + q) * hplane + static_cast<size_t>(r) * cols + c;
        double a = 0.0;
        for (int t = 0; t < win; ++t) a += c_met_g[t] * hq[static_cast<size_t>(t) * cols];
        m[q] = a;
    }
    const double mx = m[0], my = m[1];
    const double vx = m[2] - mx * mx, vy = m[3] - my * my, cov = m[4] - mx * my;
    const double a1 = 2.0 * mx * my + c1, b1 = mx * mx + my * my + c1;
    const double a2 = 2.0 * cov + c2, b2 = vx + vy + c2;
    S[static_cast<size_t>(j) * rows * cols + static_cast<size_t>(r) * cols + c] = (a1 * a2) / (b1 * b2);
}

__global__ void k_met_final(int n_img, int P, double max_val, const double* __restrict__ part,
                            const double* __restrict__ ssim, double* __restrict__ out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n_img) return;
    double l1 = 0.0, sq = 0.0;
    for (int b = 0; b < kMetParts; ++b) {
        l1 += part[(static_cast<size_t>(j) * kMetParts + b) * 2];
        sq += part[(static_cast<size_t>(j) * kMetParts + b) * 2 + 1];
    }
    const double mse = sq / static_cast<double>(P);
    out[4 * j] = l1 / static_cast<double>(P);
    out[4 * j + 1] = mse;
    out[4 * j + 2] = mse == 0.0 ? 300.0 : 10.0 * log10(max_val * max_val / mse);  // kDbSentinel (metrics.hpp:12)
    out[4 * j + 3] = ssim ? ssim[j] : nan("");
}

}  // namespace

size_t image_metrics_ws_bytes(int n_img, int h, int w, int win) {
    size_t b = sizeof(double) * static_cast<size_t>(n_img) * kMetParts * 2;
    if (win > 0) {
        const size_t cols = w - win + 1, rows = h - win + 1;
        b += sizeof(double) * static_cast<size_t>(n_img) * (5 * h * cols + rows * cols + 1);
    }
    return b;
}

cudaError_t launch_image_metrics(int n_img, int h, int w, const void* pred, bool pred_f32, const double* gt,
                                 double max_val, int win, double sigma, double dyn, void* ws, double* out,
                                 cudaStream_t s) {
    const int P = h * w;
    double* part = static_cast<double*>(ws);
    double* ssim = nullptr;
    if (pred_f32)
        k_met_sums<float><<<dim3(kMetParts, n_img), 256, 0, s>>>(P, static_cast<const float*>(pred), gt, part);
    else
        k_met_sums<double><<<dim3(kMetParts, n_img), 256, 0, s>>>(P, static_cast<const double*>(pred), gt, part);
    if (win > 0) {
        if (win > kMetMaxWin) return cudaErrorInvalidValue;
        double g[kMetMaxWin], sum = 0.0;  // gaussian_window (metrics.cpp:38-51), 1-D factor
        const int half = win / 2;
        for (int t = 0; t < win; ++t) {
            const double d = t - half;
            g[t] = std::exp(-(d * d) / (2.0 * sigma * sigma));
            sum += g[t];
        }
        for (int t = 0; t < win; ++t) g[t] /= sum;
        cudaError_t e = cudaMemcpyToSymbolAsync(c_met_g, g, sizeof(double) * win, 0, cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return e;
        const int cols = w - win + 1, rows = h - win + 1;
        double* H = part + static_cast<size_t>(n_img) * kMetParts * 2;
        double* S = H + static_cast<size_t>(n_img) * 5 * h * cols;
        ssim = S + static_cast<size_t>(n_img) * rows * cols;
        const double c1 = 0.01 * dyn * 0.01 * dyn, c2 = 0.03 * dyn * 0.03 * dyn;
        const int tb = 128;
        if (pred_f32)
            k_met_ssim_h<float><<<dim3((cols + tb - 1) / tb, h, n_img), tb, 0, s>>>(h, w, win,
                                                                                 static_cast<const float*>(pred), gt, H);
        else
            k_met_ssim_h<double><<<dim3((cols + tb - 1) / tb, h, n_img), tb, 0, s>>>(
                h, w, win, static_cast<const double*>(pred), gt, H);
        k_met_ssim_v<<<dim3((cols + tb - 1) / tb, rows, n_img), tb, 0, s>>>(h, w, win, c1, c2, H, S);
        k_ssim_mean<<<n_img, 256, 0, s>>>(rows, cols, S, ssim);
    }
    k_met_final<<<(n_img + 127) / 128, 128, 0, s>>>(n_img, P, max_val, part, ssim, out);
    return cudaGetLastError();
}

}  // namespace rxgs_b200
