// Per-tile front-to-back compositing (render_field, sphraster.cpp:255-315)
// for a whole receiver batch, with the spectrum / RSSI / CSI epilogues of
// aggregate_modality (sphraster.cpp:323-381) fused in.
//
// The FP64 walk (k_walk.cu) has already turned every tile into its blend
// weight matrix tw[pos][cell] (= T_prev * w, zero after each cell's exit), so
// for receiver column j
//     field[cell][j] = sum_{pos < W_tile} tw[pos][cell] * s[list[pos]][j]
// -- a (64 cells x W) x (W x cols) product per tile, cols = n_rx * C complex.
// One CTA per (tile, 64-cell block, 32-column chunk); list chunks of 32
// positions are staged through shared memory (tw rows coalesced, signal rows
// gathered by list index, 256 B contiguous each), double-buffered through
// registers; 256 threads each own 4 cells x 2 complex columns.
#include "rxgs_internal.cuh"

namespace rxgs_b200 {
namespace {

constexpr int kP = 32;      // list positions per stage
constexpr int kCols = 32;   // complex columns per CTA
constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads)
    k_composite(DevGrid g, const int64_t* __restrict__ tile_offsets, const int* __restrict__ list,
                const float* __restrict__ tw, const int* __restrict__ walk_len,
                const float2* __restrict__ sig, int n_rx, int C, float* __restrict__ spectrum,
                float* __restrict__ rssi_partial, double* __restrict__ values,
                float* __restrict__ csi_partial, float* __restrict__ field32) {
    __shared__ __align__(16) float s_tw[2][kP][kMaxCellsPerBlock];
    __shared__ __align__(16) float2 s_sig[2][kP][kCols];
    const int tile = blockIdx.x, cb = blockIdx.y, chunk = blockIdx.z;
    const int tid = threadIdx.x;
    const int cg = tid & 15;   // cells 4cg .. 4cg+3
    const int colg = tid >> 4; // complex columns 2colg, 2colg+1
    const int n_cols = n_rx * C;
    const int col0 = chunk * kCols;
    const int tb = tile * g.cell_blocks + cb;
    const int W = walk_len[tb];
    const int64_t begin = tile_offsets[tile];
    const size_t tw_stride = static_cast<size_t>(g.cell_blocks) * kMaxCellsPerBlock;
    const float* twb = tw + static_cast<size_t>(begin) * tw_stride + static_cast<size_t>(cb) * kMaxCellsPerBlock;

    float acc[4][2][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.f;

    // loader mapping: tw -> 2 float4 per thread ((kP*64)/4 = 512 float4);
    // sig -> 2 float4 (= 4 complex) per thread (kP*kCols/2 = 512 float4)
    float4 rtw[2], rsg[2];
    auto load = [&](int p0) {
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int idx = tid + r * kThreads;  // 0..511
            const int pos = idx >> 4, c4 = idx & 15;
            rtw[r] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (p0 + pos < W)
                rtw[r] = *reinterpret_cast<const float4*>(twb + static_cast<size_t>(p0 + pos) * tw_stride + 4 * c4);
            const int c2 = idx & 15;  // pair of complex columns
            rsg[r] = make_float4(0.f, 0.f, 0.f, 0.f);
            const int col = col0 + 2 * c2;
            if (p0 + pos < W && col < n_cols) {
                const int k = list[begin + p0 + pos];
                const float2* row = sig + static_cast<size_t>(k) * n_cols;
                if (col + 1 < n_cols && (n_cols & 1) == 0) {
                    rsg[r] = *reinterpret_cast<const float4*>(row + col);
                } else {
                    const float2 v = row[col];
                    const float2 u = col + 1 < n_cols ? row[col + 1] : make_float2(0.f, 0.f);
                    rsg[r] = make_float4(v.x, v.y, u.x, u.y);
                }
            }
        }
    };
    auto store = [&](int buf) {
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int idx = tid + r * kThreads;
            const int pos = idx >> 4, c4 = idx & 15;
            *reinterpret_cast<float4*>(&s_tw[buf][pos][4 * c4]) = rtw[r];
            *reinterpret_cast<float4*>(&s_sig[buf][pos][2 * c4]) = rsg[r];
        }
    };
    int buf = 0;
    if (W > 0) {
        load(0);
        store(0);
    }
    __syncthreads();
    for (int p0 = 0; p0 < W; p0 += kP) {
        const bool more = p0 + kP < W;
        if (more) load(p0 + kP);
        const int np_ = min(kP, W - p0);
#pragma unroll 8
        for (int p = 0; p < np_; ++p) {
            const float4 t = *reinterpret_cast<const float4*>(&s_tw[buf][p][4 * cg]);
            const float4 sv = *reinterpret_cast<const float4*>(&s_sig[buf][p][2 * colg]);
            const float tv[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                acc[a][0][0] = fmaf(tv[a], sv.x, acc[a][0][0]);
                acc[a][0][1] = fmaf(tv[a], sv.y, acc[a][0][1]);
                acc[a][1][0] = fmaf(tv[a], sv.z, acc[a][1][0]);
                acc[a][1][1] = fmaf(tv[a], sv.w, acc[a][1][1]);
            }
        }
        if (more) {
            store(buf ^ 1);
            __syncthreads();
            buf ^= 1;
        }
    }

    // ---------------- epilogue
    const int tt = tile / g.tiles_p, tp = tile % g.tiles_p;
    float pw[2] = {0.f, 0.f};
    float cr[2] = {0.f, 0.f}, ci[2] = {0.f, 0.f};
    const size_t plane = static_cast<size_t>(g.nt) * g.np;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int lc = cb * kMaxCellsPerBlock + 4 * cg + a;
        const int lr = lc / g.ts, lcol = lc % g.ts;
        const int row = tt * g.ts + lr, col = tp * g.ts + lcol;
        const bool valid = lc < g.cpt && row < g.nt && col < g.np;
        if (!valid) continue;
        const size_t cell = static_cast<size_t>(row) * g.np + col;
        const float dom = static_cast<float>(sin(g.tmin + (row + 0.5) * g.dth) * g.dth * g.dph);
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            const int colx = col0 + 2 * colg + b;
            if (colx >= n_cols) continue;
            const float re = acc[a][b][0], im = acc[a][b][1];
            const int j = colx / C, ch = colx % C;
            if (spectrum) spectrum[static_cast<size_t>(j) * plane + cell] = sqrtf(re * re + im * im + static_cast<float>(kAmpEps));
            if (values) {
                const size_t base = (static_cast<size_t>(j) * C + ch) * 2 * plane;
                values[base + cell] = re;
                values[base + plane + cell] = im;
            }
            if (field32) {
                const size_t base = (static_cast<size_t>(j) * C + ch) * 2 * plane;
                field32[base + cell] = re;
                field32[base + plane + cell] = im;
            }
            pw[b] += (re * re + im * im) * dom;
            cr[b] += re * dom;
            ci[b] += im * dom;
        }
    }
    if (rssi_partial || csi_partial) {
        // reduce over the 16 cell groups (lanes sharing colg), fixed order
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int off = 8; off >= 1; off >>= 1) {
                pw[b] += __shfl_xor_sync(0xffffffffu, pw[b], off);
                cr[b] += __shfl_xor_sync(0xffffffffu, cr[b], off);
                ci[b] += __shfl_xor_sync(0xffffffffu, ci[b], off);
            }
        if (cg == 0) {
            const int n_tb = g.n_tiles * g.cell_blocks;
#pragma unroll
            for (int b = 0; b < 2; ++b) {
                const int colx = col0 + 2 * colg + b;
                if (colx >= n_cols) continue;
                if (rssi_partial) rssi_partial[static_cast<size_t>(colx) * n_tb + tb] = pw[b];
                if (csi_partial) {
                    csi_partial[(static_cast<size_t>(colx) * n_tb + tb) * 2] = cr[b];
                    csi_partial[(static_cast<size_t>(colx) * n_tb + tb) * 2 + 1] = ci[b];
                }
            }
        }
    }
}

// rssi[j] = 10 log10(sum_tb partial[j][tb] + 1e-12): one warp per receiver,
// fixed-order FP64 reduction (deterministic, no atomics).
__global__ void k_rssi_finalize(const float* __restrict__ partial, int n_tb, int n_rx,
                                float* __restrict__ rssi, double* __restrict__ rssi64) {
    const int j = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (j >= n_rx) return;
    double s = 0.0;
    for (int t = lane; t < n_tb; t += 32) s += partial[static_cast<size_t>(j) * n_tb + t];
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) {
        const double v = 10.0 * log10(s + kRssiFloor);
        if (rssi) rssi[j] = static_cast<float>(v);
        if (rssi64) rssi64[j] = v;
    }
}

// aggregate_modality on a materialised f64 field (sphraster.cpp:323-381):
// one CTA per (receiver, channel); FP64 block reduction.
__global__ void k_aggregate(DevGrid g, int modality, int n_rx, int C, const double* __restrict__ values,
                            double* __restrict__ out) {
    __shared__ double red[3][256];
    const int jc = blockIdx.x;
    const int j = jc / C, ch = jc % C;
    const size_t plane = static_cast<size_t>(g.nt) * g.np;
    const double* re_p = values + (static_cast<size_t>(j) * C + ch) * 2 * plane;
    const double* im_p = re_p + plane;
    double pw = 0.0, sr = 0.0, si = 0.0;
    for (size_t cell = threadIdx.x; cell < plane; cell += blockDim.x) {
        const double re = re_p[cell], im = im_p[cell];
        if (modality == 2) {
            out[static_cast<size_t>(j) * plane + cell] = sqrt(re * re + im * im + kAmpEps);
        } else {
            const int row = static_cast<int>(cell / g.np);
            const double dom = sin(g.tmin + (row + 0.5) * g.dth) * g.dth * g.dph;
            pw += (re * re + im * im) * dom;
            sr += re * dom;
            si += im * dom;
        }
    }
    if (modality == 2) return;
    red[0][threadIdx.x] = pw;
    red[1][threadIdx.x] = sr;
    red[2][threadIdx.x] = si;
    __syncthreads();
    for (int st = blockDim.x / 2; st > 0; st >>= 1) {
        if (threadIdx.x < st)
            for (int q = 0; q < 3; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + st];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (modality == 0) {
            out[j] = 10.0 * log10(red[0][0] + kRssiFloor);
        } else {
            out[(static_cast<size_t>(j) * C + ch) * 2] = red[1][0];
            out[(static_cast<size_t>(j) * C + ch) * 2 + 1] = red[2][0];
        }
    }
}

__global__ void k_check_field(long long n, const double* __restrict__ v, int* __restrict__ err) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i < n && !isfinite(v[i])) atomicMin(err, 0);
}

__global__ void k_fill_T(size_t plane, int n_rx, const double* __restrict__ cell_T, double* __restrict__ T) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= plane * n_rx) return;
    T[i] = cell_T[i % plane];
}

}  // namespace

cudaError_t launch_composite(const rxgs_txstate_s& st, const float2* d_sig, int n_rx,
                             const CompositeOut& out, cudaStream_t s) {
    const DevGrid& g = st.grid;
    const int n_cols = n_rx * st.channels;
    dim3 grid(g.n_tiles, g.cell_blocks, (n_cols + kCols - 1) / kCols);
    k_composite<<<grid, kThreads, 0, s>>>(g, st.tile_offsets.as<int64_t>(), st.list.as<int>(),
                                          st.tw.as<float>(), st.walk_len.as<int>(), d_sig, n_rx,
                                          st.channels, out.spectrum, out.rssi_partial, out.values,
                                          out.csi_partial, out.field32);
    return cudaGetLastError();
}

cudaError_t launch_rssi_finalize(const float* d_partial, int n_tb, int n_rx, float* d_rssi,
                                 double* d_rssi64, cudaStream_t s) {
    k_rssi_finalize<<<(n_rx + 7) / 8, 256, 0, s>>>(d_partial, n_tb, n_rx, d_rssi, d_rssi64);
    return cudaGetLastError();
}

cudaError_t launch_aggregate(const DevGrid& g, int modality, int n_rx, int channels,
                             const double* d_values, double* d_out, int* d_err, bool reduce,
                             cudaStream_t s) {
    const long long n = static_cast<long long>(n_rx) * channels * 2 * g.nt * g.np;
    if (n > 0)
        k_check_field<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(n, d_values, d_err);
    if (reduce && n_rx * channels > 0)
        k_aggregate<<<n_rx * channels, 256, 0, s>>>(g, modality, n_rx, channels, d_values, d_out);
    return cudaGetLastError();
}

cudaError_t launch_fill_transmittance(const rxgs_txstate_s& st, int n_rx, double* d_T,
                                      cudaStream_t s) {
    const size_t plane = static_cast<size_t>(st.grid.nt) * st.grid.np;
    const size_t n = plane * n_rx;
    if (n == 0) return cudaSuccess;
    k_fill_T<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(plane, n_rx, st.cell_T.as<double>(), d_T);
    return cudaGetLastError();
}

}  // namespace rxgs_b200
