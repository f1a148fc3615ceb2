// Materialised conditioning adjoint in FP64 (conditioning.cpp:472-587,
// mlp_backward :33-70): d_out (K x L x C complex, one receiver) -> d_base and
// the packed ConditioningGrads (freqs | global MLP | embed | local MLP, the
// rxgs_cond_create parameter order).
//   k_cb_global_fwd    global branch forward per component, workspace kept
//   k_cb_local         local features + MLP forward, local affine adjoint,
//                      MLP adjoint; weight gradients reduced per CTA over the
//                      CTA's rows in a fixed order (no atomics)
//   k_cb_reduce_parts  CTA partials -> local gradients, fixed order
//   k_cb_global_dy     global affine adjoint per (component, channel): d_base
//                      and the reductions over K (fixed tree)
//   k_cb_global_bwd    global MLP adjoint per component
//   k_cb_global_params weight / embed / frequency gradients, summed over
//                      components in order
// The occupancy probe (T, rho features) is the FP32 one of the forward; all
// other arithmetic is FP64.
#include "cond_common.cuh"
#include "rxgs_internal.cuh"

namespace rxgs_b200 {
namespace {

using namespace cond_dev;

constexpr int kRows = 64;  // rows (Gaussians) per k_cb_local tile

__device__ __forceinline__ int comp_degree(int comp) {
    int l = static_cast<int>(sqrt(static_cast<double>(comp)));
    while ((l + 1) * (l + 1) <= comp) ++l;
    while (l * l > comp) --l;
    return l;
}

// workspace per component: in[gin] h1[H] h2[H] y[4C]
__host__ __device__ inline int gws_stride(int gin, int H, int C) { return gin + 2 * H + 4 * C; }

__global__ void k_cb_global_fwd(CondDev c, int l_max, const double* __restrict__ rx, double* __restrict__ gws) {
    const int comp = blockIdx.x * blockDim.x + threadIdx.x;
    if (comp >= c.L) return;
    const double* p = c.p64;
    const int H = c.H, gin = c.gin, F = c.F;
    double* in = gws + static_cast<size_t>(comp) * gws_stride(gin, H, c.C);
    double* h1 = in + gin;
    double* h2 = h1 + H;
    double* y = h2 + H;
    for (int a = 0; a < 3; ++a)
        for (int band = 0; band < F; ++band) {
            const double arg = p[c.o_freq + band * 3 + a] * rx[a];
            in[(a * F + band) * 2] = sin(arg);
            in[(a * F + band) * 2 + 1] = cos(arg);
        }
    const double denom = l_max > 0 ? static_cast<double>(l_max) : 1.0;
    const int l = comp_degree(comp), m = comp - l * l - l;
    in[6 * F] = l / denom;
    in[6 * F + 1] = m / denom;
    for (int e = 0; e < c.dc; ++e) in[6 * F + 2 + e] = p[c.o_emb + comp * c.dc + e];
    for (int o = 0; o < H; ++o) {
        double a = p[c.o_gb1 + o];
        for (int i = 0; i < gin; ++i) a += p[c.o_gw1 + o * gin + i] * in[i];
        h1[o] = a > 0.0 ? a : 0.0;
    }
    for (int o = 0; o < H; ++o) {
        double a = p[c.o_gb2 + o];
        for (int i = 0; i < H; ++i) a += p[c.o_gw2 + o * H + i] * h1[i];
        h2[o] = a > 0.0 ? a : 0.0;
    }
    for (int o = 0; o < 4 * c.C; ++o) {
        double a = p[c.o_gb3 + o];
        for (int i = 0; i < H; ++i) a += p[c.o_gw3 + o * H + i] * h2[i];
        y[o] = a;
    }
}

__device__ __forceinline__ void affine(double zr, double zi, double ar, double ai, double br, double bi, double& o_r,
                                       double& o_i) {  // conditioning.cpp:271-275
    o_r = zr + (ar * zr - ai * zi + br);
    o_i = zi + (ai * zr + ar * zi + bi);
}

// smem per row: x[6] h1[H] h2[H] dpre1[H] dpre2[H] dy[4C]
__host__ __device__ inline int row_stride(int H, int C) { return 6 + 4 * H + 4 * C; }

__global__ void __launch_bounds__(kRows) k_cb_local(CondDev c, int K, const double* __restrict__ pos,
                                                    const double* __restrict__ rx, const double* __restrict__ base,
                                                    const double* __restrict__ gws, const double* __restrict__ d_out,
                                                    double* __restrict__ d_mid, double* __restrict__ part,
                                                    int n_lp) {
    extern __shared__ double srow[];
    const int t = threadIdx.x, H = c.H, C = c.C, L = c.L;
    const int rs = row_stride(H, C);
    const double* p = c.p64;
    double* my = srow + t * rs;
    double* x = my;
    double* h1 = x + 6;
    double* h2 = h1 + H;
    double* dp1 = h2 + H;
    double* dp2 = dp1 + H;
    double* dy = dp2 + H;
    double* mypart = part + static_cast<size_t>(blockIdx.x) * n_lp;
    for (int i = t; i < n_lp; i += kRows) mypart[i] = 0.0;
    const int gst = gws_stride(c.gin, H, C);
    for (int tile0 = blockIdx.x * kRows; tile0 < K; tile0 += gridDim.x * kRows) {
        const int k = tile0 + t;
        const int n_rows = K - tile0 < kRows ? K - tile0 : kRows;
        if (k < K) {
            // features (conditioning.cpp:376-396): FP64 direction / distance, FP32 probe
            const double px = pos[3 * k], py = pos[3 * k + 1], pz = pos[3 * k + 2];
            const double dx = rx[0] - px, dy_ = rx[1] - py, dz = rx[2] - pz;
            const double d = sqrt(dx * dx + dy_ * dy_ + dz * dz);
            float xf[6];
            local_features<false>(c, c.occ, static_cast<float>(px), static_cast<float>(py), static_cast<float>(pz),
                                  static_cast<float>(rx[0]), static_cast<float>(rx[1]), static_cast<float>(rx[2]),
                                  xf);
            x[0] = dx / d;
            x[1] = dy_ / d;
            x[2] = dz / d;
            x[3] = d;
            x[4] = c.probe ? static_cast<double>(xf[4]) : 1.0;
            x[5] = c.probe ? static_cast<double>(xf[5]) : 0.0;
            for (int o = 0; o < H; ++o) {
                double a = p[c.o_lb1 + o];
                for (int i = 0; i < 6; ++i) a += p[c.o_lw1 + o * 6 + i] * x[i];
                h1[o] = a > 0.0 ? a : 0.0;
            }
            for (int o = 0; o < H; ++o) {
                double a = p[c.o_lb2 + o];
                for (int i = 0; i < H; ++i) a += p[c.o_lw2 + o * H + i] * h1[i];
                h2[o] = a > 0.0 ? a : 0.0;
            }
            // local affine adjoint (conditioning.cpp:493-519)
            for (int ch = 0; ch < C; ++ch) {
                double y[4];
                for (int q = 0; q < 4; ++q) {
                    double a = p[c.o_lb3 + 4 * ch + q];
                    for (int i = 0; i < H; ++i) a += p[c.o_lw3 + (4 * ch + q) * H + i] * h2[i];
                    y[q] = a;
                }
                const double ar = c.additive ? 0.0 : y[0], ai = c.additive ? 0.0 : y[1];
                double dar = 0.0, dai = 0.0, dbr = 0.0, dbi = 0.0;
                for (int comp = 0; comp < L; ++comp) {
                    const size_t idx = ((static_cast<size_t>(k) * L + comp) * C + ch) * 2;
                    double zr = base[idx], zi = base[idx + 1];
                    if (c.use_global) {
                        const double* gy = gws + static_cast<size_t>(comp) * gst + c.gin + 2 * H + 4 * ch;
                        const double gar = c.additive ? 0.0 : gy[0], gai = c.additive ? 0.0 : gy[1];
                        double mr, mi;
                        affine(zr, zi, gar, gai, gy[2], gy[3], mr, mi);
                        zr = mr;
                        zi = mi;
                    }
                    const double gr = d_out[idx], gi = d_out[idx + 1];
                    d_mid[idx] = gr * (1.0 + ar) + gi * ai;
                    d_mid[idx + 1] = -gr * ai + gi * (1.0 + ar);
                    dar += gr * zr + gi * zi;
                    dai += -gr * zi + gi * zr;
                    dbr += gr;
                    dbi += gi;
                }
                dy[4 * ch] = c.additive ? 0.0 : dar;
                dy[4 * ch + 1] = c.additive ? 0.0 : dai;
                dy[4 * ch + 2] = dbr;
                dy[4 * ch + 3] = dbi;
            }
            // MLP adjoint (conditioning.cpp:33-70)
            for (int i = 0; i < H; ++i) {
                double a = 0.0;
                for (int o = 0; o < 4 * C; ++o) a += p[c.o_lw3 + o * H + i] * dy[o];
                dp2[i] = h2[i] <= 0.0 ? 0.0 : a;
            }
            for (int i = 0; i < H; ++i) {
                double a = 0.0;
                for (int o = 0; o < H; ++o) a += p[c.o_lw2 + o * H + i] * dp2[o];
                dp1[i] = h1[i] <= 0.0 ? 0.0 : a;
            }
        }
        __syncthreads();
        // weight gradients: thread-owned parameters, rows in order
        const int n_w1 = H * 6, n_w2 = H * H, n_w3 = 4 * C * H;
        for (int idx = t; idx < n_lp; idx += kRows) {
            int off = idx;
            double acc = 0.0;
            if (off < n_w1) {
                const int o = off / 6, i = off % 6;
                for (int r = 0; r < n_rows; ++r) acc += srow[r * rs + 6 + 2 * H + o] * srow[r * rs + i];
            } else if ((off -= n_w1) < H) {
                for (int r = 0; r < n_rows; ++r) acc += srow[r * rs + 6 + 2 * H + off];
            } else if ((off -= H) < n_w2) {
                const int o = off / H, i = off % H;
                for (int r = 0; r < n_rows; ++r) acc += srow[r * rs + 6 + 3 * H + o] * srow[r * rs + 6 + i];
            } else if ((off -= n_w2) < H) {
                for (int r = 0; r < n_rows; ++r) acc += srow[r * rs + 6 + 3 * H + off];
            } else if ((off -= H) < n_w3) {
                const int o = off / H, i = off % H;
                for (int r = 0; r < n_rows; ++r) acc += srow[r * rs + 6 + 4 * H + o] * srow[r * rs + 6 + H + i];
            } else {
                off -= n_w3;
                for (int r = 0; r < n_rows; ++r) acc += srow[r * rs + 6 + 4 * H + off];
            }
            mypart[idx] += acc;
        }
        __syncthreads();
    }
}

__global__ void k_cb_reduce_parts(int n_parts, int n, const double* __restrict__ part, double* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;
    for (int b = 0; b < n_parts; ++b) s += part[static_cast<size_t>(b) * n + i];
    out[i] = s;
}

// global affine adjoint (conditioning.cpp:530-560), one CTA per (comp, channel)
__global__ void k_cb_global_dy(CondDev c, int K, const double* __restrict__ base, const double* __restrict__ gws,
                               const double* __restrict__ d_mid, double* __restrict__ d_base,
                               double* __restrict__ gdy) {
    __shared__ double red[4][256];
    const int comp = blockIdx.x / c.C, ch = blockIdx.x % c.C, L = c.L, C = c.C, H = c.H;
    const double* gy = gws + static_cast<size_t>(comp) * gws_stride(c.gin, H, C) + c.gin + 2 * H + 4 * ch;
    const double ar = c.additive ? 0.0 : gy[0], ai = c.additive ? 0.0 : gy[1];
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
        const size_t idx = ((static_cast<size_t>(k) * L + comp) * C + ch) * 2;
        const double gr = d_mid[idx], gi = d_mid[idx + 1];
        const double zr = base[idx], zi = base[idx + 1];
        d_base[idx] = gr * (1.0 + ar) + gi * ai;
        d_base[idx + 1] = -gr * ai + gi * (1.0 + ar);
        s0 += gr * zr + gi * zi;
        s1 += -gr * zi + gi * zr;
        s2 += gr;
        s3 += gi;
    }
    red[0][threadIdx.x] = s0;
    red[1][threadIdx.x] = s1;
    red[2][threadIdx.x] = s2;
    red[3][threadIdx.x] = s3;
    __syncthreads();
    for (int st = blockDim.x / 2; st > 0; st >>= 1) {
        if (threadIdx.x < st)
            for (int q = 0; q < 4; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + st];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double* o = gdy + static_cast<size_t>(comp) * 4 * C + 4 * ch;
        o[0] = c.additive ? 0.0 : red[0][0];
        o[1] = c.additive ? 0.0 : red[1][0];
        o[2] = red[2][0];
        o[3] = red[3][0];
    }
}

// per component: dpre2[H] dpre1[H] d_in[gin]
__global__ void k_cb_global_bwd(CondDev c, const double* __restrict__ gws, const double* __restrict__ gdy,
                                double* __restrict__ gbw) {
    const int comp = blockIdx.x * blockDim.x + threadIdx.x;
    if (comp >= c.L) return;
    const double* p = c.p64;
    const int H = c.H, gin = c.gin, C = c.C;
    const double* in = gws + static_cast<size_t>(comp) * gws_stride(gin, H, C);
    const double* h1 = in + gin;
    const double* h2 = h1 + H;
    const double* dy = gdy + static_cast<size_t>(comp) * 4 * C;
    double* dp2 = gbw + static_cast<size_t>(comp) * (2 * H + gin);
    double* dp1 = dp2 + H;
    double* din = dp1 + H;
    for (int i = 0; i < H; ++i) {
        double a = 0.0;
        for (int o = 0; o < 4 * C; ++o) a += p[c.o_gw3 + o * H + i] * dy[o];
        dp2[i] = h2[i] <= 0.0 ? 0.0 : a;
    }
    for (int i = 0; i < H; ++i) {
        double a = 0.0;
        for (int o = 0; o < H; ++o) a += p[c.o_gw2 + o * H + i] * dp2[o];
        dp1[i] = h1[i] <= 0.0 ? 0.0 : a;
    }
    for (int i = 0; i < gin; ++i) {
        double a = 0.0;
        for (int o = 0; o < H; ++o) a += p[c.o_gw1 + o * gin + i] * dp1[o];
        din[i] = a;
    }
}

// packed global gradients: freqs, w1 b1 w2 b2 w3 b3, embed
__global__ void k_cb_global_params(CondDev c, const double* __restrict__ rx, const double* __restrict__ gws,
                                   const double* __restrict__ gdy, const double* __restrict__ gbw,
                                   double* __restrict__ dpar) {
    const int H = c.H, gin = c.gin, C = c.C, L = c.L, F = c.F;
    const int gst = gws_stride(gin, H, C), bst = 2 * H + gin;
    const int n_w1 = H * gin, n_w2 = H * H, n_w3 = 4 * C * H;
    const int n_glob = n_w1 + H + n_w2 + H + n_w3 + 4 * C;
    const int n_total = 3 * F + n_glob + L * c.dc;
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n_total) return;
    if (idx < 3 * F) {  // Fourier adjoint (conditioning.cpp:573-583)
        const int band = idx / 3, a = idx % 3;
        double ds = 0.0, dc = 0.0;
        for (int comp = 0; comp < L; ++comp) {
            const double* din = gbw + static_cast<size_t>(comp) * bst + 2 * H;
            ds += din[(a * F + band) * 2];
            dc += din[(a * F + band) * 2 + 1];
        }
        const double arg = c.p64[c.o_freq + idx] * rx[a];
        dpar[c.o_freq + idx] = ds * rx[a] * cos(arg) - dc * rx[a] * sin(arg);
        return;
    }
    int off = idx - 3 * F;
    if (off >= n_glob) {  // component embedding slice of d_in
        off -= n_glob;
        const int comp = off / c.dc, e = off % c.dc;
        dpar[c.o_emb + off] = gbw[static_cast<size_t>(comp) * bst + 2 * H + 6 * F + 2 + e];
        return;
    }
    const int pidx = off;
    double acc = 0.0;
    if (off < n_w1) {
        const int o = off / gin, i = off % gin;
        for (int comp = 0; comp < L; ++comp)
            acc += gbw[static_cast<size_t>(comp) * bst + H + o] * gws[static_cast<size_t>(comp) * gst + i];
    } else if ((off -= n_w1) < H) {
        for (int comp = 0; comp < L; ++comp) acc += gbw[static_cast<size_t>(comp) * bst + H + off];
    } else if ((off -= H) < n_w2) {
        const int o = off / H, i = off % H;
        for (int comp = 0; comp < L; ++comp)
            acc += gbw[static_cast<size_t>(comp) * bst + o] * gws[static_cast<size_t>(comp) * gst + gin + i];
    } else if ((off -= n_w2) < H) {
        for (int comp = 0; comp < L; ++comp) acc += gbw[static_cast<size_t>(comp) * bst + off];
    } else if ((off -= H) < n_w3) {
        const int o = off / H, i = off % H;
        for (int comp = 0; comp < L; ++comp)
            acc += gdy[static_cast<size_t>(comp) * 4 * C + o] * gws[static_cast<size_t>(comp) * gst + gin + H + i];
    } else {
        off -= n_w3;
        for (int comp = 0; comp < L; ++comp) acc += gdy[static_cast<size_t>(comp) * 4 * C + off];
    }
    dpar[c.o_gw1 + pidx] = acc;  // g.w1 .. g.b3 are contiguous from o_gw1
}

}  // namespace

size_t cond_backward_ws_bytes(const rxgs_cond_s& cs, int K, int sms) {
    const int H = cs.hidden;
    const int n_lp = H * 6 + H + H * H + H + 4 * cs.C * H + 4 * cs.C;
    const size_t nb = static_cast<size_t>(std::min((K + kRows - 1) / kRows, 2 * sms));
    const size_t gst = gws_stride(cs.gin, H, cs.C);
    return sizeof(double) * (cs.L * gst + cs.L * 4 * cs.C + cs.L * (2 * H + cs.gin) +
                             std::max<size_t>(nb, 1) * n_lp) +
           sizeof(double) * static_cast<size_t>(K) * cs.L * cs.C * 2 + 1024;
}

cudaError_t launch_cond_backward(const rxgs_cond_s& cs, const rxgs_scene_s& sc, const double* d_rx,
                                 const double* d_out, double* d_base, double* d_params, void* ws, int sms,
                                 cudaStream_t s) {
    const CondDev c = make_dev(cs);
    const int K = sc.k, L = cs.L, C = cs.C, H = cs.hidden;
    const int n_lp = H * 6 + H + H * H + H + 4 * C * H + 4 * C;
    const int nb = std::max(1, std::min((K + kRows - 1) / kRows, 2 * sms));
    double* gws = static_cast<double*>(ws);
    double* gdy = gws + static_cast<size_t>(L) * gws_stride(cs.gin, H, C);
    double* gbw = gdy + static_cast<size_t>(L) * 4 * C;
    double* part = gbw + static_cast<size_t>(L) * (2 * H + cs.gin);
    double* d_mid = part + static_cast<size_t>(nb) * n_lp;
    const size_t n_params = cs.h_params.size();
    cudaMemsetAsync(d_params, 0, n_params * sizeof(double), s);
    const double* base = sc.d_coeffs64.as<double>();
    if (cs.use_global()) k_cb_global_fwd<<<(L + 63) / 64, 64, 0, s>>>(c, cs.l_max, d_rx, gws);
    const double* dm = d_out;
    if (cs.use_local() && K > 0) {
        const size_t smem = sizeof(double) * kRows * row_stride(H, C);
        cudaFuncSetAttribute(k_cb_local, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        k_cb_local<<<nb, kRows, smem, s>>>(c, K, sc.d_pos.as<double>(), d_rx, base, gws, d_out, d_mid, part, n_lp);
        k_cb_reduce_parts<<<(n_lp + 255) / 256, 256, 0, s>>>(nb, n_lp, part, d_params + cs.o_lw1);
        dm = d_mid;
    }
    const size_t nco = static_cast<size_t>(K) * L * C * 2;
    if (cs.use_global()) {
        k_cb_global_dy<<<L * C, 256, 0, s>>>(c, K, base, gws, dm, d_base, gdy);
        k_cb_global_bwd<<<(L + 63) / 64, 64, 0, s>>>(c, gws, gdy, gbw);
        const int n_total = 3 * cs.F + H * cs.gin + H + H * H + H + 4 * C * H + 4 * C + L * cs.dc;
        k_cb_global_params<<<(n_total + 127) / 128, 128, 0, s>>>(c, d_rx, gws, gdy, gbw, d_params);
    } else if (nco) {
        cudaMemcpyAsync(d_base, dm, nco * sizeof(double), cudaMemcpyDeviceToDevice, s);
    }
    return cudaGetLastError();
}

}  // namespace rxgs_b200
