// FP64 device kernels behind the reference-shaped single-call API (the
// materialised conditioning, the occupancy / probe helpers, blend_ray): the
// functions a caller of rxgs::raster / rxgs::cond uses outside the fused
// query path, computed on the B200 in the reference's FP64 operation order
// (compiled with -fmad=false, like k_geometry.cu), so the reference's own
// test suites hold at their tolerances (1e-12 .. 1e-15, bitwise where they
// compare bitwise) and finite differences of the materialised forward agree
// with condition_backward.
//
//   k_blend_ray        blend_ray (sphraster.cpp:174-185)
//   k_occ_sample       OccupancyGrid::sample_trilinear / sample_nearest
//                      (conditioning.cpp:74-112)
//   k_probe64          probe_segment (conditioning.cpp:163-178)
//   k_fourier64        fourier_encode (conditioning.cpp:255-265)
//   k_mlp_layer64      MlpLayer::forward (conditioning.cpp:12-19)
//   k_cond_global64    the global branch (conditioning.cpp:317-361): per
//                      (receiver, component) the MLP in mlp_forward's order
//   k_cond_forward64   per (receiver, Gaussian) the local features, the local
//                      MLP and both affines (conditioning.cpp:365-421)
#include "cond_common.cuh"
#include "rxgs_internal.cuh"

namespace rxgs_b200 {
using namespace cond_dev;
namespace {

__device__ __forceinline__ double clampd(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }

__global__ void k_blend_ray(int n, const double* __restrict__ w, const double* __restrict__ sig,
                            double* __restrict__ out) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    double cr = 0.0, ci = 0.0, T = 1.0;
    for (int i = 0; i < n; ++i) {
        const double wi = clampd(w[i], 0.0, 0.999);  // kWeightClamp
        const double tw = T * wi;
        cr += tw * sig[2 * i];
        ci += tw * sig[2 * i + 1];
        T *= 1.0 - wi;
        if (T < 1e-4) break;  // kEarlyExitT
    }
    out[0] = cr;
    out[1] = ci;
    out[2] = T;
}

struct Occ64 {
    const double* dens;  // R^3, (ix * R + iy) * R + iz; nullptr = empty grid
    int R;
    double lo[3], ext[3];
};

__device__ double sample_trilinear64(const Occ64& g, double px, double py, double pz) {
    if (!g.dens) return 0.0;
    const int r = g.R;
    const double p[3] = {px, py, pz};
    double u[3], f[3];
    int i0[3];
    for (int a = 0; a < 3; ++a) {
        const double cell = g.ext[a] / r;
        u[a] = (p[a] - g.lo[a]) / cell - 0.5;
        i0[a] = static_cast<int>(floor(u[a]));
        f[a] = u[a] - i0[a];
    }
    double acc = 0.0;
    for (int dx = 0; dx < 2; ++dx)
        for (int dy = 0; dy < 2; ++dy)
            for (int dz = 0; dz < 2; ++dz) {
                const int ix = i0[0] + dx, iy = i0[1] + dy, iz = i0[2] + dz;
                if (ix < 0 || iy < 0 || iz < 0 || ix >= r || iy >= r || iz >= r) continue;
                const double wgt = (dx ? f[0] : 1 - f[0]) * (dy ? f[1] : 1 - f[1]) * (dz ? f[2] : 1 - f[2]);
                acc += wgt * g.dens[(static_cast<size_t>(ix) * r + iy) * r + iz];
            }
    return acc;
}

__device__ double sample_nearest64(const Occ64& g, double px, double py, double pz) {
    if (!g.dens) return 0.0;
    const int r = g.R;
    const double p[3] = {px, py, pz};
    int idx[3];
    for (int a = 0; a < 3; ++a) {
        const double cell = g.ext[a] / r;
        const int i = static_cast<int>(floor((p[a] - g.lo[a]) / cell));
        if (i < 0 || i >= r) return 0.0;
        idx[a] = i;
    }
    return g.dens[(static_cast<size_t>(idx[0]) * r + idx[1]) * r + idx[2]];
}

__device__ void probe64(const Occ64& g, const double* from, const double* to, int samples, bool nearest,
                        double* T, double* mean) {
    double tr = 1.0, sum = 0.0;
    for (int s = 0; s < samples; ++s) {
        const double t = samples == 1 ? 0.5 : 0.05 + 0.9 * static_cast<double>(s) / (samples - 1);
        // Vec3 q = from + t * (to - from)
        const double qx = from[0] + t * (to[0] - from[0]);
        const double qy = from[1] + t * (to[1] - from[1]);
        const double qz = from[2] + t * (to[2] - from[2]);
        const double v = nearest ? sample_nearest64(g, qx, qy, qz) : sample_trilinear64(g, qx, qy, qz);
        tr *= 1.0 - v;
        sum += v;
    }
    *T = tr;
    *mean = sum / samples;
}

__global__ void k_occ_sample(Occ64 g, int n, const double* __restrict__ pts, int nearest, double* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double* p = pts + 3 * static_cast<size_t>(i);
    out[i] = nearest ? sample_nearest64(g, p[0], p[1], p[2]) : sample_trilinear64(g, p[0], p[1], p[2]);
}

__global__ void k_probe64(Occ64 g, int n, const double* __restrict__ from, const double* __restrict__ to,
                          int samples, int nearest, double* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    probe64(g, from + 3 * static_cast<size_t>(i), to + 3 * static_cast<size_t>(i), samples, nearest != 0,
            out + 2 * static_cast<size_t>(i), out + 2 * static_cast<size_t>(i) + 1);
}

__global__ void k_fourier64(int F, const double* __restrict__ freqs, int n, const double* __restrict__ r,
                            double* __restrict__ out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * 3 * F) return;
    const int i = t / (3 * F), a = (t % (3 * F)) / F, band = t % F;
    const double arg = freqs[band * 3 + a] * r[3 * static_cast<size_t>(i) + a];
    double* o = out + static_cast<size_t>(i) * 6 * F + (static_cast<size_t>(a) * F + band) * 2;
    o[0] = sin(arg);
    o[1] = cos(arg);
}

__global__ void k_mlp_layer64(int in, int nout, const double* __restrict__ w, const double* __restrict__ b, int n,
                              const double* __restrict__ x, double* __restrict__ y) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * nout) return;
    const int i = t / nout, o = t % nout;
    double acc = b[o];
    const double* row = w + static_cast<size_t>(o) * in;
    const double* xi = x + static_cast<size_t>(i) * in;
    for (int q = 0; q < in; ++q) acc += row[q] * xi[q];
    y[t] = acc;
}

// mlp_forward (conditioning.cpp:23-29) on one input vector, FP64
template <int MAXH>
__device__ void mlp64(const double* p, int o_w1, int o_b1, int o_w2, int o_b2, int o_w3, int o_b3, int in, int H,
                      int NY, const double* x, double* y) {
    double h1[MAXH], h2[MAXH];
    for (int o = 0; o < H; ++o) {
        double acc = p[o_b1 + o];
        const double* row = p + o_w1 + static_cast<size_t>(o) * in;
        for (int i = 0; i < in; ++i) acc += row[i] * x[i];
        h1[o] = acc > 0.0 ? acc : 0.0;  // std::max(0.0, h)
    }
    for (int o = 0; o < H; ++o) {
        double acc = p[o_b2 + o];
        const double* row = p + o_w2 + static_cast<size_t>(o) * H;
        for (int i = 0; i < H; ++i) acc += row[i] * h1[i];
        h2[o] = acc > 0.0 ? acc : 0.0;
    }
    for (int o = 0; o < NY; ++o) {
        double acc = p[o_b3 + o];
        const double* row = p + o_w3 + static_cast<size_t>(o) * H;
        for (int i = 0; i < H; ++i) acc += row[i] * h2[i];
        y[o] = acc;
    }
}

constexpr int kMaxHidden64 = 128;
constexpr int kMaxGin64 = 6 * 16 + 2 + 64;

// ag[(j * L + comp) * 4C + o]: the global MLP output for receiver j, component comp
__global__ void k_cond_global64(CondDev c, const double* __restrict__ rx, int n_rx, double* __restrict__ ag) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_rx * c.L) return;
    const int j = t / c.L, comp = t % c.L;
    const double* p = c.p64;
    double in[kMaxGin64];
    const int F = c.F;
    for (int a = 0; a < 3; ++a)  // fourier_encode
        for (int band = 0; band < F; ++band) {
            const double arg = p[c.o_freq + band * 3 + a] * rx[3 * static_cast<size_t>(j) + a];
            in[(a * F + band) * 2] = sin(arg);
            in[(a * F + band) * 2 + 1] = cos(arg);
        }
    int l_max = 0;
    while ((l_max + 1) * (l_max + 1) < c.L) ++l_max;
    const double den = l_max > 0 ? static_cast<double>(l_max) : 1.0;
    int l = 0;
    while ((l + 1) * (l + 1) <= comp) ++l;
    in[6 * F] = l / den;
    in[6 * F + 1] = (comp - l * l - l) / den;
    for (int e = 0; e < c.dc; ++e) in[6 * F + 2 + e] = p[c.o_emb + comp * c.dc + e];
    double y[4 * kCMax];
    const int NY = 4 * c.C;
    mlp64<kMaxHidden64>(p, c.o_gw1, c.o_gb1, c.o_gw2, c.o_gb2, c.o_gw3, c.o_gb3, c.gin, c.H, NY, in, y);
    for (int o = 0; o < NY; ++o) ag[static_cast<size_t>(t) * NY + o] = y[o];
}

// out[j][k][l][c][2] = the conditioned coefficients (conditioning.cpp:365-421)
__global__ void k_cond_forward64(CondDev c, Occ64 g, int K, const double* __restrict__ pos,
                                 const double* __restrict__ rx, int n_rx, const double* __restrict__ base,
                                 const double* __restrict__ ag, double* __restrict__ out,
                                 double* __restrict__ local_in) {
    const long long row = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (row >= static_cast<long long>(K) * n_rx) return;
    const int j = static_cast<int>(row / K), k = static_cast<int>(row % K);
    const int C = c.C, L = c.L, NY = 4 * C;
    double y[4 * kCMax];
    if (c.use_local) {
        const double* p = pos + 3 * static_cast<size_t>(k);
        const double* r = rx + 3 * static_cast<size_t>(j);
        const double dx = r[0] - p[0], dy = r[1] - p[1], dz = r[2] - p[2];  // Vec3 diff = rx - p
        const double d = sqrt(dx * dx + dy * dy + dz * dz);
        double in[6] = {dx / d, dy / d, dz / d, d, 1.0, 0.0};
        if (c.probe) probe64(g, p, r, c.S, c.nearest != 0, &in[4], &in[5]);
        mlp64<kMaxHidden64>(c.p64, c.o_lw1, c.o_lb1, c.o_lw2, c.o_lb2, c.o_lw3, c.o_lb3, 6, c.H, NY, in, y);
        if (local_in && j == 0)
            for (int i = 0; i < 6; ++i) local_in[static_cast<size_t>(k) * 6 + i] = in[i];
    }
    const size_t stride = static_cast<size_t>(L) * C * 2;
    for (int comp = 0; comp < L; ++comp)
        for (int ch = 0; ch < C; ++ch) {
            const size_t idx = static_cast<size_t>(k) * stride + (static_cast<size_t>(comp) * C + ch) * 2;
            const double zr = base[idx], zi = base[idx + 1];
            double mr = zr, mi = zi;
            if (c.use_global) {
                const double* a = ag + (static_cast<size_t>(j) * L + comp) * NY + 4 * ch;
                const double ar = c.additive ? 0.0 : a[0], ai = c.additive ? 0.0 : a[1];
                mr = zr + (ar * zr - ai * zi + a[2]);
                mi = zi + (ai * zr + ar * zi + a[3]);
            }
            double orr = mr, oi = mi;
            if (c.use_local) {
                const double ar = c.additive ? 0.0 : y[4 * ch], ai = c.additive ? 0.0 : y[4 * ch + 1];
                orr = mr + (ar * mr - ai * mi + y[4 * ch + 2]);
                oi = mi + (ai * mr + ar * mi + y[4 * ch + 3]);
            }
            const size_t o = static_cast<size_t>(j) * K * stride + idx;
            out[o] = orr;
            out[o + 1] = oi;
        }
}

// ---- materialised render_field in FP64 (sphraster.cpp:190-315)
__device__ __forceinline__ double wrap_pm_pi64(double a) {  // linalg.hpp:152-157
    if (!(fabs(a) < kTwoPi)) a = fmod(a, kTwoPi);  // fmod returns a exactly below 2 pi
    if (a > kPi) a -= kTwoPi;
    if (a <= -kPi) a += kTwoPi;
    return a;
}

// s[(k * n_rx + j) * C + c] = sum_comp cplx{a, b} * basis (reduce_signals)
__global__ void k_reduce_signals64(int K, int L, int C, int n_rx, const int* __restrict__ culled,
                                   const double* __restrict__ basis64, const double* __restrict__ co,
                                   double2* __restrict__ sig) {
    const long long row = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (row >= static_cast<long long>(K) * n_rx) return;
    const int k = static_cast<int>(row / n_rx), j = static_cast<int>(row % n_rx);
    const size_t stride = static_cast<size_t>(L) * C * 2;
    const double* cb = co + (static_cast<size_t>(j) * K + k) * stride;
    const double* b = basis64 + static_cast<size_t>(k) * L * 2;
    for (int ch = 0; ch < C; ++ch) {
        double sr = 0.0, si = 0.0;
        if (!culled[k])
            for (int l = 0; l < L; ++l) {
                const double a = cb[(l * C + ch) * 2], bb = cb[(l * C + ch) * 2 + 1];
                sr += a * b[2 * l] - bb * b[2 * l + 1];
                si += a * b[2 * l + 1] + bb * b[2 * l];
            }
        sig[(static_cast<size_t>(k) * n_rx + j) * C + ch] = make_double2(sr, si);
    }
}

// One thread per (receiver, cell): the reference's per-cell front-to-back
// walk (gaussian_weight, min(w, 0.999), contribute, update T, exit below 1e-4).
__global__ void k_render64(DevGrid g, int n_rx, int C, const GaussRec* __restrict__ rec,
                           const int64_t* __restrict__ offsets, const int* __restrict__ list,
                           const double2* __restrict__ sig, double* __restrict__ values, double* __restrict__ tout) {
    const size_t plane = static_cast<size_t>(g.nt) * g.np;
    const long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (t >= static_cast<long long>(n_rx) * plane) return;
    const int j = static_cast<int>(t / plane);
    const size_t cell = static_cast<size_t>(t % plane);
    const int row = static_cast<int>(cell / g.np), col = static_cast<int>(cell % g.np);
    const int tile = (row / g.ts) * g.tiles_p + col / g.ts;
    const double theta_r = g.tmin + (row + 0.5) * g.dth;  // SphericalGrid::theta_at
    const double phi_r = (col + 0.5) * g.dph;             // phi_at
    double ar[kCMax], ai[kCMax];
    for (int c = 0; c < C; ++c) ar[c] = ai[c] = 0.0;
    double T = 1.0;
    for (int64_t p = offsets[tile]; p < offsets[tile + 1]; ++p) {
        const int k = list[p];
        const GaussRec r = rec[k];
        const double dt = theta_r - r.theta;
        const double dpraw = wrap_pm_pi64(phi_r - r.phi);
        const double dp = r.sin_theta * dpraw;
        const double m2 = r.pa * dt * dt + r.pbc * dt * dp + r.pd * dp * dp;
        double w = r.tau * exp(-0.5 * m2);
        w = 0.999 < w ? 0.999 : w;  // std::min(w, kWeightClamp)
        const double tw = T * w;
        const double2* s = sig + (static_cast<size_t>(k) * n_rx + j) * C;
        for (int c = 0; c < C; ++c) {
            ar[c] += tw * s[c].x;
            ai[c] += tw * s[c].y;
        }
        T *= 1.0 - w;
        if (T < 1e-4) break;
    }
    for (int c = 0; c < C; ++c) {
        const size_t base = (static_cast<size_t>(j) * C + c) * 2 * plane;
        values[base + cell] = ar[c];
        values[base + plane + cell] = ai[c];
    }
    if (tout) tout[static_cast<size_t>(j) * plane + cell] = T;
}

Occ64 make_occ64(const rxgs_cond_s* c, const double* dens, int R, const double* lo, const double* hi) {
    Occ64 g{};
    g.dens = dens;
    g.R = R;
    for (int a = 0; a < 3; ++a) {
        g.lo[a] = lo[a];
        g.ext[a] = hi[a] - lo[a];  // Aabb::extent
    }
    (void)c;
    return g;
}

}  // namespace

cudaError_t launch_render64(const rxgs_txstate_s& st, const double* d_co, int n_rx, double2* d_sig, double* values,
                            double* tout, cudaStream_t s) {
    const long long rows = static_cast<long long>(st.k) * n_rx;
    if (rows > 0)
        k_reduce_signals64<<<static_cast<unsigned>((rows + 255) / 256), 256, 0, s>>>(
            st.k, st.L, st.channels, n_rx, st.culled.as<int>(), st.basis64.as<double>(), d_co, d_sig);
    const long long t = static_cast<long long>(n_rx) * st.grid.nt * st.grid.np;
    if (t > 0)
        k_render64<<<static_cast<unsigned>((t + 127) / 128), 128, 0, s>>>(st.grid, n_rx, st.channels,
                                                                          st.rec.as<GaussRec>(),
                                                                          st.tile_offsets.as<int64_t>(),
                                                                          st.list.as<int>(), d_sig, values, tout);
    return cudaGetLastError();
}

cudaError_t launch_blend_ray(int n, const double* w, const double* sig, double* out, cudaStream_t s) {
    k_blend_ray<<<1, 1, 0, s>>>(n, w, sig, out);
    return cudaGetLastError();
}

cudaError_t launch_occ_sample(int R, const double* lo, const double* hi, const double* dens, int n, const double* pts,
                              int nearest, double* out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_occ_sample<<<(n + 127) / 128, 128, 0, s>>>(make_occ64(nullptr, dens, R, lo, hi), n, pts, nearest, out);
    return cudaGetLastError();
}

cudaError_t launch_probe64(int R, const double* lo, const double* hi, const double* dens, int n, const double* from,
                           const double* to, int samples, int nearest, double* out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_probe64<<<(n + 127) / 128, 128, 0, s>>>(make_occ64(nullptr, dens, R, lo, hi), n, from, to, samples, nearest,
                                              out);
    return cudaGetLastError();
}

cudaError_t launch_fourier64(int F, const double* freqs, int n, const double* r, double* out, cudaStream_t s) {
    const int t = n * 3 * F;
    if (t == 0) return cudaSuccess;
    k_fourier64<<<(t + 127) / 128, 128, 0, s>>>(F, freqs, n, r, out);
    return cudaGetLastError();
}

cudaError_t launch_mlp_layer64(int in, int nout, const double* w, const double* b, int n, const double* x, double* y,
                               cudaStream_t s) {
    const int t = n * nout;
    if (t == 0) return cudaSuccess;
    k_mlp_layer64<<<(t + 127) / 128, 128, 0, s>>>(in, nout, w, b, n, x, y);
    return cudaGetLastError();
}

cudaError_t launch_cond_forward64(const rxgs_cond_s& c, const rxgs_scene_s& sc, const double* d_rx, int n_rx,
                                  const double* base, double* ag64, double* out, double* local_in, cudaStream_t s) {
    if (c.hidden > kMaxHidden64 || c.gin > kMaxGin64 || c.C > kCMax) return cudaErrorInvalidValue;
    CondDev d = make_dev(c);
    if (c.use_global() && n_rx * c.L > 0)
        k_cond_global64<<<(n_rx * c.L + 63) / 64, 64, 0, s>>>(d, d_rx, n_rx, ag64);
    const long long rows = static_cast<long long>(sc.k) * n_rx;
    if (rows == 0) return cudaGetLastError();
    const Occ64 g = make_occ64(&c, c.has_occ ? c.d_occ64.as<double>() : nullptr, c.R, c.lo, c.hi);
    k_cond_forward64<<<static_cast<unsigned>((rows + 127) / 128), 128, 0, s>>>(
        d, g, sc.k, sc.d_pos.as<double>(), d_rx, n_rx, base, ag64, out, local_in);
    return cudaGetLastError();
}

}  // namespace rxgs_b200
