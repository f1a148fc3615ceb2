// Exact adjoints of the render path in FP64 (the materialised API):
//   aggregate_modality_backward (sphraster.cpp:383-449)      -> k_aggregate_bwd
//   backward_render             (sphraster.cpp:509-733)      -> k_bwd_walk,
//                                                               k_bwd_gauss_reduce,
//                                                               k_bwd_finalize
// The reference re-walks every cell and runs a reverse pass with per-(rx, c)
// suffix sums.  Here the suffix is obtained in a second FORWARD walk as
// suffix(pos) = C_total - C_upto(pos) (C_total from a first walk), so no per
// cell walk history is stored; both walks are FP64 with the reference's
// operation order for w and T (same early exit).  Per-entry contributions are
// reduced over the tile's cells in a fixed tree, regrouped per Gaussian in
// tile order (no floating-point atomics), then the per-Gaussian geometry
// chain (basis jet, precision -> covariance -> scale/quaternion, frame and
// depth terms, tau logit) runs one thread per Gaussian.
#include "rxgs_internal.cuh"

namespace rxgs_b200 {
namespace {

#ifndef RXGS_BWD_NC
#define RXGS_BWD_NC 4  // A/B (2, 4, 8) on the joint step: 4 (with the reduce-scatter: 4 = 5.8 ms, 8 = 6.4 ms, 195 registers)
#endif
constexpr int kNC = RXGS_BWD_NC;  // (receiver, channel) pairs per walk pass (one receiver chunk)

__device__ __forceinline__ double wrap_pm_pi(double a) {  // linalg.hpp:152-157
    // fmod(a, 2 pi) returns a exactly when |a| < 2 pi (always, for two
    // azimuths in [0, 2 pi)): the software FP64 fmod is skipped there
    if (!(fabs(a) < kTwoPi)) a = fmod(a, kTwoPi);
    if (a > kPi) a -= kTwoPi;
    if (a <= -kPi) a += kTwoPi;
    return a;
}

// ------------------------------------------------------------------ aggregate adjoint
__global__ void k_aggregate_bwd(DevGrid g, int modality, int n_rx, int C, const double* __restrict__ values,
                                const double* __restrict__ up, double* __restrict__ dv) {
    __shared__ double red[256];
    const int jc = blockIdx.x, j = jc / C, ch = jc % C;
    const size_t plane = static_cast<size_t>(g.nt) * g.np;
    const double* re_p = values + (static_cast<size_t>(j) * C + ch) * 2 * plane;
    const double* im_p = re_p + plane;
    double* dre = dv + (static_cast<size_t>(j) * C + ch) * 2 * plane;
    double* dim = dre + plane;
    if (modality == 0) {  // rssi: d = up * 10 / (ln 10 (power + floor))
        double pw = 0.0;
        for (size_t cell = threadIdx.x; cell < plane; cell += blockDim.x) {
            const int row = static_cast<int>(cell / g.np);
            const double dom = sin(g.tmin + (row + 0.5) * g.dth) * g.dth * g.dph;
            pw += (re_p[cell] * re_p[cell] + im_p[cell] * im_p[cell]) * dom;
        }
        red[threadIdx.x] = pw;
        __syncthreads();
        for (int s = blockDim.x / 2; s > 0; s >>= 1) {
            if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
            __syncthreads();
        }
        const double d_power = up[j] * 10.0 / (log(10.0) * (red[0] + kRssiFloor));
        for (size_t cell = threadIdx.x; cell < plane; cell += blockDim.x) {
            const int row = static_cast<int>(cell / g.np);
            const double dom = sin(g.tmin + (row + 0.5) * g.dth) * g.dth * g.dph;
            dre[cell] = d_power * 2.0 * re_p[cell] * dom;
            dim[cell] = d_power * 2.0 * im_p[cell] * dom;
        }
    } else if (modality == 1) {  // csi: d = conj-free complex upstream * dOmega
        const double gr = up[(static_cast<size_t>(j) * C + ch) * 2], gi = up[(static_cast<size_t>(j) * C + ch) * 2 + 1];
        for (size_t cell = threadIdx.x; cell < plane; cell += blockDim.x) {
            const int row = static_cast<int>(cell / g.np);
            const double dom = sin(g.tmin + (row + 0.5) * g.dth) * g.dth * g.dph;
            dre[cell] = gr * dom;
            dim[cell] = gi * dom;
        }
    } else {  // spectrum: d = up * re / amp
        for (size_t cell = threadIdx.x; cell < plane; cell += blockDim.x) {
            const double re = re_p[cell], im = im_p[cell];
            const double amp = sqrt(re * re + im * im + kAmpEps);
            const double u = up[static_cast<size_t>(j) * plane + cell];
            dre[cell] = u * re / amp;
            dim[cell] = u * im / amp;
        }
    }
}

// ------------------------------------------------------------------ signals in FP64
// rows: all K x n_rx (rows == nullptr) or the state's needed Gaussians only
// (the re-walk reads the signals of walked entries, all among them)
__global__ void k_signals64(int K, int L, int C, int n_rx, const int* __restrict__ culled,
                            const double* __restrict__ basis64, const double* __restrict__ co, double2* __restrict__ sig,
                            const int* __restrict__ rows, const int* __restrict__ n_rows) {
    const long long row = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    const long long n_k = rows ? *n_rows : K;
    if (row >= n_k * n_rx) return;
    const int k = rows ? rows[row / n_rx] : static_cast<int>(row / n_rx), j = static_cast<int>(row % n_rx);
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

// One halving step of a warp reduce-scatter: lanes with bit `off` clear keep
// the low half of the N values, the others the high half, each adding its
// partner's copy of the half it keeps.
template <int N>
__device__ __forceinline__ void rs_step(const double (&in)[N], double (&out)[N / 2], int wl, int off) {
    const bool up = (wl & off) != 0;
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
        const double lo = in[i], hi = in[i + N / 2];
        out[i] = (up ? hi : lo) + __shfl_xor_sync(0xffffffffu, up ? lo : hi, off);
    }
}
// kV <= 16 values: 8 + 4 + 2 + 1 exchanges, then lanes l and l^1 add (both
// hold value 8 b4 + 4 b3 + 2 b2 + b1 of their lane index)
template <int kV>
__device__ __forceinline__ double reduce_scatter16(const double* v, int wl) {
    double a[16], b[8], c[4], d[2];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = i < kV ? v[i] : 0.0;
    rs_step<16>(a, b, wl, 16);
    rs_step<8>(b, c, wl, 8);
    rs_step<4>(c, d, wl, 4);
    const bool up2 = (wl & 2) != 0;
    double h = (up2 ? d[1] : d[0]) + __shfl_xor_sync(0xffffffffu, up2 ? d[0] : d[1], 2);
    return h + __shfl_xor_sync(0xffffffffu, h, 1);
}
// kV <= 32 values: 16 + 8 + 4 + 2 + 1 exchanges; lane l holds value
// 16 b4 + 8 b3 + 4 b2 + 2 b1 + b0
template <int kV>
__device__ __forceinline__ double reduce_scatter32(const double* v, int wl) {
    double a[32], b[16], c[8], d[4], e[2];
#pragma unroll
    for (int i = 0; i < 32; ++i) a[i] = i < kV ? v[i] : 0.0;
    rs_step<32>(a, b, wl, 16);
    rs_step<16>(b, c, wl, 8);
    rs_step<8>(c, d, wl, 4);
    rs_step<4>(d, e, wl, 2);
    const bool up1 = (wl & 1) != 0;
    return (up1 ? e[1] : e[0]) + __shfl_xor_sync(0xffffffffu, up1 ? e[0] : e[1], 1);
}

// ------------------------------------------------------------------ per-cell walks
// One CTA per (tile, 64-cell block).  jc0..jc0+nc are the (receiver, channel)
// pairs of this pass; entry records are zeroed beforehand and accumulated
// (geometry terms are linear in dw, so passes and cell blocks add).
// ent_geo[e] = d_tau_act, d_prec (a, b, c, d), d_theta, d_phi;
// ent_ds[e][jc] = d signal.  Blocks of one tile run in launch order on the
// same stream (blockIdx.y outer launches), so the sums are deterministic.
__global__ void __launch_bounds__(64) k_bwd_walk(DevGrid g, int cb, const int64_t* __restrict__ tile_offsets,
                                                 const int* __restrict__ list, const GaussRec* __restrict__ rec,
                                                 const int* __restrict__ walk_len, const double2* __restrict__ sig,
                                                 int n_jc, const double* __restrict__ dvals, int64_t n_ent,
                                                 double* __restrict__ ent_geo, double2* __restrict__ ent_ds) {
    constexpr int kV = 7 + 2 * kNC;
    // per-warp block sums of the last 32 positions, flushed to the entry
    // records 32 positions at a time by all threads (red[0] + red[1], then
    // accumulated: the order of the former per-position flush)
    __shared__ double ring[2][32][kV];
    // the walk records and this chunk's signals of 64 list positions, staged
    // cooperatively (every cell of the block reads the same entries)
    constexpr int kStage = 64;
    __shared__ GaussRec srec[kStage];
    __shared__ double2 ssig[kStage][kNC];
    const int tile = blockIdx.x, lane = threadIdx.x;
    // receiver chunk blockIdx.y: its own slice of the per-entry geometry sums
    const int jc0 = blockIdx.y * kNC, nc = n_jc - jc0 < kNC ? n_jc - jc0 : kNC;
    ent_geo += static_cast<size_t>(blockIdx.y) * n_ent * 7;
    const int tt = tile / g.tiles_p, tp = tile % g.tiles_p;
    const int lc = cb * kMaxCellsPerBlock + lane;
    const int row = tt * g.ts + lc / g.ts, col = tp * g.ts + lc % g.ts;
    const bool valid = lc < g.cpt && row < g.nt && col < g.np;
    const int64_t begin = tile_offsets[tile];
    const int W = walk_len[tile * g.cell_blocks + cb];
    const size_t plane = static_cast<size_t>(g.nt) * g.np;
    const size_t cell = valid ? static_cast<size_t>(row) * g.np + col : 0;
    const double theta_r = valid ? g.tmin + (row + 0.5) * g.dth : 0.0;
    const double phi_r = valid ? (col + 0.5) * g.dph : 0.0;
    double gre[kNC], gim[kNC], Cr[kNC], Ci[kNC];
#pragma unroll
    for (int q = 0; q < kNC; ++q) {
        gre[q] = gim[q] = Cr[q] = Ci[q] = 0.0;
        if (valid && q < nc) {
            const int jc = jc0 + q;  // values index [j][c][re/im][cell]
            gre[q] = dvals[static_cast<size_t>(jc) * 2 * plane + cell];
            gim[q] = dvals[static_cast<size_t>(jc) * 2 * plane + plane + cell];
        }
    }
    auto stage_chunk = [&](int c0) {  // positions c0 .. c0 + 63 -> srec / ssig
        __syncthreads();  // the previous chunk has been consumed
        if (c0 + lane < W) {
            const int k = list[begin + c0 + lane];
            srec[lane] = rec[k];
#pragma unroll
            for (int q = 0; q < kNC; ++q)
                ssig[lane][q] = q < nc ? sig[static_cast<size_t>(k) * n_jc + jc0 + q] : make_double2(0.0, 0.0);
        }
        __syncthreads();
    };
    // pass 1: C_total (forward walk, identical exit)
    int len = 0;
    {
        double T = 1.0;
        bool alive = valid;
        for (int c0 = 0; c0 < W; c0 += kStage) {
            if (!__syncthreads_or(alive)) break;
            stage_chunk(c0);
            const int m = W - c0 < kStage ? W - c0 : kStage;
            for (int e = 0; e < m && alive; ++e) {
                const GaussRec& r = srec[e];
                const double dt = theta_r - r.theta;
                const double dpraw = wrap_pm_pi(phi_r - r.phi);
                const double dp = r.sin_theta * dpraw;
                const double m2 = r.pa * dt * dt + r.pbc * dt * dp + r.pd * dp * dp;
                double w = r.tau * exp(-0.5 * m2);
                w = kWeightClamp < w ? kWeightClamp : w;
                const double tw = T * w;
#pragma unroll
                for (int q = 0; q < kNC; ++q)
                    if (q < nc) {
                        const double2 sv = ssig[e][q];
                        Cr[q] += tw * sv.x;
                        Ci[q] += tw * sv.y;
                    }
                T *= 1.0 - w;
                len = c0 + e + 1;
                if (T < kEarlyExitT) alive = false;
            }
        }
    }
    // pass 2: per-entry adjoints with suffix = C_total - C_upto(p), reduced
    // over the block's cells per position in a fixed tree
    double T = 1.0;
    double Ur[kNC], Ui[kNC];
#pragma unroll
    for (int q = 0; q < kNC; ++q) Ur[q] = Ui[q] = 0.0;
    const int warp = lane >> 5, wl = lane & 31;
    for (int c0 = 0; c0 < W; c0 += kStage) {
    stage_chunk(c0);
    const int m_ch = W - c0 < kStage ? W - c0 : kStage;
    for (int e = 0; e < m_ch; ++e) {
        const int p = c0 + e;
        double v[7 + 2 * kNC];
#pragma unroll
        for (int i = 0; i < 7 + 2 * kNC; ++i) v[i] = 0.0;
        if (p < len) {
            const GaussRec& r = srec[e];
            const double dt = theta_r - r.theta;
            const double dpraw = wrap_pm_pi(phi_r - r.phi);
            const double dp = r.sin_theta * dpraw;
            const double m2 = r.pa * dt * dt + r.pbc * dt * dp + r.pd * dp * dp;
            const double w_raw = r.tau * exp(-0.5 * m2);
            const bool clamped = w_raw > kWeightClamp;
            const double w = clamped ? kWeightClamp : w_raw;
            const double gg = r.tau > 0.0 ? w_raw / r.tau : 0.0;
            const double t_prev = T;
            const double inv_rest = 1.0 / (1.0 - w);
            double dw = 0.0;
#pragma unroll
            for (int q = 0; q < kNC; ++q)
                if (q < nc) {
                    const double2 s = ssig[e][q];
                    v[7 + 2 * q] = gre[q] * t_prev * w;
                    v[8 + 2 * q] = gim[q] * t_prev * w;
                    Ur[q] += t_prev * w * s.x;
                    Ui[q] += t_prev * w * s.y;
                    const double sr = Cr[q] - Ur[q], si = Ci[q] - Ui[q];  // beyond this entry
                    dw += gre[q] * (t_prev * s.x - sr * inv_rest);
                    dw += gim[q] * (t_prev * s.y - si * inv_rest);
                }
            T = t_prev * (1.0 - w);
            if (!clamped) {
                const double dm2 = dw * r.tau * (-0.5) * gg;
                const double st = r.sin_theta, ct = r.cos_theta;  // = cos(theta), computed once in k_tx_prep
                v[0] = dw * gg;
                v[1] = dm2 * dt * dt;
                v[2] = dm2 * dt * dp;
                v[3] = dm2 * dt * dp;
                v[4] = dm2 * dp * dp;
                const double d_dt = dm2 * (2.0 * r.pa * dt + r.pbc * dp);
                const double d_dp = dm2 * (r.pbc * dt + 2.0 * r.pd * dp);
                v[5] = -d_dt + d_dp * ct * dpraw;
                v[6] = -d_dp * st;
            }
        }
        // reduce-scatter of the kV values by recursive halving (VP/2 + ... + 1
        // exchanges; for VP = 16 a final pair add): lane l ends with the warp sum
        // of value rs_index(l); fixed order
        if constexpr (kV <= 16) {
            const double h1 = reduce_scatter16<kV>(v, wl);
            const int idx = 8 * ((wl >> 4) & 1) + 4 * ((wl >> 3) & 1) + 2 * ((wl >> 2) & 1) + ((wl >> 1) & 1);
            if ((wl & 1) == 0 && idx < 7 + 2 * nc) ring[warp][p & 31][idx] = h1;
        } else {
            const double h1 = reduce_scatter32<kV>(v, wl);
            const int idx = 16 * ((wl >> 4) & 1) + 8 * ((wl >> 3) & 1) + 4 * ((wl >> 2) & 1) + 2 * ((wl >> 1) & 1) +
                            (wl & 1);
            if (idx < 7 + 2 * nc) ring[warp][p & 31][idx] = h1;
        }
        if ((p & 31) == 31 || p == W - 1) {
            __syncthreads();
            const int p0 = p & ~31, np = p - p0 + 1, nv = 7 + 2 * nc;
            for (int idx = lane; idx < np * nv; idx += 64) {
                const int pp = idx / nv, i = idx % nv;
                const int64_t e = begin + p0 + pp;
                const double x = ring[0][pp][i] + ring[1][pp][i];
                double* dst = i < 7 ? ent_geo + e * 7 + i
                                    : reinterpret_cast<double*>(ent_ds) + (e * n_jc + jc0 + (i - 7) / 2) * 2 + (i - 7) % 2;
                *dst += x;
            }
            __syncthreads();
        }
    }
    }
}

// per-Gaussian sums of the walked entries, in tile order
// One thread per (Gaussian, output value): the 7 geometry terms (receiver
// chunks summed in order per entry) and the n_jc signal adjoints, each summed
// over the Gaussian's entries in tile order -- the same per-value order as one
// thread per Gaussian, with 7 + n_jc times the parallelism for the gathers.
__global__ void k_bwd_gauss_reduce(int K, int n_jc, int n_chunks, int64_t n_ent, const int* __restrict__ goff,
                                   const int* __restrict__ gent, const double* __restrict__ ent_geo,
                                   const double2* __restrict__ ent_ds, double* __restrict__ raw_geo,
                                   double2* __restrict__ raw_ds) {
    const int nv = 7 + n_jc;
    const long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (t >= static_cast<long long>(K) * nv) return;
    const int k = static_cast<int>(t / nv), i = static_cast<int>(t - static_cast<long long>(k) * nv);
    const int e0 = goff[k], e1 = goff[k + 1];
    if (i < 7) {
        double acc = 0.0;
        for (int e = e0; e < e1; ++e) {
            const int ge = gent[e];
            double v = ent_geo[static_cast<size_t>(ge) * 7 + i];  // receiver chunks in order
            for (int ch = 1; ch < n_chunks; ++ch) v += ent_geo[(static_cast<size_t>(ch) * n_ent + ge) * 7 + i];
            acc += v;
        }
        raw_geo[static_cast<size_t>(k) * 7 + i] = acc;
    } else {
        const int q = i - 7;
        double2 a = make_double2(0.0, 0.0);
        for (int e = e0; e < e1; ++e) {
            const double2 v = ent_ds[static_cast<size_t>(gent[e]) * n_jc + q];
            a.x += v.x;
            a.y += v.y;
        }
        raw_ds[static_cast<size_t>(k) * n_jc + q] = a;
    }
}

__device__ __forceinline__ double normalization(int l, int am) {  // radiance.cpp:9-14
    double ratio = 1.0;
    for (int i = l - am + 1; i <= l + am; ++i) ratio /= static_cast<double>(i);
    return sqrt((2.0 * l + 1.0) / (4.0 * kPi) * ratio);
}

// Per-Gaussian finalisation (sphraster.cpp:615-731).  LT > 0: l_max == LT
// at compile time -- the Legendre tables stay in registers and each
// component's basis derivatives (normalization, cos / sin of m phi) are
// formed once per Gaussian instead of once per receiver; the same
// expressions in the same order, so the results are bit-identical.
template <int LT>
__global__ void k_bwd_finalize(int K, int l_max_rt, int C, int n_rx, const int* __restrict__ culled,
                               const double* __restrict__ geom, const double* __restrict__ basis64,
                               const double* __restrict__ coeffs, const double* __restrict__ raw_geo,
                               const double2* __restrict__ raw_ds, const double* __restrict__ ls,
                               const double* __restrict__ quat, double* __restrict__ d_pos, double* __restrict__ d_ls,
                               double* __restrict__ d_q, double* __restrict__ d_tau, double* __restrict__ d_coeffs) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    const int l_max = LT > 0 ? LT : l_max_rt;
    const int L = (l_max + 1) * (l_max + 1);
    for (int a = 0; a < 3; ++a) d_pos[3 * k + a] = d_ls[3 * k + a] = 0.0;
    for (int a = 0; a < 4; ++a) d_q[4 * k + a] = 0.0;
    d_tau[k] = 0.0;
    const size_t stride = static_cast<size_t>(L) * C * 2;
    if (d_coeffs)
        for (int j = 0; j < n_rx; ++j)
            for (size_t i = 0; i < stride; ++i) d_coeffs[(static_cast<size_t>(j) * K + k) * stride + i] = 0.0;
    if (culled[k]) return;
    const double* gm = geom + 12 * static_cast<size_t>(k);
    const double theta = gm[0], phi = gm[1], depth = gm[2];
    const double* rg = raw_geo + 7 * static_cast<size_t>(k);
    double d_theta = rg[5], d_phi = rg[6];

    // ---- basis jet (radiance.cpp:39-77, 94-114) and coefficient gradients
    constexpr int kPT = LT > 0 ? (LT + 1) * (LT + 2) / 2 : (kMaxLmax + 1) * (kMaxLmax + 2) / 2;
    double P[kPT], D[kPT];
    {
        const double x = cos(theta), s = sin(theta);
#define AT(l, m) P[(l) * ((l) + 1) / 2 + (m)]
#define DAT(l, m) D[(l) * ((l) + 1) / 2 + (m)]
        AT(0, 0) = 1.0;
        DAT(0, 0) = 0.0;
        for (int m = 1; m <= l_max; ++m) {
            const double c = 2.0 * m - 1.0;
            AT(m, m) = AT(m - 1, m - 1) * c * s;
            DAT(m, m) = c * (DAT(m - 1, m - 1) * s + AT(m - 1, m - 1) * x);
        }
        for (int m = 0; m < l_max; ++m) {
            const double c = 2.0 * m + 1.0;
            AT(m + 1, m) = x * c * AT(m, m);
            DAT(m + 1, m) = c * (-s * AT(m, m) + x * DAT(m, m));
        }
        for (int m = 0; m <= l_max; ++m)
            for (int l = m + 2; l <= l_max; ++l) {
                const double a = 2.0 * l - 1.0, b = l + m - 1.0, inv = 1.0 / (l - m);
                AT(l, m) = (x * a * AT(l - 1, m) - b * AT(l - 2, m)) * inv;
                DAT(l, m) = (a * (-s * AT(l - 1, m) + x * DAT(l - 1, m)) - b * DAT(l - 2, m)) * inv;
            }
    }
    const double* B = basis64 + static_cast<size_t>(k) * L * 2;
    if constexpr (LT > 0) {
        constexpr int LL = (LT + 1) * (LT + 1);
        double tb[LL][4];  // per component: d/dtheta (re, im) and d/dphi (re, im) of the basis
#pragma unroll
        for (int l = 0; l <= LT; ++l)
#pragma unroll
            for (int m = -l; m <= l; ++m) {
                const int comp = l * l + m + l, am = m < 0 ? -m : m;
                const double nrm = normalization(l, am);
                const double cm = cos(m * phi), sm = sin(m * phi);
                const double dth = nrm * DAT(l, am);
                const double bre = nrm * AT(l, am) * cm, bim = nrm * AT(l, am) * sm;
                tb[comp][0] = dth * cm;
                tb[comp][1] = dth * sm;
                tb[comp][2] = -m * bim;
                tb[comp][3] = m * bre;
            }
        for (int j = 0; j < n_rx; ++j)
            for (int c = 0; c < C; ++c) {
                const double2 ds = raw_ds[(static_cast<size_t>(k) * n_rx + j) * C + c];
                if (ds.x == 0.0 && ds.y == 0.0) continue;
                const size_t cbase = (static_cast<size_t>(j) * K + k) * stride;
#pragma unroll
                for (int comp = 0; comp < LL; ++comp) {
                    const size_t ci = cbase + (static_cast<size_t>(comp) * C + c) * 2;
                    const double br = B[2 * comp], bi = B[2 * comp + 1];
                    if (d_coeffs) {
                        d_coeffs[ci] += ds.x * br + ds.y * bi;
                        d_coeffs[ci + 1] += -ds.x * bi + ds.y * br;
                    }
                    const double a_co = coeffs[ci], b_co = coeffs[ci + 1];
                    const double db_re = ds.x * a_co + ds.y * b_co;
                    const double db_im = -ds.x * b_co + ds.y * a_co;
                    d_theta += db_re * tb[comp][0] + db_im * tb[comp][1];
                    d_phi += db_re * tb[comp][2] + db_im * tb[comp][3];
                }
            }
    } else
    for (int j = 0; j < n_rx; ++j)
        for (int c = 0; c < C; ++c) {
            const double2 ds = raw_ds[(static_cast<size_t>(k) * n_rx + j) * C + c];
            if (ds.x == 0.0 && ds.y == 0.0) continue;
            const size_t cbase = (static_cast<size_t>(j) * K + k) * stride;
            for (int l = 0; l <= l_max; ++l)
                for (int m = -l; m <= l; ++m) {
                    const int comp = l * l + m + l, am = m < 0 ? -m : m;
                    const size_t ci = cbase + (static_cast<size_t>(comp) * C + c) * 2;
                    const double br = B[2 * comp], bi = B[2 * comp + 1];
                    if (d_coeffs) {
                        d_coeffs[ci] += ds.x * br + ds.y * bi;
                        d_coeffs[ci + 1] += -ds.x * bi + ds.y * br;
                    }
                    const double a_co = coeffs[ci], b_co = coeffs[ci + 1];
                    const double db_re = ds.x * a_co + ds.y * b_co;
                    const double db_im = -ds.x * b_co + ds.y * a_co;
                    const double nrm = normalization(l, am);
                    const double cm = cos(m * phi), sm = sin(m * phi);
                    const double dth = nrm * DAT(l, am);  // d/dtheta of N P e^{jm phi} = nrm dP (cm, sm)
                    const double bth_re = dth * cm, bth_im = dth * sm;
                    const double bre = nrm * AT(l, am) * cm, bim = nrm * AT(l, am) * sm;
                    const double bph_re = -m * bim, bph_im = m * bre;  // j m B
                    d_theta += db_re * bth_re + db_im * bth_im;
                    d_phi += db_re * bph_re + db_im * bph_im;
                }
        }
#undef AT
#undef DAT
    // ---- precision -> covariance: dA = -P dP P
    const double pa = gm[7], pb = gm[8], pc = gm[9], pd = gm[10];
    const double qa = rg[1], qb = rg[2], qc = rg[3], qd = rg[4];
    // t = P dP
    const double t_a = pa * qa + pb * qc, t_b = pa * qb + pb * qd, t_c = pc * qa + pd * qc, t_d = pc * qb + pd * qd;
    const double da[2][2] = {{-(t_a * pa + t_b * pc), -(t_a * pb + t_b * pd)},
                             {-(t_c * pa + t_d * pc), -(t_c * pb + t_d * pd)}};
    const double st = sin(theta), ct = cos(theta), sp = sin(phi), cp = cos(phi);
    const double et[3] = {ct * cp, ct * sp, -st};
    const double ep[3] = {-sp, cp, 0.0};
    const double uh[3] = {st * cp, st * sp, ct};
    const double inv_d2 = 1.0 / (depth * depth);
    const double* frame[2] = {et, ep};
    double dsig[9];
    for (int i = 0; i < 9; ++i) dsig[i] = 0.0;
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
            for (int r = 0; r < 3; ++r)
                for (int c2 = 0; c2 < 3; ++c2) dsig[r * 3 + c2] += da[a][b] * frame[a][r] * frame[b][c2] * inv_d2;
    const double acov[2][2] = {{gm[3], gm[4]}, {gm[5], gm[6]}};
    double d_depth = 0.0;
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) d_depth += da[a][b] * acov[a][b] * (-2.0 / depth);
    // covariance of the Gaussian (scene.cpp:42-51)
    const double* lsk = ls + 3 * static_cast<size_t>(k);
    const double* qk = quat + 4 * static_cast<size_t>(k);
    const double qn_ = sqrt(qk[0] * qk[0] + qk[1] * qk[1] + qk[2] * qk[2] + qk[3] * qk[3]);
    const double w = qk[0] / qn_, x = qk[1] / qn_, y = qk[2] / qn_, z = qk[3] / qn_;
    const double R[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z),     2 * (x * z + w * y),
                         2 * (x * y + w * z),     1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                         2 * (x * z - w * y),     2 * (y * z + w * x),     1 - 2 * (x * x + y * y)};
    const double sc[3] = {exp(lsk[0]), exp(lsk[1]), exp(lsk[2])};
    double M[9], S[9];
    for (int r = 0; r < 3; ++r)
        for (int c2 = 0; c2 < 3; ++c2) M[r * 3 + c2] = R[r * 3 + c2] * sc[c2];
    for (int i = 0; i < 3; ++i)
        for (int j2 = 0; j2 < 3; ++j2) {
            double s2 = 0.0;
            for (int kk = 0; kk < 3; ++kk) s2 += M[i * 3 + kk] * M[j2 * 3 + kk];
            S[i * 3 + j2] = s2;
        }
    // frame dependence on the centre angles
    const double gvec[3] = {cp, sp, 0.0};
    const double zero3[3] = {0.0, 0.0, 0.0};
    const double m_uh[3] = {-uh[0], -uh[1], -uh[2]};
    const double ep_ct[3] = {ep[0] * ct, ep[1] * ct, ep[2] * ct};
    const double m_g[3] = {-gvec[0], -gvec[1], -gvec[2]};
    const double* dft[2] = {m_uh, zero3};
    const double* dfp[2] = {ep_ct, m_g};
    auto mv = [&](const double* v, double* o) {
        for (int i = 0; i < 3; ++i) o[i] = S[i * 3] * v[0] + S[i * 3 + 1] * v[1] + S[i * 3 + 2] * v[2];
    };
    auto dot = [](const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; };
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) {
            double t1[3], t2[3];
            mv(frame[b], t1);
            mv(dft[b], t2);
            d_theta += da[a][b] * (dot(t1, dft[a]) * inv_d2 + dot(t2, frame[a]) * inv_d2);
            mv(dfp[b], t2);
            d_phi += da[a][b] * (dot(t1, dfp[a]) * inv_d2 + dot(t2, frame[a]) * inv_d2);
        }
    // centre angles and depth back to the position
    const double ux = st * cp * depth, uy = st * sp * depth, uz = ct * depth;
    const double rho = sqrt(ux * ux + uy * uy);
    double dp3[3] = {0.0, 0.0, 0.0};
    if (rho > 1e-300) {
        const double gth[3] = {uz * ux / (rho * depth * depth), uz * uy / (rho * depth * depth), -rho / (depth * depth)};
        const double gph[3] = {-uy / (rho * rho), ux / (rho * rho), 0.0};
        for (int a = 0; a < 3; ++a) dp3[a] += gth[a] * d_theta + gph[a] * d_phi;
    }
    for (int a = 0; a < 3; ++a) d_pos[3 * k + a] = dp3[a] + uh[a] * d_depth;
    // covariance_from_backward (scene.cpp:68-104): dM = (G + G^T) M
    double dM[9];
    for (int i = 0; i < 3; ++i)
        for (int j2 = 0; j2 < 3; ++j2) {
            double s2 = 0.0;
            for (int kk = 0; kk < 3; ++kk) s2 += (dsig[i * 3 + kk] + dsig[kk * 3 + i]) * M[kk * 3 + j2];
            dM[i * 3 + j2] = s2;
        }
    double dR[9], dlsk[3] = {0.0, 0.0, 0.0};
    for (int r = 0; r < 3; ++r)
        for (int c2 = 0; c2 < 3; ++c2) {
            dR[r * 3 + c2] = dM[r * 3 + c2] * sc[c2];
            dlsk[c2] += dM[r * 3 + c2] * R[r * 3 + c2] * sc[c2];
        }
    const double part[4][9] = {{0, -z, y, z, 0, -x, -y, x, 0},
                               {0, y, z, y, -2 * x, -w, z, w, -2 * x},
                               {-2 * y, x, w, x, 0, z, -w, z, -2 * y},
                               {-2 * z, -w, x, w, -2 * z, y, x, y, 0}};
    double dqn[4];
    for (int i = 0; i < 4; ++i) {
        double acc = 0.0;
        for (int e = 0; e < 9; ++e) acc += dR[e] * (part[i][e] * 2.0);
        dqn[i] = acc;
    }
    const double qv[4] = {w, x, y, z};
    double dotq = 0.0;
    for (int i = 0; i < 4; ++i) dotq += qv[i] * dqn[i];
    for (int i = 0; i < 4; ++i) d_q[4 * k + i] = (dqn[i] - qv[i] * dotq) / qn_;
    for (int a = 0; a < 3; ++a) d_ls[3 * k + a] = dlsk[a];
    const double tau = gm[11];
    d_tau[k] = rg[0] * tau * (1.0 - tau);
}

}  // namespace

size_t bwd_geo_bytes(int64_t entries, int n_jc) {
    return sizeof(double) * 7 * static_cast<size_t>(std::max<int64_t>(entries, 1)) * ((n_jc + kNC - 1) / kNC);
}

cudaError_t launch_aggregate_bwd(const DevGrid& g, int modality, int n_rx, int channels, const double* values,
                                 const double* up, double* dv, cudaStream_t s) {
    if (n_rx * channels == 0) return cudaSuccess;
    k_aggregate_bwd<<<n_rx * channels, 256, 0, s>>>(g, modality, n_rx, channels, values, up, dv);
    return cudaGetLastError();
}

cudaError_t launch_backward_render(const rxgs_txstate_s& st, const rxgs_scene_s& sc, const double* d_coeffs_in,
                                   int n_rx, const double* d_values, double2* sig64, double* ent_geo,
                                   double2* ent_ds, double* raw_geo, double2* raw_ds, double* d_pos, double* d_ls,
                                   double* d_q, double* d_tau, double* d_coeffs, cudaStream_t s, bool needed_only) {
    const DevGrid& g = st.grid;
    const int K = st.k, C = st.channels, L = st.L;
    const int n_jc = n_rx * C;
    const long long n_k = needed_only ? (st.needed_host >= 0 ? st.needed_host : st.visible) : K;
    const long long rows = n_k * n_rx;
    if (rows > 0)
        k_signals64<<<static_cast<unsigned>((rows + 255) / 256), 256, 0, s>>>(
            K, L, C, n_rx, st.culled.as<int>(), st.basis64.as<double>(), d_coeffs_in, sig64,
            needed_only ? st.needed_order.as<int>() : nullptr, needed_only ? st.needed_count.as<int>() : nullptr);
    const int n_chunks = (n_jc + kNC - 1) / kNC;
    if (st.entries > 0) {
        cudaMemsetAsync(ent_geo, 0, sizeof(double) * 7 * st.entries * n_chunks, s);
        cudaMemsetAsync(ent_ds, 0, sizeof(double2) * n_jc * st.entries, s);
        // receiver chunks run concurrently (disjoint ent_ds columns, own ent_geo slices)
        for (int cb = 0; cb < g.cell_blocks; ++cb)
            k_bwd_walk<<<dim3(g.n_tiles, n_chunks), 64, 0, s>>>(g, cb, st.tile_offsets.as<int64_t>(),
                                                                 st.list.as<int>(), st.rec.as<GaussRec>(),
                                                                 st.walk_len.as<int>(), sig64, n_jc, d_values,
                                                                 st.entries, ent_geo, ent_ds);
    }
    if (K > 0) {
        const long long nt = static_cast<long long>(K) * (7 + n_jc);
        k_bwd_gauss_reduce<<<static_cast<unsigned>((nt + 255) / 256), 256, 0, s>>>(K, n_jc, n_chunks, st.entries,
                                                                                  st.gauss_off.as<int>(),
                                                          st.gauss_ent.as<int>(), ent_geo, ent_ds, raw_geo, raw_ds);
        auto fin = st.l_max == 2 ? k_bwd_finalize<2> : k_bwd_finalize<0>;
        fin<<<(K + 63) / 64, 64, 0, s>>>(K, st.l_max, C, n_rx, st.culled.as<int>(), st.geom.as<double>(),
                                                    st.basis64.as<double>(), d_coeffs_in, raw_geo, raw_ds,
                                                    sc.d_ls.as<double>(), sc.d_q.as<double>(), d_pos, d_ls, d_q,
                                                    d_tau, d_coeffs);
    }
    return cudaGetLastError();
}

}  // namespace rxgs_b200
