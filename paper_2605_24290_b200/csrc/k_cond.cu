// Receiver conditioning on sm_100a (conditioning.cpp:284-423).
//
//   k_cond_global      global branch: fourier_encode (:255-265) + the per-
//                      component MLP (:317-361) for every (receiver, l);
//                      tiny (N*L rows), run in FP64.
//   k_cond_signal      THE hot kernel of the query path: per (Gaussian,
//                      receiver) the local features (:376-396, probe_segment
//                      :163-178 over an occupancy grid held in shared memory),
//                      the local MLP 6->H->H->4C (:397), both complex affines
//                      (:271-275) and the FLE reduction of reduce_signals
//                      (sphraster.cpp:190-226), fused so the N*K*L*C*2
//                      coefficient tensor is never materialised:
//                        s = (1+aL) * sum_l[(1+aG_l) (B_l base_l) + bG_l B_l]
//                            + bL * sum_l B_l
//                      FP32 SIMT, persistent CTAs, one warp = 32 receivers of
//                      one Gaussian (Gaussian data broadcast, receiver data
//                      per lane).
//   k_cond_materialize condition_forward's materialised output (FP64 affine
//                      on the FP64 base, so zero branches are bitwise identity
//                      exactly as in the reference).
#include "cond_common.cuh"
#include "rxgs_internal.cuh"

namespace rxgs_b200 {
namespace {

using namespace cond_dev;


// ------------------------------------------------------------------ global branch (FP64)
// Persistent CTAs loop over receivers.  Per receiver the Fourier part of
// layer 1 (the first 6F inputs, shared by all L components) is summed once;
// then the components go through the MLP CP at a time: thread (o, group)
// carries FOUR components' dot products for output unit o (four independent
// FP64 chains sharing each weight load -- the chains, not the FLOP count,
// bound this kernel), and layer 3 splits each (component, output) sum over
// a few lanes joined by shuffles.  W2 is staged transposed in shared memory
// once per CTA.  The outputs are rounded to f32 (ag), so the summation order
// only moves the FP64 rounding, far below that.
constexpr int kGlobThreads = 256;
constexpr int kGlobChains = 4;

__global__ void __launch_bounds__(kGlobThreads) k_cond_global(CondDev c, const double* __restrict__ rx, int n_rx,
                                                              float* __restrict__ ag) {
    extern __shared__ double sm[];
    const int H = c.H, F6 = 6 * c.F, G = kGlobThreads / H, CP = G * kGlobChains, gin = c.gin, NY = 4 * c.C;
    // every weight of the global MLP staged once per CTA, transposed so a
    // warp's 32 output units read consecutive words
    double* w1t = sm;                    // [i][o], gin x H
    double* w2t = w1t + gin * H;         // [i][o], H x H
    double* w3 = w2t + H * H;            // [oo][i], NY x H
    double* emb = w3 + NY * H;           // L x dc
    double* b1 = emb + c.L * c.dc;       // H
    double* b2 = b1 + H;                 // H
    double* b3 = b2 + H;                 // NY
    double* gam = b3 + NY;               // 6F
    double* pre = gam + F6;              // H
    double* h1 = pre + H;                // CP x H
    double* h2 = h1 + CP * H;            // CP x H
    const double* p = c.p64;
    const int tid = threadIdx.x;
    // staging: several loads in flight per thread (a one-receiver call is
    // one CTA, latency-bound on this)
#pragma unroll 8
    for (int i = tid; i < gin * H; i += blockDim.x) w1t[(i % gin) * H + i / gin] = p[c.o_gw1 + i];
#pragma unroll 8
    for (int i = tid; i < H * H; i += blockDim.x) w2t[(i % H) * H + i / H] = p[c.o_gw2 + i];
#pragma unroll 4
    for (int i = tid; i < NY * H; i += blockDim.x) w3[i] = p[c.o_gw3 + i];
#pragma unroll 4
    for (int i = tid; i < c.L * c.dc; i += blockDim.x) emb[i] = p[c.o_emb + i];
    for (int i = tid; i < H; i += blockDim.x) {
        b1[i] = p[c.o_gb1 + i];
        b2[i] = p[c.o_gb2 + i];
    }
    for (int i = tid; i < NY; i += blockDim.x) b3[i] = p[c.o_gb3 + i];
    int l_max = 0;
    while ((l_max + 1) * (l_max + 1) < c.L) ++l_max;
    const double den = l_max > 0 ? static_cast<double>(l_max) : 1.0;  // conditioning.cpp:328
    const int o = tid % H, grp = tid / H;
    // layer 3: (component, output) pairs of a pass, TP lanes each (power of two <= 32)
    const int pairs = CP * NY;
    int TP = 1;
    while (TP * 2 <= 32 && pairs * TP * 2 <= kGlobThreads) TP *= 2;
    for (int j = blockIdx.x; j < n_rx; j += gridDim.x) {
        __syncthreads();
        for (int i = tid; i < F6; i += blockDim.x) {  // fourier_encode, conditioning.cpp:255-265
            const int a = i / (2 * c.F), band = (i % (2 * c.F)) / 2;
            const double arg = p[c.o_freq + band * 3 + a] * rx[3 * j + a];
            gam[i] = (i % 2) ? cos(arg) : sin(arg);
        }
        __syncthreads();
        if (tid < H) {  // the Fourier part of layer 1, shared by every component
            double acc = b1[tid];
            for (int i = 0; i < F6; ++i) acc += w1t[i * H + tid] * gam[i];
            pre[tid] = acc;
        }
        for (int c0 = 0; c0 < c.L; c0 += CP) {
            __syncthreads();
            if (grp < G) {  // layer 1 tail: [l/l_max, m/l_max, e_l]
#pragma unroll
                for (int q = 0; q < kGlobChains; ++q) {
                    const int cl = grp * kGlobChains + q, comp = c0 + cl;
                    if (comp >= c.L) break;
                    int l = 0;
                    while ((l + 1) * (l + 1) <= comp) ++l;
                    const int m = comp - l * l - l;
                    double acc = pre[o];
                    acc += w1t[F6 * H + o] * (l / den);
                    acc += w1t[(F6 + 1) * H + o] * (m / den);
                    for (int e = 0; e < c.dc; ++e) acc += w1t[(F6 + 2 + e) * H + o] * emb[comp * c.dc + e];
                    h1[cl * H + o] = acc > 0.0 ? acc : 0.0;
                }
            }
            __syncthreads();
            if (grp < G) {  // layer 2: four chains per thread
                double acc[kGlobChains];
#pragma unroll
                for (int q = 0; q < kGlobChains; ++q) acc[q] = b2[o];
                const double* hb = h1 + grp * kGlobChains * H;
                for (int i = 0; i < H; ++i) {
                    const double w = w2t[i * H + o];
#pragma unroll
                    for (int q = 0; q < kGlobChains; ++q) acc[q] += w * hb[q * H + i];
                }
#pragma unroll
                for (int q = 0; q < kGlobChains; ++q) h2[(grp * kGlobChains + q) * H + o] = acc[q] > 0.0 ? acc[q] : 0.0;
            }
            __syncthreads();
            // layer 3: pair = (component cl, output oo), lanes sub = 0..TP-1 split the sum
            for (int t = tid; t < pairs * TP; t += blockDim.x) {
                const int pr = t / TP, sub = t % TP;
                const int cl = pr / NY, oo = pr % NY, comp = c0 + cl;
                double acc = 0.0;
                for (int i = sub; i < H; i += TP) acc += w3[oo * H + i] * h2[cl * H + i];
                for (int off = 1; off < TP; off <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off, TP);
                if (sub == 0 && comp < c.L) {
                    acc += b3[oo];
                    if (c.additive && (oo % 4) < 2) acc = 0.0;
                    ag[(static_cast<size_t>(j) * c.L + comp) * NY + oo] = static_cast<float>(acc);
                }
            }
        }
    }
}

// ------------------------------------------------------------------ trilinear cell table
// Cell (cx, cy, cz) in [-1, R]^3 (the cells a clamped or in-grid sample can
// fall in) -> the coefficients of v = a + b w0 + c w1 + d w2 + e w0 w1 +
// f w0 w2 + g w1 w2 + h w0 w1 w2 (out-of-grid corners read 0, as in
// sample_trilinear, conditioning.cpp:74-98), stored [a, d, b, f, c, g, e, h]
// so the probe evaluates it with three FFMA2 and one FFMA (k_cond_tc.cu).
// Computed in FP64 from the FP32 grid values, rounded once.
__global__ void k_occ_cubes(int R, const float* __restrict__ occ, float* __restrict__ cube) {
    const int P = R + 2;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P * P * P) return;
    const int cx = i / (P * P) - 1, cy = (i / P) % P - 1, cz = i % P - 1;
    auto q = [&](int x, int y, int z) -> double {
        return (x < 0 || y < 0 || z < 0 || x >= R || y >= R || z >= R) ? 0.0 : occ[(x * R + y) * R + z];
    };
    const double q000 = q(cx, cy, cz), q001 = q(cx, cy, cz + 1), q010 = q(cx, cy + 1, cz), q011 = q(cx, cy + 1, cz + 1);
    const double q100 = q(cx + 1, cy, cz), q101 = q(cx + 1, cy, cz + 1), q110 = q(cx + 1, cy + 1, cz),
                 q111 = q(cx + 1, cy + 1, cz + 1);
    float* o = cube + 8 * static_cast<size_t>(i);
    o[0] = static_cast<float>(q000);                                      // a
    o[1] = static_cast<float>(q001 - q000);                               // d (z)
    o[2] = static_cast<float>(q100 - q000);                               // b (x)
    o[3] = static_cast<float>(q101 - q100 - q001 + q000);                 // f (xz)
    o[4] = static_cast<float>(q010 - q000);                               // c (y)
    o[5] = static_cast<float>(q011 - q010 - q001 + q000);                 // g (yz)
    o[6] = static_cast<float>(q110 - q100 - q010 + q000);                 // e (xy)
    o[7] = static_cast<float>(q111 - q110 - q101 - q011 + q100 + q010 + q001 - q000);  // h (xyz)
}

// ------------------------------------------------------------------ local branch helpers

// ------------------------------------------------------------------ fused hot kernel
template <int HT, int CT>
__global__ void __launch_bounds__(512, 1)
    k_cond_signal(CondDev c, const int* __restrict__ n_rows, const int* __restrict__ vis, const float4* __restrict__ pos32,
                  const double* __restrict__ rx, int n_rx, const float2* __restrict__ B,
                  const float2* __restrict__ GB, const float* __restrict__ ag,
                  SigOut sig) {
    extern __shared__ __align__(16) float smem[];
    const int H = HT > 0 ? HT : c.H;
    const int C = CT > 0 ? CT : c.C;
    // the specialised path probes the trilinear cell table (cube_features, the
    // same features as the training backward); the generic one the smem grid
    const bool cubep = HT > 0 && c.probe && !c.nearest && c.cube != nullptr;
    const int R3 = c.probe && !cubep ? c.R * c.R * c.R : 0;
    // layout: w2 (H*H) | w1 (H*6) | b1 (H) | b2 (H) | w3 (4C*H) | b3 (4C) | occ (R^3)
    float* s_w2 = smem;
    float* s_w1 = s_w2 + H * H;
    float* s_b1 = s_w1 + H * 6;
    float* s_b2 = s_b1 + H;
    float* s_w3 = s_b2 + H;
    float* s_b3 = s_w3 + 4 * C * H;
    float* s_occ = s_b3 + ((4 * C + 3) & ~3);
    // HT == 64, CT == 1: W2 as output pairs, transposed (local_mlp64_t), after the grid
    const int occ_floats = R3 ? padded_dim(c.R) * padded_dim(c.R) * padded_dim(c.R) : 0;
    float2* s_w2t2 = reinterpret_cast<float2*>(s_occ + ((occ_floats + 3) & ~3));
    const float* p = c.p32;
    if (c.use_local) {
        if (HT == 64 && CT == 1)
            for (int i = threadIdx.x; i < H * H / 2; i += blockDim.x) {
                const int ii = i / (H / 2), op = i % (H / 2);
                s_w2t2[i] = make_float2(p[c.o_lw2 + (2 * op) * H + ii], p[c.o_lw2 + (2 * op + 1) * H + ii]);
            }
        for (int i = threadIdx.x; i < H * H; i += blockDim.x) s_w2[i] = p[c.o_lw2 + i];
        for (int i = threadIdx.x; i < H * 6; i += blockDim.x) s_w1[i] = p[c.o_lw1 + i];
        for (int i = threadIdx.x; i < H; i += blockDim.x) {
            s_b1[i] = p[c.o_lb1 + i];
            s_b2[i] = p[c.o_lb2 + i];
        }
        for (int i = threadIdx.x; i < 4 * C * H; i += blockDim.x) s_w3[i] = p[c.o_lw3 + i];
        for (int i = threadIdx.x; i < 4 * C; i += blockDim.x) s_b3[i] = p[c.o_lb3 + i];
        if (R3) load_padded_occ(c, s_occ);
    }
    __syncthreads();
    const LocalSmem w{s_occ, s_w1, s_b1, s_w2, s_b2, s_w3, s_b3};

    const int lane = threadIdx.x & 31;
    const int warps_per_block = blockDim.x >> 5;
    // a warp takes 32 consecutive rows of the (needed Gaussian, receiver)
    // space, receivers fastest: no idle lanes when n_rx is not a multiple
    // of 32 (training batches of 16)
    const long long rows_total = static_cast<long long>(*n_rows) * n_rx;
    const long long items = (rows_total + 31) >> 5;
    const long long stride = static_cast<long long>(gridDim.x) * warps_per_block;
    const int L = c.L;
    constexpr int YM = CT > 0 ? 4 * CT : 4 * kCMax;
    for (long long it = static_cast<long long>(blockIdx.x) * warps_per_block + (threadIdx.x >> 5);
         it < items; it += stride) {
        const long long row = it * 32 + lane;
        const bool act = row < rows_total;
        const long long rowc = act ? row : rows_total - 1;
        const int vi = static_cast<int>(rowc / n_rx);
        const int j = static_cast<int>(rowc - static_cast<long long>(vi) * n_rx);
        const int k = vis[vi];
        const float4 pk = pos32[k];
        const int jr = act ? j : 0;
        const float rxx = static_cast<float>(rx[3 * jr]);
        const float rxy = static_cast<float>(rx[3 * jr + 1]);
        const float rxz = static_cast<float>(rx[3 * jr + 2]);
        float y[YM];
        float in[6];
        if (c.use_local && cubep) {  // warp-uniform: the probe votes over all lanes
            if (c.S == 16 && c.R == 32)
                cube_features<16, 32>(c, act, pk, rxx, rxy, rxz, in);
            else
                cube_features<0, 0>(c, act, pk, rxx, rxy, rxz, in);
        }
        if (!act) continue;
        if (c.use_local) {
            if (!cubep) local_features<true>(c, s_occ, pk.x, pk.y, pk.z, rxx, rxy, rxz, in);
            if constexpr (HT == 64 && CT == 1)
                local_mlp64_t(w, s_w2t2, in, y);
            else
                local_mlp<HT, CT>(c, w, in, y);
        } else {
#pragma unroll
            for (int q = 0; q < YM; ++q) y[q] = 0.f;
        }
        for (int ch = 0; ch < C; ++ch) {
            float2 M = make_float2(0.f, 0.f), Bs = make_float2(0.f, 0.f);
            const float4* a4 = reinterpret_cast<const float4*>(ag) + static_cast<size_t>(j) * L * C + ch;
            for (int l = 0; l < L; ++l) {
                const float2 b = B[static_cast<size_t>(k) * L + l];
                const float2 gb = GB[(static_cast<size_t>(k) * L + l) * C + ch];
                const float4 a = a4[static_cast<size_t>(l) * C];
                const float2 one_a = make_float2(1.f + a.x, a.y);
                const float2 t0 = cmul(one_a, gb), t1 = cmul(make_float2(a.z, a.w), b);
                M.x += t0.x + t1.x;
                M.y += t0.y + t1.y;
                Bs.x += b.x;
                Bs.y += b.y;
            }
            const float ar = c.additive ? 0.f : y[4 * ch], ai = c.additive ? 0.f : y[4 * ch + 1];
            const float2 s0 = cmul(make_float2(1.f + ar, ai), M);
            const float2 s1 = cmul(make_float2(y[4 * ch + 2], y[4 * ch + 3]), Bs);
            store_sig(sig, k, n_rx, j, C, ch, make_float2(s0.x + s1.x, s0.y + s1.y));
        }
    }
}

// ------------------------------------------------------------------ materialised output
__global__ void k_cond_materialize(CondDev c, int K, const float4* __restrict__ pos32,
                                   const double* __restrict__ rx, int n_rx,
                                   const double* __restrict__ base, const float* __restrict__ ag,
                                   double* __restrict__ out, double* __restrict__ local_in,
                                   const int* __restrict__ rows = nullptr, const int* __restrict__ n_rows = nullptr) {
    extern __shared__ __align__(16) float smem[];
    const int H = c.H, C = c.C, L = c.L;
    const int R3 = (c.probe && c.use_local) ? c.R * c.R * c.R : 0;
    float* s_w2 = smem;
    float* s_w1 = s_w2 + H * H;
    float* s_b1 = s_w1 + H * 6;
    float* s_b2 = s_b1 + H;
    float* s_w3 = s_b2 + H;
    float* s_b3 = s_w3 + 4 * C * H;
    float* s_occ = s_b3 + ((4 * C + 3) & ~3);
    const float* p = c.p32;
    if (c.use_local) {
        for (int i = threadIdx.x; i < H * H; i += blockDim.x) s_w2[i] = p[c.o_lw2 + i];
        for (int i = threadIdx.x; i < H * 6; i += blockDim.x) s_w1[i] = p[c.o_lw1 + i];
        for (int i = threadIdx.x; i < H; i += blockDim.x) {
            s_b1[i] = p[c.o_lb1 + i];
            s_b2[i] = p[c.o_lb2 + i];
        }
        for (int i = threadIdx.x; i < 4 * C * H; i += blockDim.x) s_w3[i] = p[c.o_lw3 + i];
        for (int i = threadIdx.x; i < 4 * C; i += blockDim.x) s_b3[i] = p[c.o_lb3 + i];
        if (R3) load_padded_occ(c, s_occ);
    }
    __syncthreads();
    const LocalSmem w{s_occ, s_w1, s_b1, s_w2, s_b2, s_w3, s_b3};
    const long long row = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    int j, k;
    if (rows) {  // only the listed rows (the TxState's needed Gaussians, Morton order)
        const int n = *n_rows;
        if (row >= static_cast<long long>(n) * n_rx) return;
        j = static_cast<int>(row / n);
        k = rows[row % n];
    } else {
        if (row >= static_cast<long long>(K) * n_rx) return;
        j = static_cast<int>(row / K);
        k = static_cast<int>(row % K);
    }
    float y[4 * kCMax];
    for (int q = 0; q < 4 * C; ++q) y[q] = 0.f;
    if (c.use_local) {
        const float4 pk = pos32[k];
        float in[6];
        local_features<true>(c, s_occ, pk.x, pk.y, pk.z, static_cast<float>(rx[3 * j]),
                       static_cast<float>(rx[3 * j + 1]), static_cast<float>(rx[3 * j + 2]), in);
        local_mlp<0, 0>(c, w, in, y);
        if (local_in && j == 0)
            for (int i = 0; i < 6; ++i) local_in[static_cast<size_t>(k) * 6 + i] = in[i];
    }
    const size_t stride = static_cast<size_t>(L) * C * 2;
    for (int l = 0; l < L; ++l)
        for (int ch = 0; ch < C; ++ch) {
            const size_t idx = static_cast<size_t>(k) * stride + (static_cast<size_t>(l) * C + ch) * 2;
            const double zr = base[idx], zi = base[idx + 1];
            double mr = zr, mi = zi;
            if (c.use_global) {
                const float* a = ag + (static_cast<size_t>(j) * L + l) * 4 * C + 4 * ch;
                const double ar = a[0], ai = a[1], br = a[2], bi = a[3];
                mr = zr + (ar * zr - ai * zi + br);
                mi = zi + (ai * zr + ar * zi + bi);
            }
            double orr = mr, oi = mi;
            if (c.use_local) {
                const double ar = c.additive ? 0.0 : y[4 * ch], ai = c.additive ? 0.0 : y[4 * ch + 1];
                const double br = y[4 * ch + 2], bi = y[4 * ch + 3];
                orr = mr + (ar * mr - ai * mi + br);
                oi = mi + (ai * mr + ar * mi + bi);
            }
            const size_t o = static_cast<size_t>(j) * K * stride + idx;
            out[o] = orr;
            out[o + 1] = oi;
        }
}

// condition_forward's materialised output (conditioning.cpp:340-421) of the
// needed rows from the local branch's (alpha_L, beta_L) y[k][j] (tcgen05,
// launch_local_y_rows): out = affine_L(affine_G(base)) in FP64, the
// reference's operation order; C == 1.
__global__ void k_materialize_y(CondDev c, int K, int L, int n_rx, const int* __restrict__ rows,
                                const int* __restrict__ n_rows, const double* __restrict__ base,
                                const float* __restrict__ ag, const float4* __restrict__ y,
                                double* __restrict__ out) {
    const long long row = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    const int n = *n_rows;
    if (row >= static_cast<long long>(n) * n_rx) return;
    const int j = static_cast<int>(row / n);
    const int k = rows[row % n];
    const float4 yl = c.use_local ? y[static_cast<size_t>(k) * n_rx + j] : make_float4(0.f, 0.f, 0.f, 0.f);
    const double ar = c.additive ? 0.0 : yl.x, ai = c.additive ? 0.0 : yl.y, br = yl.z, bi = yl.w;
    const size_t stride = static_cast<size_t>(L) * 2;
    for (int l = 0; l < L; ++l) {
        const size_t idx = static_cast<size_t>(k) * stride + static_cast<size_t>(l) * 2;
        const double zr = base[idx], zi = base[idx + 1];
        double mr = zr, mi = zi;
        if (c.use_global) {
            const float* a = ag + (static_cast<size_t>(j) * L + l) * 4;
            const double gar = a[0], gai = a[1], gbr = a[2], gbi = a[3];
            mr = zr + (gar * zr - gai * zi + gbr);
            mi = zi + (gai * zr + gar * zi + gbi);
        }
        double orr = mr, oi = mi;
        if (c.use_local) {
            orr = mr + (ar * mr - ai * mi + br);
            oi = mi + (ai * mr + ar * mi + bi);
        }
        const size_t o = static_cast<size_t>(j) * K * stride + idx;
        out[o] = orr;
        out[o + 1] = oi;
    }
}

__global__ void k_probe(CondDev c, int n, const double* __restrict__ from,
                        const double* __restrict__ to, double* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float px = static_cast<float>(from[3 * i]), py = static_cast<float>(from[3 * i + 1]),
                pz = static_cast<float>(from[3 * i + 2]);
    float in[6];
    local_features(c, c.occ, px, py, pz, static_cast<float>(to[3 * i]),
                   static_cast<float>(to[3 * i + 1]), static_cast<float>(to[3 * i + 2]), in);
    out[2 * i] = in[4];
    out[2 * i + 1] = in[5];
}

// reduce_signals (sphraster.cpp:190-226) from the materialised f64 tensor.
__global__ void k_reduce_signals(int K, int L, int C, int n_rx, const int* __restrict__ culled,
                                 const double* __restrict__ basis64, const double* __restrict__ co,
                                 float2* __restrict__ sig) {
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
        sig[(static_cast<size_t>(k) * n_rx + j) * C + ch] =
            make_float2(static_cast<float>(sr), static_cast<float>(si));
    }
}

__global__ void k_check_finite(long long n, long long per_row, const double* __restrict__ co,
                               int* __restrict__ err) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    if (!isfinite(co[i])) atomicMin(err, static_cast<int>(i / per_row));
}

__global__ void k_check_coincide(int K, const double* __restrict__ pos, const double* __restrict__ rx,
                                 int n_rx, int* __restrict__ err) {
    const long long row = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (row >= static_cast<long long>(K) * n_rx) return;
    const int j = static_cast<int>(row / K), k = static_cast<int>(row % K);
    const double dx = rx[3 * j] - pos[3 * k], dy = rx[3 * j + 1] - pos[3 * k + 1],
                 dz = rx[3 * j + 2] - pos[3 * k + 2];
    if (sqrt(dx * dx + dy * dy + dz * dz) == 0.0) atomicMin(err, static_cast<int>(row));
}

size_t local_smem_bytes(const CondDev& d, bool with_occ) {
    const size_t f = static_cast<size_t>(d.H) * d.H + d.H * 6 + 2 * d.H + 4 * d.C * d.H +
                     ((4 * d.C + 3) & ~3) + (with_occ ? static_cast<size_t>(padded_dim(d.R)) * padded_dim(d.R) * padded_dim(d.R) : 0);
    return f * sizeof(float);
}

}  // namespace

cudaError_t launch_cond_global(const rxgs_cond_s& c, const double* d_rx, int n_rx, float* d_ag,
                               cudaStream_t s) {
    if (n_rx == 0) return cudaSuccess;
    if (!c.use_global()) return cudaMemsetAsync(d_ag, 0, sizeof(float) * n_rx * c.L * 4 * c.C, s);
    const CondDev d = make_dev(c);
    const int H = c.hidden;
    if (H > kGlobThreads) return cudaErrorInvalidValue;
    const int CP = (kGlobThreads / H) * kGlobChains, NY = 4 * c.C;
    const size_t smem = sizeof(double) * (static_cast<size_t>(c.gin) * H + static_cast<size_t>(H) * H + NY * H +
                                          static_cast<size_t>(c.L) * c.dc + 2 * H + NY + 6 * c.F + H +
                                          2 * static_cast<size_t>(CP) * H);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaFuncSetAttribute(k_cond_global, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
#ifndef RXGS_GLOB_CTAS_PER_SM
#define RXGS_GLOB_CTAS_PER_SM 2  // weights staged in shared memory (~90 KB at L = 100): 2 CTAs per SM
#endif
    k_cond_global<<<std::min(n_rx, RXGS_GLOB_CTAS_PER_SM * sms), kGlobThreads, smem, s>>>(d, d_rx, n_rx, d_ag);
    return cudaGetLastError();
}

cudaError_t launch_cond_signal(const rxgs_cond_s* c, const rxgs_scene_s& sc,
                               const rxgs_txstate_s& st, const double* d_rx, int n_rx,
                               const float* d_ag, SigOut d_sig, int* d_err, cudaStream_t s) {
    (void)d_err;
    if (st.visible == 0 || n_rx == 0) return cudaSuccess;
    if (sc.ctx->cond_kernel != 1 && cond_tc_eligible(c))
        return launch_cond_signal_tc(*c, sc, st, d_rx, n_rx, d_ag, d_sig, s);
    CondDev d{};
    if (c) {
        d = make_dev(*c);
    } else {  // unconditioned model: identity branches
        d.H = 1; d.C = sc.channels; d.L = sc.L; d.use_global = 0; d.use_local = 0; d.probe = 0;
    }
    const size_t smem = d.use_local ? local_smem_bytes(d, d.probe) : 16;
    int dev = 0;
    cudaGetDevice(&dev);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long items = static_cast<long long>(st.visible) * ((n_rx + 31) / 32);
    const int threads = 512;
    const long long want = (items + (threads / 32) - 1) / (threads / 32);
    const int blocks = static_cast<int>(want < sms ? want : sms);
    const bool fast = d.use_local && d.H == 64 && d.C == 1;
    if (fast) {
        const bool cubep = d.probe && !d.nearest && d.cube != nullptr;
        const size_t smem_f = (cubep ? local_smem_bytes(d, false) : smem) + sizeof(float) * (64 * 64 + 4);
        cudaFuncSetAttribute(k_cond_signal<64, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem_f));
        k_cond_signal<64, 1><<<blocks, threads, smem_f, s>>>(
            d, st.needed_count.as<int>(), st.needed_order.as<int>(), sc.d_pos32.as<float4>(), d_rx, n_rx,
            st.basis32.as<float2>(), st.gb32.as<float2>(), d_ag, d_sig);
    } else {
        if (d.H > kHMax || d.C > kCMax) return cudaErrorInvalidValue;
        cudaFuncSetAttribute(k_cond_signal<0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
        k_cond_signal<0, 0><<<blocks, threads, smem, s>>>(
            d, st.needed_count.as<int>(), st.needed_order.as<int>(), sc.d_pos32.as<float4>(), d_rx, n_rx,
            st.basis32.as<float2>(), st.gb32.as<float2>(), d_ag, d_sig);
    }
    return cudaGetLastError();
}

cudaError_t launch_cond_materialize(const rxgs_cond_s& c, const rxgs_scene_s& sc,
                                    const double* d_rx, int n_rx, const float* d_ag, double* d_out,
                                    double* d_local_in, int* d_err, cudaStream_t s) {
    (void)d_err;
    if (sc.k == 0 || n_rx == 0) return cudaSuccess;
    const CondDev d = make_dev(c);
    if (d.H > kHMax || d.C > kCMax) return cudaErrorInvalidValue;
    const size_t smem = local_smem_bytes(d, d.probe && d.use_local);
    cudaFuncSetAttribute(k_cond_materialize, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    const long long rows = static_cast<long long>(sc.k) * n_rx;
    k_cond_materialize<<<static_cast<unsigned>((rows + 255) / 256), 256, smem, s>>>(
        d, sc.k, sc.d_pos32.as<float4>(), d_rx, n_rx, sc.d_coeffs64.as<double>(), d_ag, d_out,
        d_local_in);
    return cudaGetLastError();
}

cudaError_t launch_materialize_y(const rxgs_cond_s& c, const rxgs_scene_s& sc, const rxgs_txstate_s& st, int n_rx,
                                 const float* d_ag, const float4* y, double* d_out, cudaStream_t s) {
    if (st.visible == 0 || n_rx == 0) return cudaSuccess;
    const long long bound = static_cast<long long>(st.visible) * n_rx;
    k_materialize_y<<<static_cast<unsigned>((bound + 255) / 256), 256, 0, s>>>(
        make_dev(c), sc.k, sc.L, n_rx, st.needed_order.as<int>(), st.needed_count.as<int>(),
        sc.d_coeffs64.as<double>(), d_ag, y, d_out);
    return cudaGetLastError();
}

cudaError_t launch_cond_materialize_needed(const rxgs_cond_s& c, const rxgs_scene_s& sc, const rxgs_txstate_s& st,
                                           const double* d_rx, int n_rx, const float* d_ag, double* d_out,
                                           cudaStream_t s) {
    if (st.visible == 0 || n_rx == 0) return cudaSuccess;
    const CondDev d = make_dev(c);
    if (d.H > kHMax || d.C > kCMax) return cudaErrorInvalidValue;
    const size_t smem = local_smem_bytes(d, d.probe && d.use_local);
    cudaFuncSetAttribute(k_cond_materialize, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    const long long bound = static_cast<long long>(st.visible) * n_rx;
    k_cond_materialize<<<static_cast<unsigned>((bound + 255) / 256), 256, smem, s>>>(
        d, sc.k, sc.d_pos32.as<float4>(), d_rx, n_rx, sc.d_coeffs64.as<double>(), d_ag, d_out, nullptr,
        st.needed_order.as<int>(), st.needed_count.as<int>());
    return cudaGetLastError();
}

cudaError_t launch_occ_cubes(rxgs_cond_s& c, cudaStream_t s) {
    const int P = c.R + 2;
    const size_t n = static_cast<size_t>(P) * P * P;
    cudaError_t e = c.d_occ_cube.ensure(n * 8 * sizeof(float));
    if (e != cudaSuccess) return e;
    k_occ_cubes<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(c.R, c.d_occ32.as<float>(), c.d_occ_cube.as<float>());
    return cudaGetLastError();
}

cudaError_t launch_probe(const rxgs_cond_s& c, int n, const double* d_from, const double* d_to,
                         double* d_out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    CondDev d = make_dev(c);
    d.probe = c.has_occ ? 1 : 0;
    k_probe<<<(n + 127) / 128, 128, 0, s>>>(d, n, d_from, d_to, d_out);
    return cudaGetLastError();
}

cudaError_t launch_reduce_signals(const rxgs_txstate_s& st, const double* d_coeffs, int n_rx,
                                  float2* d_sig, int* d_err, cudaStream_t s) {
    const long long n = static_cast<long long>(n_rx) * st.k * st.L * st.channels * 2;
    if (n == 0) return cudaSuccess;
    k_check_finite<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(
        n, static_cast<long long>(st.L) * st.channels * 2, d_coeffs, d_err);
    const long long rows = static_cast<long long>(st.k) * n_rx;
    k_reduce_signals<<<static_cast<unsigned>((rows + 255) / 256), 256, 0, s>>>(
        st.k, st.L, st.channels, n_rx, st.culled.as<int>(), st.basis64.as<double>(), d_coeffs, d_sig);
    return cudaGetLastError();
}

cudaError_t launch_check_finite(long long n, long long per_row, const double* d_coeffs, int* d_err,
                                cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_check_finite<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(n, per_row, d_coeffs, d_err);
    return cudaGetLastError();
}

cudaError_t launch_check_coincide(const rxgs_scene_s& sc, const double* d_rx, int n_rx, int* d_err,
                                  cudaStream_t s) {
    const long long rows = static_cast<long long>(sc.k) * n_rx;
    if (rows == 0) return cudaSuccess;
    k_check_coincide<<<static_cast<unsigned>((rows + 255) / 256), 256, 0, s>>>(
        sc.k, sc.d_pos.as<double>(), d_rx, n_rx, d_err);
    return cudaGetLastError();
}

}  // namespace rxgs_b200
