// Device code shared by the SIMT (k_cond.cu) and tcgen05 (k_cond_tc.cu)
// conditioning kernels: parameter view, local features / occupancy probe
// (conditioning.cpp:74-98, 163-178, 376-396), the SIMT local MLP and the
// fused conditioning + FLE reduction of one (Gaussian, receiver) row.
#pragma once

#include "f32x2.cuh"
#include "rxgs_internal.cuh"

namespace rxgs_b200 {
namespace cond_dev {

constexpr int kHMax = 64;
constexpr int kCMax = 8;

struct CondDev {
    const float* p32;
    const double* p64;
    const float* occ;
    const float* cube;  // trilinear cell table (rxgs_cond_s::d_occ_cube)
    int F, H, dc, S, R, nearest, mode, L, C, gin;
    int o_freq, o_gw1, o_gb1, o_gw2, o_gb2, o_gw3, o_gb3, o_emb, o_lw1, o_lb1, o_lw2, o_lb2, o_lw3, o_lb3;
    int probe;  // 1 = sample the occupancy grid, 0 = T=1, rho=0
    int use_global, use_local, additive;
    float lo[3], cell[3];
};

inline CondDev make_dev(const rxgs_cond_s& c) {
    CondDev d{};
    d.p32 = c.d_params32.as<float>();
    d.p64 = c.d_params64.as<double>();
    d.occ = c.d_occ32.as<float>();
    d.cube = c.d_occ_cube.as<float>();
    d.F = c.F; d.H = c.hidden; d.dc = c.dc; d.S = c.S; d.R = c.R; d.nearest = c.nearest;
    d.mode = c.mode; d.L = c.L; d.C = c.C; d.gin = c.gin;
    d.o_freq = static_cast<int>(c.o_freq); d.o_gw1 = static_cast<int>(c.o_gw1);
    d.o_gb1 = static_cast<int>(c.o_gb1); d.o_gw2 = static_cast<int>(c.o_gw2);
    d.o_gb2 = static_cast<int>(c.o_gb2); d.o_gw3 = static_cast<int>(c.o_gw3);
    d.o_gb3 = static_cast<int>(c.o_gb3); d.o_emb = static_cast<int>(c.o_emb);
    d.o_lw1 = static_cast<int>(c.o_lw1); d.o_lb1 = static_cast<int>(c.o_lb1);
    d.o_lw2 = static_cast<int>(c.o_lw2); d.o_lb2 = static_cast<int>(c.o_lb2);
    d.o_lw3 = static_cast<int>(c.o_lw3); d.o_lb3 = static_cast<int>(c.o_lb3);
    d.probe = c.no_occ() ? 0 : 1;
    d.use_global = c.use_global();
    d.use_local = c.use_local();
    d.additive = c.additive();
    for (int a = 0; a < 3; ++a) {
        d.lo[a] = static_cast<float>(c.lo[a]);
        d.cell[a] = static_cast<float>((c.hi[a] - c.lo[a]) / c.R);
    }
    return d;
}

struct LocalSmem {
    const float* occ;
    const float* w1;
    const float* b1;
    const float* w2;
    const float* b2;
    const float* w3;
    const float* b3;
};

__device__ __forceinline__ float sample_tri(const CondDev& c, const float* occ, float qx, float qy,
                                            float qz) {
    const int R = c.R;
    const float u0 = (qx - c.lo[0]) / c.cell[0] - 0.5f;
    const float u1 = (qy - c.lo[1]) / c.cell[1] - 0.5f;
    const float u2 = (qz - c.lo[2]) / c.cell[2] - 0.5f;
    const float f0 = floorf(u0), f1 = floorf(u1), f2 = floorf(u2);
    const int i0 = static_cast<int>(f0), i1 = static_cast<int>(f1), i2 = static_cast<int>(f2);
    const float a0 = u0 - f0, a1 = u1 - f1, a2 = u2 - f2;
    float acc = 0.f;
#pragma unroll
    for (int dx = 0; dx < 2; ++dx)
#pragma unroll
        for (int dy = 0; dy < 2; ++dy)
#pragma unroll
            for (int dz = 0; dz < 2; ++dz) {
                const int ix = i0 + dx, iy = i1 + dy, iz = i2 + dz;
                if (ix < 0 || iy < 0 || iz < 0 || ix >= R || iy >= R || iz >= R) continue;
                const float w = (dx ? a0 : 1.f - a0) * (dy ? a1 : 1.f - a1) * (dz ? a2 : 1.f - a2);
                acc += w * occ[(ix * R + iy) * R + iz];
            }
    return acc;
}

// Occupancy held with a zero border -- one voxel below, two above: a
// (R+3)^3 grid.  A trilinear sample then needs no per-corner bounds test:
// each voxel coordinate u is clamped to [-1, R]; every corner of the clamped
// sample is either real data or border, and a clamped axis lands on the
// border with weight 1, which reproduces the reference's "out-of-bounds
// corners read 0" (conditioning.cpp:91) exactly.
__host__ __device__ constexpr int padded_dim(int R) { return R + 3; }
__device__ __forceinline__ int padded_index(int R, int ix, int iy, int iz) {
    const int P = padded_dim(R);
    return ((ix + 1) * P + (iy + 1)) * P + (iz + 1);
}

// Fill the padded copy of the R^3 grid (called by all threads of a CTA).
__device__ __forceinline__ void load_padded_occ(const CondDev& c, float* dst) {
    const int R = c.R, P = padded_dim(R), n = P * P * P;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int ix = i / (P * P) - 1, iy = (i / P) % P - 1, iz = i % P - 1;
        const bool in = ix >= 0 && iy >= 0 && iz >= 0 && ix < R && iy < R && iz < R;
        dst[i] = in ? c.occ[(ix * R + iy) * R + iz] : 0.f;
    }
}

// probe_segment (conditioning.cpp:163-178), trilinear, on the padded grid.
// The segment p -> p + d is walked in voxel units; ST / RT > 0 specialise the
// sample count / resolution at compile time (fully unrolled, immediate
// corner offsets), 0 = runtime values.
template <int ST, int RT, bool CLAMP>
__device__ __forceinline__ void probe_walk(const float* occ, int R, int S, float b0, float b1, float b2, float s0,
                                           float s1, float s2, float& tr, float& sum) {
    const int P = padded_dim(R);
    const float hi = static_cast<float>(R);
    const float cidx = static_cast<float>(P * P + P + 1);  // the +1 border offset of each axis
    const float dt = S == 1 ? 0.f : 0.9f / static_cast<float>(S - 1);
#pragma unroll
    for (int s = 0; s < (ST > 0 ? ST : 1); ++s) {
        for (int si = (ST > 0 ? s : 0); si < (ST > 0 ? s + 1 : S); ++si) {
            const float t = S == 1 ? 0.5f : fmaf(static_cast<float>(si), dt, 0.05f);
            float u0 = fmaf(t, s0, b0), u1 = fmaf(t, s1, b1), u2 = fmaf(t, s2, b2);
            if (CLAMP) {
                u0 = fminf(fmaxf(u0, -1.f), hi);
                u1 = fminf(fmaxf(u1, -1.f), hi);
                u2 = fminf(fmaxf(u2, -1.f), hi);
            }
            const float f0 = floorf(u0), f1 = floorf(u1), f2 = floorf(u2);
            const float w0 = u0 - f0, w1 = u1 - f1, w2 = u2 - f2;
            // padded linear index, exact in FP32 (P^3 < 2^24)
            const int idx = static_cast<int>(
                fmaf(f0, static_cast<float>(P * P), fmaf(f1, static_cast<float>(P), f2 + cidx)));
            const float* q = occ + idx;
            const float c00 = fmaf(w2, q[1] - q[0], q[0]);
            const float c01 = fmaf(w2, q[P + 1] - q[P], q[P]);
            const float c10 = fmaf(w2, q[P * P + 1] - q[P * P], q[P * P]);
            const float c11 = fmaf(w2, q[P * P + P + 1] - q[P * P + P], q[P * P + P]);
            const float c0 = fmaf(w1, c01 - c00, c00);
            const float c1 = fmaf(w1, c11 - c10, c10);
            const float v = fmaf(w0, c1 - c0, c0);
            tr *= 1.f - v;
            sum += v;
        }
    }
}

template <int ST = 0, int RT = 0>
__device__ __forceinline__ void probe_padded(const CondDev& c, const float* occ, float px, float py, float pz,
                                             float dx, float dy, float dz, float& T, float& rho) {
    const int R = RT > 0 ? RT : c.R;
    const int S = ST > 0 ? ST : c.S;
    const float i0 = 1.f / c.cell[0], i1 = 1.f / c.cell[1], i2 = 1.f / c.cell[2];
    const float b0 = (px - c.lo[0]) * i0 - 0.5f, b1 = (py - c.lo[1]) * i1 - 0.5f, b2 = (pz - c.lo[2]) * i2 - 0.5f;
    const float s0 = dx * i0, s1 = dy * i1, s2 = dz * i2;
    float tr = 1.f, sum = 0.f;
    probe_walk<ST, RT, true>(occ, R, S, b0, b1, b2, s0, s1, s2, tr, sum);
    T = tr;
    rho = sum / static_cast<float>(S);
}

__device__ __forceinline__ float sample_near(const CondDev& c, const float* occ, float qx, float qy,
                                             float qz) {
    const int R = c.R;
    const int ix = static_cast<int>(floorf((qx - c.lo[0]) / c.cell[0]));
    const int iy = static_cast<int>(floorf((qy - c.lo[1]) / c.cell[1]));
    const int iz = static_cast<int>(floorf((qz - c.lo[2]) / c.cell[2]));
    if (ix < 0 || iy < 0 || iz < 0 || ix >= R || iy >= R || iz >= R) return 0.f;
    return occ[(ix * R + iy) * R + iz];
}

// Local features [v_hat, d, T, rho] (conditioning.cpp:377-396).  PADDED:
// occ is the (R+2)^3 zero-bordered copy (trilinear fast path); otherwise the
// plain R^3 grid.
template <bool PADDED = false, int ST = 0, int RT = 0>
__device__ __forceinline__ void local_features(const CondDev& c, const float* occ, float px,
                                               float py, float pz, float rx, float ry, float rz,
                                               float* in) {
    const float dx = rx - px, dy = ry - py, dz = rz - pz;
    const float d = sqrtf(dx * dx + dy * dy + dz * dz);
    const float inv = 1.f / d;
    in[0] = dx * inv;
    in[1] = dy * inv;
    in[2] = dz * inv;
    in[3] = d;
    float T = 1.f, rho = 0.f;
    if (PADDED && c.probe && !c.nearest) {
        probe_padded<ST, RT>(c, occ, px, py, pz, dx, dy, dz, T, rho);
    } else if (c.probe) {
        float sum = 0.f;
        for (int s = 0; s < c.S; ++s) {
            const float t = c.S == 1 ? 0.5f : 0.05f + 0.9f * static_cast<float>(s) / (c.S - 1);
            const float qx = px + dx * t, qy = py + dy * t, qz = pz + dz * t;
            float v;
            if (PADDED) {  // nearest lookup on the padded grid
                const int ix = static_cast<int>(floorf((qx - c.lo[0]) / c.cell[0]));
                const int iy = static_cast<int>(floorf((qy - c.lo[1]) / c.cell[1]));
                const int iz = static_cast<int>(floorf((qz - c.lo[2]) / c.cell[2]));
                const bool in_ = ix >= 0 && iy >= 0 && iz >= 0 && ix < c.R && iy < c.R && iz < c.R;
                v = in_ ? occ[padded_index(c.R, ix, iy, iz)] : 0.f;
            } else {
                v = c.nearest ? sample_near(c, occ, qx, qy, qz) : sample_tri(c, occ, qx, qy, qz);
            }
            T *= 1.f - v;
            sum += v;
        }
        rho = sum / c.S;
    }
    in[4] = T;
    in[5] = rho;
}

// Local MLP 6 -> H -> H -> 4C (mlp_forward :23-29) in FP32; y has 4C outputs.
template <int HT, int CT>
__device__ __forceinline__ void local_mlp(const CondDev& c, const LocalSmem& w, const float* in,
                                          float* y) {
    constexpr int HM = HT > 0 ? HT : kHMax;
    constexpr int YM = CT > 0 ? 4 * CT : 4 * kCMax;
    const int H = HT > 0 ? HT : c.H;
    const int NY = CT > 0 ? 4 * CT : 4 * c.C;
    float h1[HM];
#pragma unroll
    for (int o = 0; o < HM; ++o) {
        if (HT == 0 && o >= H) break;
        float acc = w.b1[o];
#pragma unroll
        for (int i = 0; i < 6; ++i) acc = fmaf(w.w1[o * 6 + i], in[i], acc);
        h1[o] = fmaxf(acc, 0.f);
    }
#pragma unroll
    for (int q = 0; q < YM; ++q)
        if (q < NY) y[q] = w.b3[q];
#pragma unroll 2
    for (int o = 0; o < H; ++o) {
        const float* row = w.w2 + o * H;
        float acc = w.b2[o];
        if (HT > 0) {
#pragma unroll
            for (int i = 0; i < HM; i += 4) {
                const float4 wv = *reinterpret_cast<const float4*>(row + i);
                acc = fmaf(wv.x, h1[i], acc);
                acc = fmaf(wv.y, h1[i + 1], acc);
                acc = fmaf(wv.z, h1[i + 2], acc);
                acc = fmaf(wv.w, h1[i + 3], acc);
            }
        } else {
            for (int i = 0; i < H; ++i) acc = fmaf(row[i], h1[i], acc);
        }
        const float h2 = fmaxf(acc, 0.f);
#pragma unroll
        for (int q = 0; q < YM; ++q)
            if (q < NY) y[q] = fmaf(w.w3[q * H + o], h2, y[q]);
    }
}

// local_mlp<64, 1> on W2 transposed into output pairs, w2t2[i][o / 2] =
// (W2[o][i], W2[o + 1][i]): eight outputs at a time as four independent
// FFMA2 chains (the row kernel's pattern); per output the sum still runs
// over i in ascending order with fmaf, so the result is bit-identical.
__device__ __forceinline__ void local_mlp64_t(const LocalSmem& w, const float2* __restrict__ w2t2, const float* in,
                                              float* y) {
    constexpr int H = 64;
    float h1[H];
#pragma unroll
    for (int o = 0; o < H; ++o) {
        float acc = w.b1[o];
#pragma unroll
        for (int i = 0; i < 6; ++i) acc = fmaf(w.w1[o * 6 + i], in[i], acc);
        h1[o] = fmaxf(acc, 0.f);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) y[q] = w.b3[q];
#pragma unroll 1
    for (int op0 = 0; op0 < H / 2; op0 += 4) {  // output pairs op0 .. op0 + 3 (outputs 2 op0 .. 2 op0 + 7)
        float2 ac[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) ac[u] = make_float2(w.b2[2 * (op0 + u)], w.b2[2 * (op0 + u) + 1]);
#pragma unroll
        for (int i = 0; i < H; ++i) {
            const float4* wq = reinterpret_cast<const float4*>(w2t2 + i * (H / 2) + op0);
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
#pragma unroll
            for (int q = 0; q < 4; ++q) y[q] = fmaf(w.w3[q * H + o], hv0, y[q]);
#pragma unroll
            for (int q = 0; q < 4; ++q) y[q] = fmaf(w.w3[q * H + o + 1], hv1, y[q]);
        }
    }
}

// Store one signal value (k, j, channel ch) in the requested format.
__device__ __forceinline__ void store_sig(const SigOut& o, int k, int n_rx, int j, int C, int ch, float2 v) {
    const size_t i = (static_cast<size_t>(k) * n_rx + j) * C + ch;
    if (o.split) {  // C == 1
        uint32_t h, l;
        asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(v.y), "f"(v.x));
        const float hx = __uint_as_float(h << 16), hy = __uint_as_float(h & 0xFFFF0000u);
        asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(l) : "f"(v.y - hy), "f"(v.x - hx));
        o.split[i] = make_uint2(h, l);
    } else {
        o.f2[i] = v;
    }
}

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// The receiver-dependent but MLP-independent half of the fused signal:
// M = sum_l [(1+aG_l) GB_l + bG_l B_l] = sum_l mid_l B_l and Bs = sum_l B_l.
__device__ __forceinline__ void fle_reduce(int k, int j, int ch, int L, int C, const float2* __restrict__ B,
                                           const float2* __restrict__ GB, const float* __restrict__ ag, float2& M,
                                           float2& Bs) {
    M = make_float2(0.f, 0.f);
    Bs = make_float2(0.f, 0.f);
    const float4* a4 = reinterpret_cast<const float4*>(ag) + static_cast<size_t>(j) * L * C + ch;
    for (int l = 0; l < L; ++l) {
        const float2 b = B[static_cast<size_t>(k) * L + l];
        const float2 gb = GB[(static_cast<size_t>(k) * L + l) * C + ch];
        const float4 a = a4[static_cast<size_t>(l) * C];
        const float2 t0 = cmul(make_float2(1.f + a.x, a.y), gb), t1 = cmul(make_float2(a.z, a.w), b);
        M.x += t0.x + t1.x;
        M.y += t0.y + t1.y;
        Bs.x += b.x;
        Bs.y += b.y;
    }
}

// s = (1+aL) M + bL Bs, y = local MLP output (4C) for channel ch.
__device__ __forceinline__ float2 local_affine(const CondDev& c, int ch, float2 M, float2 Bs, const float* y) {
    const float ar = c.additive ? 0.f : y[4 * ch], ai = c.additive ? 0.f : y[4 * ch + 1];
    const float2 s0 = cmul(make_float2(1.f + ar, ai), M);
    const float2 s1 = cmul(make_float2(y[4 * ch + 2], y[4 * ch + 3]), Bs);
    return make_float2(s0.x + s1.x, s0.y + s1.y);
}

// s = (1+aL) * sum_l[(1+aG_l) GB_l + bG_l B_l] + bL * sum_l B_l for one
// (Gaussian k, receiver j, channel ch); y = local MLP output (4C).
__device__ __forceinline__ float2 fused_signal(const CondDev& c, int k, int j, int ch, int L, int C,
                                               const float2* __restrict__ B, const float2* __restrict__ GB,
                                               const float* __restrict__ ag, const float* y) {
    float2 M, Bs;
    fle_reduce(k, j, ch, L, C, B, GB, ag, M, Bs);
    return local_affine(c, ch, M, Bs, y);
}

// ---- the same probes on the trilinear cell table (RXGS_PROBE_CUBE): one
// 256-bit read-only load per sample (the cell's 8 polynomial coefficients,
// k_occ_cubes) and v = (a + w0 b + w1 (c + w0 e)) + w2 (d + w0 f + w1 (g + w0 h))
// in three FFMA2 + one FFMA, instead of 8 shared-memory corner loads and 7
// lerps.  Cells are [-1, R]^3, i.e. exactly the padded grid's cell range.
__device__ __forceinline__ float cube_eval(const float* cell, float w0, float w1, float w2) {
    float c0, c1, c2, c3, c4, c5, c6, c7;
    asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(c0), "=f"(c1), "=f"(c2), "=f"(c3), "=f"(c4), "=f"(c5), "=f"(c6), "=f"(c7)
        : "l"(cell));
    const float2 x13 = x2::fma(x2::bc(w0), make_float2(c2, c3), make_float2(c0, c1));  // (a + w0 b, d + w0 f)
    const float2 x24 = x2::fma(x2::bc(w0), make_float2(c6, c7), make_float2(c4, c5));  // (c + w0 e, g + w0 h)
    const float2 y = x2::fma(x2::bc(w1), x24, x13);
    return fmaf(w2, y.y, y.x);
}

template <int ST, int RT, int P0, int P1>
__device__ __forceinline__ void probe_pairs_cube(const float* __restrict__ cube, float b0, float b1, float b2,
                                                 float s0, float s1, float s2, float2& tr2, float2& sum2) {
    static_assert(ST >= 2 && ST % 2 == 0 && RT > 0, "paired probe needs an even, static sample count");
    constexpr int P = RT + 2;
    constexpr float cidx = static_cast<float>(P * P + P + 1);
    constexpr float dt = 0.9f / static_cast<float>(ST - 1);
#pragma unroll
    for (int sp = P0; sp < P1; ++sp) {
        const float2 t = make_float2(fmaf(static_cast<float>(2 * sp), dt, 0.05f),
                                     fmaf(static_cast<float>(2 * sp + 1), dt, 0.05f));
        const float2 u0 = x2::fma(t, x2::bc(s0), x2::bc(b0));
        const float2 u1 = x2::fma(t, x2::bc(s1), x2::bc(b1));
        const float2 u2 = x2::fma(t, x2::bc(s2), x2::bc(b2));
        const float2 f0 = make_float2(floorf(u0.x), floorf(u0.y));
        const float2 f1 = make_float2(floorf(u1.x), floorf(u1.y));
        const float2 f2 = make_float2(floorf(u2.x), floorf(u2.y));
        const float2 w0 = x2::sub(u0, f0), w1 = x2::sub(u1, f1), w2 = x2::sub(u2, f2);
        const float2 fi = x2::fma(f0, x2::bc(static_cast<float>(P * P)),
                                  x2::fma(f1, x2::bc(static_cast<float>(P)), x2::add(f2, x2::bc(cidx))));
        const float va = cube_eval(cube + 8 * static_cast<int>(fi.x), w0.x, w1.x, w2.x);
        const float vb = cube_eval(cube + 8 * static_cast<int>(fi.y), w0.y, w1.y, w2.y);
        const float2 v = make_float2(va, vb);
        tr2 = x2::mul(tr2, x2::sub(x2::bc(1.f), v));
        sum2 = x2::add(sum2, v);
    }
}

template <int ST, int RT, bool CLAMP>
__device__ __forceinline__ void probe_seg_cube(const float* __restrict__ cube, int R, int S, float b0, float b1,
                                               float b2, float s0, float s1, float s2, float& tr, float& sum) {
    const int P = (RT > 0 ? RT : R) + 2;
    const float hi = static_cast<float>(RT > 0 ? RT : R);
    const float cidx = static_cast<float>(P * P + P + 1);
    const int NS = ST > 0 ? ST : S;
    const float dt = NS == 1 ? 0.f : 0.9f / static_cast<float>(NS - 1);
#pragma unroll 1
    for (int si = 0; si < NS; ++si) {
        const float t = NS == 1 ? 0.5f : fmaf(static_cast<float>(si), dt, 0.05f);
        float u0 = fmaf(t, s0, b0), u1 = fmaf(t, s1, b1), u2 = fmaf(t, s2, b2);
        if (CLAMP) {
            u0 = fminf(fmaxf(u0, -1.f), hi);
            u1 = fminf(fmaxf(u1, -1.f), hi);
            u2 = fminf(fmaxf(u2, -1.f), hi);
        }
        const float f0 = floorf(u0), f1 = floorf(u1), f2 = floorf(u2);
        const int idx = static_cast<int>(fmaf(f0, static_cast<float>(P * P), fmaf(f1, static_cast<float>(P), f2 + cidx)));
        const float v = cube_eval(cube + 8 * idx, u0 - f0, u1 - f1, u2 - f2);
        tr *= 1.f - v;
        sum += v;
    }
}


// Local features [v_hat, d, T, rho] of one (Gaussian, receiver) with the
// occupancy probe on the trilinear cell table (as the tcgen05 kernel: the
// paired fast path when the whole warp's segments lie inside the grid); the
// generic probe for nearest lookup.  Called by every lane (warp vote);
// inactive lanes get dummy features.  Used by the training forward and
// backward, so both see the same features.
template <int ST, int RT>
__device__ __forceinline__ void cube_features(const CondDev& c, bool active, float4 pk, float qx, float qy, float qz,
                                             float* x) {
    const bool cube = c.probe && !c.nearest && c.cube != nullptr;
    if (!cube) {
        if (active) local_features<false>(c, c.occ, pk.x, pk.y, pk.z, qx, qy, qz, x);
        return;
    }
    const float px = active ? pk.x : 0.f, py = active ? pk.y : 0.f, pz = active ? pk.z : 0.f;
    if (!active) {
        qx = 1.f;
        qy = qz = 0.f;
    }
    const float dx = qx - px, dy = qy - py, dz = qz - pz;
    const float d = sqrtf(dx * dx + dy * dy + dz * dz);
    const float inv = 1.f / d;
    x[0] = dx * inv;
    x[1] = dy * inv;
    x[2] = dz * inv;
    x[3] = d;
    float ic[3], bl[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        ic[a] = 1.f / c.cell[a];
        bl[a] = __fadd_rn(__fmul_rn(c.lo[a], ic[a]), 0.5f);
    }
    const float b0 = fmaf(px, ic[0], -bl[0]), b1 = fmaf(py, ic[1], -bl[1]), b2 = fmaf(pz, ic[2], -bl[2]);
    const float s0 = dx * ic[0], s1 = dy * ic[1], s2 = dz * ic[2];
    const int R = RT > 0 ? RT : c.R, S = ST > 0 ? ST : c.S;
    const float hiR = static_cast<float>(R);
    const float tlast = S == 1 ? 0.5f : fmaf(static_cast<float>(S - 1), 0.9f / static_cast<float>(S - 1), 0.05f);
    const float tfirst = S == 1 ? 0.5f : 0.05f;
    auto inside = [&](float t) {
        const float u0 = fmaf(t, s0, b0), u1 = fmaf(t, s1, b1), u2 = fmaf(t, s2, b2);
        return u0 >= -1.f && u0 <= hiR && u1 >= -1.f && u1 <= hiR && u2 >= -1.f && u2 <= hiR;
    };
    const bool ok = !active || (inside(tfirst) && inside(tlast));
    float tr = 1.f, sum = 0.f;
    if (__all_sync(0xffffffffu, ok)) {
        if constexpr (ST >= 2 && ST % 2 == 0 && RT > 0) {
            float2 tr2 = make_float2(1.f, 1.f), sum2 = make_float2(0.f, 0.f);
            if (active) probe_pairs_cube<ST, RT, 0, ST / 2>(c.cube, b0, b1, b2, s0, s1, s2, tr2, sum2);
            tr = tr2.x * tr2.y;
            sum = sum2.x + sum2.y;
        } else {
            if (active) probe_seg_cube<ST, RT, false>(c.cube, R, S, b0, b1, b2, s0, s1, s2, tr, sum);
        }
    } else if (active) {
        probe_seg_cube<ST, RT, true>(c.cube, R, S, b0, b1, b2, s0, s1, s2, tr, sum);
    }
    x[4] = tr;
    x[5] = sum * (1.f / static_cast<float>(S));
}


// activations per row as bf16 hi/lo feature planes act[plane][f][row]
// (hi = bf16(v), lo = bf16(v - hi)); the feature order groups the operands
// of k_cond_grads_tc's two GEMMs over rows: [dh2 | dh1] (A of GEMM 1),
// [h1 | x] (B of GEMM 1), h2 (A of GEMM 2), dy (B of GEMM 2)
constexpr int kActF = 4 * 64 + 6 + 4;  // activation features per row
constexpr int kAdh2 = 0, kAdh1 = 64, kAh1 = 128, kAx = 192, kAh2 = 198, kAdy = 262;
constexpr int kActRowAlign = 64;       // rows padded to the grads kernel's K chunk

__device__ __forceinline__ uint32_t act_bf16(float v) {  // bf16 round to nearest, in the low half
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(0.f), "f"(v));
    return r;
}
struct ActOut {
    uint16_t* p;
    long long rpad;
    __device__ __forceinline__ void put(long long row, int f, float v) const {
        const uint32_t h = act_bf16(v) & 0xFFFFu;
        const uint32_t l = act_bf16(v - __uint_as_float(h << 16)) & 0xFFFFu;
        p[static_cast<size_t>(f) * rpad + row] = static_cast<uint16_t>(h);
        p[static_cast<size_t>(kActF + f) * rpad + row] = static_cast<uint16_t>(l);
    }
    // a value already split into bf16 hi / lo
    __device__ __forceinline__ void put_bits(long long row, int f, uint32_t hi16, uint32_t lo16) const {
        p[static_cast<size_t>(f) * rpad + row] = static_cast<uint16_t>(hi16);
        p[static_cast<size_t>(kActF + f) * rpad + row] = static_cast<uint16_t>(lo16);
    }
};


}  // namespace cond_dev
}  // namespace rxgs_b200
