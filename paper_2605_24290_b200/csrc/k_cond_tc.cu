// Conditioning hot kernel on the 5th-gen tensor cores (tcgen05 + TMEM).
//
// Same math as k_cond_signal (k_cond.cu): per (Gaussian k, receiver j) row
// the local features + occupancy probe, the local MLP 6 -> 64 -> 64 -> 4 and
// the fused affine + FLE reduction (conditioning.cpp:369-421 with
// reduce_signals, sphraster.cpp:190-226).  The 64x64 hidden layer (86% of
// the MLP FLOPs) runs on tcgen05:
//   * a CTA owns the whole SM (512 threads = 4 independent 128-row groups);
//     each group's 128 rows map 1:1 to the 128 TMEM lanes;
//   * every thread writes its row of h1 = relu(W1 x + b1), split into bf16
//     hi + lo parts, straight into TMEM with tcgen05.st (A operand in TMEM:
//     no shared-memory staging);
//   * W2 (hi/lo, bf16, no-swizzle K-major core matrices) sits in shared
//     memory for the whole kernel;
//   * one elected thread per group issues 12 tcgen05.mma (4 K-steps x
//     {hi*hi, hi*lo, lo*hi}: ~2^-17 relative error, FP32-class accuracy for
//     the 1e-4 parity bar) into a 64-column FP32 accumulator, commits to the
//     group's mbarrier; the group reads the accumulator back with tcgen05.ld;
//   * layers 1 and 3 and the biases are FFMAs with constant-bank operands
//     (the weights travel as a __grid_constant__ kernel parameter);
//   * while one group waits on its MMAs the other three run their SIMT parts.
// TMEM: 512 columns per CTA = 4 groups x (64 accumulator + 32 A-hi + 32 A-lo).
// Shared memory: W2 hi/lo (16 KB) + the occupancy grid (R^3 FP32, 128 KB).
#include "cond_common.cuh"
#include "rxgs_internal.cuh"
#include "tc_util.cuh"

namespace rxgs_b200 {
namespace {

using namespace cond_dev;

constexpr int kH = 64;
constexpr int kGroups = 4;
constexpr int kThreads = 128 * kGroups;
constexpr uint32_t kIdesc = tc::idesc_bf16_f32(128, kH);
constexpr int kW2Bytes = kH * kH * 2;  // one bf16 64x64 matrix
constexpr int kW1Bytes = kH * 16 * 2;  // one bf16 64x16 matrix

struct LocalW {
    float w1[kH * 6];
    float b1[kH];
    float b2[kH];
    float w3[4 * kH];
    float b3[4];
};

// byte offset of element (row r, k) in a no-swizzle K-major canonical tile
// with 64 K-elements per row: core matrices of 8 rows x 8 k (128 B), K-chunks
// contiguous (LBO = 128 B), 8-row groups 1 KB apart (SBO = 1024 B).
__device__ __forceinline__ uint32_t canon_off(int r, int k) {
    return static_cast<uint32_t>(((r >> 3) * 8 + (k >> 3)) * 128 + (r & 7) * 16 + (k & 7) * 2);
}

// byte offset of element (row r, k) in a no-swizzle K-major tile with 16
// K-elements per row (2 K-chunks): LBO = 128 B, SBO = 256 B.
__device__ __forceinline__ uint32_t canon_off16(int r, int k) {
    return static_cast<uint32_t>(((r >> 3) * 2 + (k >> 3)) * 128 + (r & 7) * 16 + (k & 7) * 2);
}

__device__ __forceinline__ void split_store(uint8_t* hi_base, uint8_t* lo_base, uint32_t off, float w) {
    const float hi = tc::bf16_round(w);
    *reinterpret_cast<uint16_t*>(hi_base + off) = static_cast<uint16_t>(tc::pack_bf16(hi, 0.f) & 0xFFFFu);
    *reinterpret_cast<uint16_t*>(lo_base + off) = static_cast<uint16_t>(tc::pack_bf16(w - hi, 0.f) & 0xFFFFu);
}

// YOUT: rows are all K Gaussians (vis unused) and the local-branch output
// y = (alpha_L, beta_L) is written to ycache[k][j] instead of the signal (the
// Tx-independent cache of the coverage workload).
template <int ST, int RT, bool YOUT>
__global__ void __launch_bounds__(kThreads, 1)
    k_cond_tc(const __grid_constant__ LocalW W, CondDev c, const int* __restrict__ n_rows, const int* __restrict__ vis,
              const float4* __restrict__ pos32, const double* __restrict__ rx, int n_rx,
              const float2* __restrict__ Bm, const float2* __restrict__ GB, const float* __restrict__ ag,
              float2* __restrict__ sig, float4* __restrict__ ycache, int n_all) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* w2hi = smem;
    uint8_t* w2lo = smem + kW2Bytes;
    uint8_t* w1hi = smem + 2 * kW2Bytes;           // [W1 | b1 | 0] : 64 x 16 bf16
    uint8_t* w1lo = w1hi + kW1Bytes;
    float* s_occ = reinterpret_cast<float*>(smem + 2 * kW2Bytes + 2 * kW1Bytes);
    __shared__ uint64_t bars[kGroups];
    __shared__ uint32_t tbase_s;

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int g = warp >> 2, wl = warp & 3;

    // ---- one-time setup: W1 (+bias column) and W2 as bf16 hi/lo core matrices, occupancy
    for (int i = tid; i < kH * kH; i += kThreads) split_store(w2hi, w2lo, canon_off(i / kH, i % kH), c.p32[c.o_lw2 + i]);
    for (int i = tid; i < kH * 16; i += kThreads) {
        const int n = i / 16, k = i % 16;
        const float w = k < 6 ? c.p32[c.o_lw1 + n * 6 + k] : (k == 6 ? c.p32[c.o_lb1 + n] : 0.f);
        split_store(w1hi, w1lo, canon_off16(n, k), w);
    }
    if (c.probe) load_padded_occ(c, s_occ);
    if (warp == 0) {
        tc::tmem_alloc(&tbase_s, 512);
        tc::tmem_relinquish();
    }
    if (tid == 0) {
        for (int q = 0; q < kGroups; ++q) tc::mbar_init(&bars[q], 1);
        tc::fence_mbar_init();
    }
    tc::fence_proxy_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();

    const uint32_t tbase = tbase_s;
    const uint32_t lane_off = static_cast<uint32_t>(32 * wl) << 16;
    const uint32_t tm_d = tbase + 128 * g;       // 64 f32 columns (layer-1 then layer-2 accumulator)
    const uint32_t tm_ahi = tm_d + 64;           // 32 columns = 64 bf16 (layer-1 A uses the first 8)
    const uint32_t tm_alo = tm_d + 96;
    const uint32_t w2hi_a = tc::smem_u32(w2hi), w2lo_a = tc::smem_u32(w2lo);
    const uint32_t w1hi_a = tc::smem_u32(w1hi), w1lo_a = tc::smem_u32(w1lo);

    const int n_jc = (n_rx + 31) >> 5;
    const long long items = static_cast<long long>(YOUT ? n_all : *n_rows) * n_jc;
    const long long tiles = (items + 3) >> 2;
    const long long step = static_cast<long long>(gridDim.x) * kGroups;
    const int L = c.L;
    uint32_t phase = 0;

    for (long long tile = static_cast<long long>(blockIdx.x) * kGroups + g; tile < tiles; tile += step) {
        const long long item = tile * 4 + wl;
        const bool valid_item = item < items;
        const int vi = valid_item ? static_cast<int>(item / n_jc) : 0;
        const int jc = valid_item ? static_cast<int>(item % n_jc) : 0;
        const int j = jc * 32 + lane;
        const bool active = valid_item && j < n_rx;
        const int k = valid_item ? (YOUT ? vi : vis[vi]) : 0;

        float in[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (active) {
            const float4 pk = pos32[k];
            local_features<true, ST, RT>(c, s_occ, pk.x, pk.y, pk.z, static_cast<float>(rx[3 * j]),
                                         static_cast<float>(rx[3 * j + 1]), static_cast<float>(rx[3 * j + 2]), in);
        }
        // ---- layer 1 on the tensor cores: A1 = [x, 1, 0...] (K = 16) hi/lo -> TMEM
        {
            uint32_t hi[8], lo[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const float xa = 2 * q < 6 ? in[2 * q] : (2 * q == 6 ? 1.f : 0.f);
                const float xb = 2 * q + 1 < 6 ? in[2 * q + 1] : 0.f;
                hi[q] = tc::pack_bf16(xa, xb);
                lo[q] = tc::pack_bf16(xa - __uint_as_float(hi[q] << 16), xb - __uint_as_float(hi[q] & 0xFFFF0000u));
            }
            tc::tmem_st8(tm_ahi + lane_off, hi);
            tc::tmem_st8(tm_alo + lane_off, lo);
        }
        tc::wait_st();
        tc::fence_before_sync();
        tc::named_bar_sync(1 + g, 128);
        if (wl == 0 && lane == 0) {
            tc::fence_after_sync();
            const uint64_t bh = tc::sdesc_kmajor_noswizzle(w1hi_a, 128, 256);
            const uint64_t bl = tc::sdesc_kmajor_noswizzle(w1lo_a, 128, 256);
            tc::mma_ts(tm_d, tm_ahi, bh, kIdesc, 0u);
            tc::mma_ts(tm_d, tm_ahi, bl, kIdesc, 1u);
            tc::mma_ts(tm_d, tm_alo, bh, kIdesc, 1u);
            tc::mma_commit(&bars[g]);
        }
        tc::mbar_wait(&bars[g], phase);
        phase ^= 1u;
        tc::fence_after_sync();
        // ---- ReLU(h1) -> bf16 hi/lo -> TMEM (layer-2 A operand; overwrites A1)
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
            uint32_t r[16];
            tc::tmem_ld16(tm_d + lane_off + 16 * ch, r);
            tc::wait_ld();
            uint32_t hi[8], lo[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const float ha = fmaxf(__uint_as_float(r[2 * q]), 0.f);
                const float hb = fmaxf(__uint_as_float(r[2 * q + 1]), 0.f);
                hi[q] = tc::pack_bf16(ha, hb);
                lo[q] = tc::pack_bf16(ha - __uint_as_float(hi[q] << 16), hb - __uint_as_float(hi[q] & 0xFFFF0000u));
            }
            tc::tmem_st8(tm_ahi + lane_off + 8 * ch, hi);
            tc::tmem_st8(tm_alo + lane_off + 8 * ch, lo);
        }
        tc::wait_st();
        tc::fence_before_sync();
        tc::named_bar_sync(1 + g, 128);
        // ---- layer 2 on the tensor cores: D = Ahi Bhi + Ahi Blo + Alo Bhi
        if (wl == 0 && lane == 0) {
            tc::fence_after_sync();
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                const uint64_t bh = tc::sdesc_kmajor_noswizzle(w2hi_a + 256 * s, 128, 1024);
                const uint64_t bl = tc::sdesc_kmajor_noswizzle(w2lo_a + 256 * s, 128, 1024);
                tc::mma_ts(tm_d, tm_ahi + 8 * s, bh, kIdesc, s > 0 ? 1u : 0u);
                tc::mma_ts(tm_d, tm_ahi + 8 * s, bl, kIdesc, 1u);
                tc::mma_ts(tm_d, tm_alo + 8 * s, bh, kIdesc, 1u);
            }
            tc::mma_commit(&bars[g]);
        }
        // FLE reduction (global loads) overlaps the layer-2 MMAs
        tc::mbar_wait(&bars[g], phase);
        phase ^= 1u;
        tc::fence_after_sync();
        // ---- layer-2 bias + ReLU, layer 3 (FFMA) from the TMEM accumulator
        float y[4] = {W.b3[0], W.b3[1], W.b3[2], W.b3[3]};
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
            uint32_t r[16];
            tc::tmem_ld16(tm_d + lane_off + 16 * ch, r);
            tc::wait_ld();
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const int o = 16 * ch + q;
                const float h2 = fmaxf(__uint_as_float(r[q]) + W.b2[o], 0.f);
#pragma unroll
                for (int t = 0; t < 4; ++t) y[t] = fmaf(W.w3[t * kH + o], h2, y[t]);
            }
        }
        tc::fence_before_sync();  // the next tile's layer-1 MMA overwrites D after the barrier
        if (YOUT) {
            if (active) ycache[static_cast<size_t>(k) * n_rx + j] = make_float4(y[0], y[1], y[2], y[3]);
        } else if (active) {  // FLE reduction after the MMAs (measured faster than overlapping them)
            float2 M, Bs;
            fle_reduce(k, j, 0, L, 1, Bm, GB, ag, M, Bs);
            sig[static_cast<size_t>(k) * n_rx + j] = local_affine(c, 0, M, Bs, y);
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tbase, 512);
}

// ------------------------------------------------------------------ self test
// 128x64x64 bf16 GEMM through both operand paths (A in TMEM and A in shared
// memory) against FP32 FMA of the same bf16 values.
__global__ void __launch_bounds__(128) k_tc_selftest(float* __restrict__ err, int mode) {
    __shared__ __align__(1024) uint8_t sB[kW2Bytes];
    __shared__ __align__(1024) uint8_t sA[128 * kH * 2];
    __shared__ uint64_t bar;
    __shared__ uint32_t tb;
    const int tid = threadIdx.x, warp = tid >> 5;
    // mode 0: smooth values; mode 1: small integers (products and sums exact in FP32)
    auto Aval = [mode](int m, int k) {
        return mode ? static_cast<float>((m + 3 * k) % 5 - 2) : tc::bf16_round(sinf(0.37f * m + 0.11f * k));
    };
    auto Bval = [mode](int n, int k) {
        return mode ? static_cast<float>((2 * n + k) % 7 - 3) : tc::bf16_round(cosf(0.23f * n - 0.07f * k));
    };
    for (int i = tid; i < kH * kH; i += 128) {
        const int n = i / kH, k = i % kH;
        *reinterpret_cast<uint16_t*>(sB + canon_off(n, k)) =
            static_cast<uint16_t>(tc::pack_bf16(Bval(n, k), 0.f) & 0xFFFFu);
    }
    for (int i = tid; i < 128 * kH; i += 128) {
        const int m = i / kH, k = i % kH;
        *reinterpret_cast<uint16_t*>(sA + canon_off(m, k)) =
            static_cast<uint16_t>(tc::pack_bf16(Aval(m, k), 0.f) & 0xFFFFu);
    }
    if (warp == 0) {
        tc::tmem_alloc(&tb, 256);
        tc::tmem_relinquish();
    }
    if (tid == 0) {
        tc::mbar_init(&bar, 1);
        tc::fence_mbar_init();
    }
    tc::fence_proxy_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t base = tb;
    const uint32_t lo = static_cast<uint32_t>(32 * warp) << 16;
    // A row tid into TMEM columns [128, 160)
#pragma unroll
    for (int c0 = 0; c0 < 32; c0 += 8) {
        uint32_t r[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) r[q] = tc::pack_bf16(Aval(tid, 2 * (c0 + q)), Aval(tid, 2 * (c0 + q) + 1));
        tc::tmem_st8(base + lo + 128 + c0, r);
    }
    tc::wait_st();
    tc::fence_before_sync();
    __syncthreads();
    if (tid == 0) {
        tc::fence_after_sync();
        const uint32_t ba = tc::smem_u32(sB), aa = tc::smem_u32(sA);
        for (int s = 0; s < 4; ++s) {
            tc::mma_ts(base + 0, base + 128 + 8 * s, tc::sdesc_kmajor_noswizzle(ba + 256 * s, 128, 1024), kIdesc,
                       s > 0);
            tc::mma_ss(base + 64, tc::sdesc_kmajor_noswizzle(aa + 256 * s, 128, 1024),
                       tc::sdesc_kmajor_noswizzle(ba + 256 * s, 128, 1024), kIdesc, s > 0);
        }
        tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, 0);
    tc::fence_after_sync();
    float e_ts = 0.f, e_ss = 0.f;
    for (int c0 = 0; c0 < kH; c0 += 16) {
        uint32_t r[16], r2[16];
        tc::tmem_ld16(base + lo + c0, r);
        tc::tmem_ld16(base + lo + 64 + c0, r2);
        tc::wait_ld();
        for (int q = 0; q < 16; ++q) {
            const int n = c0 + q;
            float ref = 0.f;
            for (int k = 0; k < kH; ++k) {  // from the stored bf16 operands
                const float a = __uint_as_float(static_cast<uint32_t>(*reinterpret_cast<const uint16_t*>(sA + canon_off(tid, k))) << 16);
                const float b = __uint_as_float(static_cast<uint32_t>(*reinterpret_cast<const uint16_t*>(sB + canon_off(n, k))) << 16);
                ref = fmaf(a, b, ref);
            }
            e_ts = fmaxf(e_ts, fabsf(__uint_as_float(r[q]) - ref));
            e_ss = fmaxf(e_ss, fabsf(__uint_as_float(r2[q]) - ref));
        }
    }
    atomicMax(reinterpret_cast<int*>(err), __float_as_int(e_ts));
    atomicMax(reinterpret_cast<int*>(err) + 1, __float_as_int(e_ss));
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(base, 256);
}

}  // namespace

bool cond_tc_eligible(const rxgs_cond_s* c) {
    return c && c->use_local() && c->hidden == kH && c->C == 1 && padded_dim(c->R) * padded_dim(c->R) * padded_dim(c->R) <= 48000;
}

namespace {

template <bool YOUT>
cudaError_t launch_tc(const rxgs_cond_s& cs, const rxgs_scene_s& sc, const int* n_rows, const int* vis,
                      long long rows_host, const double* d_rx, int n_rx, const float2* basis32, const float2* gb32,
                      const float* d_ag, float2* d_sig, float4* ycache, cudaStream_t s) {
    if (rows_host == 0 || n_rx == 0) return cudaSuccess;
    const CondDev d = make_dev(cs);
    LocalW w{};
    const std::vector<double>& p = cs.h_params;
    for (int i = 0; i < kH * 6; ++i) w.w1[i] = static_cast<float>(p[cs.o_lw1 + i]);
    for (int i = 0; i < kH; ++i) {
        w.b1[i] = static_cast<float>(p[cs.o_lb1 + i]);
        w.b2[i] = static_cast<float>(p[cs.o_lb2 + i]);
    }
    for (int i = 0; i < 4 * kH; ++i) w.w3[i] = static_cast<float>(p[cs.o_lw3 + i]);
    for (int i = 0; i < 4; ++i) w.b3[i] = static_cast<float>(p[cs.o_lb3 + i]);
    const size_t P = static_cast<size_t>(padded_dim(d.R));
    const size_t smem = 2 * kW2Bytes + 2 * kW1Bytes + (d.probe ? P * P * P * sizeof(float) : 0);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long items = rows_host * ((n_rx + 31) / 32);
    const long long tiles = (items + 3) / 4;
    const long long want = (tiles + kGroups - 1) / kGroups;
    const int blocks = static_cast<int>(want < sms ? want : sms);
    const bool fast = d.S == 16 && d.R == 32 && !d.nearest;
    auto kern = fast ? k_cond_tc<16, 32, YOUT> : k_cond_tc<0, 0, YOUT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    kern<<<blocks, kThreads, smem, s>>>(w, d, n_rows, vis, sc.d_pos32.as<float4>(), d_rx, n_rx, basis32, gb32, d_ag,
                                        d_sig, ycache, static_cast<int>(rows_host));
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_cond_signal_tc(const rxgs_cond_s& cs, const rxgs_scene_s& sc, const rxgs_txstate_s& st,
                                  const double* d_rx, int n_rx, const float* d_ag, float2* d_sig,
                                  cudaStream_t s) {
    return launch_tc<false>(cs, sc, st.needed_count.as<int>(), st.needed_order.as<int>(), st.visible, d_rx, n_rx,
                            st.basis32.as<float2>(), st.gb32.as<float2>(), d_ag, d_sig, nullptr, s);
}

cudaError_t launch_local_cache_tc(const rxgs_cond_s& cs, const rxgs_scene_s& sc, const double* d_rx, int n_rx,
                                  float4* ycache, cudaStream_t s) {
    return launch_tc<true>(cs, sc, nullptr, nullptr, sc.k, d_rx, n_rx, nullptr, nullptr, nullptr, nullptr, ycache, s);
}

cudaError_t launch_tc_selftest(float* d_err, cudaStream_t s) {
    k_tc_selftest<<<1, 128, 0, s>>>(d_err, 0);
    k_tc_selftest<<<1, 128, 0, s>>>(d_err + 2, 1);
    return cudaGetLastError();
}

}  // namespace rxgs_b200
