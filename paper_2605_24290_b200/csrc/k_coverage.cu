// Coverage table (BASELINE config 3: n_tx transmitters x n_rx receivers ->
// RSSI).  The local conditioning branch has no transmitter input
// (conditioning.cpp:369-421), so its output y = (alpha_L, beta_L) per
// (Gaussian, receiver) is computed once and kept in HBM (K x N float4); the
// global branch (alpha_G, beta_G) per receiver likewise.  Per transmitter only
// the factorised signal remains:
//   s = (1+alpha_L) sum_l [(1+alpha_G,l) B_l base_l + beta_G,l B_l] + beta_L sum_l B_l
// which k_cov_signal evaluates for the Tx's needed Gaussians, followed by
// the tcgen05 compositor in RSSI-only mode.
//   k_ycache_simt  local-branch cache for configurations the tcgen05 kernel
//                  does not cover (hidden != 64); FP32 SIMT
//   k_cov_signal   per (needed Gaussian, receiver) signal from the caches
#include "cond_common.cuh"
#include "rxgs_internal.cuh"
#include "f32x2.cuh"

namespace rxgs_b200 {
namespace {

using namespace cond_dev;

__global__ void k_ycache_simt(CondDev c, int K, const float4* __restrict__ pos32, const double* __restrict__ rx,
                              int n_rx, float4* __restrict__ ycache) {
    const long long row = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (row >= static_cast<long long>(K) * n_rx) return;
    const int k = static_cast<int>(row / n_rx), j = static_cast<int>(row % n_rx);
    const float* p = c.p32;
    LocalSmem w{c.occ, p + c.o_lw1, p + c.o_lb1, p + c.o_lw2, p + c.o_lb2, p + c.o_lw3, p + c.o_lb3};
    const float4 pk = pos32[k];
    float in[6], y[4 * kCMax];
    local_features<false>(c, c.occ, pk.x, pk.y, pk.z, static_cast<float>(rx[3 * j]), static_cast<float>(rx[3 * j + 1]),
                          static_cast<float>(rx[3 * j + 2]), in);
    local_mlp<0, 1>(c, w, in, y);
    ycache[row] = make_float4(y[0], y[1], y[2], y[3]);
}

// (alpha_G, beta_G) transposed to [l][j] so a warp (32 receivers of one
// Gaussian) reads 512 contiguous bytes per degree
__global__ void k_ag_transpose(int n_rx, int L, const float4* __restrict__ ag, float4* __restrict__ agT) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_rx * L) return;
    const int l = i / n_rx, j = i % n_rx;
    agT[i] = ag[static_cast<size_t>(j) * L + l];
}

// One CTA = 32 conditioning rows (Morton order) x 256 receivers; thread =
// one receiver.  The receiver's global-branch terms (alpha_G, beta_G) for all
// l stay in registers for the 32 rows; the rows' (basis*base, basis) pairs
// are staged in shared memory and read as broadcasts.  Per (row, receiver):
// one coalesced 16-byte y read, L x 4 FFMA2, one coalesced signal store --
// HBM-bound on the y cache.
constexpr int kCovRows = 32;
constexpr int kCovThreads = 256;

// LT > 0: L == LT, the receiver's (alpha_G, beta_G) held in registers;
// LT == 0 (other l_max): re-read per row from the transposed cache.
template <int LT>
#ifndef RXGS_COV_MINB
#define RXGS_COV_MINB 4  // A/B (config 3, ms per table / cov_signal phase): 3 CTAs + 8 ahead 111.2 / 42,
                          // 4 + 4 107.3 / 36, 4 + 8 (spills) 115.2 / 46, 5 + 4 125 / 55; 2 + 4 (earlier) 43.7 phase
#endif
#ifndef RXGS_COV_AHEAD
#define RXGS_COV_AHEAD 4
#endif
__global__ void __launch_bounds__(kCovThreads, RXGS_COV_MINB) k_cov_signal(CondDev c, const int* __restrict__ n_rows,
                                                            const int* __restrict__ rows, int n_rx, int L,
                                                            const float2* __restrict__ B, const float2* __restrict__ GB,
                                                            const float4* __restrict__ agT,
                                                            const float4* __restrict__ ycache, SigOut sig) {
    extern __shared__ float4 s_e_dyn[];  // (GB, B) per (row, l): [kCovRows][L], then s_a
    __shared__ float4 s_sum[kCovRows];          // (sum_l GB, sum_l B)
    __shared__ int s_k[kCovRows];
    const int nr = *n_rows;
    const int r0 = blockIdx.x * kCovRows;
    if (r0 >= nr) return;
    const int tid = threadIdx.x;
#pragma unroll 1
    for (int i = tid; i < kCovRows * L; i += kCovThreads) {
        const int rr = i / L, l = i % L;
        const int r = r0 + rr;
        const int k = r < nr ? rows[r] : 0;
        const float2 b = B[static_cast<size_t>(k) * L + l], gb = GB[static_cast<size_t>(k) * L + l];
        s_e_dyn[rr * L + l] = make_float4(gb.x, gb.y, b.x, b.y);
    }
    __syncthreads();
    if (tid < kCovRows) {
        const int r = r0 + tid;
        s_k[tid] = r < nr ? rows[r] : -1;
        float4 sm = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
        for (int l = 0; l < L; ++l) {  // same l order as fle_reduce
            const float4 e = s_e_dyn[tid * L + l];
            sm.x += e.x;
            sm.y += e.y;
            sm.z += e.z;
            sm.w += e.w;
        }
        s_sum[tid] = sm;
    }
    const int j = blockIdx.y * kCovThreads + tid;
    const bool jok = j < n_rx;
    // this receiver's (alpha_G, beta_G) per l, [l][thread] in shared memory
    float4* s_a = s_e_dyn + kCovRows * L;
#pragma unroll 1
    for (int l = 0; l < LT; ++l)
        s_a[l * kCovThreads + tid] = jok ? agT[static_cast<size_t>(l) * n_rx + j] : make_float4(0.f, 0.f, 0.f, 0.f);
    __syncthreads();
    if (!jok) return;
    auto load_y = [&](int rr) {
        const int k = rr < kCovRows ? s_k[rr] : -1;
        return (ycache && k >= 0) ? ycache[static_cast<size_t>(k) * n_rx + j] : make_float4(0.f, 0.f, 0.f, 0.f);
    };
    // the receiver's (alpha_G, beta_G) for all l in registers for the 32 rows
    float4 areg[LT > 0 ? LT : 1];
#pragma unroll
    for (int l = 0; l < LT; ++l) areg[l] = s_a[l * kCovThreads + tid];
    constexpr int kAhead = RXGS_COV_AHEAD;  // y-cache rows in flight per thread
    static_assert(kCovRows % kAhead == 0, "the y-cache ring walks whole 32-row blocks");
    float4 yq[kAhead];
#pragma unroll
    for (int q = 0; q < kAhead; ++q) yq[q] = load_y(q);
#pragma unroll 1
    for (int rr0 = 0; rr0 < kCovRows; rr0 += kAhead) {
#pragma unroll
    for (int q = 0; q < kAhead; ++q) {
        const int rr = rr0 + q;
        const int k = s_k[rr];
        if (k < 0) return;
        const float4 y = yq[q];
        yq[q] = load_y(rr + kAhead);  // kAhead rows ahead
        const float4 sm = s_sum[rr];
        // M = sum_l [(1 + aG_l) GB_l + bG_l B_l] = sum_l GB_l + sum_l [aG_l GB_l + bG_l B_l]
        float2 M = make_float2(sm.x, sm.y), M1 = make_float2(0.f, 0.f);
        auto term = [](float2 acc, float4 e, float4 al) {
            acc = x2::fma(x2::bc(al.x), make_float2(e.x, e.y), acc);
            acc = x2::fma(make_float2(-e.y, e.x), x2::bc(al.y), acc);
            acc = x2::fma(x2::bc(al.z), make_float2(e.z, e.w), acc);
            return x2::fma(make_float2(-e.w, e.z), x2::bc(al.w), acc);
        };
        if constexpr (LT > 0) {
#pragma unroll
            for (int l = 0; l < LT; ++l) {
                if (l & 1) M1 = term(M1, s_e_dyn[rr * LT + l], areg[l]);
                else M = term(M, s_e_dyn[rr * LT + l], areg[l]);
            }
        } else {
            for (int l = 0; l < L; ++l) {
                const float4 al = agT[static_cast<size_t>(l) * n_rx + j];
                if (l & 1) M1 = term(M1, s_e_dyn[rr * L + l], al);
                else M = term(M, s_e_dyn[rr * L + l], al);
            }
        }
        M = x2::add(M, M1);
        // s = (1 + aL) M + bL Bs (local_affine; additive mode: aL = 0)
        const float ar = c.additive ? 0.f : y.x, ai = c.additive ? 0.f : y.y;
        float2 sg = x2::fma(x2::bc(ar), M, M);
        sg = x2::fma(make_float2(-M.y, M.x), x2::bc(ai), sg);
        sg = x2::fma(x2::bc(y.z), make_float2(sm.z, sm.w), sg);
        sg = x2::fma(make_float2(-sm.w, sm.z), x2::bc(y.w), sg);
        store_sig(sig, k, n_rx, j, 1, 0, sg);
    }
    }
}

// s = (1 + aL) M + bL Bs from the FLE GEMM's M[row][j]: one thread per (row,
// receiver), receivers fastest -- coalesced y, M and signal streams.
__global__ void __launch_bounds__(256) k_cov_affine(CondDev c, const int* __restrict__ n_rows,
                                                    const int* __restrict__ rows, int n_rx,
                                                    const float2* __restrict__ M, const float4* __restrict__ rS,
                                                    const float4* __restrict__ ycache, SigOut sig) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= static_cast<long long>(*n_rows) * n_rx) return;
    const int r = static_cast<int>(i / n_rx), j = static_cast<int>(i % n_rx);
    const int k = rows[r];
    const float2 m = M[i];
    const float4 sm = rS[r];
    const float4 y = ycache ? ycache[static_cast<size_t>(k) * n_rx + j] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float ar = c.additive ? 0.f : y.x, ai = c.additive ? 0.f : y.y;
    float2 sg = x2::fma(x2::bc(ar), m, m);
    sg = x2::fma(make_float2(-m.y, m.x), x2::bc(ai), sg);
    sg = x2::fma(x2::bc(y.z), make_float2(sm.z, sm.w), sg);
    sg = x2::fma(make_float2(-sm.w, sm.z), x2::bc(y.w), sg);
    store_sig(sig, k, n_rx, j, 1, 0, sg);
}

}  // namespace

cudaError_t launch_cov_signal_gemm(const rxgs_cond_s* cs, const rxgs_scene_s& sc, const rxgs_txstate_s& st, int n_rx,
                                   const float* d_ag, const float4* ycache, SigOut d_sig, cudaStream_t s) {
    const long long bound = st.needed_host >= 0 ? st.needed_host : st.visible;
    if (bound == 0 || n_rx == 0) return cudaSuccess;
    rxgs_ctx ctx = sc.ctx;
    cudaError_t e;
    if ((e = gather_rows(sc, st, s)) != cudaSuccess) return e;
    if ((e = ctx->fle_m.ensure(sizeof(float2) * static_cast<size_t>(st.k) * n_rx)) != cudaSuccess) return e;
    if ((e = launch_fle_gemm(ctx, st.needed_count.as<int>(), bound, st.k, st.L, n_rx, ctx->row_GB.as<float4>(),
                             ctx->row_S.as<float4>(), d_ag, ctx->fle_m.as<float2>(), s, st.version, true)) != cudaSuccess)
        return e;
    CondDev d{};
    if (cs) d = make_dev(*cs);
    const long long n = bound * n_rx;
    k_cov_affine<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(d, st.needed_count.as<int>(),
                                                                      st.needed_order.as<int>(), n_rx,
                                                                      ctx->fle_m.as<float2>(), ctx->row_S.as<float4>(),
                                                                      ycache, d_sig);
    ctx->launches += 1;
    return cudaGetLastError();
}

cudaError_t launch_local_cache(const rxgs_cond_s& cs, const rxgs_scene_s& sc, const double* d_rx, int n_rx,
                               float4* ycache, cudaStream_t s) {
    if (cond_tc_eligible(&cs)) return launch_local_cache_tc(cs, sc, d_rx, n_rx, ycache, s);
    const long long rows = static_cast<long long>(sc.k) * n_rx;
    if (rows == 0) return cudaSuccess;
    k_ycache_simt<<<static_cast<unsigned>((rows + 127) / 128), 128, 0, s>>>(make_dev(cs), sc.k,
                                                                            sc.d_pos32.as<float4>(), d_rx, n_rx,
                                                                            ycache);
    return cudaGetLastError();
}

cudaError_t launch_ag_transpose(int n_rx, int L, const float* d_ag, float* d_agT, cudaStream_t s) {
    if (n_rx * L == 0) return cudaSuccess;
    k_ag_transpose<<<(n_rx * L + 255) / 256, 256, 0, s>>>(n_rx, L, reinterpret_cast<const float4*>(d_ag),
                                                          reinterpret_cast<float4*>(d_agT));
    return cudaGetLastError();
}

cudaError_t launch_cov_signal(const rxgs_cond_s* cs, const rxgs_txstate_s& st, int n_rx, const float* d_agT,
                              const float4* ycache, SigOut d_sig, cudaStream_t s) {
    // upper bound on the rows; the exact count is on the device
    const long long bound = st.needed_host >= 0 ? st.needed_host : st.visible;
    if (bound == 0 || n_rx == 0) return cudaSuccess;
    CondDev d{};
    if (cs) d = make_dev(*cs);
    dim3 grid(static_cast<unsigned>((bound + kCovRows - 1) / kCovRows), (n_rx + kCovThreads - 1) / kCovThreads);
    const bool reg = st.L == 9 || st.L == 4 || st.L == 1;  // specialised: alpha_G / beta_G staged per thread
    const size_t smem = sizeof(float4) * (kCovRows + (reg ? kCovThreads : 0)) * st.L;
    auto kern = st.L == 9 ? k_cov_signal<9> : (st.L == 4 ? k_cov_signal<4> : (st.L == 1 ? k_cov_signal<1> : k_cov_signal<0>));
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    kern<<<grid, kCovThreads, smem, s>>>(d, st.needed_count.as<int>(), st.needed_order.as<int>(), n_rx, st.L,
                                              st.basis32.as<float2>(), st.gb32.as<float2>(),
                                              reinterpret_cast<const float4*>(d_agT), ycache, d_sig);
    return cudaGetLastError();
}

}  // namespace rxgs_b200
