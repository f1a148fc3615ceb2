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

__global__ void __launch_bounds__(256) k_cov_signal(CondDev c, const int* __restrict__ n_rows,
                                                    const int* __restrict__ rows, int n_rx, int L,
                                                    const float2* __restrict__ B, const float2* __restrict__ GB,
                                                    const float4* __restrict__ agT, const float4* __restrict__ ycache,
                                                    float2* __restrict__ sig) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= static_cast<long long>(*n_rows) * n_rx) return;
    const int k = rows[i / n_rx], j = static_cast<int>(i % n_rx);
    float2 M = make_float2(0.f, 0.f), Bs = make_float2(0.f, 0.f);
    for (int l = 0; l < L; ++l) {  // fle_reduce (cond_common.cuh) with the transposed global branch
        const float2 b = B[static_cast<size_t>(k) * L + l];
        const float2 gb = GB[static_cast<size_t>(k) * L + l];
        const float4 a = agT[static_cast<size_t>(l) * n_rx + j];
        const float2 t0 = cmul(make_float2(1.f + a.x, a.y), gb), t1 = cmul(make_float2(a.z, a.w), b);
        M.x += t0.x + t1.x;
        M.y += t0.y + t1.y;
        Bs.x += b.x;
        Bs.y += b.y;
    }
    float y[4] = {0.f, 0.f, 0.f, 0.f};
    if (ycache) {
        const float4 v = ycache[static_cast<size_t>(k) * n_rx + j];
        y[0] = v.x;
        y[1] = v.y;
        y[2] = v.z;
        y[3] = v.w;
    }
    sig[static_cast<size_t>(k) * n_rx + j] = local_affine(c, 0, M, Bs, y);
}

}  // namespace

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
                              const float4* ycache, float2* d_sig, cudaStream_t s) {
    const long long rows = static_cast<long long>(st.visible) * n_rx;  // upper bound; exact count on device
    if (rows == 0) return cudaSuccess;
    CondDev d{};
    if (cs) d = make_dev(*cs);
    k_cov_signal<<<static_cast<unsigned>((rows + 255) / 256), 256, 0, s>>>(
        d, st.needed_count.as<int>(), st.needed_order.as<int>(), n_rx, st.L, st.basis32.as<float2>(),
        st.gb32.as<float2>(), reinterpret_cast<const float4*>(d_agT), ycache, d_sig);
    return cudaGetLastError();
}

}  // namespace rxgs_b200
