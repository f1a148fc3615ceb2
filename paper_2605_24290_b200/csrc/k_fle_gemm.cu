// The FLE reduction of the query path as one tensor-core GEMM per receiver
// batch (used for high l_max, where the per-row loop of k_cond_tc would
// stream L float4 pairs per (Gaussian, receiver) row from L1/L2):
//
//   M[r][j] = sum_l [(1 + aG_jl) GB_rl + bG_jl B_rl]            (fle_reduce,
//           = sum_l GB_rl + sum_l [aG_jl GB_rl + bG_jl B_rl]     cond_common.cuh)
//
// as a real product D[r][n] = sum_kk A[r][kk] Bm[n][kk] with K = 4L:
//   A[r][4l + (0..3)]    = (Re GB_rl, Im GB_rl, Re B_rl, Im B_rl)
//   Bm[2j][4l + (0..3)]   = (Re aG, -Im aG, Re bG, -Im bG)_jl   -> Re M
//   Bm[2j+1][4l + (0..3)] = (Im aG,  Re aG, Im bG,  Re bG)_jl   -> Im M
// then M = D + sum_l GB_rl, written [j][row] for k_cond_tc's coalesced read
// (or [row][j] for the coverage signal kernel).
// tcgen05: 128 rows x 256 columns (128 receivers, re/im) per CTA, K in
// steps of 16, bf16x3 (Ahi Bhi + Ahi Blo + Alo Bhi, ~2^-17 relative,
// FP32-class) into a 256-column TMEM accumulator.  The pack kernels write
// the operands pre-tiled: every (128-row or 256-row block, 16-wide K step)
// slab is the exact image of the no-swizzle K-major canonical layout, so
// one thread moves a whole stage (A hi / lo 4 KB each, B hi / lo 8 KB each)
// with four bulk copies on the TMA engine (cp.async.bulk, completion
// counted in bytes on the stage's mbarrier) and the MMAs of a stage start
// as soon as its bytes have landed; three stages in flight.
#include "rxgs_internal.cuh"
#include "tc_util.cuh"

namespace rxgs_b200 {
namespace {

constexpr int kTM = 128, kTN = 256, kTK = 16, kStages = 3, kThr = 128;
constexpr int kASlab = kTM * kTK * 2;  // 4 KB
constexpr int kBSlab = kTN * kTK * 2;  // 8 KB
constexpr int kStage = 2 * kASlab + 2 * kBSlab;
constexpr uint32_t kIdesc = tc::idesc_bf16_f32(kTM, kTN);

__device__ __forceinline__ uint32_t slab_off(int r, int k) {  // K = 16: LBO 128 B, SBO 256 B
    return static_cast<uint32_t>(((r >> 3) * 2 + (k >> 3)) * 128 + (r & 7) * 16 + (k & 7) * 2);
}
// element index of (row r, k) in the pre-tiled operand: blocks of `rows`
// rows, each a run of Kp / 16 slabs (rows x 16 bf16) in the canonical layout
__device__ __forceinline__ size_t slab_elem(int r, int k, int rows, int Kp) {
    const size_t slab = static_cast<size_t>(r / rows) * (Kp / kTK) + k / kTK;
    return slab * rows * kTK + slab_off(r % rows, k % kTK) / 2;
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ uint16_t bf16_bits(float x) { return static_cast<uint16_t>(tc::pack_bf16(x, 0.f) & 0xFFFFu); }
__device__ __forceinline__ void split(float x, uint16_t& hi, uint16_t& lo) {
    const float h = tc::bf16_round(x);
    hi = bf16_bits(h);
    lo = bf16_bits(x - h);
}

// A rows from the gathered (GB, B) pairs ([l][row] float4, k_gather_rows)
__global__ void k_fle_pack_a(const int* __restrict__ n_rows, int cap, int L, int Kp, const float4* __restrict__ rGB,
                             uint16_t* __restrict__ a_hi, uint16_t* __restrict__ a_lo) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    const int nq = Kp / 4;
    const long long r = i / nq;
    const int l = static_cast<int>(i % nq);
    if (r >= *n_rows) return;
    const float4 e = l < L ? rGB[static_cast<size_t>(l) * cap + r] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float v[4] = {e.x, e.y, e.z, e.w};
    uint16_t h[4], lo[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) split(v[q], h[q], lo[q]);
    const size_t o = slab_elem(static_cast<int>(r), 4 * l, kTM, Kp);
    *reinterpret_cast<uint2*>(a_hi + o) = make_uint2(h[0] | (uint32_t(h[1]) << 16), h[2] | (uint32_t(h[3]) << 16));
    *reinterpret_cast<uint2*>(a_lo + o) = make_uint2(lo[0] | (uint32_t(lo[1]) << 16), lo[2] | (uint32_t(lo[3]) << 16));
}

// Bm rows from the global branch ag[j][l] = (aG, bG) (k_cond_global)
__global__ void k_fle_pack_b(int n_rx, int L, int Kp, const float4* __restrict__ ag, uint16_t* __restrict__ b_hi,
                             uint16_t* __restrict__ b_lo) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    const int nq = Kp / 4;
    const long long n = i / nq;
    const int l = static_cast<int>(i % nq);
    if (n >= 2LL * n_rx) return;
    const int j = static_cast<int>(n >> 1);
    const float4 a = l < L ? ag[static_cast<size_t>(j) * L + l] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float v[4] = {(n & 1) ? a.y : a.x, (n & 1) ? a.x : -a.y, (n & 1) ? a.w : a.z, (n & 1) ? a.z : -a.w};
    uint16_t h[4], lo[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) split(v[q], h[q], lo[q]);
    const size_t o = slab_elem(static_cast<int>(n), 4 * l, kTN, Kp);
    *reinterpret_cast<uint2*>(b_hi + o) = make_uint2(h[0] | (uint32_t(h[1]) << 16), h[2] | (uint32_t(h[3]) << 16));
    *reinterpret_cast<uint2*>(b_lo + o) = make_uint2(lo[0] | (uint32_t(lo[1]) << 16), lo[2] | (uint32_t(lo[3]) << 16));
}

__global__ void __launch_bounds__(kThr) k_fle_gemm(const int* __restrict__ n_rows_dev, int cap, int n_rx, int Kp,
                                                   const uint16_t* __restrict__ a_hi, const uint16_t* __restrict__ a_lo,
                                                   const uint16_t* __restrict__ b_hi, const uint16_t* __restrict__ b_lo,
                                                   const float4* __restrict__ rS, float2* __restrict__ Mout,
                                                   int row_major) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bars[kStages];  // MMAs of the stage done (buffer free)
    __shared__ uint64_t full[kStages];  // the stage's bytes landed
    __shared__ uint32_t tbase_s;
    const int n_rows = *n_rows_dev;
    const int r0 = blockIdx.x * kTM;
    if (r0 >= n_rows) return;
    const int n0 = blockIdx.y * kTN;  // first column (2 j0)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) {
        tc::tmem_alloc(&tbase_s, kTN);
        tc::tmem_relinquish();
    }
    if (tid == 0) {
        for (int q = 0; q < kStages; ++q) {
            tc::mbar_init(&bars[q], 1);
            tc::mbar_init(&full[q], 1);
        }
        tc::fence_mbar_init();
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm = tbase_s;
    const uint32_t s0 = tc::smem_u32(smem);
    const int nk = Kp / kTK;

    // one thread runs the whole pipeline: bulk copies of stage ks + kStages
    // into the buffer stage ks used, once its MMAs are done (empty[b]); the
    // MMAs of stage ks once its bytes have landed (full[b])
    if (tid == 0) {
        const uint16_t* pa_hi = a_hi + static_cast<size_t>(blockIdx.x) * nk * (kASlab / 2);
        const uint16_t* pa_lo = a_lo + static_cast<size_t>(blockIdx.x) * nk * (kASlab / 2);
        const uint16_t* pb_hi = b_hi + static_cast<size_t>(blockIdx.y) * nk * (kBSlab / 2);
        const uint16_t* pb_lo = b_lo + static_cast<size_t>(blockIdx.y) * nk * (kBSlab / 2);
        auto load = [&](int ks) {
            const int b = ks % kStages;
            const uint32_t base = s0 + b * kStage;
            mbar_expect_tx(&full[b], kStage);
            const uint32_t fb = tc::smem_u32(&full[b]);
            bulk_g2s(base, pa_hi + static_cast<size_t>(ks) * (kASlab / 2), kASlab, fb);
            bulk_g2s(base + kASlab, pa_lo + static_cast<size_t>(ks) * (kASlab / 2), kASlab, fb);
            bulk_g2s(base + 2 * kASlab, pb_hi + static_cast<size_t>(ks) * (kBSlab / 2), kBSlab, fb);
            bulk_g2s(base + 2 * kASlab + kBSlab, pb_lo + static_cast<size_t>(ks) * (kBSlab / 2), kBSlab, fb);
        };
        for (int ks = 0; ks < kStages && ks < nk; ++ks) load(ks);
        for (int ks = 0; ks < nk; ++ks) {
            const int b = ks % kStages;
            tc::mbar_wait(&full[b], static_cast<uint32_t>((ks / kStages) & 1));
            tc::fence_after_sync();
            const uint32_t ah = s0 + b * kStage, al = ah + kASlab, bh = ah + 2 * kASlab, bl = bh + kBSlab;
            const uint64_t dah = tc::sdesc_kmajor_noswizzle(ah, 128, 256), dal = tc::sdesc_kmajor_noswizzle(al, 128, 256);
            const uint64_t dbh = tc::sdesc_kmajor_noswizzle(bh, 128, 256), dbl = tc::sdesc_kmajor_noswizzle(bl, 128, 256);
            tc::mma_ss(tm, dah, dbh, kIdesc, ks > 0 ? 1u : 0u);
            tc::mma_ss(tm, dah, dbl, kIdesc, 1u);
            tc::mma_ss(tm, dal, dbh, kIdesc, 1u);
            tc::mma_commit(&bars[b]);
            if (ks + kStages < nk) {
                tc::mbar_wait(&bars[b], static_cast<uint32_t>((ks / kStages) & 1));  // its MMAs read the buffer
                load(ks + kStages);
            }
        }
    }
    // the last commit tracks every MMA before it.  Only thread 0 has seen
    // every earlier phase of that barrier (a parity wait by the others could
    // match an older phase), so it waits and releases the CTA.
    if (tid == 0 && nk >= 1) {
        const int lb = (nk - 1) % kStages;
        tc::mbar_wait(&bars[lb], static_cast<uint32_t>(((nk - 1) / kStages) & 1));
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    // ---- epilogue: lane = row, column pairs = (Re, Im) of receiver j0 + c/2
    const int r = r0 + 32 * warp + lane;
    const bool rok = r < n_rows;
    const float4 gs = rok ? rS[r] : make_float4(0.f, 0.f, 0.f, 0.f);
    const int j0 = n0 >> 1;
#pragma unroll 1
    for (int ch = 0; ch < kTN / 16; ++ch) {
        uint32_t v[16];
        if (nk > 0) {
            tc::tmem_ld16(tm + (static_cast<uint32_t>(32 * warp) << 16) + 16 * ch, v);
            tc::wait_ld();
        } else {
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = 0u;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int j = j0 + 8 * ch + q;
            if (rok && j < n_rx)
                Mout[row_major ? static_cast<size_t>(r) * n_rx + j : static_cast<size_t>(j) * cap + r] =
                    make_float2(__uint_as_float(v[2 * q]) + gs.x, __uint_as_float(v[2 * q + 1]) + gs.y);
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tm, kTN);
}

}  // namespace

int fle_gemm_kpad(int L) { return (4 * L + kTK - 1) / kTK * kTK; }

cudaError_t launch_fle_gemm(rxgs_ctx ctx, const int* n_rows_dev, long long rows_bound, int cap, int L, int n_rx,
                            const float4* rGB, const float4* rS, const float* d_ag, float2* Mout, cudaStream_t s,
                            uint64_t a_version, bool row_major) {
    if (rows_bound == 0 || n_rx == 0) return cudaSuccess;
    const int Kp = fle_gemm_kpad(L);
    cudaError_t e;
    // pre-tiled operands: rows padded to the 128-row A blocks and the
    // 256-column B blocks (the padding rows feed only unused outputs)
    const size_t rows_p = (static_cast<size_t>(cap) + kTM - 1) / kTM * kTM;
    const size_t cols_p = (2 * static_cast<size_t>(n_rx) + kTN - 1) / kTN * kTN;
    if ((e = ctx->fle_a.ensure(sizeof(uint16_t) * 2 * rows_p * Kp)) != cudaSuccess) return e;
    if ((e = ctx->fle_b.ensure(sizeof(uint16_t) * 2 * cols_p * Kp)) != cudaSuccess) return e;
    uint16_t* a_hi = ctx->fle_a.as<uint16_t>();
    uint16_t* a_lo = a_hi + rows_p * Kp;
    uint16_t* b_hi = ctx->fle_b.as<uint16_t>();
    uint16_t* b_lo = b_hi + cols_p * Kp;
    const long long na = rows_bound * (Kp / 4), nb = 2LL * n_rx * (Kp / 4);
    if (a_version == 0 || ctx->fle_a_version != a_version) {  // A depends on the state only
        k_fle_pack_a<<<static_cast<unsigned>((na + 255) / 256), 256, 0, s>>>(n_rows_dev, cap, L, Kp, rGB, a_hi, a_lo);
        ctx->fle_a_version = a_version;
    }
    k_fle_pack_b<<<static_cast<unsigned>((nb + 255) / 256), 256, 0, s>>>(n_rx, L, Kp,
                                                                          reinterpret_cast<const float4*>(d_ag), b_hi, b_lo);
    const size_t smem = kStages * kStage;
    if ((e = cudaFuncSetAttribute(k_fle_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem))) !=
        cudaSuccess)
        return e;
    dim3 grid(static_cast<unsigned>((rows_bound + kTM - 1) / kTM), (2 * n_rx + kTN - 1) / kTN);
    k_fle_gemm<<<grid, kThr, smem, s>>>(n_rows_dev, cap, n_rx, Kp, a_hi, a_lo, b_hi, b_lo, rS, Mout, row_major ? 1 : 0);
    ctx->launches += 3;
    return cudaGetLastError();
}

}  // namespace rxgs_b200
