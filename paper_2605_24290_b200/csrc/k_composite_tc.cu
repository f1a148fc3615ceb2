// Per-tile compositing on the tensor cores (tcgen05), the query-path
// counterpart of k_composite (k_composite.cu; render_field,
// sphraster.cpp:255-315, with the aggregate_modality epilogues :323-381).
//
// For one 8x8-cell tile and a chunk of 64 receivers:
//     D[m][cell] = sum_{pos < W} A[m][pos] * B[cell][pos]
//     A[m][pos]  = s[list[pos]][j0 + m/2].{re, im}   (m = 2 j + re/im)   M = 128
//     B[cell][pos] = tw[pos][cell]                                        N = 64
// i.e. the transposed tile product with receivers on the 128 TMEM lanes.
// Both operands are staged through shared memory in the no-swizzle
// MN-major canonical layout (8 MN-elements x 8 K-rows core matrices) as
// bf16 hi/lo (D = Ahi Bhi + Ahi Blo + Alo Bhi, ~2^-17 relative).  The
// signals arrive pre-split by the conditioning kernel (SigOut::presplit:
// {bf16x2 hi, bf16x2 lo} per receiver, the same 8 bytes as complex f32), so
// staging A is register moves only; the blend weights are split on the fly.
// 32 list positions per stage, two stages in flight: the MMAs of
// stage i (6 x tcgen05.mma M128 N64 K16, committed to the stage's mbarrier)
// overlap the gather/convert of stage i+1.  Epilogue: tcgen05.ld, re/im lane
// pairs exchanged with shuffles, spectrum amplitude, RSSI partial per tile,
// optional f32 field (training forward).
#include "rxgs_internal.cuh"
#include "tc_util.cuh"

namespace rxgs_b200 {
namespace {

constexpr int kM = 128;       // 64 receivers x {re, im}
constexpr int kN = 64;        // cells of an 8x8 tile
constexpr int kKS = 32;       // list positions per stage
constexpr int kThr = 128;
constexpr int kABytes = (kKS / 8) * (kM / 8) * 144;  // one bf16 operand stage (9 KB with SBO padding)
constexpr int kBBytes = (kKS / 8) * (kN / 8) * 144;  // 4.5 KB
constexpr int kStageBytes = 2 * kABytes + 2 * kBBytes;  // hi + lo of A and B (24 KB)
// MN-major no-swizzle: core matrix = 8 K-rows x 16 B (128 B contiguous);
// MN groups SBO apart, K groups LBO apart.  SBO = 144 B (not 128): the 16 B
// stores of one K-row across MN groups then spread over all 32 banks
// (2 wavefronts per warp instead of a 16-way conflict).
constexpr uint32_t kSBO = 144;
constexpr uint32_t kALBO = (kM / 8) * kSBO;  // 2304
constexpr uint32_t kBLBO = (kN / 8) * kSBO;  // 1152
constexpr uint32_t kIdesc = tc::idesc_bf16_f32(kM, kN) | (1u << 15) | (1u << 16);  // A, B MN-major

__device__ __forceinline__ uint32_t mn_off(int mn, int k, uint32_t lbo) {
    return static_cast<uint32_t>((k >> 3) * lbo + (mn >> 3) * kSBO + (k & 7) * 16 + (mn & 7) * 2);
}

#ifndef RXGS_COMP_WAIT
#define RXGS_COMP_WAIT tc::mbar_wait
#endif
#ifndef RXGS_COMP_RX_FAST
#define RXGS_COMP_RX_FAST 1
#endif

template <bool FIELD>
__global__ void __launch_bounds__(kThr) k_composite_tc(DevGrid g, const int64_t* __restrict__ tile_offsets,
                                                       const int* __restrict__ list, const float* __restrict__ tw,
                                                       const int* __restrict__ walk_len,
                                                       const uint2* __restrict__ sig, int n_rx,
                                                       float* __restrict__ spectrum, float* __restrict__ rssi_partial,
                                                       float* __restrict__ field32) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bars[2];
    __shared__ uint32_t tbase_s;
    __shared__ float s_dom[8];  // solid angle of the tile's 8 rows
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
#if RXGS_COMP_RX_FAST  // receiver blocks of one tile back to back: its weight rows stay in L2
    const int tile = blockIdx.y;
#else
    const int tile = blockIdx.x;
#endif
    if (tid < 8) {  // zero for rows past the grid (partial last tile row)
        const int row = (tile / g.tiles_p) * 8 + tid;
        s_dom[tid] = row < g.nt ? static_cast<float>(sin(g.tmin + (row + 0.5) * g.dth) * g.dth * g.dph) : 0.f;
    }
#if RXGS_COMP_RX_FAST
    const int j0 = blockIdx.x * (kM / 2);
#else
    const int j0 = blockIdx.y * (kM / 2);
#endif
    const int W = walk_len[tile];
    const int64_t begin = tile_offsets[tile];

    if (warp == 0) {
        tc::tmem_alloc(&tbase_s, 64);
        tc::tmem_relinquish();
    }
    if (tid == 0) {
        tc::mbar_init(&bars[0], 1);
        tc::mbar_init(&bars[1], 1);
        tc::fence_mbar_init();
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm_d = tbase_s;
    const int n_stages = (W + kKS - 1) / kKS;
    uint32_t ph[2] = {0u, 0u};

    // Loader: warp w stages list positions 8w .. 8w+7 of a stage.  A: one
    // coalesced 512 B row (64 receivers, complex) per position, lane l holding
    // receivers j0+2l, j0+2l+1 (= m-values 4l..4l+3); B: one 256 B blend-weight
    // row per half-warp (lane holds cells 4(l%16)..+3).  Loads for stage s+1
    // are issued before stage s's barrier/MMA so their latency is hidden.
    uint4 ra[8];
    float4 rb[4];
    const bool even_n = (n_rx & 1) == 0;
    // list indices of a whole stage in one coalesced load (lane i <-> position i)
    auto load_idx = [&](int st) {
        const int pos = st * kKS + lane;
        return pos < W ? list[begin + pos] : 0;
    };
    int kidx = n_stages > 0 ? load_idx(0) : 0;
    // A: lane holds receivers j0 + 4 (lane % 16) .. +3 of list position
    // 8w + 2i + lane / 16 (i = 0..3): two 16-byte loads of {hi, lo} pairs,
    // regrouped into one 16-byte row (4 receivers re/im) per bf16 plane.
    auto load = [&](int st) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int pp = 8 * warp + 2 * i + (lane >> 4);
            const int pos = st * kKS + pp;
            const int k = __shfl_sync(0xffffffffu, kidx, pp);
            ra[2 * i] = ra[2 * i + 1] = make_uint4(0u, 0u, 0u, 0u);
            if (pos < W) {
                const int jj = j0 + 4 * (lane & 15);
                const uint2* rowp = sig + static_cast<size_t>(k) * n_rx + jj;
                if (even_n && jj + 3 < n_rx) {
                    ra[2 * i] = *reinterpret_cast<const uint4*>(rowp);
                    ra[2 * i + 1] = *reinterpret_cast<const uint4*>(rowp + 2);
                } else {
                    uint2 t[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) t[q] = jj + q < n_rx ? rowp[q] : make_uint2(0u, 0u);
                    ra[2 * i] = make_uint4(t[0].x, t[0].y, t[1].x, t[1].y);
                    ra[2 * i + 1] = make_uint4(t[2].x, t[2].y, t[3].x, t[3].y);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int pos = st * kKS + 8 * warp + 2 * i + (lane >> 4);
            rb[i] = pos < W ? *reinterpret_cast<const float4*>(tw + static_cast<size_t>(begin + pos) * kN + 4 * (lane & 15))
                            : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        kidx = st + 1 < n_stages ? load_idx(st + 1) : 0;  // next stage's indices, one stage early
    };
    auto split4 = [](float4 v, uint2& hi, uint2& lo) {
        hi.x = tc::pack_bf16(v.x, v.y);
        hi.y = tc::pack_bf16(v.z, v.w);
        lo.x = tc::pack_bf16(v.x - __uint_as_float(hi.x << 16), v.y - __uint_as_float(hi.x & 0xFFFF0000u));
        lo.y = tc::pack_bf16(v.z - __uint_as_float(hi.y << 16), v.w - __uint_as_float(hi.y & 0xFFFF0000u));
    };
    if (n_stages > 0) load(0);
    for (int st = 0; st < n_stages; ++st) {
        const int buf = st & 1;
        uint8_t* base = smem + buf * kStageBytes;
        uint8_t* a_hi = base;
        uint8_t* a_lo = base + kABytes;
        uint8_t* b_hi = base + 2 * kABytes;
        uint8_t* b_lo = base + 2 * kABytes + kBBytes;
        if (st >= 2) {  // the MMAs that read this buffer two stages ago must be done
            RXGS_COMP_WAIT(&bars[buf], ph[buf]);
            ph[buf] ^= 1u;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {  // {hi0, lo0, hi1, lo1}, {hi2, lo2, hi3, lo3} -> (hi0..hi3), (lo0..lo3)
            const uint32_t off = mn_off(8 * (lane & 15), 8 * warp + 2 * i + (lane >> 4), kALBO);
            *reinterpret_cast<uint4*>(a_hi + off) = make_uint4(ra[2 * i].x, ra[2 * i].z, ra[2 * i + 1].x, ra[2 * i + 1].z);
            *reinterpret_cast<uint4*>(a_lo + off) = make_uint4(ra[2 * i].y, ra[2 * i].w, ra[2 * i + 1].y, ra[2 * i + 1].w);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            uint2 hi, lo;
            split4(rb[i], hi, lo);
            const uint32_t off = mn_off(4 * (lane & 15), 8 * warp + 2 * i + (lane >> 4), kBLBO);
            *reinterpret_cast<uint2*>(b_hi + off) = hi;
            *reinterpret_cast<uint2*>(b_lo + off) = lo;
        }
        if (st + 1 < n_stages) load(st + 1);
        tc::fence_proxy_async_smem();
        tc::fence_before_sync();
        __syncthreads();
        if (tid == 0) {
            tc::fence_after_sync();
            const uint32_t ah = tc::smem_u32(a_hi), al = tc::smem_u32(a_lo);
            const uint32_t bh = tc::smem_u32(b_hi), bl = tc::smem_u32(b_lo);
#pragma unroll
            for (int ks = 0; ks < kKS / 16; ++ks) {
                const uint64_t dah = tc::sdesc_kmajor_noswizzle(ah + 2 * kALBO * ks, kALBO, kSBO);
                const uint64_t dal = tc::sdesc_kmajor_noswizzle(al + 2 * kALBO * ks, kALBO, kSBO);
                const uint64_t dbh = tc::sdesc_kmajor_noswizzle(bh + 2 * kBLBO * ks, kBLBO, kSBO);
                const uint64_t dbl = tc::sdesc_kmajor_noswizzle(bl + 2 * kBLBO * ks, kBLBO, kSBO);
                const uint32_t acc0 = (st > 0 || ks > 0) ? 1u : 0u;
                tc::mma_ss(tm_d, dah, dbh, kIdesc, acc0);
                tc::mma_ss(tm_d, dah, dbl, kIdesc, 1u);
                tc::mma_ss(tm_d, dal, dbh, kIdesc, 1u);
            }
            tc::mma_commit(&bars[buf]);
        }
    }
    // ---- wait for the last stage(s)
    if (n_stages >= 2) {
        const int b2 = (n_stages - 2) & 1;
        RXGS_COMP_WAIT(&bars[b2], ph[b2]);
    }
    if (n_stages >= 1) {
        const int b1 = (n_stages - 1) & 1;
        RXGS_COMP_WAIT(&bars[b1], ph[b1]);
    }
    tc::fence_after_sync();

    // ---- epilogue: lane m = 32 warp + lane holds row m = 2 jl + (re|im)
    const int m = 32 * warp + lane;
    const int jl = m >> 1;
    const int j = j0 + jl;
    const bool is_im = m & 1;
    const int tt = tile / g.tiles_p, tp = tile % g.tiles_p;
    const size_t plane = static_cast<size_t>(g.nt) * g.np;
    float* s_amp = reinterpret_cast<float*>(smem);  // [64 receivers][68] (stage buffers are free now)
    constexpr int kAmpStride = 68;                  // 16 B aligned rows, bank-spread
    // Lanes 2j / 2j+1 hold re / im of receiver j for every cell.  For each
    // column pair (q, q+1) one exchange gives the even lane (re, im) of cell
    // q and the odd lane (re, im) of cell q+1: every lane finishes one cell
    // per pair, no divergence.
    float pw = 0.f;
#pragma unroll
    for (int ch = 0; ch < 4; ++ch) {
        uint32_t r[16];
        if (n_stages > 0) {
            tc::tmem_ld16(tm_d + (static_cast<uint32_t>(32 * warp) << 16) + 16 * ch, r);
            tc::wait_ld();
        } else {
#pragma unroll
            for (int q = 0; q < 16; ++q) r[q] = 0u;
        }
        if (FIELD) {
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const int cell = 16 * ch + q;
                const int row = tt * 8 + (cell >> 3), col = tp * 8 + (cell & 7);
                if (row < g.nt && col < g.np && j < n_rx)
                    field32[(static_cast<size_t>(j) * 2 + (is_im ? 1 : 0)) * plane + static_cast<size_t>(row) * g.np + col] =
                        __uint_as_float(r[q]);
            }
        }
#pragma unroll
        for (int q = 0; q < 16; q += 2) {
            const float v0 = __uint_as_float(r[q]), v1 = __uint_as_float(r[q + 1]);
            const float got = __shfl_xor_sync(0xffffffffu, is_im ? v0 : v1, 1);
            const float re = is_im ? got : v0, im = is_im ? v1 : got;
            const int cell = 16 * ch + q + (is_im ? 1 : 0);
            const float p2 = fmaf(re, re, im * im);
            float amp;
            asm("sqrt.approx.f32 %0, %1;" : "=f"(amp) : "f"(p2 + static_cast<float>(kAmpEps)));
            s_amp[jl * kAmpStride + cell] = amp;
            pw = fmaf(p2, s_dom[cell >> 3], pw);  // rows past the grid have s_dom = 0
        }
    }
    pw += __shfl_xor_sync(0xffffffffu, pw, 1);
    if (rssi_partial && !is_im && j < n_rx) rssi_partial[static_cast<size_t>(j) * g.n_tiles + tile] = pw;
    if (spectrum) {
        __syncthreads();
        // 64 receivers x 8 tile rows = 512 row segments of 8 cells (32 B)
        for (int sgm = tid; sgm < 64 * 8; sgm += kThr) {
            const int r8 = sgm & 7, jr = sgm >> 3;
            const int jg = j0 + jr, row = tt * 8 + r8, col0 = tp * 8;
            if (jg >= n_rx || row >= g.nt) continue;
            const float* src = s_amp + jr * kAmpStride + r8 * 8;
            float* dst = spectrum + static_cast<size_t>(jg) * plane + static_cast<size_t>(row) * g.np + col0;
            if (col0 + 8 <= g.np && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
                *reinterpret_cast<float4*>(dst) = *reinterpret_cast<const float4*>(src);
                *reinterpret_cast<float4*>(dst + 4) = *reinterpret_cast<const float4*>(src + 4);
            } else {
                for (int c = 0; c < 8 && col0 + c < g.np; ++c) dst[c] = src[c];
            }
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tm_d, 64);
}

// 128x64x64 GEMM with A and B both MN-major in shared memory (the
// composite's operand layout), small-integer data: must be exact.
__global__ void __launch_bounds__(128) k_tc_selftest_mn(float* __restrict__ err) {
    __shared__ __align__(1024) uint8_t sA[8 * (128 / 8) * 144];
    __shared__ __align__(1024) uint8_t sB[8 * (64 / 8) * 144];
    __shared__ uint64_t bar;
    __shared__ uint32_t tb;
    const int tid = threadIdx.x, warp = tid >> 5;
    auto Av = [](int m, int k) { return static_cast<float>((m + 3 * k) % 5 - 2); };
    auto Bv = [](int n, int k) { return static_cast<float>((2 * n + k) % 7 - 3); };
    for (int i = tid; i < 128 * 64; i += 128) {
        const int m = i % 128, k = i / 128;
        *reinterpret_cast<uint16_t*>(sA + mn_off(m, k, kALBO)) = static_cast<uint16_t>(tc::pack_bf16(Av(m, k), 0.f));
    }
    for (int i = tid; i < 64 * 64; i += 128) {
        const int n = i % 64, k = i / 64;
        *reinterpret_cast<uint16_t*>(sB + mn_off(n, k, kBLBO)) = static_cast<uint16_t>(tc::pack_bf16(Bv(n, k), 0.f));
    }
    if (warp == 0) {
        tc::tmem_alloc(&tb, 64);
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
    if (tid == 0) {
        for (int ks = 0; ks < 4; ++ks)
            tc::mma_ss(tb, tc::sdesc_kmajor_noswizzle(tc::smem_u32(sA) + 2 * kALBO * ks, kALBO, kSBO),
                       tc::sdesc_kmajor_noswizzle(tc::smem_u32(sB) + 2 * kBLBO * ks, kBLBO, kSBO), kIdesc, ks > 0);
        tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, 0);
    tc::fence_after_sync();
    float e = 0.f;
    for (int c0 = 0; c0 < 64; c0 += 16) {
        uint32_t r[16];
        tc::tmem_ld16(tb + (static_cast<uint32_t>(32 * warp) << 16) + c0, r);
        tc::wait_ld();
        for (int q = 0; q < 16; ++q) {
            float ref = 0.f;
            for (int k = 0; k < 64; ++k) ref += Av(tid, k) * Bv(c0 + q, k);
            e = fmaxf(e, fabsf(__uint_as_float(r[q]) - ref));
        }
    }
    atomicMax(reinterpret_cast<int*>(err), __float_as_int(e));
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tb, 64);
}

}  // namespace

cudaError_t launch_tc_selftest_mn(float* d_err, cudaStream_t s) {
    k_tc_selftest_mn<<<1, 128, 0, s>>>(d_err);
    return cudaGetLastError();
}

bool composite_tc_eligible(const rxgs_txstate_s& st) { return st.grid.cell_blocks == 1 && st.grid.ts == 8 && st.channels == 1; }

cudaError_t launch_composite_tc(const rxgs_txstate_s& st, const uint2* d_sig, int n_rx, const CompositeOut& out,
                                cudaStream_t s) {
    const DevGrid& g = st.grid;
    const size_t smem = 2 * kStageBytes;
    auto kern = out.field32 ? k_composite_tc<true> : k_composite_tc<false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
#if RXGS_COMP_RX_FAST
    dim3 grid((n_rx + kM / 2 - 1) / (kM / 2), g.n_tiles);
#else
    dim3 grid(g.n_tiles, (n_rx + kM / 2 - 1) / (kM / 2));
#endif
    kern<<<grid, kThr, smem, s>>>(g, st.tile_offsets.as<int64_t>(), st.list.as<int>(), st.tw.as<float>(),
                                            st.walk_len.as<int>(), d_sig, n_rx, out.spectrum, out.rssi_partial,
                                            out.field32);
    return cudaGetLastError();
}

}  // namespace rxgs_b200
