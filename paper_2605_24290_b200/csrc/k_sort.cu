// Tile binning: the device form of bin_and_sort (sphraster.cpp:85-102),
// hand-written (no CUB).
//
// The reference pushes Gaussian indices into each covered tile in index
// order and std::stable_sort's every list by FP64 depth, i.e. each list is
// ordered by (depth, index).  On the device:
//   1. depth rank: a stable LSD radix sort (8-bit digits, 4 passes) of the
//      Gaussians by a 32-bit order-preserving key of their FP64 depth -- the
//      depth bits minus the smallest visible depth's bits, shifted right
//      just far enough that every visible key fits in 31 bits (culled ->
//      0xFFFFFFFF, last).  The input is in index order, so equal keys keep
//      index order.  Keys that collide after the shift (Gaussians whose
//      depths agree to ~1e-9 relative) form short runs that k_depth_final
//      re-orders by the full 64-bit depth bits (then index): the result is
//      exactly the (FP64 depth, index) order -- rank[g];
//   2. per rank the Gaussian's tile count, exclusive scan -> the first list
//      entry of every rank (entries are laid out in rank order);
//   3. one stable counting-sort pass by tile id over the E entries, the
//      entries generated on the fly from the rank-ordered spans (entry ->
//      rank by a binary search of the scan in shared memory): per-block
//      tile histograms, a scan over (tile, block), and a scatter that ranks
//      equal tiles inside the block with warp ballots and warp-private
//      counters, so within a tile the rank order survives.  It writes the
//      lists, the 64-bit keys (tile << 32) | rank the north star asks to be
//      bit-exact, and the tile offsets directly.
//   Grids with more than kFusedTiles tiles take a generic path instead:
//   (tile, rank) pairs, LSD passes on the tile id, then lists and keys.
//
// Stable scatter (every pass): block b owns a contiguous run of items; warp
// w a contiguous sub-run, processed 32 at a time in lane order, so (block,
// warp, round, lane) is input order.  Lanes with the same digit find each
// other with ballots on the digit bits; a warp-private shared-memory counter per
// digit carries the count across rounds; an exclusive prefix over the warps
// plus the block's offset from the (digit, block) scan gives each item its
// output position.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "rxgs_internal.cuh"

namespace rxgs_b200 {
namespace {

constexpr int kRadixBits = 8;
constexpr int kBins = 1 << kRadixBits;
constexpr int kPassWarps = 8;
constexpr int kPassThreads = kPassWarps * 32;
#ifndef RXGS_PASS_SMALL_N
#define RXGS_PASS_SMALL_N 400000
#endif
#ifndef RXGS_PASS_SMALL_M
#define RXGS_PASS_SMALL_M 512  // A/B at K = 100k (config-2 step): 2048 3.285 ms, 1024 3.291, 512 3.260
#endif

constexpr int kTileWarps = 8;
constexpr int kTileThreads = kTileWarps * 32;
// entries per block of the emit / tile-scatter passes: the template
// parameter M (2048 or 8192, by entry count; bin_tiles)
constexpr int kFusedTiles = 4096;                      // tile ids of the fused pass: 12 bits

// elements per block of the K scans: the template parameter CH, 2048, or
// 512 up to RXGS_PASS_SMALL_N elements (scan_chunk)

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Lanes of the warp holding the same low BITS bits of d (valid lanes only):
// BITS + 1 ballots, the warp-level multisplit of a radix pass (MATCH.ANY
// measured latency-bound here).
template <int BITS>
__device__ __forceinline__ unsigned match_digit(unsigned d, bool ok) {
    const unsigned v = __ballot_sync(0xffffffffu, ok);
    unsigned m = ok ? v : ~v;
#pragma unroll
    for (int b = 0; b < BITS; ++b) {
        const unsigned bal = __ballot_sync(0xffffffffu, (d >> b) & 1u);
        m &= ((d >> b) & 1u) ? bal : ~bal;
    }
    return m;
}

// Block-wide inclusive scan of one value per thread (blockDim.x multiple of
// 32, <= 1024); returns the thread's inclusive prefix, *total the block sum.
template <typename T>
__device__ __forceinline__ T block_incl_scan(T v, T* warp_sums, T* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    if (lane == 31) warp_sums[warp] = v;
    __syncthreads();
    if (warp == 0) {
        T w = lane < nw ? warp_sums[lane] : T(0);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const T u = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += u;
        }
        if (lane < nw) warp_sums[lane] = w;
    }
    __syncthreads();
    if (warp > 0) v += warp_sums[warp - 1];
    *total = warp_sums[nw - 1];
    __syncthreads();
    return v;
}

// ---------------------------------------------------------------- generic LSD pass
// hist[d * nb + b] = number of items of block b with digit d.
template <int M>
__global__ void __launch_bounds__(kPassThreads) k_radix_hist(int n, int nb, const uint32_t* __restrict__ kin,
                                                              int shift, int* __restrict__ hist) {
    __shared__ int h[kBins];
    for (int d = threadIdx.x; d < kBins; d += kPassThreads) h[d] = 0;
    __syncthreads();
    const int b = blockIdx.x;
    const int i1 = min(n, (b + 1) * M);
    for (int i = b * M + threadIdx.x; i < i1; i += kPassThreads)
        atomicAdd(&h[(kin[i] >> shift) & (kBins - 1)], 1);
    __syncthreads();
    for (int d = threadIdx.x; d < kBins; d += kPassThreads) hist[d * nb + b] = h[d];
}

// Exclusive scan of the row-major (rows x nb) count matrix, rows in order
// then blocks: block r scans row r in place and posts the row total; the
// last block to finish scans the totals into base[r] (and base[rows] =
// grand total).  off(r, b) = base[r] + mat[r][b].
__global__ void k_matrix_scan(int rows, int nb, int* __restrict__ mat, int* __restrict__ tot, int* __restrict__ base,
                              unsigned* __restrict__ counter) {
    __shared__ int ws[32];
    __shared__ bool last;
    int* row = mat + static_cast<size_t>(blockIdx.x) * nb;
    int carry = 0;
    for (int c0 = 0; c0 < nb; c0 += blockDim.x) {
        const int i = c0 + threadIdx.x;
        const int v = i < nb ? row[i] : 0;
        int t;
        const int inc = block_incl_scan(v, ws, &t);
        if (i < nb) row[i] = carry + inc - v;
        carry += t;
    }
    if (threadIdx.x == 0) {
        tot[blockIdx.x] = carry;
        __threadfence();
        last = atomicAdd(counter, 1u) == static_cast<unsigned>(rows - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    carry = 0;
    for (int c0 = 0; c0 < rows; c0 += blockDim.x) {
        const int i = c0 + threadIdx.x;
        const int v = i < rows ? *reinterpret_cast<volatile int*>(tot + i) : 0;
        int t;
        const int inc = block_incl_scan(v, ws, &t);
        if (i < rows) base[i] = carry + inc - v;
        carry += t;
    }
    if (threadIdx.x == 0) {
        base[rows] = carry;
        *counter = 0u;  // reusable by the next pass on this stream
    }
}

// Stable scatter of one LSD pass (see the file header).  The block's items
// are staged in shared memory in (digit, input) order and written out with
// consecutive threads on consecutive output positions (runs of one digit).
template <int M>
__global__ void __launch_bounds__(kPassThreads) k_radix_scatter(int n, int nb, const uint32_t* __restrict__ kin,
                                                                 const int* __restrict__ vin, uint32_t* __restrict__ kout,
                                                                 int* __restrict__ vout, int shift,
                                                                 const int* __restrict__ mat,
                                                                 const int* __restrict__ base) {
    __shared__ int wc[kPassWarps][kBins];
    __shared__ int gb[kBins], lb[kBins];  // global / local start of the block's run of each digit
    constexpr int kRounds = M / kPassThreads;
    __shared__ uint32_t sk[M];
    __shared__ int sv[M];
    __shared__ int wsum[kPassWarps];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < kPassWarps * kBins; i += kPassThreads) (&wc[0][0])[i] = 0;
    __syncthreads();
    const int b = blockIdx.x;
    const int i0 = b * M + warp * (M / kPassWarps);
    const unsigned lt = lanemask_lt();
    uint32_t kk[kRounds];
    int vv[kRounds], loc[kRounds];
#pragma unroll
    for (int it = 0; it < kRounds; ++it) {  // all loads in flight before the ranking
        const int i = i0 + it * 32 + lane;
        kk[it] = i < n ? __ldg(kin + i) : 0u;
        vv[it] = i < n ? __ldg(vin + i) : 0;
    }
#pragma unroll
    for (int it = 0; it < kRounds; ++it) {
        const bool ok = i0 + it * 32 + lane < n;
        const int d = static_cast<int>((kk[it] >> shift) & (kBins - 1));
        const unsigned peers = match_digit<kRadixBits>(static_cast<unsigned>(d), ok);
        const int c = ok ? wc[warp][d] : 0;
        __syncwarp();
        if (ok && lane == __ffs(peers) - 1) wc[warp][d] = c + __popc(peers);
        __syncwarp();
        loc[it] = c + __popc(peers & lt);
    }
    __syncthreads();
    static_assert(kBins == kPassThreads, "one digit per thread");
    {
        const int d = threadIdx.x;
        gb[d] = base[d] + mat[d * nb + b];
        int s = 0;
#pragma unroll
        for (int w = 0; w < kPassWarps; ++w) {
            const int t = wc[w][d];
            wc[w][d] = s;
            s += t;
        }
        int tot = 0;
        const int inc = block_incl_scan<int>(s, wsum, &tot);  // over digits
        lb[d] = inc - s;
    }
    __syncthreads();
    const int n_blk = n - b * M < M ? n - b * M : M;
#pragma unroll
    for (int it = 0; it < kRounds; ++it) {
        if (i0 + it * 32 + lane >= n) continue;
        const int d = static_cast<int>((kk[it] >> shift) & (kBins - 1));
        const int lp = lb[d] + wc[warp][d] + loc[it];
        sk[lp] = kk[it];
        sv[lp] = vv[it];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n_blk; i += kPassThreads) {
        const uint32_t k = sk[i];
        const int d = static_cast<int>((k >> shift) & (kBins - 1));
        const int pos = gb[d] + (i - lb[d]);
        kout[pos] = k;
        vout[pos] = sv[i];
    }
}

// ---------------------------------------------------------------- depth rank
__global__ void k_depth_minmax(int K, const uint64_t* __restrict__ dk, unsigned long long* __restrict__ mm) {
    __shared__ unsigned long long slo[32], shi[32];
    unsigned long long lo = ~0ull, hi = 0ull;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < K; i += gridDim.x * blockDim.x) {
        const unsigned long long v = dk[i];
        if (v != ~0ull) {
            lo = v < lo ? v : lo;
            hi = v > hi ? v : hi;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, lo, o), c = __shfl_xor_sync(0xffffffffu, hi, o);
        lo = a < lo ? a : lo;
        hi = c > hi ? c : hi;
    }
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        slo[w] = lo;
        shi[w] = hi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < nw; ++i) {
            lo = slo[i] < lo ? slo[i] : lo;
            hi = shi[i] > hi ? shi[i] : hi;
        }
        if (lo != ~0ull) atomicMin(mm, lo);
        if (hi != 0ull) atomicMax(mm + 1, hi);
    }
}

__device__ __forceinline__ int depth_shift(unsigned long long lo, unsigned long long hi) {
    if (lo > hi) return 0;  // nothing visible
    const unsigned long long span = hi - lo;
    const int bits = span ? 64 - __clzll(static_cast<long long>(span)) : 0;
    return bits > 31 ? bits - 31 : 0;
}

// 32-bit order-preserving depth keys (index-ordered input) + the first
// pass's histogram.
template <int M>
__global__ void __launch_bounds__(kPassThreads) k_depth_keys(int K, int nb, const uint64_t* __restrict__ dk,
                                                              const unsigned long long* __restrict__ mm,
                                                              uint32_t* __restrict__ key, int* __restrict__ val,
                                                              int* __restrict__ hist) {
    __shared__ int h[kBins];
    for (int d = threadIdx.x; d < kBins; d += kPassThreads) h[d] = 0;
    __syncthreads();
    const unsigned long long lo = mm[0], hi = mm[1];
    const int sh = depth_shift(lo, hi);
    const int b = blockIdx.x;
    const int i1 = min(K, (b + 1) * M);
    for (int i = b * M + threadIdx.x; i < i1; i += kPassThreads) {
        const unsigned long long v = dk[i];
        const uint32_t k = v == ~0ull ? 0xFFFFFFFFu : static_cast<uint32_t>((v - lo) >> sh);
        key[i] = k;
        val[i] = i;
        atomicAdd(&h[k & (kBins - 1)], 1);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < kBins; d += kPassThreads) hist[d * nb + b] = h[d];
}

// Final depth order: runs of equal 32-bit keys among visible Gaussians are
// re-ordered by (full FP64 depth bits, index) -- insertion sort, stable, in
// place (the run belongs to the thread at its start); then order, the
// per-rank tile counts and spans (coalesced writes), and the visible count.
__device__ __forceinline__ int64_t span_count(int4 sp) {
    return static_cast<int64_t>(max(0, sp.y - sp.x + 1)) * max(0, sp.w - sp.z + 1);
}

__global__ void k_depth_final(int K, const uint32_t* __restrict__ ks, int* __restrict__ vs,
                              const uint64_t* __restrict__ dk, const int4* __restrict__ spans,
                              int* __restrict__ order,
                              int64_t* __restrict__ cnt_sorted, int4* __restrict__ spans_sorted,
                              int64_t* __restrict__ visible) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r > K) return;
    if (r == K) {
        cnt_sorted[K] = 0;
        if (K == 0 || ks[K - 1] != 0xFFFFFFFFu) *visible = K;
        return;
    }
    const uint32_t k = ks[r];
    if (k == 0xFFFFFFFFu) {  // culled: index order already, no entries
        if (r == 0 || ks[r - 1] != 0xFFFFFFFFu) *visible = r;
        order[r] = vs[r];
        cnt_sorted[r] = 0;
        spans_sorted[r] = make_int4(0, -1, 0, -1);
        return;
    }
    const bool head = r == 0 || ks[r - 1] != k;
    const bool run = (r + 1 < K && ks[r + 1] == k) || !head;
    if (!run) {
        const int g = vs[r];
        const int4 sp = spans[g];
        order[r] = g;
        spans_sorted[r] = sp;
        cnt_sorted[r] = span_count(sp);
        return;
    }
    if (!head) return;  // inside a run: its head handles it
    int e = r + 1;
    while (e < K && ks[e] == k) ++e;
    for (int i = r + 1; i < e; ++i) {  // stable insertion sort by full depth bits
        const int g = vs[i];
        const uint64_t d = dk[g];
        int j = i - 1;
        while (j >= r && dk[vs[j]] > d) {
            vs[j + 1] = vs[j];
            --j;
        }
        vs[j + 1] = g;
    }
    for (int i = r; i < e; ++i) {
        const int g = vs[i];
        const int4 sp = spans[g];
        order[i] = g;
        spans_sorted[i] = sp;
        cnt_sorted[i] = span_count(sp);
    }
}

// ---------------------------------------------------------------- K scans (int64)
// Block-local exclusive scan of CH elements; block totals to bsum.
// Warp w scans its contiguous chunk 32 elements at a time (coalesced,
// register shuffles), then adds the totals of the earlier warps.
// T = int64_t or int (int sums accumulate in int64 and are written back narrowed).
template <typename T, int CH>
__global__ void __launch_bounds__(256) k_scan_blocks(int64_t n, const T* __restrict__ in, T* __restrict__ out,
                                                     int64_t* __restrict__ bsum) {
    __shared__ int64_t wt[8];
    constexpr int SEG = CH / 8;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t b0 = blockIdx.x * static_cast<int64_t>(CH) + warp * SEG;
    int64_t v[SEG / 32];
    int64_t carry = 0;
#pragma unroll
    for (int r = 0; r < SEG / 32; ++r) {
        const int64_t i = b0 + r * 32 + lane;
        const int64_t x = i < n ? static_cast<int64_t>(in[i]) : 0;
        int64_t inc = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
        }
        v[r] = carry + inc - x;
        carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) wt[warp] = carry;
    __syncthreads();
    int64_t prev = 0, tot = 0;
    for (int w = 0; w < 8; ++w) {
        if (w < warp) prev += wt[w];
        tot += wt[w];
    }
#pragma unroll
    for (int r = 0; r < SEG / 32; ++r) {
        const int64_t i = b0 + r * 32 + lane;
        if (i < n) out[i] = static_cast<T>(v[r] + prev);
    }
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

// out += sum of the block totals before this block.
template <typename T, int CH>
__global__ void k_scan_add(int64_t n, T* __restrict__ out, const int64_t* __restrict__ bsum) {
    __shared__ int64_t ws[32];
    int64_t p = 0;
    for (int i = threadIdx.x; i < static_cast<int>(blockIdx.x); i += blockDim.x) p += bsum[i];
    int64_t t;
    block_incl_scan(p, ws, &t);
    if (t == 0) return;
    const int64_t b0 = blockIdx.x * static_cast<int64_t>(CH);
    for (int i = threadIdx.x; i < CH; i += blockDim.x)
        if (b0 + i < n) out[b0 + i] += static_cast<T>(t);
}

// ---------------------------------------------------------------- tile pass
struct EntryMap {
    int r0, nseg;
    bool glob;  // ranks do not fit the shared window: search the scan in global memory
};

// Block-wide inclusive max-scan of own[0..n) in place (kTileThreads threads,
// n <= M): warp w scans its contiguous M / kTileWarps elements 32 at
// a time (lane-contiguous, conflict-free), then applies the max of the
// earlier warps' totals.
template <int M>
__device__ __forceinline__ void block_max_scan(int* own, int n) {
    __shared__ int wm[kTileWarps];
    constexpr int SEG = M / kTileWarps;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int* seg = own + warp * SEG;
    const int len = min(SEG, max(0, n - warp * SEG));
    int carry = -1;
    for (int c0 = 0; c0 < len; c0 += 32) {
        int v = c0 + lane < len ? seg[c0 + lane] : -1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) v = max(v, __shfl_up_sync(0xffffffffu, v, o));
        v = max(v, carry);
        if (c0 + lane < len) seg[c0 + lane] = v;
        carry = __shfl_sync(0xffffffffu, v, 31);
    }
    if (lane == 0) wm[warp] = carry;
    __syncthreads();
    int prev = -1;
    for (int w = 0; w < warp; ++w) prev = max(prev, wm[w]);
    if (prev >= 0)
        for (int i = lane; i < len; i += 32) seg[i] = max(seg[i], prev);
    __syncthreads();
}

// Entry -> rank for the entries [e0, e0 + n) of this block, without a search
// per entry: the scan values of ranks r0 .. r0 + nseg - 1 (relative to e0)
// go to seg[], every rank marks its first entry in own[], and a max-scan
// spreads the marks -- own[q] = rank index (from r0) of entry q.  Every rank
// with tiles has >= 1 entry, so M + 2 ranks cover a block unless
// zero-count ranks sit between them (only possible through the host-span
// API); then the entries binary-search the scan in global memory instead.
template <int M>
__device__ __forceinline__ EntryMap map_entries(const int* __restrict__ bfirst, const int* __restrict__ blast,
                                                int64_t e0, int n, const int64_t* __restrict__ scan, int* seg,
                                                int* own) {
    const int r0 = bfirst[blockIdx.x];
    const int need = blast[blockIdx.x] - r0 + 1;
    if (need > M + 2) return {r0, need, true};
    for (int i = threadIdx.x; i < need; i += blockDim.x) seg[i] = static_cast<int>(scan[r0 + i] - e0);
    for (int q = threadIdx.x; q < n; q += blockDim.x) own[q] = 0;
    __syncthreads();
    for (int i = threadIdx.x + 1; i < need; i += blockDim.x)
        if (seg[i] < n) atomicMax(&own[seg[i]], i);
    __syncthreads();
    block_max_scan<M>(own, n);
    return {r0, need, false};
}

// bfirst[b] / blast[b]: the ranks holding the first and the last entry of
// block b (blocks of M entries), from the scan in one pass over the
// ranks -- no per-block binary search.
template <int M>
__global__ void k_block_ranks(int K, int64_t E, const int64_t* __restrict__ scan, int* __restrict__ bfirst,
                              int* __restrict__ blast) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= K) return;
    const int64_t a = scan[r], c = scan[r + 1];
    if (c <= a) return;
    const int64_t nb = (E + M - 1) / M;
    for (int64_t b = (a + M - 1) / M; b * M < c; ++b) bfirst[b] = r;
    // block b ends at entry min(E, (b + 1) M) - 1
    for (int64_t b = a / M; b < nb; ++b) {
        const int64_t last = min(E, (b + 1) * M) - 1;
        if (last >= c) break;
        if (last >= a) blast[b] = r;
    }
}

// rank index (from r0) of entry q and its position j inside that rank
__device__ __forceinline__ int entry_rank(int q, int64_t e0, const int* seg, const int* own,
                                          const int64_t* __restrict__ scan, const EntryMap& m, int* j) {
    if (!m.glob) {
        const int i = own[q];
        *j = q - seg[i];
        return i;
    }
    const int64_t e = e0 + q;
    int lo = 0, hi = m.nseg - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (scan[m.r0 + mid] <= e) lo = mid;
        else hi = mid - 1;
    }
    *j = static_cast<int>(e - scan[m.r0 + lo]);
    return lo;
}

__device__ __forceinline__ int entry_tile(int j, int4 sp, int tiles_p) {
    const int w = sp.w - sp.z + 1;
    const int tt = sp.x + j / w;
    const int pp = sp.z + j % w;
    return tt * tiles_p + pp % tiles_p;
}

// (tile, rank) of every entry, in entry (= rank) order, coalesced; with
// hist != nullptr also the block's tile histogram hist[t * nb + b] (the
// fused counting-sort path, n_tiles <= kFusedTiles).
template <int M>
__global__ void __launch_bounds__(kTileThreads) k_emit_entries(int64_t E, int nb, int n_tiles, int tiles_p,
                                                                const int64_t* __restrict__ scan,
                                                                const int* __restrict__ bfirst,
                                                                const int* __restrict__ blast,
                                                                const int4* __restrict__ spans_sorted,
                                                                uint32_t* __restrict__ tkey, int* __restrict__ tval,
                                                                int* __restrict__ hist) {
    extern __shared__ int sm[];
    int* seg = sm;                  // M + 2
    int* own = seg + M + 2;         // M
    int* h = own + M;               // n_tiles (hist only)
    if (hist)
        for (int t = threadIdx.x; t < n_tiles; t += kTileThreads) h[t] = 0;
    const int64_t e0 = static_cast<int64_t>(blockIdx.x) * M;
    const int n = static_cast<int>(E - e0 < M ? E - e0 : int64_t{M});
    const EntryMap m = map_entries<M>(bfirst, blast, e0, n, scan, seg, own);
    for (int q = threadIdx.x; q < n; q += kTileThreads) {
        int j;
        const int i = entry_rank(q, e0, seg, own, scan, m, &j);
        const int t = entry_tile(j, __ldg(spans_sorted + m.r0 + i), tiles_p);
        tkey[e0 + q] = static_cast<uint32_t>(t);
        tval[e0 + q] = m.r0 + i;
        if (hist) atomicAdd(&h[t], 1);
    }
    if (!hist) return;
    __syncthreads();
    for (int t = threadIdx.x; t < n_tiles; t += kTileThreads) hist[t * nb + blockIdx.x] = h[t];
}

// Stable scatter of the entries by tile (rank order within a tile) from the
// emitted (tile, rank) arrays; writes list[pos] = Gaussian, keys[pos] =
// (tile << 32) | rank, and the tile offsets.
// Stable counting-sort pass by tile of one block's M entries.  The
// ranking (warp ballots, warp-private counters) gives every entry its output
// position; the entries are then staged in shared memory in (tile, rank)
// order, aliased over the consumed per-warp counters, and written out so
// that consecutive threads write consecutive list / key positions (runs of
// one tile) instead of 32 scattered tiles per warp store.
template <int M>
__global__ void __launch_bounds__(kTileThreads) k_tile_scatter(int64_t E, int nb, int n_tiles,
                                                                const uint32_t* __restrict__ tkey,
                                                                const int* __restrict__ tval,
                                                                const int* __restrict__ order,
                                                                const int* __restrict__ mat,
                                                                const int* __restrict__ base, int* __restrict__ list,
                                                                uint64_t* __restrict__ keys,
                                                                int64_t* __restrict__ tile_offsets) {
    extern __shared__ int sm[];
    int* tb = sm;                          // n_tiles: global offset of this block's run of each tile
    int* ls = tb + n_tiles;                // n_tiles: local (block) start of each tile's run
    int* s_tot = ls + n_tiles;             // kTileThreads: scan scratch
    uint16_t* wc = reinterpret_cast<uint16_t*>(s_tot + kTileThreads);  // kTileWarps x n_tiles (< 8192 each)
    int* st_r = reinterpret_cast<int*>(wc);                                // staged ranks (aliases wc)
    uint16_t* st_t = reinterpret_cast<uint16_t*>(st_r + M);                // staged tiles
    constexpr int kRounds = M / kTileThreads;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < kTileWarps * n_tiles; i += kTileThreads) wc[i] = 0;
    if (blockIdx.x == 0)
        for (int t = threadIdx.x; t <= n_tiles; t += kTileThreads) tile_offsets[t] = base[t];
    __syncthreads();
    const int64_t e0 = static_cast<int64_t>(blockIdx.x) * M;
    const int n = static_cast<int>(E - e0 < M ? E - e0 : int64_t{M});
    const int q0 = warp * (M / kTileWarps);
    const unsigned lt = lanemask_lt();
    uint32_t pk[kRounds];  // tile, then tile << 12 | local rank (< 1024 per warp)
#pragma unroll
    for (int it = 0; it < kRounds; ++it) {
        const int q = q0 + it * 32 + lane;
        pk[it] = q < n ? __ldg(tkey + e0 + q) : 0u;
    }
    int rv[kRounds];
#pragma unroll
    for (int it = 0; it < kRounds; ++it) {
        const int q = q0 + it * 32 + lane;
        rv[it] = q < n ? __ldg(tval + e0 + q) : 0;
    }
#pragma unroll
    for (int it = 0; it < kRounds; ++it) {
        const bool ok = q0 + it * 32 + lane < n;
        const int t = static_cast<int>(pk[it]);
        const unsigned peers = match_digit<12>(static_cast<unsigned>(t), ok);
        const int c = ok ? wc[warp * n_tiles + t] : 0;
        __syncwarp();
        if (ok && lane == __ffs(peers) - 1) wc[warp * n_tiles + t] = static_cast<uint16_t>(c + __popc(peers));
        __syncwarp();
        pk[it] = (static_cast<uint32_t>(t) << 12) | static_cast<uint32_t>(c + __popc(peers & lt));
    }
    __syncthreads();
    // per tile: global base, exclusive prefix over warps, and the block count;
    // the block counts' exclusive scan over tiles -> local starts
    const int per = (n_tiles + kTileThreads - 1) / kTileThreads;  // tiles per thread (contiguous)
    int my_sum = 0;
    for (int u = 0; u < per; ++u) {
        const int t = threadIdx.x * per + u;
        if (t >= n_tiles) break;
        tb[t] = base[t] + mat[t * nb + blockIdx.x];
        int acc = 0;
#pragma unroll
        for (int w = 0; w < kTileWarps; ++w) {
            const int v = wc[w * n_tiles + t];
            wc[w * n_tiles + t] = static_cast<uint16_t>(acc);
            acc += v;
        }
        ls[t] = acc;  // block count for now
        my_sum += acc;
    }
    s_tot[threadIdx.x] = my_sum;
    __syncthreads();
    if (threadIdx.x == 0) {  // exclusive scan of the thread sums (kTileThreads values)
        int a = 0;
        for (int i = 0; i < kTileThreads; ++i) {
            const int v = s_tot[i];
            s_tot[i] = a;
            a += v;
        }
    }
    __syncthreads();
    {
        int a = s_tot[threadIdx.x];
        for (int u = 0; u < per; ++u) {
            const int t = threadIdx.x * per + u;
            if (t >= n_tiles) break;
            const int v = ls[t];
            ls[t] = a;
            a += v;
        }
    }
    __syncthreads();
    // local position of every entry (reads wc), then stage over wc
    int lp[kRounds];
#pragma unroll
    for (int it = 0; it < kRounds; ++it) {
        const int t = static_cast<int>(pk[it] >> 12);
        lp[it] = ls[t] + wc[warp * n_tiles + t] + static_cast<int>(pk[it] & 0xFFFu);
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < kRounds; ++it) {
        if (q0 + it * 32 + lane >= n) continue;
        st_r[lp[it]] = rv[it];
        st_t[lp[it]] = static_cast<uint16_t>(pk[it] >> 12);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += kTileThreads) {
        const int t = st_t[i], r = st_r[i];
        const int pos = tb[t] + (i - ls[t]);
        list[pos] = __ldg(order + r);
        keys[pos] = (static_cast<uint64_t>(t) << 32) | static_cast<uint32_t>(r);
    }
}

__global__ void k_pairs_final(int64_t E, const uint32_t* __restrict__ tks, const int* __restrict__ rks,
                              const int* __restrict__ order, int* __restrict__ list, uint64_t* __restrict__ keys) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= E) return;
    const int r = rks[i];
    list[i] = order[r];
    keys[i] = (static_cast<uint64_t>(tks[i]) << 32) | static_cast<uint32_t>(r);
}

// tile_offsets[t] = first position of tile t in the tile-sorted pairs.
__global__ void k_offsets(int64_t n, int n_tiles, const uint32_t* __restrict__ tks, int64_t* __restrict__ off) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i > n) return;
    const int prev = i == 0 ? -1 : static_cast<int>(tks[i - 1]);
    const int cur = i == n ? n_tiles : static_cast<int>(tks[i]);
    for (int t = prev + 1; t <= cur; ++t) off[t] = i;
}

int bits_for(int64_t n) {
    int b = 1;
    while ((int64_t{1} << b) < n) ++b;
    return b;
}

size_t al256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

}  // namespace

// Stable LSD radix sort of (u32 key, int value) pairs on the low `bits` key
// bits: kin/vin -> kin/vin (ping-ponging through ktmp/vtmp).  work: int
// scratch of radix_sort_work_ints(n) (count matrix, totals, base, counter).
// items per block of the LSD passes: blocks enough for the SMs at small n
// (RXGS_PASS_SMALL_M below RXGS_PASS_SMALL_N items); RXGS_PASS_M overrides (512 / 1024 / 2048)
static int pass_m(int n) {
    static const int forced = [] {
        const char* v = std::getenv("RXGS_PASS_M");
        return v ? std::atoi(v) : 0;
    }();
    if (forced == 512 || forced == 1024 || forced == 2048) return forced;
    return n <= RXGS_PASS_SMALL_N ? RXGS_PASS_SMALL_M : 2048;
}

size_t radix_sort_work_ints(int n) {
    const int nb = (n + pass_m(n) - 1) / pass_m(n);
    return static_cast<size_t>(kBins) * std::max(nb, 1) + 2 * (kBins + 1) + 64;
}

cudaError_t radix_sort_pairs(int n, int bits, uint32_t* kin, int* vin, uint32_t* ktmp, int* vtmp, int* work,
                             bool hist_ready, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const int M = pass_m(n);
    const int nb = (n + M - 1) / M;
    auto hist_k = M == 512 ? k_radix_hist<512> : (M == 1024 ? k_radix_hist<1024> : k_radix_hist<2048>);
    auto scat_k = M == 512 ? k_radix_scatter<512> : (M == 1024 ? k_radix_scatter<1024> : k_radix_scatter<2048>);
    int* mat = work;
    int* tot = mat + static_cast<size_t>(kBins) * nb;
    int* base = tot + kBins + 1;
    unsigned* counter = reinterpret_cast<unsigned*>(base + kBins + 1);
    const int passes = (bits + kRadixBits - 1) / kRadixBits;
    uint32_t* ka = kin;
    uint32_t* kb = ktmp;
    int* va = vin;
    int* vb = vtmp;
    for (int p = 0; p < passes; ++p) {
        const int shift = p * kRadixBits;
        if (!(p == 0 && hist_ready)) hist_k<<<nb, kPassThreads, 0, s>>>(n, nb, ka, shift, mat);
        k_matrix_scan<<<kBins, 256, 0, s>>>(kBins, nb, mat, tot, base, counter);
        scat_k<<<nb, kPassThreads, 0, s>>>(n, nb, ka, va, kb, vb, shift, mat, base);
        std::swap(ka, kb);
        std::swap(va, vb);
    }
    if (ka != kin) {  // odd pass count: result is in the temporaries
        cudaMemcpyAsync(kin, ka, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, s);
        cudaMemcpyAsync(vin, va, sizeof(int) * n, cudaMemcpyDeviceToDevice, s);
    }
    return cudaGetLastError();
}

// Exclusive scan of n int64 / int (in -> out, may alias); bsum: scan_bsum_count(n) int64.
static int scan_chunk(int64_t n) { return n <= RXGS_PASS_SMALL_N ? 512 : 2048; }

template <typename T, int CH>
static cudaError_t scan_chunks(int64_t n, const T* in, T* out, int64_t* bsum, cudaStream_t s) {
    const unsigned nb = static_cast<unsigned>((n + CH - 1) / CH);
    k_scan_blocks<T, CH><<<nb, 256, 0, s>>>(n, in, out, bsum);
    if (nb > 1) k_scan_add<T, CH><<<nb, 256, 0, s>>>(n, out, bsum);
    return cudaGetLastError();
}

template <typename T>
static cudaError_t scan_any(int64_t n, const T* in, T* out, int64_t* bsum, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    return scan_chunk(n) == 512 ? scan_chunks<T, 512>(n, in, out, bsum, s) : scan_chunks<T, 2048>(n, in, out, bsum, s);
}
cudaError_t scan_i64(int64_t n, const int64_t* in, int64_t* out, int64_t* bsum, cudaStream_t s) {
    return scan_any(n, in, out, bsum, s);
}
cudaError_t scan_i32(int64_t n, const int* in, int* out, int64_t* bsum, cudaStream_t s) {
    return scan_any(n, in, out, bsum, s);
}
size_t scan_bsum_count(int64_t n) { return static_cast<size_t>(n / scan_chunk(n) + 2); }

int bin_tiles(rxgs_ctx ctx, rxgs_txstate_s& st, cudaStream_t s) {
    const int K = st.k;
    const int n_tiles = st.grid.n_tiles;
    RXGS_CUDA(st.order.ensure(sizeof(int) * (K + 1)));
    RXGS_CUDA(st.scan.ensure(sizeof(int64_t) * (K + 1)));
    RXGS_CUDA(st.tile_offsets.ensure(sizeof(int64_t) * (n_tiles + 1)));

    // scratch_a: keys/values x2 | cnt_sorted | spans_sorted | radix work | block sums | [minmax, visible]
    const int pm = pass_m(K);  // the same blocks as radix_sort_pairs (the first pass's histogram)
    const int nbk = (K + pm - 1) / pm;
    const size_t o_k1 = 0, o_v1 = al256(4 * (K + 1)), o_k2 = o_v1 + al256(4 * (K + 1)),
                 o_v2 = o_k2 + al256(4 * (K + 1)), o_cnt = o_v2 + al256(4 * (K + 1)),
                 o_sp = o_cnt + al256(8 * (K + 2)), o_work = o_sp + al256(16 * (K + 1)),
                 o_bs = o_work + al256(4 * radix_sort_work_ints(K)),
                 o_red = o_bs + al256(8 * scan_bsum_count(K + 1));
    RXGS_CUDA(ctx->scratch_a.ensure(o_red + 256));
    char* base = ctx->scratch_a.as<char>();
    uint32_t* k1 = reinterpret_cast<uint32_t*>(base + o_k1);
    int* v1 = reinterpret_cast<int*>(base + o_v1);
    uint32_t* k2 = reinterpret_cast<uint32_t*>(base + o_k2);
    int* v2 = reinterpret_cast<int*>(base + o_v2);
    int64_t* cnt_sorted = reinterpret_cast<int64_t*>(base + o_cnt);
    int4* spans_sorted = reinterpret_cast<int4*>(base + o_sp);
    int* work = reinterpret_cast<int*>(base + o_work);
    int64_t* bsum = reinterpret_cast<int64_t*>(base + o_bs);
    unsigned long long* mm = reinterpret_cast<unsigned long long*>(base + o_red);
    int64_t* visible = reinterpret_cast<int64_t*>(base + o_red + 16);
    // the matrix-scan counter lives at the end of work and must start at 0
    RXGS_CUDA(cudaMemsetAsync(work, 0, 4 * radix_sort_work_ints(K), s));

    if (K > 0) {
        const unsigned long long init[2] = {~0ull, 0ull};
        RXGS_CUDA(cudaMemcpyAsync(mm, init, sizeof init, cudaMemcpyHostToDevice, s));
        k_depth_minmax<<<std::min((K + 255) / 256, 2 * ctx->sm_count), 256, 0, s>>>(K, st.depth_key.as<uint64_t>(),
                                                                                      mm);
        auto dk_k = pm == 512 ? k_depth_keys<512> : (pm == 1024 ? k_depth_keys<1024> : k_depth_keys<2048>);
        dk_k<<<nbk, kPassThreads, 0, s>>>(K, nbk, st.depth_key.as<uint64_t>(), mm, k1, v1, work);
        RXGS_CUDA(radix_sort_pairs(K, 32, k1, v1, k2, v2, work, true, s));
        k_depth_final<<<(K + 1 + 255) / 256, 256, 0, s>>>(K, k1, v1, st.depth_key.as<uint64_t>(),
                                                          st.spans.as<int4>(), st.order.as<int>(), cnt_sorted,
                                                          spans_sorted, visible);
        RXGS_CUDA(scan_i64(K + 1, cnt_sorted, st.scan.as<int64_t>(), bsum, s));
    }
    int64_t total = 0, vis = 0;
    if (K > 0) {
        RXGS_CUDA(cudaMemcpyAsync(&total, st.scan.as<int64_t>() + K, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        RXGS_CUDA(cudaMemcpyAsync(&vis, visible, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        RXGS_CUDA(cudaStreamSynchronize(s));
    }
    if (total >= (int64_t{1} << 31)) return fail(RXGS_ERR_INVALID, "bin_and_sort: more than 2^31 tile entries");
    st.entries = total;
    st.visible = vis;
    RXGS_CUDA(st.list.ensure(sizeof(int) * (total + 1)));
    RXGS_CUDA(st.keys.ensure(sizeof(uint64_t) * (total + 1)));
    const int64_t E = total;
    if (E == 0) {
        RXGS_CUDA(cudaMemsetAsync(st.tile_offsets.p, 0, sizeof(int64_t) * (n_tiles + 1), s));
        return RXGS_OK;
    }
    // entries per block of the emit / tile-scatter passes: 2048 below ~1.2M
    // entries (config 2: 169 blocks instead of 43 on 148 SMs), else 8192; the
    // stable counting sort gives the same lists and keys for either
    auto bin_entries = [&](auto m_c) -> int {
        constexpr int M = decltype(m_c)::value;
        const int nbt = static_cast<int>((E + M - 1) / M);
        RXGS_CUDA(st.rank.ensure(sizeof(int) * 2 * (nbt + 1)));  // per-block first / last ranks
        int* bfirst = st.rank.as<int>();
        int* blast = bfirst + nbt + 1;
        k_block_ranks<M><<<(K + 255) / 256, 256, 0, s>>>(K, E, st.scan.as<int64_t>(), bfirst, blast);
        // entries (tile, rank) | pair temporaries | count matrix etc. in scratch_b
        const size_t o_v = al256(4 * (E + 1)), o_kt = o_v + al256(4 * (E + 1)), o_vt = o_kt + al256(4 * (E + 1)),
                     o_w = o_vt + al256(4 * (E + 1));
        const bool fused = n_tiles <= kFusedTiles;
        const size_t mat_ints = fused ? static_cast<size_t>(n_tiles) * nbt + 2 * (n_tiles + 1) + 64
                                      : radix_sort_work_ints(static_cast<int>(E));
        RXGS_CUDA(ctx->scratch_b.ensure(o_w + 4 * mat_ints));
        char* pb = ctx->scratch_b.as<char>();
        uint32_t* tk = reinterpret_cast<uint32_t*>(pb);
        int* tv = reinterpret_cast<int*>(pb + o_v);
        int* mat = reinterpret_cast<int*>(pb + o_w);
        const size_t sm_e = 4 * (2 * static_cast<size_t>(M) + 2 + (fused ? n_tiles : 0));
        RXGS_CUDA(cudaFuncSetAttribute(k_emit_entries<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm_e)));
        if (fused) {
            int* tot = mat + static_cast<size_t>(n_tiles) * nbt;
            int* tbase = tot + n_tiles + 1;
            unsigned* counter = reinterpret_cast<unsigned*>(tbase + n_tiles + 1);
            RXGS_CUDA(cudaMemsetAsync(counter, 0, 4, s));
            k_emit_entries<M><<<nbt, kTileThreads, sm_e, s>>>(E, nbt, n_tiles, st.grid.tiles_p, st.scan.as<int64_t>(), bfirst,
                                                           blast, spans_sorted, tk, tv, mat);
            k_matrix_scan<<<n_tiles, 256, 0, s>>>(n_tiles, nbt, mat, tot, tbase, counter);
            const size_t sm_s = 4 * (2 * static_cast<size_t>(n_tiles) + kTileThreads) +
                                std::max(2 * static_cast<size_t>(kTileWarps) * n_tiles, 6 * static_cast<size_t>(M));
            RXGS_CUDA(cudaFuncSetAttribute(k_tile_scatter<M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(sm_s)));
            k_tile_scatter<M><<<nbt, kTileThreads, sm_s, s>>>(E, nbt, n_tiles, tk, tv, st.order.as<int>(), mat, tbase,
                                                           st.list.as<int>(), st.keys.as<uint64_t>(),
                                                           st.tile_offsets.as<int64_t>());
        } else {
            // generic: LSD passes on the tile id, then lists / keys / offsets
            const int En = static_cast<int>(E);
            RXGS_CUDA(cudaMemsetAsync(mat, 0, 4 * mat_ints, s));
            k_emit_entries<M><<<nbt, kTileThreads, sm_e, s>>>(E, nbt, n_tiles, st.grid.tiles_p, st.scan.as<int64_t>(), bfirst,
                                                           blast, spans_sorted, tk, tv, nullptr);
            RXGS_CUDA(radix_sort_pairs(En, bits_for(n_tiles), tk, tv, reinterpret_cast<uint32_t*>(pb + o_kt),
                                       reinterpret_cast<int*>(pb + o_vt), mat, false, s));
            k_pairs_final<<<static_cast<unsigned>((E + 255) / 256), 256, 0, s>>>(E, tk, tv, st.order.as<int>(),
                                                                                 st.list.as<int>(),
                                                                                 st.keys.as<uint64_t>());
            k_offsets<<<static_cast<unsigned>((E + 1 + 255) / 256), 256, 0, s>>>(E, n_tiles, tk,
                                                                                  st.tile_offsets.as<int64_t>());
        }
        return RXGS_OK;
    };
    {
        const int rc = E < (int64_t{1} << 20) + (int64_t{1} << 18) ? bin_entries(std::integral_constant<int, 2048>{})
                                                                  : bin_entries(std::integral_constant<int, 8192>{});
        if (rc) return rc;
    }
    ctx->launches += 20;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? RXGS_OK : cuda_fail(e, "bin_tiles");
}

}  // namespace rxgs_b200

// ---------------------------------------------------------------- needed rows
namespace rxgs_b200 {
namespace {

__global__ void k_mark_needed(DevGrid g, const int64_t* __restrict__ tile_offsets, const int* __restrict__ list,
                              const int* __restrict__ walk_len, unsigned char* __restrict__ needed) {
    const int tile = blockIdx.x;
    int w = 0;
    for (int b = 0; b < g.cell_blocks; ++b) w = max(w, walk_len[tile * g.cell_blocks + b]);
    const int64_t begin = tile_offsets[tile];
    for (int p = threadIdx.x; p < w; p += blockDim.x) needed[list[begin + p]] = 1;
}

// flag of the r-th Gaussian in Morton order (int64 for the scan); flags[n] = 0
__global__ void k_flags_in_order(int n, const int* __restrict__ order, const unsigned char* __restrict__ needed,
                                 int64_t* __restrict__ flags) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) flags[r] = needed[order[r]];
    else if (r == n) flags[r] = 0;
}

__global__ void k_compact(int n, const int* __restrict__ order, const unsigned char* __restrict__ needed,
                          const int64_t* __restrict__ pos, int* __restrict__ out, int* __restrict__ count) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n && needed[order[r]]) out[pos[r]] = order[r];
    if (r == n) *count = static_cast<int>(pos[n]);
}

}  // namespace

int compact_needed(rxgs_ctx ctx, const rxgs_scene_s& sc, rxgs_txstate_s& st, cudaStream_t s) {
    const int K = st.k;
    RXGS_CUDA(st.needed.ensure(static_cast<size_t>(K + 1)));
    RXGS_CUDA(st.needed_order.ensure(sizeof(int) * (K + 1)));
    RXGS_CUDA(st.needed_count.ensure(sizeof(int) * 4));
    RXGS_CUDA(st.scan.ensure(sizeof(int64_t) * (K + 2)));  // free after binning: the flag scan
    RXGS_CUDA(ctx->scratch_b.ensure(sizeof(int64_t) * scan_bsum_count(K + 1)));
    unsigned char* needed = st.needed.as<unsigned char>();
    RXGS_CUDA(cudaMemsetAsync(needed, 0, static_cast<size_t>(K + 1), s));
    RXGS_CUDA(cudaMemsetAsync(st.needed_count.p, 0, sizeof(int), s));
    if (st.entries > 0)
        k_mark_needed<<<st.grid.n_tiles, 128, 0, s>>>(st.grid, st.tile_offsets.as<int64_t>(), st.list.as<int>(),
                                                       st.walk_len.as<int>(), needed);
    if (st.visible > 0 && K > 0) {
        // compact in the scene's spatial (Morton) order: consecutive
        // conditioning rows are nearby Gaussians (k_cond_tc.cu)
        int64_t* pos = st.scan.as<int64_t>();
        k_flags_in_order<<<(K + 1 + 255) / 256, 256, 0, s>>>(K, sc.d_morton.as<int>(), needed, pos);
        RXGS_CUDA(scan_i64(K + 1, pos, pos, ctx->scratch_b.as<int64_t>(), s));
        k_compact<<<(K + 1 + 255) / 256, 256, 0, s>>>(K, sc.d_morton.as<int>(), needed, pos,
                                                     st.needed_order.as<int>(), st.needed_count.as<int>());
    }
    st.needed_host = -1;
    if (ctx->profile) {  // roofline bookkeeping only: the row count of the next conditioning launch
        int h = 0;
        RXGS_CUDA(cudaMemcpyAsync(&h, st.needed_count.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        RXGS_CUDA(cudaStreamSynchronize(s));
        st.needed_host = h;
    }
    ctx->launches += 4;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? RXGS_OK : cuda_fail(e, "compact_needed");
}

// ------------------------------------------------------------- scene order
// Morton (Z-order) permutation of the scene's Gaussians over their bounding
// box, 10 bits per axis: the spatial order the conditioning kernel walks
// rows in, so a warp's 32 occupancy probes stay within a few voxels.
namespace {
__device__ __forceinline__ uint32_t spread3(uint32_t v) {
    v &= 0x3FFu;
    v = (v | (v << 16)) & 0x030000FFu;
    v = (v | (v << 8)) & 0x0300F00Fu;
    v = (v | (v << 4)) & 0x030C30C3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}
__global__ void k_morton(int K, const float4* __restrict__ pos, float lx, float ly, float lz, float sx, float sy,
                         float sz, uint32_t* __restrict__ key, int* __restrict__ idx) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    const float4 p = pos[k];
    auto q = [](float v, float lo, float sc) {
        const float u = (v - lo) * sc;
        return static_cast<uint32_t>(fminf(fmaxf(u, 0.f), 1023.f));
    };
    key[k] = (spread3(q(p.x, lx, sx)) << 2) | (spread3(q(p.y, ly, sy)) << 1) | spread3(q(p.z, lz, sz));
    idx[k] = k;
}
__global__ void k_gather_pos(int K, const int* __restrict__ order, const float4* __restrict__ pos,
                             float4* __restrict__ out) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < K) out[r] = pos[order[r]];
}
}  // namespace

int build_scene_order(rxgs_ctx ctx, rxgs_scene_s& sc, cudaStream_t s) {
    const int K = sc.k;
    RXGS_CUDA(sc.d_morton.ensure(sizeof(int) * std::max(K, 1)));
    RXGS_CUDA(sc.d_mpos32.ensure(sizeof(float4) * std::max(K, 1)));
    if (K == 0) return RXGS_OK;
    double lo[3], hi[3];
    for (int a = 0; a < 3; ++a) {
        lo[a] = 1.7976931348623157e308;
        hi[a] = -1.7976931348623157e308;
    }
    for (int k = 0; k < K; ++k)
        for (int a = 0; a < 3; ++a) {
            lo[a] = std::min(lo[a], sc.h_pos[3 * k + a]);
            hi[a] = std::max(hi[a], sc.h_pos[3 * k + a]);
        }
    float scale[3];
    for (int a = 0; a < 3; ++a) scale[a] = hi[a] > lo[a] ? static_cast<float>(1024.0 / (hi[a] - lo[a])) : 0.f;
    const size_t wi = radix_sort_work_ints(K);
    DevBuf keys;
    RXGS_CUDA(keys.ensure(static_cast<size_t>(K) * 4 * 3 + 4 * wi));
    uint32_t* k_in = keys.as<uint32_t>();
    uint32_t* k_tmp = k_in + K;
    int* i_tmp = reinterpret_cast<int*>(k_tmp + K);
    int* work = i_tmp + K;
    RXGS_CUDA(cudaMemsetAsync(work, 0, 4 * wi, s));
    k_morton<<<(K + 255) / 256, 256, 0, s>>>(K, sc.d_pos32.as<float4>(), static_cast<float>(lo[0]),
                                              static_cast<float>(lo[1]), static_cast<float>(lo[2]), scale[0],
                                              scale[1], scale[2], k_in, sc.d_morton.as<int>());
    RXGS_CUDA(radix_sort_pairs(K, 30, k_in, sc.d_morton.as<int>(), k_tmp, i_tmp, work, false, s));
    k_gather_pos<<<(K + 255) / 256, 256, 0, s>>>(K, sc.d_morton.as<int>(), sc.d_pos32.as<float4>(),
                                                  sc.d_mpos32.as<float4>());
    RXGS_CUDA(cudaStreamSynchronize(s));  // keys is freed on return
    return RXGS_OK;
}

}  // namespace rxgs_b200
