// Receiver-independent front-to-back blend weights, FP64 (-fmad=false).
//
// render_field (sphraster.cpp:278-298) walks each cell's tile list, computing
// w = min(tau * exp(-m2/2), 0.999) (gaussian_weight :239-251), accumulating
// T*w*s for every receiver, updating T *= 1-w and stopping once T < 1e-4.
// Neither w nor T depends on the receiver, so the walk is done ONCE per
// transmitter here, in FP64 with the reference's operation order (the exit
// decision is a discontinuity: it must be taken exactly where the reference
// takes it).  The result is the blend-weight matrix of every tile,
//     tw[entry][cell] = T_prev(cell, entry) * w(cell, entry)    (f32),
// zero past each cell's exit, truncated at the tile's longest walk.  The
// per-receiver composite is then a plain (cells x walk) x (walk x receivers)
// product (k_composite.cu).
//
// One CTA per (tile, 64-cell block), 256 threads.  Records are staged
// through shared memory in chunks of 64 list entries.  Only the
// transmittance recurrence is sequential, so each chunk runs in two phases:
//   A. all 256 threads evaluate the weights of the chunk's (entry, cell)
//      pairs of still-alive cells (4 threads per cell, 16 independent exp
//      chains each) into shared memory;
//   B. the 64 cell owners run T through the chunk in list order, exactly as
//      the reference does, writing tw and stopping at T < 1e-4.
// The kernel's duration is set by the longest tile walk, so phase A's 4-way
// parallelism is what shortens it.  The CTA stops loading as soon as every
// cell has exited.
#include "rxgs_internal.cuh"

namespace rxgs_b200 {
namespace {

#ifndef RXGS_WALK_CHUNK
#define RXGS_WALK_CHUNK 128  // A/B: 128 > 64 > 32 (config-3 walk 17.5 / 18.6 / 21.1 ms)
#endif
[[maybe_unused]] constexpr int kChunk = RXGS_WALK_CHUNK;
#ifndef RXGS_WALK_THREADS
#define RXGS_WALK_THREADS 384  // A/B (walk ms, config 2 / config 5): 512: 0.118 / 0.377, 384: 0.114 / 0.336, 256: 0.131 / 0.357
#endif
constexpr int kWalkThreads = RXGS_WALK_THREADS;
constexpr int kLanesPerCell = kWalkThreads / kMaxCellsPerBlock;

__device__ __forceinline__ double wrap_pm_pi(double a) {  // linalg.hpp:152-157
    // fmod(a, 2 pi) is exact and returns a itself when |a| < 2 pi -- always
    // the case for two azimuths in [0, 2 pi) -- so the call is skipped there
    if (!(fabs(a) < kTwoPi)) a = fmod(a, kTwoPi);
    if (a > kPi) a -= kTwoPi;
    if (a <= -kPi) a += kTwoPi;
    return a;
}

#ifndef RXGS_WALK_PIPE
#define RXGS_WALK_PIPE 1
#endif
#if !RXGS_WALK_PIPE
__global__ void __launch_bounds__(kWalkThreads) k_walk(DevGrid g, const int64_t* __restrict__ tile_offsets,
                                                       const int* __restrict__ list,
                                                       const GaussRec* __restrict__ rec, float* __restrict__ tw,
                                                       int* __restrict__ walk_len, double* __restrict__ cell_T,
                                                       int* __restrict__ cell_len) {
    extern __shared__ __align__(16) uint8_t walk_smem[];
    GaussRec* srec = reinterpret_cast<GaussRec*>(walk_smem);
    double(*sw)[kMaxCellsPerBlock] = reinterpret_cast<double(*)[kMaxCellsPerBlock]>(walk_smem + sizeof(GaussRec) * kChunk);
    __shared__ int s_alive[kMaxCellsPerBlock];
    __shared__ int s_len[kMaxCellsPerBlock];
    __shared__ int s_max, s_min;
    const int tile = blockIdx.x;
    const int cb = blockIdx.y;
    const int tid = threadIdx.x;
    const int cl = tid % kMaxCellsPerBlock;  // this thread's cell in phase A
    const int tt = tile / g.tiles_p, tp = tile % g.tiles_p;
    const int lc = cb * kMaxCellsPerBlock + cl;
    const int row = tt * g.ts + lc / g.ts;
    const int col = tp * g.ts + lc % g.ts;
    const bool valid = lc < g.cpt && (lc / g.ts) < g.ts && row < g.nt && col < g.np;
    const int64_t begin = tile_offsets[tile];
    const int n = static_cast<int>(tile_offsets[tile + 1] - begin);
    const size_t stride = static_cast<size_t>(g.cell_blocks) * kMaxCellsPerBlock;
    float* out = tw + static_cast<size_t>(begin) * stride + static_cast<size_t>(cb) * kMaxCellsPerBlock + cl;
    const bool owner = tid < kMaxCellsPerBlock;

    const double theta_r = valid ? g.tmin + (row + 0.5) * g.dth : 0.0;
    const double phi_r = valid ? (col + 0.5) * g.dph : 0.0;
    double T = 1.0;
    int len = valid ? n : 0;
    bool alive = owner && valid && n > 0;
    if (owner) s_alive[cl] = alive ? 1 : 0;
    if (tid == 0) {
        s_max = 0;
        s_min = 0x7fffffff;
    }
    for (int c0 = 0; c0 < n; c0 += kChunk) {
        if (!__syncthreads_or(alive)) break;
        const int m = min(kChunk, n - c0);
        for (int q = tid; q < m; q += kWalkThreads) srec[q] = rec[list[begin + c0 + q]];
        __syncthreads();
        if (s_alive[cl]) {  // phase A: weights (gaussian_weight, sphraster.cpp:239-251)
            for (int e = tid / kMaxCellsPerBlock; e < m; e += kLanesPerCell) {
                const GaussRec& r = srec[e];
                const double dt = theta_r - r.theta;
                const double dpraw = wrap_pm_pi(phi_r - r.phi);
                const double dp = r.sin_theta * dpraw;
                const double m2 = r.pa * dt * dt + r.pbc * dt * dp + r.pd * dp * dp;
                const double w = r.tau * exp(-0.5 * m2);
                sw[e][cl] = kWeightClamp < w ? kWeightClamp : w;  // std::min(w, 0.999)
            }
        }
        __syncthreads();
        if (alive) {  // phase B: the front-to-back recurrence (render_field :285-298)
            for (int e = 0; e < m; ++e) {
                const double w = sw[e][cl];
                out[static_cast<size_t>(c0 + e) * stride] = static_cast<float>(T * w);
                T *= 1.0 - w;
                if (T < kEarlyExitT) {
                    len = c0 + e + 1;
                    alive = false;
                    break;
                }
            }
            s_alive[cl] = alive ? 1 : 0;
        }
    }
    if (owner) {
        s_len[cl] = len;
        atomicMax(&s_max, len);
        atomicMin(&s_min, len);
    }
    __syncthreads();
    const int wmax = s_max;
    // zero the rows past each cell's exit up to the tile's longest walk
    for (int e = s_min + tid / kMaxCellsPerBlock; e < wmax; e += kLanesPerCell)
        if (e >= s_len[cl]) out[static_cast<size_t>(e) * stride] = 0.0f;
    if (tid == 0) walk_len[tile * g.cell_blocks + cb] = wmax;
    if (owner && valid) {
        const size_t cell = static_cast<size_t>(row) * g.np + col;
        cell_T[cell] = T;
        cell_len[cell] = len;
    }
}

#endif  // !RXGS_WALK_PIPE

// Pipelined variant (RXGS_WALK_PIPE, default): the two phases run
// concurrently on different warps -- warps 0-1 (the 64 cell owners) run the
// recurrence of chunk c while warps 2-15 stage the records of chunk c+1 and
// evaluate its weights into the other half of a double buffer -- so a chunk
// costs max(A, B) instead of A + B.  The producers skip cells that had
// exited by the end of chunk c-1 (a cell exiting during chunk c costs at
// most one chunk of unneeded weights).  Same arithmetic, same order: the
// output is identical to the two-phase kernel.
#ifndef RXGS_WALK_PCHUNK
#define RXGS_WALK_PCHUNK 64
#endif
constexpr int kPipeChunk = RXGS_WALK_PCHUNK;
constexpr int kProducers = kWalkThreads - kMaxCellsPerBlock;  // 320

__global__ void __launch_bounds__(kWalkThreads) k_walk_pipe(DevGrid g, const int64_t* __restrict__ tile_offsets,
                                                            const int* __restrict__ list,
                                                            const GaussRec* __restrict__ rec, float* __restrict__ tw,
                                                            int* __restrict__ walk_len, double* __restrict__ cell_T,
                                                            int* __restrict__ cell_len) {
    extern __shared__ __align__(16) uint8_t walk_smem[];
    GaussRec* srec = reinterpret_cast<GaussRec*>(walk_smem);  // [2][kPipeChunk]
    double(*sw)[kMaxCellsPerBlock] =
        reinterpret_cast<double(*)[kMaxCellsPerBlock]>(walk_smem + sizeof(GaussRec) * 2 * kPipeChunk);  // [2 * chunk][64]
    __shared__ int s_alive[kMaxCellsPerBlock];
    __shared__ int s_len[kMaxCellsPerBlock];
    __shared__ int s_max, s_min;
    const int tile = blockIdx.x;
    const int cb = blockIdx.y;
    const int tid = threadIdx.x;
    const bool owner = tid < kMaxCellsPerBlock;
    const int cl = tid % kMaxCellsPerBlock;  // owner: its cell; producer: the cell it evaluates
    const int tt = tile / g.tiles_p, tp = tile % g.tiles_p;
    const int lc = cb * kMaxCellsPerBlock + cl;
    const int row = tt * g.ts + lc / g.ts;
    const int col = tp * g.ts + lc % g.ts;
    const bool valid = lc < g.cpt && (lc / g.ts) < g.ts && row < g.nt && col < g.np;
    const int64_t begin = tile_offsets[tile];
    const int n = static_cast<int>(tile_offsets[tile + 1] - begin);
    const size_t stride = static_cast<size_t>(g.cell_blocks) * kMaxCellsPerBlock;
    float* out = tw + static_cast<size_t>(begin) * stride + static_cast<size_t>(cb) * kMaxCellsPerBlock + cl;
    const double theta_r = valid ? g.tmin + (row + 0.5) * g.dth : 0.0;
    const double phi_r = valid ? (col + 0.5) * g.dph : 0.0;
    double T = 1.0;
    int len = valid ? n : 0;
    bool alive = owner && valid && n > 0;
    if (owner) s_alive[cl] = alive ? 1 : 0;
    if (tid == 0) {
        s_max = 0;
        s_min = 0x7fffffff;
    }
    __syncthreads();
    const int n_ch = (n + kPipeChunk - 1) / kPipeChunk;
    const int ptid = tid - kMaxCellsPerBlock;  // producer index (owners: negative)
    // producer step: records of chunk ch into half ch % 2, then its weights
    auto produce = [&](int ch) {
        const int h = ch & 1;
        const int c0 = ch * kPipeChunk;
        const int m = min(kPipeChunk, n - c0);
        for (int q = ptid; q < m; q += kProducers) srec[h * kPipeChunk + q] = rec[list[begin + c0 + q]];
        asm volatile("bar.sync 1, %0;" ::"n"(kProducers) : "memory");  // producers only
        if (!*reinterpret_cast<volatile int*>(&s_alive[cl])) return;  // exited (by the end of the chunk before last)
        for (int e = ptid / kMaxCellsPerBlock; e < m; e += kProducers / kMaxCellsPerBlock) {
            const GaussRec& r = srec[h * kPipeChunk + e];
            const double dt = theta_r - r.theta;
            const double dpraw = wrap_pm_pi(phi_r - r.phi);
            const double dp = r.sin_theta * dpraw;
            const double m2 = r.pa * dt * dt + r.pbc * dt * dp + r.pd * dp * dp;
            const double w = r.tau * exp(-0.5 * m2);
            sw[h * kPipeChunk + e][cl] = kWeightClamp < w ? kWeightClamp : w;  // std::min(w, 0.999)
        }
    };
    if (!owner && n_ch > 0) produce(0);
    for (int ch = 0; ch < n_ch; ++ch) {
        if (!__syncthreads_or(alive)) break;  // chunk ch's weights are ready; every cell exited -> stop
        if (owner) {
            if (alive) {  // the front-to-back recurrence (render_field :285-298)
                const int h = ch & 1, c0 = ch * kPipeChunk, m = min(kPipeChunk, n - c0);
                for (int e = 0; e < m; ++e) {
                    const double w = sw[h * kPipeChunk + e][cl];
                    out[static_cast<size_t>(c0 + e) * stride] = static_cast<float>(T * w);
                    T *= 1.0 - w;
                    if (T < kEarlyExitT) {
                        len = c0 + e + 1;
                        alive = false;
                        break;
                    }
                }
                s_alive[cl] = alive ? 1 : 0;
            }
        } else if (ch + 1 < n_ch) {
            produce(ch + 1);
        }
    }
    if (owner) {
        s_len[cl] = len;
        atomicMax(&s_max, len);
        atomicMin(&s_min, len);
    }
    __syncthreads();
    const int wmax = s_max;
    // zero the rows past each cell's exit up to the tile's longest walk
    for (int e = s_min + tid / kMaxCellsPerBlock; e < wmax; e += kLanesPerCell)
        if (e >= s_len[cl]) out[static_cast<size_t>(e) * stride] = 0.0f;
    if (tid == 0) walk_len[tile * g.cell_blocks + cb] = wmax;
    if (owner && valid) {
        const size_t cell = static_cast<size_t>(row) * g.np + col;
        cell_T[cell] = T;
        cell_len[cell] = len;
    }
}

}  // namespace

cudaError_t launch_walk(rxgs_txstate_s& st, cudaStream_t s) {
    const DevGrid& g = st.grid;
    dim3 grid(g.n_tiles, g.cell_blocks);
#if RXGS_WALK_PIPE
    const size_t smem = 2 * (sizeof(GaussRec) * kPipeChunk + sizeof(double) * kPipeChunk * kMaxCellsPerBlock);
    cudaFuncSetAttribute(k_walk_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k_walk_pipe<<<grid, kWalkThreads, smem, s>>>(g, st.tile_offsets.as<int64_t>(), st.list.as<int>(),
                                                  st.rec.as<GaussRec>(), st.tw.as<float>(), st.walk_len.as<int>(),
                                                  st.cell_T.as<double>(), st.cell_len.as<int>());
#else
    const size_t smem = sizeof(GaussRec) * kChunk + sizeof(double) * kChunk * kMaxCellsPerBlock;
    cudaFuncSetAttribute(k_walk, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k_walk<<<grid, kWalkThreads, smem, s>>>(g, st.tile_offsets.as<int64_t>(), st.list.as<int>(),
                               st.rec.as<GaussRec>(), st.tw.as<float>(), st.walk_len.as<int>(),
                               st.cell_T.as<double>(), st.cell_len.as<int>());
#endif
    return cudaGetLastError();
}

}  // namespace rxgs_b200
