// Stage-I densification: densify_and_prune
// (scene.cpp:178-274), DensifyState::accumulate (scene.cpp:141-151) and
// reset_transmittance (scene.cpp:276-279) on the device.
//
// densify_and_prune as stream compaction over the Gaussians:
//   k_dens_classify  mean |dL/dp| and size -> keep / clone / split
//   2 exclusive scans appended rank (clone + split) and split rank
//   k_dens_build     the merged scene of K + A rows: row i in place (the
//                    first child for a split), row K + rank_i appended (the
//                    clone, or the second child); the split sign is the
//                    split's own draw of the "scene.densify" stream, taken by
//                    random access (SplitMix64: the r-th state is s0 + (r+1) g);
//                    each merged row gets its prune flag
//   1 exclusive scan surviving rank
//   k_dens_compact   survivors in merged order + their source rows
// Compiled without FMA contraction (like the FP64 geometry) so positions and
// scales follow the reference's rounding.

#include <cmath>

#include "rxgs_internal.cuh"

namespace rxgs_b200 {
namespace {

// detail::mix64 / Rng::uniform (rng.hpp:20-31, 58-62)
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ double uniform_at(uint64_t s0, uint64_t r) {
    return static_cast<double>(mix64(s0 + (r + 1) * 0x9e3779b97f4a7c15ull) >> 11) * 0x1.0p-53;
}

// gaussian_size (scene.cpp:155-158): exp of the largest log scale
__device__ __forceinline__ double gsize(const double* ls) {
    double m = ls[0];
    if (ls[1] > m) m = ls[1];
    if (ls[2] > m) m = ls[2];
    return exp(m);
}

__global__ void k_dens_classify(int K, const double* __restrict__ accum, const int* __restrict__ count,
                                const double* __restrict__ ls, double grad_thr, double size_bound,
                                uint8_t* __restrict__ op, int* __restrict__ app, int* __restrict__ spl) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= K) return;
    const double mean = count[i] > 0 ? accum[i] / static_cast<double>(count[i]) : 0.0;
    uint8_t o = 0;
    if (!(mean <= grad_thr)) o = gsize(ls + 3 * static_cast<size_t>(i)) < size_bound ? 1 : 2;
    op[i] = o;
    app[i] = o != 0;
    spl[i] = o == 2;
}

struct SceneRows {
    double *pos, *ls, *q, *tau, *co;
};

__device__ __forceinline__ void copy_row(const SceneRows& s, int i, const SceneRows& d, int r, int stride) {
    for (int a = 0; a < 3; ++a) d.pos[3 * static_cast<size_t>(r) + a] = s.pos[3 * static_cast<size_t>(i) + a];
    for (int a = 0; a < 3; ++a) d.ls[3 * static_cast<size_t>(r) + a] = s.ls[3 * static_cast<size_t>(i) + a];
    for (int a = 0; a < 4; ++a) d.q[4 * static_cast<size_t>(r) + a] = s.q[4 * static_cast<size_t>(i) + a];
    d.tau[r] = s.tau[i];
    for (int a = 0; a < stride; ++a)
        d.co[static_cast<size_t>(r) * stride + a] = s.co[static_cast<size_t>(i) * stride + a];
}

__global__ void k_dens_build(int K, int stride, SceneRows src, SceneRows mrg, const uint8_t* __restrict__ op,
                             const int* __restrict__ app_rank, const int* __restrict__ split_rank, uint64_t s0,
                             double shrink, double prune_bound, int* __restrict__ msrc, int* __restrict__ keep) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= K) return;
    const uint8_t o = op[i];
    copy_row(src, i, mrg, i, stride);
    msrc[i] = o == 2 ? -1 : i;
    if (o != 0) {
        const int r2 = K + app_rank[i];
        copy_row(src, i, mrg, r2, stride);
        msrc[r2] = -1;
        if (o == 2) {
            // quat_to_rotation (linalg.hpp:122-131), column of the largest scale
            const double* q = src.q + 4 * static_cast<size_t>(i);
            const double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
            const double w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
            const double rm[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z),     2 * (x * z + w * y),
                                  2 * (x * y + w * z),     1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                                  2 * (x * z - w * y),     2 * (y * z + w * x),     1 - 2 * (x * x + y * y)};
            const double* ls = src.ls + 3 * static_cast<size_t>(i);
            int axis = 0;
            for (int a = 1; a < 3; ++a)
                if (ls[a] > ls[axis]) axis = a;
            const double sigma = exp(ls[axis]);
            const double side = uniform_at(s0, static_cast<uint64_t>(split_rank[i])) < 0.5 ? 1.0 : -1.0;
            for (int a = 0; a < 3; ++a) {
                mrg.pos[3 * static_cast<size_t>(i) + a] += side * sigma * rm[a * 3 + axis];
                mrg.pos[3 * static_cast<size_t>(r2) + a] -= side * sigma * rm[a * 3 + axis];
            }
            for (int a = 0; a < 3; ++a) {
                mrg.ls[3 * static_cast<size_t>(i) + a] += shrink;
                mrg.ls[3 * static_cast<size_t>(r2) + a] += shrink;
            }
        }
        keep[r2] = !(gsize(mrg.ls + 3 * static_cast<size_t>(r2)) > prune_bound);
    }
    keep[i] = !(gsize(mrg.ls + 3 * static_cast<size_t>(i)) > prune_bound);
}

__global__ void k_dens_compact(int M, int stride, SceneRows mrg, SceneRows out, const int* __restrict__ keep,
                               const int* __restrict__ rank, const int* __restrict__ msrc, int* __restrict__ source) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= M || !keep[i]) return;
    const int r = rank[i];
    copy_row(mrg, i, out, r, stride);
    source[r] = msrc[i];
}

// DensifyState::accumulate: grad_accum += ||dL/dp_k||, accum_count += 1
__global__ void k_dens_accumulate(int K, const double* __restrict__ dpos, double* __restrict__ accum,
                                  int* __restrict__ count) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= K) return;
    const double gx = dpos[3 * static_cast<size_t>(i)], gy = dpos[3 * static_cast<size_t>(i) + 1],
                 gz = dpos[3 * static_cast<size_t>(i) + 2];
    accum[i] += sqrt(gx * gx + gy * gy + gz * gz);
    count[i] += 1;
}

__global__ void k_fill(int64_t n, double v, double* __restrict__ x) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) x[i] = v;
}

// Optimizer::remap_rows (diffengine.cpp:60-79): moments of surviving rows
// follow their source row, new rows start at zero
__global__ void k_remap_rows(int n_rows, int width, const int* __restrict__ source, const double* __restrict__ in,
                             double* __restrict__ out) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= static_cast<int64_t>(n_rows) * width) return;
    const int r = static_cast<int>(i / width), a = static_cast<int>(i % width);
    const int s = source[r];
    out[i] = s < 0 ? 0.0 : in[static_cast<int64_t>(s) * width + a];
}

unsigned blocks(int64_t n) { return static_cast<unsigned>((n + 255) / 256); }

bool on_device(const void* p) {
    cudaPointerAttributes a{};
    if (!p || cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int exclusive_sum(rxgs_ctx ctx, const int* in, int* out, int n, cudaStream_t s) {
    RXGS_CUDA(ctx->sort_tmp.ensure(sizeof(int64_t) * scan_bsum_count(n)));
    RXGS_CUDA(scan_i32(n, in, out, ctx->sort_tmp.as<int64_t>(), s));
    return RXGS_OK;
}

}  // namespace

cudaError_t launch_dens_accumulate(int K, const double* dpos, double* accum, int* count, cudaStream_t s) {
    if (K == 0) return cudaSuccess;
    k_dens_accumulate<<<blocks(K), 256, 0, s>>>(K, dpos, accum, count);
    return cudaGetLastError();
}

cudaError_t launch_remap_rows(int n_rows, int width, const int* source, const double* in, double* out,
                              cudaStream_t s) {
    const int64_t n = static_cast<int64_t>(n_rows) * width;
    if (n == 0) return cudaSuccess;
    k_remap_rows<<<blocks(n), 256, 0, s>>>(n_rows, width, source, in, out);
    return cudaGetLastError();
}

cudaError_t launch_fill64(int64_t n, double v, double* x, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_fill<<<blocks(n), 256, 0, s>>>(n, v, x);
    return cudaGetLastError();
}

int densify_scene(rxgs_ctx ctx, rxgs_scene_s* sc, const double* d_accum, const int* d_count, double extent,
                  const double thr[4], uint64_t stream_state, int report[3], DevBuf& source_out) {
    cudaStream_t s = ctx->stream;
    const int K = sc->k;
    const int stride = sc->L * sc->channels * 2;
    report[0] = report[1] = report[2] = 0;
    DevBuf op, app, spl, app_r, spl_r;
    RXGS_CUDA(op.ensure(std::max(K, 1)));
    RXGS_CUDA(app.ensure(sizeof(int) * (std::max(K, 1) + 1)));
    RXGS_CUDA(spl.ensure(sizeof(int) * (std::max(K, 1) + 1)));
    RXGS_CUDA(app_r.ensure(sizeof(int) * (std::max(K, 1) + 1)));
    RXGS_CUDA(spl_r.ensure(sizeof(int) * (std::max(K, 1) + 1)));
    // the host evaluates the thresholds exactly as the reference writes them
    const double size_bound = thr[1] * extent, prune_bound = thr[2] * extent, shrink = std::log(thr[3]);
    RXGS_CUDA(cudaMemsetAsync(app.p, 0, sizeof(int) * (K + 1), s));
    RXGS_CUDA(cudaMemsetAsync(spl.p, 0, sizeof(int) * (K + 1), s));
    if (K > 0)
        k_dens_classify<<<blocks(K), 256, 0, s>>>(K, d_accum, d_count, sc->d_ls.as<double>(), thr[0], size_bound,
                                                  op.as<uint8_t>(), app.as<int>(), spl.as<int>());
    TRY_RC(exclusive_sum(ctx, app.as<int>(), app_r.as<int>(), K + 1, s));
    TRY_RC(exclusive_sum(ctx, spl.as<int>(), spl_r.as<int>(), K + 1, s));
    int A = 0, S = 0;
    RXGS_CUDA(cudaMemcpyAsync(&A, app_r.as<int>() + K, sizeof(int), cudaMemcpyDeviceToHost, s));
    RXGS_CUDA(cudaMemcpyAsync(&S, spl_r.as<int>() + K, sizeof(int), cudaMemcpyDeviceToHost, s));
    RXGS_CUDA(cudaStreamSynchronize(s));
    const int M = K + A;
    DevBuf mp, ml, mq, mt, mc, msrc, keep, keep_r;
    RXGS_CUDA(mp.ensure(sizeof(double) * 3 * std::max(M, 1)));
    RXGS_CUDA(ml.ensure(sizeof(double) * 3 * std::max(M, 1)));
    RXGS_CUDA(mq.ensure(sizeof(double) * 4 * std::max(M, 1)));
    RXGS_CUDA(mt.ensure(sizeof(double) * std::max(M, 1)));
    RXGS_CUDA(mc.ensure(sizeof(double) * std::max<size_t>(static_cast<size_t>(M) * stride, 1)));
    RXGS_CUDA(msrc.ensure(sizeof(int) * std::max(M, 1)));
    RXGS_CUDA(keep.ensure(sizeof(int) * (M + 1)));
    RXGS_CUDA(keep_r.ensure(sizeof(int) * (M + 1)));
    RXGS_CUDA(cudaMemsetAsync(keep.p, 0, sizeof(int) * (M + 1), s));
    const SceneRows src{sc->d_pos.as<double>(), sc->d_ls.as<double>(), sc->d_q.as<double>(), sc->d_tau.as<double>(),
                        sc->d_coeffs64.as<double>()};
    const SceneRows mrg{mp.as<double>(), ml.as<double>(), mq.as<double>(), mt.as<double>(), mc.as<double>()};
    if (K > 0)
        k_dens_build<<<blocks(K), 256, 0, s>>>(K, stride, src, mrg, op.as<uint8_t>(), app_r.as<int>(),
                                               spl_r.as<int>(), stream_state, shrink, prune_bound, msrc.as<int>(),
                                               keep.as<int>());
    TRY_RC(exclusive_sum(ctx, keep.as<int>(), keep_r.as<int>(), M + 1, s));
    int K2 = 0;
    RXGS_CUDA(cudaMemcpyAsync(&K2, keep_r.as<int>() + M, sizeof(int), cudaMemcpyDeviceToHost, s));
    RXGS_CUDA(cudaStreamSynchronize(s));
    DevBuf np, nl, nq, nt, nc;
    RXGS_CUDA(np.ensure(sizeof(double) * 3 * std::max(K2, 1)));
    RXGS_CUDA(nl.ensure(sizeof(double) * 3 * std::max(K2, 1)));
    RXGS_CUDA(nq.ensure(sizeof(double) * 4 * std::max(K2, 1)));
    RXGS_CUDA(nt.ensure(sizeof(double) * std::max(K2, 1)));
    RXGS_CUDA(nc.ensure(sizeof(double) * std::max<size_t>(static_cast<size_t>(K2) * stride, 1)));
    RXGS_CUDA(source_out.ensure(sizeof(int) * std::max(K2, 1)));
    const SceneRows out{np.as<double>(), nl.as<double>(), nq.as<double>(), nt.as<double>(), nc.as<double>()};
    if (M > 0)
        k_dens_compact<<<blocks(M), 256, 0, s>>>(M, stride, mrg, out, keep.as<int>(), keep_r.as<int>(),
                                                 msrc.as<int>(), source_out.as<int>());
    RXGS_CUDA(cudaGetLastError());
    RXGS_CUDA(cudaStreamSynchronize(s));
    sc->d_pos = std::move(np);
    sc->d_ls = std::move(nl);
    sc->d_q = std::move(nq);
    sc->d_tau = std::move(nt);
    sc->d_coeffs64 = std::move(nc);
    sc->k = K2;
    sc->coeff_version += 1;
    sc->geo_version += 1;
    report[0] = A - S;
    report[1] = S;
    report[2] = M - K2;
    ctx->launches += 6;
    return scene_resized(sc);
}

}  // namespace rxgs_b200

using namespace rxgs_b200;

extern "C" {

int rxgs_densify_and_prune(rxgs_ctx ctx, rxgs_scene scene, const double* grad_accum, const int32_t* accum_count,
                           double scene_extent, const double thresholds[4], uint64_t seed, uint64_t pass_index,
                           int32_t report[3], int32_t* source_row, int32_t* new_count) {
    if (!ctx || !scene) return fail(RXGS_ERR_INVALID, "densify_and_prune: null argument");
    const int K = scene->k;
    if (K > 0 && (!grad_accum || !accum_count)) return fail(RXGS_ERR_INVALID, "densify_and_prune: state size mismatch");
    RXGS_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const double def[4] = {2e-4, 0.01, 0.1, 0.8};  // DensifyThresholds (scene.hpp:81-86)
    const double* thr = thresholds ? thresholds : def;
    DevBuf t_acc, t_cnt, src;
    const double* d_acc = grad_accum;
    const int* d_cnt = accum_count;
    if (K > 0 && !on_device(grad_accum)) {
        RXGS_CUDA(t_acc.ensure(sizeof(double) * K));
        RXGS_CUDA(cudaMemcpyAsync(t_acc.p, grad_accum, sizeof(double) * K, cudaMemcpyHostToDevice, s));
        d_acc = t_acc.as<double>();
    }
    if (K > 0 && !on_device(accum_count)) {
        RXGS_CUDA(t_cnt.ensure(sizeof(int) * K));
        RXGS_CUDA(cudaMemcpyAsync(t_cnt.p, accum_count, sizeof(int) * K, cudaMemcpyHostToDevice, s));
        d_cnt = t_cnt.as<int>();
    }
    TRY_RC(scene_sync_host(scene));  // pending optimizer updates land before the rows move
    int rep[3];
    TRY_RC(densify_scene(ctx, scene, d_acc, d_cnt, scene_extent, thr, derive_stream_state(seed, "scene.densify", pass_index),
                         rep, src));
    if (report)
        for (int a = 0; a < 3; ++a) report[a] = rep[a];
    if (new_count) *new_count = scene->k;
    if (source_row && scene->k > 0)
        RXGS_CUDA(cudaMemcpy(source_row, src.p, sizeof(int) * scene->k, cudaMemcpyDefault));
    return RXGS_OK;
}

int rxgs_reset_transmittance(rxgs_scene scene) {
    if (!scene) return fail(RXGS_ERR_INVALID, "null scene");
    RXGS_CUDA(cudaSetDevice(scene->ctx->device));
    TRY_RC(scene_sync_host(scene));
    const double v = std::log(0.01 / (1.0 - 0.01));  // logit(0.01) (scene.cpp:276-279, linalg logit)
    RXGS_CUDA(launch_fill64(scene->k, v, scene->d_tau.as<double>(), scene->ctx->stream));
    scene->geo_stale = true;
    scene->geo_version += 1;  // tau enters the states' blend weights
    return RXGS_OK;
}

}  // extern "C"
