// Coverage consumers of the config-3 RSSI table and the
// evaluation metrics (met::mae / mse / psnr / ssim, k_train.cu kernels):
// apps::coverage_fraction and apps::greedy_plan (src/apps.cpp:53-116).
// Integer work on a tx-major table of FP64 dBm values, exact like the
// reference: a threshold test per (tx, candidate), counts, and a greedy
// maximum-coverage selection whose ties break on the lower candidate index.
//   k_cover_bits   candidate c -> bitset over transmitters of table > thr
//   k_cover_count  transmitters covered by a selection (coverage_fraction)
//   k_greedy       one CTA runs every round: gains = popcount(bits & ~covered),
//                  argmax with the lowest index on ties, covered |= bits[best]
#include "rxgs_internal.cuh"

namespace rxgs_b200 {
namespace {

__global__ void k_cover_bits(int64_t tx_count, int64_t cand, int words, const double* __restrict__ table,
                             double thr, uint32_t* __restrict__ bits) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= cand * words) return;
    const int64_t c = i / words;
    const int w = static_cast<int>(i % words);
    uint32_t m = 0;
    for (int b = 0; b < 32; ++b) {
        const int64_t t = static_cast<int64_t>(w) * 32 + b;
        if (t < tx_count && table[t * cand + c] > thr) m |= 1u << b;
    }
    bits[i] = m;
}

__global__ void k_cover_count(int64_t tx_count, int64_t cand, const double* __restrict__ table, const int* __restrict__ sel,
                              int n_sel, double thr, unsigned long long* __restrict__ count) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    bool cov = false;
    if (t < tx_count)
        for (int s = 0; s < n_sel && !cov; ++s) cov = table[t * cand + sel[s]] > thr;
    const unsigned n = __popc(__ballot_sync(0xffffffffu, cov));
    if ((threadIdx.x & 31) == 0 && n) atomicAdd(count, static_cast<unsigned long long>(n));
}

constexpr int kGreedyThreads = 1024;

__global__ void __launch_bounds__(kGreedyThreads) k_greedy(int64_t cand, int words, int k, const uint32_t* __restrict__ bits,
                                                           uint32_t* __restrict__ covered, uint8_t* __restrict__ chosen,
                                                           int* __restrict__ order) {
    __shared__ unsigned long long best_s[kGreedyThreads / 32];
    __shared__ int pick;
    const int tid = threadIdx.x;
    for (int w = tid; w < words; w += blockDim.x) covered[w] = 0u;
    for (int64_t c = tid; c < cand; c += blockDim.x) chosen[c] = 0;
    __syncthreads();
    for (int round = 0; round < k; ++round) {
        // key = gain << 32 | (0xFFFFFFFF - c): the max key is the largest gain, lowest index
        unsigned long long key = 0ull;
        for (int64_t c = tid; c < cand; c += blockDim.x) {
            if (chosen[c]) continue;
            unsigned gain = 0;
            for (int w = 0; w < words; ++w) gain += __popc(bits[c * words + w] & ~covered[w]);
            const unsigned long long kk =
                (static_cast<unsigned long long>(gain) << 32) | (0xFFFFFFFFull - static_cast<unsigned long long>(c));
            key = kk > key ? kk : key;
        }
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long ot = __shfl_xor_sync(0xffffffffu, key, o);
            key = ot > key ? ot : key;
        }
        if ((tid & 31) == 0) best_s[tid >> 5] = key;
        __syncthreads();
        if (tid < 32) {
            unsigned long long v = tid < static_cast<int>(blockDim.x >> 5) ? best_s[tid] : 0ull;
            for (int o = 16; o > 0; o >>= 1) {
                const unsigned long long ot = __shfl_xor_sync(0xffffffffu, v, o);
                v = ot > v ? ot : v;
            }
            if (tid == 0) {
                pick = static_cast<int>(0xFFFFFFFFull - (v & 0xFFFFFFFFull));
                chosen[pick] = 1;
                order[round] = pick;
            }
        }
        __syncthreads();
        for (int w = tid; w < words; w += blockDim.x) covered[w] |= bits[static_cast<int64_t>(pick) * words + w];
        __syncthreads();
    }
}

}  // namespace
}  // namespace rxgs_b200

using namespace rxgs_b200;

namespace {
bool dev_ptr(const void* p) {
    cudaPointerAttributes a{};
    if (!p || cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}
}  // namespace

extern "C" {

int rxgs_coverage_fraction(rxgs_ctx ctx, const double* table, int64_t tx_count, int64_t cand_count,
                           const int32_t* selected, int n_selected, double threshold_dbm, double* out) {
    if (!ctx || !out) return fail(RXGS_ERR_INVALID, "coverage_fraction: null argument");
    if (n_selected <= 0 || !selected) return fail(RXGS_ERR_INVALID, "coverage_fraction: empty selection");
    if (!table || tx_count < 0 || cand_count < 0) return fail(RXGS_ERR_INVALID, "coverage_fraction: table shape mismatch");
    std::vector<int32_t> sel(n_selected);
    RXGS_CUDA(cudaMemcpy(sel.data(), selected, sizeof(int32_t) * n_selected, cudaMemcpyDefault));
    for (int32_t c : sel)
        if (c < 0 || c >= cand_count) return fail(RXGS_ERR_INVALID, "coverage_fraction: candidate index out of range");
    if (tx_count == 0) {
        *out = 0.0 / 0.0;  // 0 / 0, as the reference divides by tx_count
        return RXGS_OK;
    }
    RXGS_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    DevBuf t_tab, t_sel, t_cnt;
    const double* d_tab = table;
    if (!dev_ptr(table)) {
        RXGS_CUDA(t_tab.ensure(sizeof(double) * tx_count * cand_count));
        RXGS_CUDA(cudaMemcpyAsync(t_tab.p, table, sizeof(double) * tx_count * cand_count, cudaMemcpyHostToDevice, s));
        d_tab = t_tab.as<double>();
    }
    RXGS_CUDA(t_sel.ensure(sizeof(int32_t) * n_selected));
    RXGS_CUDA(cudaMemcpyAsync(t_sel.p, sel.data(), sizeof(int32_t) * n_selected, cudaMemcpyHostToDevice, s));
    RXGS_CUDA(t_cnt.ensure(sizeof(unsigned long long)));
    RXGS_CUDA(cudaMemsetAsync(t_cnt.p, 0, sizeof(unsigned long long), s));
    k_cover_count<<<static_cast<unsigned>((tx_count + 255) / 256), 256, 0, s>>>(
        tx_count, cand_count, d_tab, t_sel.as<int>(), n_selected, threshold_dbm, t_cnt.as<unsigned long long>());
    RXGS_CUDA(cudaGetLastError());
    unsigned long long n = 0;
    RXGS_CUDA(cudaMemcpyAsync(&n, t_cnt.p, sizeof(n), cudaMemcpyDeviceToHost, s));
    RXGS_CUDA(cudaStreamSynchronize(s));
    ctx->launches += 1;
    *out = static_cast<double>(n) / static_cast<double>(tx_count);
    return RXGS_OK;
}

int rxgs_greedy_plan(rxgs_ctx ctx, const double* table, int64_t tx_count, int64_t cand_count, int k,
                     double threshold_dbm, int32_t* order_out) {
    if (!ctx || !order_out) return fail(RXGS_ERR_INVALID, "greedy_plan: null argument");
    if (k < 1 || k > cand_count) return fail(RXGS_ERR_INVALID, "greedy_plan: k out of range");
    if (!table || tx_count < 0) return fail(RXGS_ERR_INVALID, "greedy_plan: table shape mismatch");
    if (cand_count > 0xFFFFFFFFll) return fail(RXGS_ERR_INVALID, "greedy_plan: too many candidates");
    RXGS_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const int words = static_cast<int>((tx_count + 31) / 32);
    DevBuf t_tab, t_bits, t_cov, t_ch, t_ord;
    const double* d_tab = table;
    if (!dev_ptr(table) && tx_count > 0) {
        RXGS_CUDA(t_tab.ensure(sizeof(double) * tx_count * cand_count));
        RXGS_CUDA(cudaMemcpyAsync(t_tab.p, table, sizeof(double) * tx_count * cand_count, cudaMemcpyHostToDevice, s));
        d_tab = t_tab.as<double>();
    }
    RXGS_CUDA(t_bits.ensure(sizeof(uint32_t) * std::max<int64_t>(cand_count * words, 1)));
    RXGS_CUDA(t_cov.ensure(sizeof(uint32_t) * std::max(words, 1)));
    RXGS_CUDA(t_ch.ensure(std::max<int64_t>(cand_count, 1)));
    RXGS_CUDA(t_ord.ensure(sizeof(int) * k));
    if (words > 0)
        k_cover_bits<<<static_cast<unsigned>((cand_count * words + 255) / 256), 256, 0, s>>>(
            tx_count, cand_count, words, d_tab, threshold_dbm, t_bits.as<uint32_t>());
    k_greedy<<<1, kGreedyThreads, 0, s>>>(cand_count, words, k, t_bits.as<uint32_t>(), t_cov.as<uint32_t>(),
                                          t_ch.as<uint8_t>(), t_ord.as<int>());
    RXGS_CUDA(cudaGetLastError());
    RXGS_CUDA(cudaMemcpyAsync(order_out, t_ord.p, sizeof(int) * k, cudaMemcpyDefault, s));
    RXGS_CUDA(cudaStreamSynchronize(s));
    ctx->launches += 2;
    return RXGS_OK;
}

int rxgs_image_metrics(rxgs_ctx ctx, const void* pred, int pred_f32, const double* gt, int n_img, int h, int w,
                       double max_val, const double ssim_opts[3], double* out) {
    if (!ctx || !out || !pred || !gt) return fail(RXGS_ERR_INVALID, "image_metrics: null argument");
    if (n_img < 1 || h < 0 || w < 0 || static_cast<int64_t>(h) * w == 0)
        return fail(RXGS_ERR_INVALID, "mae: need equal non-empty inputs");
    const int win = ssim_opts ? static_cast<int>(ssim_opts[0]) : 11;
    const double sigma = ssim_opts ? ssim_opts[1] : 1.5, dyn = ssim_opts ? ssim_opts[2] : 1.0;
    if (win > 0 && (h < win || w < win)) return fail(RXGS_ERR_INVALID, "ssim: image smaller than the window");
    if (win > 64) return fail(RXGS_ERR_INVALID, "image_metrics: ssim window above 64");
    RXGS_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const size_t n = static_cast<size_t>(n_img) * h * w;
    DevBuf t_p, t_g, t_ws, t_out;
    const void* d_p = pred;
    const double* d_g = gt;
    if (!dev_ptr(pred)) {
        const size_t b = n * (pred_f32 ? sizeof(float) : sizeof(double));
        RXGS_CUDA(t_p.ensure(b));
        RXGS_CUDA(cudaMemcpyAsync(t_p.p, pred, b, cudaMemcpyHostToDevice, s));
        d_p = t_p.p;
    }
    if (!dev_ptr(gt)) {
        RXGS_CUDA(t_g.ensure(n * sizeof(double)));
        RXGS_CUDA(cudaMemcpyAsync(t_g.p, gt, n * sizeof(double), cudaMemcpyHostToDevice, s));
        d_g = t_g.as<double>();
    }
    RXGS_CUDA(t_ws.ensure(image_metrics_ws_bytes(n_img, h, w, win > 0 ? win : 0)));
    RXGS_CUDA(t_out.ensure(sizeof(double) * 4 * n_img));
    RXGS_CUDA(launch_image_metrics(n_img, h, w, d_p, pred_f32 != 0, d_g, max_val, win > 0 ? win : 0, sigma, dyn,
                                   t_ws.p, t_out.as<double>(), s));
    RXGS_CUDA(cudaMemcpyAsync(out, t_out.p, sizeof(double) * 4 * n_img, cudaMemcpyDefault, s));
    RXGS_CUDA(cudaStreamSynchronize(s));
    ctx->launches += win > 0 ? 5 : 2;
    return RXGS_OK;
}

}  // extern "C"
