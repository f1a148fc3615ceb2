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
#include <cmath>
#include <climits>

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

// met::snr_csi (metrics.cpp:114-125) per set: err = sum |p - g|^2, sig =
// sum |g|^2 in a fixed order (per-thread strided sums, then a fixed tree).
__global__ void k_snr_csi(int64_t len, const double* __restrict__ pred, const double* __restrict__ gt,
                          double* __restrict__ es) {
    __shared__ double se[256], ss[256];
    const double* p = pred + static_cast<size_t>(blockIdx.x) * 2 * len;
    const double* g = gt + static_cast<size_t>(blockIdx.x) * 2 * len;
    double e = 0.0, sg = 0.0;
    for (int64_t i = threadIdx.x; i < len; i += blockDim.x) {
        const double dr = p[2 * i] - g[2 * i], di = p[2 * i + 1] - g[2 * i + 1];
        e += dr * dr + di * di;  // std::norm
        sg += g[2 * i] * g[2 * i] + g[2 * i + 1] * g[2 * i + 1];
    }
    se[threadIdx.x] = e;
    ss[threadIdx.x] = sg;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            se[threadIdx.x] += se[threadIdx.x + o];
            ss[threadIdx.x] += ss[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        es[2 * blockIdx.x] = se[0];
        es[2 * blockIdx.x + 1] = ss[0];
    }
}

// met::per_receiver_aggregate (metrics.cpp:127-149) on records sorted by
// receiver (stable: input order within a receiver): head[i] marks the first
// record of a receiver; its thread sums that receiver's values in input
// order (as the reference's map slots do).
__global__ void k_rx_heads(int64_t n, const uint32_t* __restrict__ key, int64_t* __restrict__ head) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) head[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
    else if (i == n) head[i] = 0;
}

__global__ void k_rx_segments(int64_t n, const uint32_t* __restrict__ key, const int* __restrict__ idx,
                              const double* __restrict__ v, const int64_t* __restrict__ seg,
                              int32_t* __restrict__ out_rx, double* __restrict__ out_mean,
                              int64_t* __restrict__ out_count) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n || (i > 0 && key[i] == key[i - 1])) return;
    double sum = 0.0;
    int64_t c = 0;
    for (int64_t q = i; q < n && key[q] == key[i]; ++q, ++c) sum += v[idx[q]];
    const int64_t u = seg[i];
    out_rx[u] = static_cast<int32_t>(key[i] ^ 0x80000000u);
    out_mean[u] = sum / static_cast<double>(c);
    out_count[u] = c;
}

// mean of the per-receiver means and their population stddev, in receiver order
__global__ void k_rx_moments(int64_t m, const double* __restrict__ means, double* __restrict__ out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double mu = 0.0;
    for (int64_t i = 0; i < m; ++i) mu += means[i];
    mu /= static_cast<double>(m);
    double var = 0.0;
    for (int64_t i = 0; i < m; ++i) {
        const double d = means[i] - mu;
        var += d * d;
    }
    out[0] = mu;
    out[1] = sqrt(var / static_cast<double>(m));
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

int rxgs_snr_csi(rxgs_ctx ctx, int n_sets, int64_t len, const double* pred, const double* gt, double* out_db) {
    if (!ctx || n_sets < 0 || (n_sets && (!pred || !gt || !out_db))) return fail(RXGS_ERR_INVALID, "snr_csi: null argument");
    if (n_sets == 0) return RXGS_OK;
    if (len < 1) return fail(RXGS_ERR_INVALID, "snr_csi: need equal non-empty inputs");
    RXGS_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const size_t n = static_cast<size_t>(n_sets) * 2 * len;
    DevBuf tp, tg, te;
    const double* dp = pred;
    const double* dg = gt;
    if (!dev_ptr(pred)) {
        RXGS_CUDA(tp.ensure(n * 8));
        RXGS_CUDA(cudaMemcpyAsync(tp.p, pred, n * 8, cudaMemcpyHostToDevice, s));
        dp = tp.as<double>();
    }
    if (!dev_ptr(gt)) {
        RXGS_CUDA(tg.ensure(n * 8));
        RXGS_CUDA(cudaMemcpyAsync(tg.p, gt, n * 8, cudaMemcpyHostToDevice, s));
        dg = tg.as<double>();
    }
    RXGS_CUDA(te.ensure(16 * static_cast<size_t>(n_sets)));
    k_snr_csi<<<n_sets, 256, 0, s>>>(len, dp, dg, te.as<double>());
    std::vector<double> es(2 * static_cast<size_t>(n_sets));
    RXGS_CUDA(cudaMemcpyAsync(es.data(), te.p, es.size() * 8, cudaMemcpyDeviceToHost, s));
    RXGS_CUDA(cudaStreamSynchronize(s));
    ctx->launches += 1;
    std::vector<double> db(static_cast<size_t>(n_sets));
    for (int i = 0; i < n_sets; ++i) {
        const double err = es[2 * i], sig = es[2 * i + 1];
        if (sig == 0.0) return fail(RXGS_ERR_INVALID, "snr_csi: zero ground-truth energy");
        db[i] = err == 0.0 ? 300.0 : -10.0 * std::log10(err / sig);  // kDbSentinel
    }
    RXGS_CUDA(cudaMemcpy(out_db, db.data(), db.size() * 8, cudaMemcpyDefault));
    return RXGS_OK;
}

int rxgs_per_receiver_aggregate(rxgs_ctx ctx, int64_t n, const int32_t* rx, const double* values, int32_t* out_rx,
                                double* out_mean, int64_t* out_count, int32_t* n_unique, double* mean,
                                double* stddev) {
    if (!ctx) return fail(RXGS_ERR_INVALID, "per_receiver_aggregate: null argument");
    if (n < 1) return fail(RXGS_ERR_INVALID, "per_receiver_aggregate: no records");
    if (!rx || !values || n > INT32_MAX) return fail(RXGS_ERR_INVALID, "per_receiver_aggregate: bad argument");
    RXGS_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const int nn = static_cast<int>(n);
    std::vector<int32_t> hrx(static_cast<size_t>(n));
    RXGS_CUDA(cudaMemcpy(hrx.data(), rx, 4 * n, cudaMemcpyDefault));
    std::vector<uint32_t> key(static_cast<size_t>(n));
    std::vector<int> idx(static_cast<size_t>(n));
    for (int i = 0; i < nn; ++i) {
        key[i] = static_cast<uint32_t>(hrx[i]) ^ 0x80000000u;  // signed order
        idx[i] = i;
    }
    const size_t wi = radix_sort_work_ints(nn);
    DevBuf buf;
    auto al = [](size_t x) { return (x + 255) & ~static_cast<size_t>(255); };
    const size_t N1 = static_cast<size_t>(n) + 2;
    const size_t o_k = 0, o_v = al(4 * N1), o_kt = o_v + al(4 * N1), o_vt = o_kt + al(4 * N1),
                 o_w = o_vt + al(4 * N1), o_val = o_w + al(4 * wi), o_seg = o_val + al(8 * N1),
                 o_bs = o_seg + al(8 * N1), o_rx = o_bs + al(8 * scan_bsum_count(static_cast<int64_t>(n) + 1)), o_mean = o_rx + al(4 * N1),
                 o_cnt = o_mean + al(8 * N1), o_mom = o_cnt + al(8 * N1);
    RXGS_CUDA(buf.ensure(o_mom + 64));
    char* b = buf.as<char>();
    auto K = reinterpret_cast<uint32_t*>(b + o_k);
    auto V = reinterpret_cast<int*>(b + o_v);
    auto W = reinterpret_cast<int*>(b + o_w);
    auto VAL = reinterpret_cast<double*>(b + o_val);
    auto SEG = reinterpret_cast<int64_t*>(b + o_seg);
    RXGS_CUDA(cudaMemcpyAsync(K, key.data(), 4 * n, cudaMemcpyHostToDevice, s));
    RXGS_CUDA(cudaMemcpyAsync(V, idx.data(), 4 * n, cudaMemcpyHostToDevice, s));
    RXGS_CUDA(cudaMemcpyAsync(VAL, values, 8 * n, cudaMemcpyDefault, s));
    RXGS_CUDA(cudaMemsetAsync(W, 0, 4 * wi, s));
    RXGS_CUDA(radix_sort_pairs(nn, 32, K, V, reinterpret_cast<uint32_t*>(b + o_kt), reinterpret_cast<int*>(b + o_vt),
                               W, false, s));
    const unsigned g = static_cast<unsigned>((n + 1 + 255) / 256);
    k_rx_heads<<<g, 256, 0, s>>>(n, K, SEG);
    RXGS_CUDA(scan_i64(n + 1, SEG, SEG, reinterpret_cast<int64_t*>(b + o_bs), s));
    auto ORX = reinterpret_cast<int32_t*>(b + o_rx);
    auto OM = reinterpret_cast<double*>(b + o_mean);
    auto OC = reinterpret_cast<int64_t*>(b + o_cnt);
    k_rx_segments<<<g, 256, 0, s>>>(n, K, V, VAL, SEG, ORX, OM, OC);
    int64_t m = 0;
    RXGS_CUDA(cudaMemcpyAsync(&m, SEG + n, 8, cudaMemcpyDeviceToHost, s));
    RXGS_CUDA(cudaStreamSynchronize(s));
    auto MOM = reinterpret_cast<double*>(b + o_mom);
    k_rx_moments<<<1, 32, 0, s>>>(m, OM, MOM);
    double mom[2];
    RXGS_CUDA(cudaMemcpyAsync(mom, MOM, 16, cudaMemcpyDeviceToHost, s));
    RXGS_CUDA(cudaStreamSynchronize(s));
    ctx->launches += 12;
    if (out_rx) RXGS_CUDA(cudaMemcpy(out_rx, ORX, 4 * m, cudaMemcpyDefault));
    if (out_mean) RXGS_CUDA(cudaMemcpy(out_mean, OM, 8 * m, cudaMemcpyDefault));
    if (out_count) RXGS_CUDA(cudaMemcpy(out_count, OC, 8 * m, cudaMemcpyDefault));
    if (n_unique) *n_unique = static_cast<int32_t>(m);
    if (mean) *mean = mom[0];
    if (stddev) *stddev = mom[1];
    return RXGS_OK;
}

}  // extern "C"
