// C-ABI layer: handles, validation with the reference's error text, host /
// device pointer handling, stream-ordered orchestration of the kernels.
// See include/rxgs_b200.h for the contract and DESIGN.md for the data flow.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <new>
#include <string>
#include <thread>
#include <mutex>
#include <condition_variable>
#include <memory>
#include <vector>

#include "rxgs_internal.cuh"

using namespace rxgs_b200;

namespace rxgs_b200 {

namespace {
thread_local std::string g_err;
}

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

uint64_t next_version() {
    static std::atomic<uint64_t> v{0};
    return ++v;
}

int cuda_fail(cudaError_t e, const char* what) {
    g_err = std::string("CUDA error: ") + cudaGetErrorString(e) + " (" + what + ")";
    return RXGS_ERR_CUDA;
}

int scene_sync_host(rxgs_scene_s* sc) {
    if (!sc->host_stale && !sc->geo_stale) return RXGS_OK;
    RXGS_CUDA(cudaSetDevice(sc->ctx->device));
    RXGS_CUDA(cudaStreamSynchronize(sc->ctx->stream));
    auto down = [](std::vector<double>& h, const DevBuf& d) {
        return h.empty() ? cudaSuccess : cudaMemcpy(h.data(), d.p, h.size() * sizeof(double), cudaMemcpyDeviceToHost);
    };
    if (sc->host_stale) {
        RXGS_CUDA(down(sc->h_coeffs, sc->d_coeffs64));
        sc->host_stale = false;
    }
    if (sc->geo_stale) {
        RXGS_CUDA(down(sc->h_pos, sc->d_pos));
        RXGS_CUDA(down(sc->h_ls, sc->d_ls));
        RXGS_CUDA(down(sc->h_q, sc->d_q));
        RXGS_CUDA(down(sc->h_tau, sc->d_tau));
        sc->pos_index.clear();
        sc->pos_index_built = false;
        sc->geo_stale = false;
    }
    return RXGS_OK;
}

void timing_begin(rxgs_ctx ctx, const char* name, cudaEvent_t* a) {
    (void)name;
    *a = nullptr;
    if (!ctx->profile) return;
    if (ctx->event_pool.empty()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        ctx->event_pool.push_back(e);
    }
    *a = ctx->event_pool.back();
    ctx->event_pool.pop_back();
    cudaEventRecord(*a, ctx->stream);
}

void timing_end(rxgs_ctx ctx, const char* name, cudaEvent_t a, double work) {
    if (!ctx->profile || !a) return;
    cudaEvent_t b;
    if (ctx->event_pool.empty()) {
        cudaEventCreate(&b);
    } else {
        b = ctx->event_pool.back();
        ctx->event_pool.pop_back();
    }
    cudaEventRecord(b, ctx->stream);
    ctx->pending.push_back({name, a, b, work});
}

}  // namespace rxgs_b200

namespace {

void resolve_timings(rxgs_ctx ctx) {
    if (ctx->pending.empty()) return;
    cudaStreamSynchronize(ctx->stream);
    for (auto& p : ctx->pending) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, p.a, p.b);
        auto& st = ctx->stats[p.name];
        st.ms += ms;
        st.launches += 1;
        st.work += p.work;
        ctx->event_pool.push_back(p.a);
        ctx->event_pool.push_back(p.b);
    }
    ctx->pending.clear();
}

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Device view of a caller array: the pointer itself if it is device memory,
// otherwise a stream-ordered copy into `tmp`.
template <typename T>
int dev_in(rxgs_ctx ctx, const T* p, size_t n, DevBuf& tmp, const T** out) {
    if (!p || n == 0) {
        *out = p;
        return RXGS_OK;
    }
    if (is_device_ptr(p)) {
        *out = p;
        return RXGS_OK;
    }
    RXGS_CUDA(tmp.ensure(n * sizeof(T)));
    RXGS_CUDA(cudaMemcpyAsync(tmp.p, p, n * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
    *out = tmp.as<T>();
    return RXGS_OK;
}

template <typename T>
int dev_out(T* p, size_t n, DevBuf& tmp, T** out) {
    if (!p) {
        *out = nullptr;
        return RXGS_OK;
    }
    if (is_device_ptr(p)) {
        *out = p;
        return RXGS_OK;
    }
    RXGS_CUDA(tmp.ensure(std::max<size_t>(n, 1) * sizeof(T)));
    *out = tmp.as<T>();
    return RXGS_OK;
}

template <typename T>
int finish_out(rxgs_ctx ctx, T* user, const T* dev, size_t n) {
    if (!user || user == dev || n == 0) return RXGS_OK;
    RXGS_CUDA(cudaMemcpyAsync(user, dev, n * sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
    return RXGS_OK;
}

template <typename T>
std::vector<T> to_host(const T* p, size_t n) {
    std::vector<T> v(n);
    if (n == 0 || !p) return v;
    if (is_device_ptr(p))
        cudaMemcpy(v.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost);
    else
        std::memcpy(v.data(), p, n * sizeof(T));
    return v;
}

int set_device(rxgs_ctx ctx) {
    RXGS_CUDA(cudaSetDevice(ctx->device));
    return RXGS_OK;
}

int validate_grid(const rxgs_grid* g) {  // SphericalGrid::validate, sphraster.cpp:14-20
    if (!g) return fail(RXGS_ERR_INVALID, "grid: null");
    if (g->n_theta < 1 || g->n_phi < 1) return fail(RXGS_ERR_INVALID, "grid: n_theta * n_phi must be >= 1");
    if (g->tile_size < 1) return fail(RXGS_ERR_INVALID, "grid: tile_size must be >= 1");
    if (!(g->radius > 0.0)) return fail(RXGS_ERR_INVALID, "grid: radius must be > 0");
    if (!(g->theta_min >= 0.0 && g->theta_max <= kPi && g->theta_min < g->theta_max))
        return fail(RXGS_ERR_INVALID, "grid: elevation span must satisfy 0 <= min < max <= pi");
    return RXGS_OK;
}

DevGrid make_grid(const rxgs_grid* g) {
    DevGrid d{};
    d.nt = g->n_theta;
    d.np = g->n_phi;
    d.ts = g->tile_size;
    d.tiles_t = (d.nt + d.ts - 1) / d.ts;
    d.tiles_p = (d.np + d.ts - 1) / d.ts;
    d.n_tiles = d.tiles_t * d.tiles_p;
    d.cpt = d.ts * d.ts;
    d.cell_blocks = (d.cpt + kMaxCellsPerBlock - 1) / kMaxCellsPerBlock;
    d.radius = g->radius;
    d.tmin = g->theta_min;
    d.tmax = g->theta_max;
    d.dth = (g->theta_max - g->theta_min) / g->n_theta;
    d.dph = kTwoPi / g->n_phi;
    return d;
}

int check_err_flag(rxgs_ctx ctx, int* d_err, int* host_val) {
    RXGS_CUDA(cudaMemcpyAsync(host_val, d_err, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    RXGS_CUDA(cudaStreamSynchronize(ctx->stream));
    return RXGS_OK;
}

int reset_err_flag(rxgs_ctx ctx) {
    RXGS_CUDA(ctx->err_flag.ensure(sizeof(int) * 4));
    const int v = INT_MAX;
    RXGS_CUDA(cudaMemcpyAsync(ctx->err_flag.p, &v, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    return RXGS_OK;
}

#define RX_TRY(expr)                 \
    do {                             \
        const int rc__ = (expr);     \
        if (rc__ != RXGS_OK) return rc__; \
    } while (0)

#define API_BEGIN try {
#define API_END                                                         \
    }                                                                   \
    catch (const std::bad_alloc&) {                                     \
        return fail(RXGS_ERR_RUNTIME, "host allocation failed");        \
    }                                                                   \
    catch (const std::exception& e) {                                   \
        return fail(RXGS_ERR_RUNTIME, e.what());                        \
    }

// Layout offsets of the packed conditioning parameters.
void layout_cond(rxgs_cond_s& c) {
    c.L = (c.l_max + 1) * (c.l_max + 1);
    c.gin = 6 * c.F + 2 + c.dc;
    size_t o = 0;
    const size_t d = c.hidden;
    c.o_freq = o; o += static_cast<size_t>(c.F) * 3;
    c.o_gw1 = o; o += d * c.gin;
    c.o_gb1 = o; o += d;
    c.o_gw2 = o; o += d * d;
    c.o_gb2 = o; o += d;
    c.o_gw3 = o; o += 4 * c.C * d;
    c.o_gb3 = o; o += 4 * c.C;
    c.o_emb = o; o += static_cast<size_t>(c.L) * c.dc;
    c.o_lw1 = o; o += d * 6;
    c.o_lb1 = o; o += d;
    c.o_lw2 = o; o += d * d;
    c.o_lb2 = o; o += d;
    c.o_lw3 = o; o += 4 * c.C * d;
    c.o_lb3 = o; o += 4 * c.C;
    c.n_params = static_cast<int64_t>(o);
}


// First (receiver j, Gaussian k) in j-major order with rx_j exactly at a
// Gaussian centre, -1 if none.  Host-side hash lookup (no device pass):
// |rx - p| == 0 in the reference (conditioning.cpp:379-382) is bitwise
// equality of the coordinates for any representable positions.
int64_t find_coincident(rxgs_scene sc, const double* rx_host, int n_rx) {
    auto key = [](double x, double y, double z) {
        std::string k(24, '\0');
        x += 0.0;  // -0 == +0
        y += 0.0;
        z += 0.0;
        std::memcpy(&k[0], &x, 8);
        std::memcpy(&k[8], &y, 8);
        std::memcpy(&k[16], &z, 8);
        return k;
    };
    if (scene_sync_host(sc) != RXGS_OK) return -2;
    if (!sc->pos_index_built) {
        sc->pos_index.reserve(static_cast<size_t>(sc->k) * 2);
        for (int k = sc->k - 1; k >= 0; --k)
            sc->pos_index[key(sc->h_pos[3 * k], sc->h_pos[3 * k + 1], sc->h_pos[3 * k + 2])] = k;
        sc->pos_index_built = true;
    }
    for (int j = 0; j < n_rx; ++j) {
        const auto it = sc->pos_index.find(key(rx_host[3 * j], rx_host[3 * j + 1], rx_host[3 * j + 2]));
        if (it != sc->pos_index.end()) return static_cast<int64_t>(j) * std::max(sc->k, 1) + it->second;
    }
    return -1;
}

int check_receivers(rxgs_ctx ctx, rxgs_scene sc, const double* rx, int n_rx) {
    std::vector<double> h = to_host(rx, 3 * static_cast<size_t>(n_rx));
    const int64_t e = find_coincident(sc, h.data(), n_rx);
    if (e == -2) return RXGS_ERR_CUDA;
    if (e >= 0)
        return fail(RXGS_ERR_INVALID, "condition_forward: receiver coincides with gaussian " +
                                          std::to_string(e % std::max(sc->k, 1)));
    (void)ctx;
    return RXGS_OK;
}

// Signals for a receiver chunk: fused conditioning (or the bare base
// coefficients when cond == nullptr).
int compute_signals(rxgs_ctx ctx, rxgs_scene sc, rxgs_cond c, rxgs_txstate st, const double* d_rx,
                    int n_rx, SigOut d_sig) {
    cudaStream_t s = ctx->stream;
    if (c && c->host_stale) {  // the tcgen05 kernel takes layers 1/3 as a kernel parameter from the host copy
        RXGS_CUDA(cudaStreamSynchronize(s));
        RXGS_CUDA(cudaMemcpy(c->h_params.data(), c->d_params64.p, c->h_params.size() * sizeof(double),
                             cudaMemcpyDeviceToHost));
        c->host_stale = false;
    }
    const size_t ag_n = static_cast<size_t>(n_rx) * sc->L * 4 * sc->channels;
    RXGS_CUDA(ctx->ag.ensure(std::max<size_t>(ag_n, 1) * sizeof(float)));
    cudaEvent_t ev;
    if (c && c->use_global()) {
        timing_begin(ctx, "cond_global", &ev);
        RXGS_CUDA(launch_cond_global(*c, d_rx, n_rx, ctx->ag.as<float>(), s));
        timing_end(ctx, "cond_global", ev, static_cast<double>(n_rx) * sc->L);
    } else {
        RXGS_CUDA(cudaMemsetAsync(ctx->ag.p, 0, ag_n * sizeof(float), s));
    }
    ctx->launches += 1;
    timing_begin(ctx, "cond_signal", &ev);
    RXGS_CUDA(launch_cond_signal(c, *sc, *st, d_rx, n_rx, ctx->ag.as<float>(), d_sig, nullptr, s));
    timing_end(ctx, "cond_signal", ev,
               static_cast<double>(st->needed_host >= 0 ? st->needed_host : st->visible) * n_rx);
    ctx->launches += 1;
    return RXGS_OK;
}

}  // namespace

extern "C" {

const char* rxgs_last_error(void) { return g_err.c_str(); }
int rxgs_version(void) { return 1; }

// ------------------------------------------------------------------ context
int rxgs_ctx_create(int device, rxgs_ctx* out) {
    API_BEGIN
    if (!out) return fail(RXGS_ERR_INVALID, "rxgs_ctx_create: null out");
    int n = 0;
    RXGS_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) return fail(RXGS_ERR_INVALID, "rxgs_ctx_create: bad device ordinal");
    RXGS_CUDA(cudaSetDevice(device));
    auto* ctx = new rxgs_ctx_s;
    ctx->device = device;
    RXGS_CUDA(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
    ctx->stream = ctx->own_stream;
    cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
    *out = ctx;
    return RXGS_OK;
    API_END
}

}  // extern "C"

namespace rxgs_b200 {
// Handles (scene, conditioning, tx state, trainer) hold a reference on their
// context; rxgs_ctx_destroy only marks it closed while any is alive, so
// destruction order (e.g. garbage-collected bindings) cannot free it early.
void ctx_retain(rxgs_ctx ctx) { ++ctx->refs; }
static void ctx_free(rxgs_ctx ctx) {
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (auto& p : ctx->pending) {
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    for (auto e : ctx->event_pool) cudaEventDestroy(e);
    for (auto* t : ctx->spare_tx) delete t;
    for (auto e : ctx->chunk_events) cudaEventDestroy(e);
    for (int i = 0; i < rxgs_ctx_s::kAuxMax; ++i) {
        if (ctx->aux_ev[i]) cudaEventDestroy(ctx->aux_ev[i]);
        if (ctx->aux_done[i]) cudaEventDestroy(ctx->aux_done[i]);
        if (ctx->aux[i]) {
            ctx->aux[i]->closed = true;
            if (ctx->aux[i]->refs == 0) ctx_free(ctx->aux[i]);
        }
    }
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;
}
void ctx_release(rxgs_ctx ctx) {
    if (--ctx->refs == 0 && ctx->closed) ctx_free(ctx);
}
void scene_release(rxgs_scene_s* sc) {
    if (--sc->refs > 0) return;
    rxgs_ctx ctx = sc->ctx;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    delete sc;
    ctx_release(ctx);
}
int ensure_tx_full(rxgs_txstate_s& st, cudaStream_t s) {
    if (st.full) return RXGS_OK;
    rxgs_scene_s* sc = st.sc;
    if (!sc) return fail(RXGS_ERR_INVALID, "tx state: no scene to complete the FP64 geometry from");
    if (sc->geo_version != st.geo_version || sc->k != st.k)
        return fail(RXGS_ERR_INVALID, "tx state: the scene geometry changed since the state was built; rebuild it");
    RXGS_CUDA(launch_tx_prep(*sc, st, s, true));  // same arithmetic: rec / spans / lists unchanged
    st.ctx->launches += 1;
    st.full = true;
    st.coeff_version = sc->coeff_version;  // basis*base recomputed from the current coefficients
    return RXGS_OK;
}
}  // namespace rxgs_b200

namespace rxgs_b200 {
int scene_resized(rxgs_scene_s* sc) {
    rxgs_ctx ctx = sc->ctx;
    RXGS_CUDA(cudaStreamSynchronize(ctx->stream));
    const size_t K = static_cast<size_t>(sc->k);
    auto down = [](std::vector<double>& h, const DevBuf& d, size_t n) {
        h.resize(n);
        return n ? cudaMemcpy(h.data(), d.p, n * sizeof(double), cudaMemcpyDeviceToHost) : cudaSuccess;
    };
    RXGS_CUDA(down(sc->h_pos, sc->d_pos, 3 * K));
    RXGS_CUDA(down(sc->h_ls, sc->d_ls, 3 * K));
    RXGS_CUDA(down(sc->h_q, sc->d_q, 4 * K));
    RXGS_CUDA(down(sc->h_tau, sc->d_tau, K));
    RXGS_CUDA(down(sc->h_coeffs, sc->d_coeffs64, K * sc->L * sc->channels * 2));
    sc->host_stale = sc->geo_stale = false;
    sc->pos_index.clear();
    sc->pos_index_built = false;
    std::vector<float> p4(4 * std::max<size_t>(K, 1), 0.f);
    for (size_t i = 0; i < K; ++i)
        for (int a = 0; a < 3; ++a) p4[4 * i + a] = static_cast<float>(sc->h_pos[3 * i + a]);
    DevBuf p32;
    RXGS_CUDA(p32.ensure(p4.size() * sizeof(float)));
    RXGS_CUDA(cudaMemcpy(p32.p, p4.data(), p4.size() * sizeof(float), cudaMemcpyHostToDevice));
    sc->d_pos32 = std::move(p32);
    sc->d_morton = DevBuf();
    sc->d_mpos32 = DevBuf();
    return build_scene_order(ctx, *sc, ctx->stream);
}
}  // namespace rxgs_b200

extern "C" {

int rxgs_ctx_destroy(rxgs_ctx ctx) {
    if (!ctx) return RXGS_OK;
    ctx->closed = true;
    if (ctx->refs == 0) ctx_free(ctx);
    return RXGS_OK;
}

int rxgs_ctx_set_stream(rxgs_ctx ctx, void* stream) {
    if (!ctx) return fail(RXGS_ERR_INVALID, "null context");
    ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
    return RXGS_OK;
}

int rxgs_ctx_synchronize(rxgs_ctx ctx) {
    if (!ctx) return fail(RXGS_ERR_INVALID, "null context");
    RX_TRY(set_device(ctx));
    RXGS_CUDA(cudaStreamSynchronize(ctx->stream));
    return RXGS_OK;
}

int rxgs_ctx_profile(rxgs_ctx ctx, int enable) {
    if (!ctx) return fail(RXGS_ERR_INVALID, "null context");
    ctx->profile = enable != 0;
    return RXGS_OK;
}

int rxgs_ctx_kernel_stats(rxgs_ctx ctx, const char* name, double* total_ms, int64_t* launches,
                          double* work) {
    if (!ctx || !name) return fail(RXGS_ERR_INVALID, "null argument");
    resolve_timings(ctx);
    const auto it = ctx->stats.find(name);
    const KStat st = it == ctx->stats.end() ? KStat{} : it->second;
    if (total_ms) *total_ms = st.ms;
    if (launches) *launches = st.launches;
    if (work) *work = st.work;
    return RXGS_OK;
}

int rxgs_ctx_reset_stats(rxgs_ctx ctx) {
    if (!ctx) return fail(RXGS_ERR_INVALID, "null context");
    resolve_timings(ctx);
    ctx->stats.clear();
    ctx->launches = 0;
    return RXGS_OK;
}

int rxgs_ctx_release_cache(rxgs_ctx ctx) {
    API_BEGIN
    if (!ctx) return fail(RXGS_ERR_INVALID, "null context");
    RX_TRY(set_device(ctx));
    RXGS_CUDA(cudaStreamSynchronize(ctx->stream));
    for (DevBuf* b : {&ctx->sort_tmp, &ctx->scratch_a, &ctx->scratch_b, &ctx->scratch_c, &ctx->scratch_d,
                      &ctx->signals, &ctx->ag, &ctx->partial, &ctx->host_in, &ctx->host_out, &ctx->ycache,
                      &ctx->fle_a, &ctx->fle_b, &ctx->fle_m, &ctx->probe_tr, &ctx->row_pos, &ctx->row_GB, &ctx->row_S}) {
        if (b->p) cudaFree(b->p);
        b->p = nullptr;
        b->bytes = 0;
    }
    for (rxgs_txstate_s* st : ctx->spare_tx) delete st;
    ctx->spare_tx.clear();
    return RXGS_OK;
    API_END
}

int64_t rxgs_ctx_launch_count(rxgs_ctx ctx) { return ctx ? ctx->launches : 0; }

int rxgs_ctx_set_cond_kernel(rxgs_ctx ctx, int which) {
    if (!ctx || which < 0 || which > 1) return fail(RXGS_ERR_INVALID, "rxgs_ctx_set_cond_kernel: bad argument");
    ctx->cond_kernel = which;
    return RXGS_OK;
}

int rxgs_ctx_set_composite_kernel(rxgs_ctx ctx, int which) {
    if (!ctx || which < 0 || which > 1) return fail(RXGS_ERR_INVALID, "rxgs_ctx_set_composite_kernel: bad argument");
    ctx->composite_kernel = which;
    return RXGS_OK;
}

int rxgs_selftest_tcgen05(rxgs_ctx ctx, double* err) {
    if (!ctx) return fail(RXGS_ERR_INVALID, "null context");
    RX_TRY(set_device(ctx));
    RXGS_CUDA(ctx->err_flag.ensure(32));
    RXGS_CUDA(cudaMemsetAsync(ctx->err_flag.p, 0, 20, ctx->stream));
    RXGS_CUDA(launch_tc_selftest(ctx->err_flag.as<float>(), ctx->stream));
    RXGS_CUDA(launch_tc_selftest_mn(ctx->err_flag.as<float>() + 4, ctx->stream));
    float e[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
    RXGS_CUDA(cudaMemcpyAsync(e, ctx->err_flag.p, 20, cudaMemcpyDeviceToHost, ctx->stream));
    RXGS_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int i = 0; i < 5; ++i) err[i] = e[i];
    return RXGS_OK;
}

// ------------------------------------------------------------------ scene
int rxgs_scene_create(rxgs_ctx ctx, int k, int l_max, int channels, int modality, const double* pos,
                      const double* ls, const double* q, const double* tau, const double* coeffs,
                      rxgs_scene* out) {
    API_BEGIN
    if (!ctx || !out) return fail(RXGS_ERR_INVALID, "rxgs_scene_create: null argument");
    if (k < 0 || l_max < 0 || channels < 1 || modality < 0 || modality > 2)
        return fail(RXGS_ERR_INVALID, "scene: per-Gaussian arrays out of alignment");
    if (l_max > kMaxLmax) return fail(RXGS_ERR_INVALID, "scene: l_max > 15 is not supported by the B200 path");
    RX_TRY(set_device(ctx));
    auto* sc = new rxgs_scene_s;
    sc->ctx = ctx;
    sc->k = k;
    sc->l_max = l_max;
    sc->channels = channels;
    sc->L = (l_max + 1) * (l_max + 1);
    sc->modality = modality;
    const size_t nc = static_cast<size_t>(k) * sc->L * channels * 2;
    sc->h_pos = to_host(pos, 3 * static_cast<size_t>(k));
    sc->h_ls = to_host(ls, 3 * static_cast<size_t>(k));
    sc->h_q = to_host(q, 4 * static_cast<size_t>(k));
    sc->h_tau = to_host(tau, static_cast<size_t>(k));
    sc->h_coeffs = to_host(coeffs, nc);
    auto up = [&](DevBuf& b, const std::vector<double>& h) -> int {
        RXGS_CUDA(b.ensure(std::max<size_t>(h.size(), 1) * sizeof(double)));
        if (!h.empty()) RXGS_CUDA(cudaMemcpy(b.p, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice));
        return RXGS_OK;
    };
    int rc = up(sc->d_pos, sc->h_pos);
    if (!rc) rc = up(sc->d_ls, sc->h_ls);
    if (!rc) rc = up(sc->d_q, sc->h_q);
    if (!rc) rc = up(sc->d_tau, sc->h_tau);
    if (!rc) rc = up(sc->d_coeffs64, sc->h_coeffs);
    if (!rc) {
        std::vector<float> p4(4 * static_cast<size_t>(std::max(k, 1)), 0.f);
        for (int i = 0; i < k; ++i)
            for (int a = 0; a < 3; ++a) p4[4 * i + a] = static_cast<float>(sc->h_pos[3 * i + a]);
        const cudaError_t e1 = sc->d_pos32.ensure(p4.size() * sizeof(float));
        if (e1 != cudaSuccess) rc = cuda_fail(e1, "scene pos32");
        else {
            const cudaError_t e2 = cudaMemcpy(sc->d_pos32.p, p4.data(), p4.size() * sizeof(float), cudaMemcpyHostToDevice);
            if (e2 != cudaSuccess) rc = cuda_fail(e2, "scene pos32 copy");
        }
    }
    if (!rc) rc = build_scene_order(ctx, *sc, ctx->stream);
    if (rc) {
        delete sc;
        return rc;
    }
    ctx_retain(ctx);
    *out = sc;
    return RXGS_OK;
    API_END
}

int rxgs_scene_destroy(rxgs_scene sc) {
    if (!sc) return RXGS_OK;
    scene_release(sc);
    return RXGS_OK;
}

int rxgs_scene_bounds(rxgs_scene sc, double inflate, double lo[3], double hi[3]) {
    if (!sc) return fail(RXGS_ERR_INVALID, "null scene");
    if (int rc = scene_sync_host(sc)) return rc;
    for (int a = 0; a < 3; ++a) {
        lo[a] = 1.7976931348623157e308;
        hi[a] = -1.7976931348623157e308;
    }
    for (int k = 0; k < sc->k; ++k)
        for (int a = 0; a < 3; ++a) {
            const double v = sc->h_pos[3 * k + a];
            lo[a] = std::min(lo[a], v);
            hi[a] = std::max(hi[a], v);
        }
    for (int a = 0; a < 3; ++a) {  // Aabb::inflated, linalg.hpp:143-147
        const double pad = (hi[a] - lo[a]) * (0.5 * inflate);
        lo[a] = lo[a] - pad;
        hi[a] = hi[a] + pad;
    }
    return RXGS_OK;
}

// ------------------------------------------------------------------ tx state
int rxgs_tx_state_build(rxgs_ctx ctx, rxgs_scene sc, const double tx[3], const rxgs_grid* grid,
                        rxgs_txstate* out) {
    API_BEGIN
    if (!ctx || !sc || !tx || !out) return fail(RXGS_ERR_INVALID, "rxgs_tx_state_build: null argument");
    RX_TRY(validate_grid(grid));
    RX_TRY(set_device(ctx));
    cudaStream_t s = ctx->stream;
    // Reuse the device buffers of the last destroyed state (grow-only), so a
    // per-transmitter rebuild does not pay cudaMalloc/cudaFree every time.
    rxgs_txstate_s* st = nullptr;
    if (!ctx->spare_tx.empty()) {
        st = ctx->spare_tx.back();
        ctx->spare_tx.pop_back();
    } else {
        st = new rxgs_txstate_s;
    }
    st->entries = st->visible = 0;
    st->needed_host = -1;
    st->regrouped = false;  // recycled buffers: per-state derived data must be rebuilt
    st->version = next_version();
    st->coeff_version = sc->coeff_version;
    st->geo_version = sc->geo_version;
    st->full = false;
    st->ctx = ctx;
    st->k = sc->k;
    st->l_max = sc->l_max;
    st->L = sc->L;
    st->channels = sc->channels;
    st->grid = make_grid(grid);
    const double txh[3] = {tx[0], tx[1], tx[2]};
    std::vector<double> txv = to_host(tx, 3);
    for (int a = 0; a < 3; ++a) st->tx[a] = txv[a];
    (void)txh;
    const size_t K = std::max(sc->k, 1);
    auto fail_st = [&](int rc) {
        delete st;
        return rc;
    };
    int rc = RXGS_OK;
#define ENS(buf, bytes)                                              \
    do {                                                             \
        const cudaError_t e__ = st->buf.ensure(bytes);               \
        if (e__ != cudaSuccess) return fail_st(cuda_fail(e__, #buf)); \
    } while (0)
    ENS(rec, K * sizeof(GaussRec));
    ENS(culled, K * sizeof(int));
    ENS(geom, K * 12 * sizeof(double));
    ENS(spans, K * sizeof(int4));
    ENS(basis64, K * sc->L * 2 * sizeof(double));
    ENS(basis32, K * sc->L * sizeof(float2));
    ENS(gb32, K * sc->L * sc->channels * sizeof(float2));
    ENS(depth_key, K * sizeof(uint64_t));
    ENS(tile_count, K * sizeof(int));
    cudaEvent_t ev;
    timing_begin(ctx, "tx_prep", &ev);
    {
        const cudaError_t e = launch_tx_prep(*sc, *st, s, false);
        if (e != cudaSuccess) return fail_st(cuda_fail(e, "tx_prep"));
    }
    timing_end(ctx, "tx_prep", ev, sc->k);
    ctx->launches += 1;
    timing_begin(ctx, "sort", &ev);
    rc = bin_tiles(ctx, *st, s);
    if (rc) return fail_st(rc);
    timing_end(ctx, "sort", ev, sc->k);
    const DevGrid& g = st->grid;
    const size_t cells = static_cast<size_t>(g.nt) * g.np;
    ENS(tw, std::max<size_t>(st->entries, 1) * g.cell_blocks * kMaxCellsPerBlock * sizeof(float));
    ENS(walk_len, static_cast<size_t>(g.n_tiles) * g.cell_blocks * sizeof(int));
    ENS(cell_T, cells * sizeof(double));
    ENS(cell_len, cells * sizeof(int));
#undef ENS
    timing_begin(ctx, "walk", &ev);
    {
        const cudaError_t e = launch_walk(*st, s);
        if (e != cudaSuccess) return fail_st(cuda_fail(e, "walk"));
    }
    timing_end(ctx, "walk", ev, static_cast<double>(cells));
    {
        const int rc = compact_needed(ctx, *sc, *st, s);
        if (rc) return fail_st(rc);
    }
    {
        const cudaError_t e = launch_basis_rows(*sc, *st, s);
        if (e != cudaSuccess) return fail_st(cuda_fail(e, "basis_rows"));
    }
    ctx->launches += 2;
    ctx_retain(ctx);
    st->sc = sc;
    sc->refs += 1;
    *out = st;
    return RXGS_OK;
    API_END
}

int rxgs_tx_state_destroy(rxgs_txstate st) {
    if (!st) return RXGS_OK;
    rxgs_ctx ctx = st->ctx;
    cudaSetDevice(ctx->device);
    if (st->sc) {
        scene_release(st->sc);
        st->sc = nullptr;
    }
    if (ctx->spare_tx.size() < 2) {
        // Keep the buffers for the next build; stream order makes reuse safe
        // (later kernels on this stream run after every reader of st).
        ctx->spare_tx.push_back(st);
    } else {
        cudaStreamSynchronize(ctx->stream);
        delete st;
    }
    ctx_release(ctx);
    return RXGS_OK;
}

int64_t rxgs_tx_state_entries(rxgs_txstate st) { return st ? st->entries : -1; }

int rxgs_tx_state_get(rxgs_txstate st, int32_t* culled, double* geom, int32_t* spans, double* basis,
                      int64_t* offsets, int32_t* indices) {
    API_BEGIN
    if (!st) return fail(RXGS_ERR_INVALID, "null tx state");
    rxgs_ctx ctx = st->ctx;
    RX_TRY(set_device(ctx));
    if ((geom || basis) && st->k) RX_TRY(ensure_tx_full(*st, ctx->stream));
    RXGS_CUDA(cudaStreamSynchronize(ctx->stream));
    const size_t K = st->k;
    if (culled && K) RXGS_CUDA(cudaMemcpy(culled, st->culled.p, K * sizeof(int), cudaMemcpyDefault));
    if (geom && K) RXGS_CUDA(cudaMemcpy(geom, st->geom.p, K * 12 * sizeof(double), cudaMemcpyDefault));
    if (spans && K) RXGS_CUDA(cudaMemcpy(spans, st->spans.p, K * 4 * sizeof(int), cudaMemcpyDefault));
    if (basis && K)
        RXGS_CUDA(cudaMemcpy(basis, st->basis64.p, K * st->L * 2 * sizeof(double), cudaMemcpyDefault));
    if (offsets)
        RXGS_CUDA(cudaMemcpy(offsets, st->tile_offsets.p, (st->grid.n_tiles + 1) * sizeof(int64_t),
                             cudaMemcpyDefault));
    if (indices && st->entries)
        RXGS_CUDA(cudaMemcpy(indices, st->list.p, st->entries * sizeof(int), cudaMemcpyDefault));
    return RXGS_OK;
    API_END
}

int rxgs_tx_state_keys(rxgs_txstate st, uint64_t* keys) {
    if (!st || !keys) return fail(RXGS_ERR_INVALID, "null argument");
    RX_TRY(set_device(st->ctx));
    RXGS_CUDA(cudaStreamSynchronize(st->ctx->stream));
    if (st->entries)
        RXGS_CUDA(cudaMemcpy(keys, st->keys.p, st->entries * sizeof(uint64_t), cudaMemcpyDefault));
    return RXGS_OK;
}

int rxgs_tx_state_stats(rxgs_txstate st, int64_t* visible, int64_t* entries, double* walk_per_cell,
                        double* tile_walk_per_cell) {
    API_BEGIN
    if (!st) return fail(RXGS_ERR_INVALID, "null tx state");
    RX_TRY(set_device(st->ctx));
    RXGS_CUDA(cudaStreamSynchronize(st->ctx->stream));
    const DevGrid& g = st->grid;
    const size_t cells = static_cast<size_t>(g.nt) * g.np;
    std::vector<int> len(cells), wl(static_cast<size_t>(g.n_tiles) * g.cell_blocks);
    RXGS_CUDA(cudaMemcpy(len.data(), st->cell_len.p, cells * sizeof(int), cudaMemcpyDeviceToHost));
    RXGS_CUDA(cudaMemcpy(wl.data(), st->walk_len.p, wl.size() * sizeof(int), cudaMemcpyDeviceToHost));
    double s = 0.0, ts = 0.0;
    for (int x : len) s += x;
    for (int t = 0; t < g.n_tiles; ++t) {
        const int tt = t / g.tiles_p, tp = t % g.tiles_p;
        const int rows = std::min(g.ts, g.nt - tt * g.ts), cols = std::min(g.ts, g.np - tp * g.ts);
        int mx = 0;
        for (int b = 0; b < g.cell_blocks; ++b) mx = std::max(mx, wl[static_cast<size_t>(t) * g.cell_blocks + b]);
        ts += static_cast<double>(mx) * rows * cols;
    }
    if (visible) *visible = st->visible;
    if (entries) *entries = st->entries;
    if (walk_per_cell) *walk_per_cell = cells ? s / cells : 0.0;
    if (tile_walk_per_cell) *tile_walk_per_cell = cells ? ts / cells : 0.0;
    return RXGS_OK;
    API_END
}

int rxgs_tx_state_needed(rxgs_txstate st, int64_t* needed) {
    if (!st || !needed) return fail(RXGS_ERR_INVALID, "null argument");
    RX_TRY(set_device(st->ctx));
    int h = 0;
    RXGS_CUDA(cudaMemcpyAsync(&h, st->needed_count.p, sizeof(int), cudaMemcpyDeviceToHost, st->ctx->stream));
    RXGS_CUDA(cudaStreamSynchronize(st->ctx->stream));
    *needed = h;
    return RXGS_OK;
}

int rxgs_tx_state_transmittance(rxgs_txstate st, double* out) {
    if (!st || !out) return fail(RXGS_ERR_INVALID, "null argument");
    RX_TRY(set_device(st->ctx));
    RXGS_CUDA(cudaStreamSynchronize(st->ctx->stream));
    const size_t cells = static_cast<size_t>(st->grid.nt) * st->grid.np;
    RXGS_CUDA(cudaMemcpy(out, st->cell_T.p, cells * sizeof(double), cudaMemcpyDefault));
    return RXGS_OK;
}

int rxgs_bin_and_sort(rxgs_ctx ctx, int k, const int32_t* culled, const double* depth,
                      const int32_t* spans, const rxgs_grid* grid, int64_t* offsets, int32_t* indices,
                      int64_t cap, int64_t* entries) {
    API_BEGIN
    if (!ctx || k < 0) return fail(RXGS_ERR_INVALID, "rxgs_bin_and_sort: bad argument");
    if (!grid || grid->tile_size < 1 || grid->n_theta < 1 || grid->n_phi < 1)
        return fail(RXGS_ERR_INVALID, "grid: n_theta * n_phi must be >= 1");
    RX_TRY(set_device(ctx));
    rxgs_txstate_s st;
    st.ctx = ctx;
    st.k = k;
    st.grid = make_grid(grid);
    const size_t K = std::max(k, 1);
    std::vector<int> cul = to_host(culled, static_cast<size_t>(k));
    std::vector<double> dep = to_host(depth, static_cast<size_t>(k));
    std::vector<int> sp = to_host(spans, 4 * static_cast<size_t>(k));
    std::vector<uint64_t> dkey(K, ~0ull);
    std::vector<int> cnt(K, 0);
    for (int i = 0; i < k; ++i) {
        if (cul[i]) continue;
        uint64_t b;
        std::memcpy(&b, &dep[i], 8);
        dkey[i] = b;
        cnt[i] = std::max(0, sp[4 * i + 1] - sp[4 * i] + 1) * std::max(0, sp[4 * i + 3] - sp[4 * i + 2] + 1);
    }
    RXGS_CUDA(st.depth_key.ensure(K * 8));
    RXGS_CUDA(st.tile_count.ensure(K * 4));
    RXGS_CUDA(st.spans.ensure(K * 16));
    RXGS_CUDA(cudaMemcpy(st.depth_key.p, dkey.data(), K * 8, cudaMemcpyHostToDevice));
    RXGS_CUDA(cudaMemcpy(st.tile_count.p, cnt.data(), K * 4, cudaMemcpyHostToDevice));
    if (k) RXGS_CUDA(cudaMemcpy(st.spans.p, sp.data(), static_cast<size_t>(k) * 16, cudaMemcpyHostToDevice));
    RX_TRY(bin_tiles(ctx, st, ctx->stream));
    RXGS_CUDA(cudaStreamSynchronize(ctx->stream));
    if (entries) *entries = st.entries;
    if (offsets)
        RXGS_CUDA(cudaMemcpy(offsets, st.tile_offsets.p, (st.grid.n_tiles + 1) * sizeof(int64_t),
                             cudaMemcpyDefault));
    if (indices && cap >= st.entries && st.entries)
        RXGS_CUDA(cudaMemcpy(indices, st.list.p, st.entries * sizeof(int), cudaMemcpyDefault));
    return RXGS_OK;
    API_END
}

// ------------------------------------------------------------------ render
// raster::render_field (sphraster.cpp:255-315), materialised: FP64 signals
// and the FP64 per-cell walk of the reference (k_refapi.cu), so the field
// matches the reference to its rounding and finite differences of it agree
// with backward_render.  The fused query path (rxgs_render_queries) is the
// throughput path.
int rxgs_render_field(rxgs_ctx ctx, rxgs_txstate st, rxgs_scene sc, const double* coeffs, int n_rx,
                      double* values, double* transmittance) {
    API_BEGIN
    if (!ctx || !st || !sc) return fail(RXGS_ERR_INVALID, "render_field: null argument");
    if (n_rx < 1) return fail(RXGS_ERR_INVALID, "render_field: n_rx must be >= 1");
    if (sc->k != st->k || sc->channels != st->channels || sc->L != st->L)
        return fail(RXGS_ERR_INVALID, "render_field: coefficient tensor has wrong size");
    RX_TRY(set_device(ctx));
    cudaStream_t s = ctx->stream;
    const size_t stride = static_cast<size_t>(sc->L) * sc->channels * 2;
    const size_t nco = static_cast<size_t>(n_rx) * sc->k * stride;
    const double* d_co = nullptr;
    RX_TRY(dev_in(ctx, coeffs, nco, ctx->host_in, &d_co));
    DevBuf sig;
    RXGS_CUDA(sig.ensure(std::max<size_t>(static_cast<size_t>(sc->k) * n_rx * sc->channels, 1) * sizeof(double2)));
    RX_TRY(reset_err_flag(ctx));
    if (nco) {
        RX_TRY(ensure_tx_full(*st, s));
        const long long n = static_cast<long long>(nco);
        RXGS_CUDA(launch_check_finite(n, static_cast<long long>(stride), d_co, ctx->err_flag.as<int>(), s));
    }
    int err = INT_MAX;
    RX_TRY(check_err_flag(ctx, ctx->err_flag.as<int>(), &err));
    if (err != INT_MAX) {
        const int j = err / std::max(sc->k, 1), k = err % std::max(sc->k, 1);
        return fail(RXGS_ERR_INVALID, "render_field: non-finite coefficient at rx " + std::to_string(j) +
                                          ", gaussian " + std::to_string(k));
    }
    const size_t plane = static_cast<size_t>(st->grid.nt) * st->grid.np;
    const size_t nv = static_cast<size_t>(n_rx) * sc->channels * 2 * plane;
    double* d_vals = nullptr;
    double* d_T = nullptr;
    RX_TRY(dev_out(values, nv, ctx->host_out, &d_vals));
    DevBuf tT;
    RX_TRY(dev_out(transmittance, static_cast<size_t>(n_rx) * plane, tT, &d_T));
    if (!d_vals) {
        RXGS_CUDA(ctx->host_out.ensure(std::max<size_t>(nv, 1) * sizeof(double)));
        d_vals = ctx->host_out.as<double>();
    }
    cudaEvent_t ev;
    timing_begin(ctx, "render_field", &ev);
    RXGS_CUDA(launch_render64(*st, d_co, n_rx, sig.as<double2>(), d_vals, d_T, s));
    timing_end(ctx, "render_field", ev, static_cast<double>(n_rx) * sc->channels);
    ctx->launches += 2;
    RX_TRY(finish_out(ctx, values, d_vals, nv));
    RX_TRY(finish_out(ctx, transmittance, d_T, static_cast<size_t>(n_rx) * plane));
    RXGS_CUDA(cudaStreamSynchronize(s));
    return RXGS_OK;
    API_END
}

int rxgs_aggregate_modality(rxgs_ctx ctx, const rxgs_grid* grid, int modality, int n_rx, int channels,
                            const double* values, double* out) {
    API_BEGIN
    if (!ctx || !grid) return fail(RXGS_ERR_INVALID, "aggregate_modality: null argument");
    RX_TRY(set_device(ctx));
    const DevGrid g = make_grid(grid);
    const size_t plane = static_cast<size_t>(g.nt) * g.np;
    const size_t nv = static_cast<size_t>(n_rx) * channels * 2 * plane;
    const double* d_v = nullptr;
    RX_TRY(dev_in(ctx, values, nv, ctx->host_in, &d_v));
    RX_TRY(reset_err_flag(ctx));
    const size_t no = modality == 0 ? n_rx : (modality == 1 ? static_cast<size_t>(n_rx) * channels * 2 : n_rx * plane);
    // finiteness first (sphraster.cpp:325-326), then the channel check (:327-328)
    RXGS_CUDA(ctx->scratch_d.ensure(std::max<size_t>(no, 1) * sizeof(double)));
    double* d_out = nullptr;
    RX_TRY(dev_out(out, no, ctx->host_out, &d_out));
    if (!d_out) d_out = ctx->scratch_d.as<double>();
    const bool ch_ok = modality == 1 || channels == 1;
    RXGS_CUDA(launch_aggregate(g, modality, n_rx, channels, d_v, d_out, ctx->err_flag.as<int>(), ch_ok,
                               ctx->stream));
    ctx->launches += 2;
    int err = INT_MAX;
    RX_TRY(check_err_flag(ctx, ctx->err_flag.as<int>(), &err));
    if (err != INT_MAX) return fail(RXGS_ERR_INVALID, "aggregate_modality: non-finite field");
    if (!ch_ok) return fail(RXGS_ERR_INVALID, "aggregate_modality: scalar modalities need channels == 1");
    RX_TRY(finish_out(ctx, out, d_out, no));
    RXGS_CUDA(cudaStreamSynchronize(ctx->stream));
    return RXGS_OK;
    API_END
}

// ------------------------------------------------------------------ adjoints (sphraster.cpp:383-733)
int rxgs_aggregate_modality_backward(rxgs_ctx ctx, const rxgs_grid* grid, int modality, int n_rx, int channels,
                                     const double* values, const double* upstream, double* d_values) {
    API_BEGIN
    if (!ctx || !grid || !values || !upstream || !d_values)
        return fail(RXGS_ERR_INVALID, "aggregate_modality_backward: null argument");
    if (n_rx < 0 || channels < 1 || modality < 0 || modality > 2)
        return fail(RXGS_ERR_INVALID, "aggregate_modality_backward: bad arguments");
    if (modality != 1 && channels != 1)
        return fail(RXGS_ERR_INVALID, "aggregate_modality_backward: scalar modalities need channels == 1");
    RX_TRY(set_device(ctx));
    const DevGrid g = make_grid(grid);
    const size_t plane = static_cast<size_t>(g.nt) * g.np;
    const size_t nv = static_cast<size_t>(n_rx) * channels * 2 * plane;
    const size_t nu = modality == 0 ? n_rx : (modality == 1 ? static_cast<size_t>(n_rx) * channels * 2 : n_rx * plane);
    DevBuf tv, tu, to;
    const double* d_v = nullptr;
    const double* d_u = nullptr;
    double* d_o = nullptr;
    RX_TRY(dev_in(ctx, values, nv, tv, &d_v));
    RX_TRY(dev_in(ctx, upstream, nu, tu, &d_u));
    RX_TRY(dev_out(d_values, nv, to, &d_o));
    RXGS_CUDA(launch_aggregate_bwd(g, modality, n_rx, channels, d_v, d_u, d_o, ctx->stream));
    ctx->launches += 1;
    RX_TRY(finish_out(ctx, d_values, d_o, nv));
    RXGS_CUDA(cudaStreamSynchronize(ctx->stream));
    return RXGS_OK;
    API_END
}

int rxgs_backward_render(rxgs_ctx ctx, rxgs_txstate st, rxgs_scene sc, const double* coeffs, int n_rx,
                         const double* d_values, double* d_positions, double* d_log_scales, double* d_quaternions,
                         double* d_tau_logits, double* d_coeffs) {
    API_BEGIN
    if (!ctx || !st || !sc || !coeffs || !d_values)
        return fail(RXGS_ERR_INVALID, "backward_render: null argument");
    if (n_rx < 1) return fail(RXGS_ERR_INVALID, "backward_render: n_rx must be >= 1");
    if (sc->k != st->k || sc->channels != st->channels || sc->L != st->L)
        return fail(RXGS_ERR_INVALID, "render_field: coefficient tensor has wrong size");
    RX_TRY(set_device(ctx));
    cudaStream_t s = ctx->stream;
    const int K = sc->k, C = sc->channels;
    const size_t stride = static_cast<size_t>(sc->L) * C * 2;
    const size_t nco = static_cast<size_t>(n_rx) * K * stride;
    const size_t plane = static_cast<size_t>(st->grid.nt) * st->grid.np;
    const size_t nv = static_cast<size_t>(n_rx) * C * 2 * plane;
    const size_t n_jc = static_cast<size_t>(n_rx) * C;
    DevBuf t_co, t_dv, b_sig, b_eg, b_eds, b_rg, b_rds, o_pos, o_ls, o_q, o_tau, o_co;
    const double* d_co = nullptr;
    const double* d_dv = nullptr;
    RX_TRY(dev_in(ctx, coeffs, nco, t_co, &d_co));
    RX_TRY(dev_in(ctx, d_values, nv, t_dv, &d_dv));
    // non-finite coefficients are rejected exactly as the forward does (sphraster.cpp:197-206)
    RXGS_CUDA(ctx->signals.ensure(std::max<size_t>(static_cast<size_t>(K) * n_jc, 1) * sizeof(float2)));
    RX_TRY(reset_err_flag(ctx));
    if (nco) {
        RX_TRY(ensure_tx_full(*st, s));
        RXGS_CUDA(launch_reduce_signals(*st, d_co, n_rx, ctx->signals.as<float2>(), ctx->err_flag.as<int>(), s));
        ctx->launches += 2;
    }
    int err = INT_MAX;
    RX_TRY(check_err_flag(ctx, ctx->err_flag.as<int>(), &err));
    if (err != INT_MAX) {
        const int j = err / std::max(K, 1), k = err % std::max(K, 1);
        return fail(RXGS_ERR_INVALID, "render_field: non-finite coefficient at rx " + std::to_string(j) +
                                          ", gaussian " + std::to_string(k));
    }
    if (!st->regrouped) RX_TRY(train_regroup(ctx, *st, s));
    const size_t E = std::max<int64_t>(st->entries, 1);
    RXGS_CUDA(b_sig.ensure(std::max<size_t>(K * n_jc, 1) * sizeof(double2)));
    RXGS_CUDA(b_eg.ensure(bwd_geo_bytes(st->entries, static_cast<int>(n_jc))));
    RXGS_CUDA(b_eds.ensure(E * n_jc * sizeof(double2)));
    RXGS_CUDA(b_rg.ensure(std::max<size_t>(K, 1) * 7 * sizeof(double)));
    RXGS_CUDA(b_rds.ensure(std::max<size_t>(K * n_jc, 1) * sizeof(double2)));
    double *dp = nullptr, *dl = nullptr, *dq = nullptr, *dt = nullptr, *dc = nullptr;
    RX_TRY(dev_out(d_positions, 3 * static_cast<size_t>(K), o_pos, &dp));
    RX_TRY(dev_out(d_log_scales, 3 * static_cast<size_t>(K), o_ls, &dl));
    RX_TRY(dev_out(d_quaternions, 4 * static_cast<size_t>(K), o_q, &dq));
    RX_TRY(dev_out(d_tau_logits, static_cast<size_t>(K), o_tau, &dt));
    RX_TRY(dev_out(d_coeffs, nco, o_co, &dc));
    // every output is produced; absent ones land in scratch
    if (!dp) { RXGS_CUDA(o_pos.ensure(std::max<size_t>(3 * K, 1) * sizeof(double))); dp = o_pos.as<double>(); }
    if (!dl) { RXGS_CUDA(o_ls.ensure(std::max<size_t>(3 * K, 1) * sizeof(double))); dl = o_ls.as<double>(); }
    if (!dq) { RXGS_CUDA(o_q.ensure(std::max<size_t>(4 * K, 1) * sizeof(double))); dq = o_q.as<double>(); }
    if (!dt) { RXGS_CUDA(o_tau.ensure(std::max<size_t>(K, 1) * sizeof(double))); dt = o_tau.as<double>(); }
    if (!dc) { RXGS_CUDA(o_co.ensure(std::max<size_t>(nco, 1) * sizeof(double))); dc = o_co.as<double>(); }
    cudaEvent_t ev;
    timing_begin(ctx, "backward_render", &ev);
    RX_TRY(ensure_tx_full(*st, s));
    RXGS_CUDA(launch_backward_render(*st, *sc, d_co, n_rx, d_dv, b_sig.as<double2>(), b_eg.as<double>(),
                                     b_eds.as<double2>(), b_rg.as<double>(), b_rds.as<double2>(), dp, dl, dq, dt, dc,
                                     s));
    timing_end(ctx, "backward_render", ev, static_cast<double>(n_rx));
    ctx->launches += 3 + st->grid.cell_blocks * static_cast<int64_t>((n_jc + 7) / 8);
    RX_TRY(finish_out(ctx, d_positions, dp, 3 * static_cast<size_t>(K)));
    RX_TRY(finish_out(ctx, d_log_scales, dl, 3 * static_cast<size_t>(K)));
    RX_TRY(finish_out(ctx, d_quaternions, dq, 4 * static_cast<size_t>(K)));
    RX_TRY(finish_out(ctx, d_tau_logits, dt, static_cast<size_t>(K)));
    RX_TRY(finish_out(ctx, d_coeffs, dc, nco));
    RXGS_CUDA(cudaStreamSynchronize(s));
    return RXGS_OK;
    API_END
}

// ------------------------------------------------------------------ conditioning
int rxgs_cond_create(rxgs_ctx ctx, const int32_t cfg[9], const double* params, const double* occ,
                     const double occ_lo[3], const double occ_hi[3], rxgs_cond* out) {
    API_BEGIN
    if (!ctx || !cfg || !params || !out) return fail(RXGS_ERR_INVALID, "rxgs_cond_create: null argument");
    if (cfg[0] < 1 || cfg[1] < 1 || cfg[2] < 1)
        return fail(RXGS_ERR_INVALID, "init_conditioning: bad dimensions");
    if (cfg[1] > 64) return fail(RXGS_ERR_INVALID, "conditioning: hidden > 64 is not supported by the B200 path");
    if (cfg[8] < 1 || cfg[8] > 8) return fail(RXGS_ERR_INVALID, "conditioning: channels must be in [1, 8]");
    if (cfg[6] < 0 || cfg[6] > 4) return fail(RXGS_ERR_INVALID, "unknown conditioning mode");
    if (cfg[3] < 1) return fail(RXGS_ERR_INVALID, "probe_segment: samples must be >= 1");
    RX_TRY(set_device(ctx));
    auto* c = new rxgs_cond_s;
    c->ctx = ctx;
    c->F = cfg[0]; c->hidden = cfg[1]; c->dc = cfg[2]; c->S = cfg[3]; c->R = cfg[4];
    c->nearest = cfg[5]; c->mode = cfg[6]; c->l_max = cfg[7]; c->C = cfg[8];
    layout_cond(*c);
    c->h_params = to_host(params, static_cast<size_t>(c->n_params));
    std::vector<float> p32(c->h_params.begin(), c->h_params.end());
    auto bad = [&](cudaError_t e, const char* w) {
        delete c;
        return cuda_fail(e, w);
    };
    cudaError_t e = c->d_params64.ensure(c->h_params.size() * sizeof(double));
    if (e != cudaSuccess) return bad(e, "params64");
    e = cudaMemcpy(c->d_params64.p, c->h_params.data(), c->h_params.size() * sizeof(double), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return bad(e, "params64 copy");
    e = c->d_params32.ensure(p32.size() * sizeof(float));
    if (e != cudaSuccess) return bad(e, "params32");
    e = cudaMemcpy(c->d_params32.p, p32.data(), p32.size() * sizeof(float), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return bad(e, "params32 copy");
    if (occ) {
        const size_t n = static_cast<size_t>(c->R) * c->R * c->R;
        std::vector<double> h = to_host(occ, n);
        c->h_occ = h;
        std::vector<float> f(h.begin(), h.end());
        e = c->d_occ32.ensure(n * sizeof(float));
        if (e != cudaSuccess) return bad(e, "occ");
        e = cudaMemcpy(c->d_occ32.p, f.data(), n * sizeof(float), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return bad(e, "occ copy");
        e = c->d_occ64.ensure(n * sizeof(double));
        if (e == cudaSuccess) e = cudaMemcpy(c->d_occ64.p, h.data(), n * sizeof(double), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return bad(e, "occ64");
        std::vector<double> lo = to_host(occ_lo, 3), hi = to_host(occ_hi, 3);
        for (int a = 0; a < 3; ++a) {
            c->lo[a] = lo[a];
            c->hi[a] = hi[a];
        }
        c->has_occ = true;
        e = launch_occ_cubes(*c, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) return bad(e, "occ cubes");
    }
    ctx_retain(ctx);
    *out = c;
    return RXGS_OK;
    API_END
}

int rxgs_cond_destroy(rxgs_cond c) {
    if (!c) return RXGS_OK;
    rxgs_ctx ctx = c->ctx;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    delete c;
    ctx_release(ctx);
    return RXGS_OK;
}

int64_t rxgs_cond_param_count(rxgs_cond c) { return c ? c->n_params : -1; }

int rxgs_cond_calls(rxgs_cond c, int64_t* g, int64_t* l) {
    if (!c) return fail(RXGS_ERR_INVALID, "null conditioning");
    if (g) *g = c->global_calls;
    if (l) *l = c->local_calls;
    return RXGS_OK;
}

int rxgs_build_occupancy(rxgs_ctx ctx, rxgs_scene sc, int R, const double lo_[3], const double hi_[3],
                         double* out, rxgs_cond attach) {
    API_BEGIN
    if (!ctx || !sc || !lo_ || !hi_) return fail(RXGS_ERR_INVALID, "build_occupancy: null argument");
    if (R < 1) return fail(RXGS_ERR_INVALID, "build_occupancy: resolution must be >= 1");
    std::vector<double> lo = to_host(lo_, 3), hi = to_host(hi_, 3);
    if (!(hi[0] - lo[0] > 0 && hi[1] - lo[1] > 0 && hi[2] - lo[2] > 0))
        return fail(RXGS_ERR_INVALID, "build_occupancy: degenerate bounds");
    RX_TRY(set_device(ctx));
    const size_t n = static_cast<size_t>(R) * R * R;
    double* d64 = nullptr;
    RX_TRY(dev_out(out, n, ctx->host_out, &d64));
    if (!d64 && attach) {  // the attached state keeps a host f64 copy (checkpoint save)
        RXGS_CUDA(ctx->host_out.ensure(n * sizeof(double)));
        d64 = ctx->host_out.as<double>();
    }
    float* d32 = nullptr;
    if (attach) {
        RXGS_CUDA(attach->d_occ32.ensure(n * sizeof(float)));
        d32 = attach->d_occ32.as<float>();
    }
    cudaEvent_t ev;
    timing_begin(ctx, "occupancy", &ev);
    RXGS_CUDA(launch_occupancy(*sc, R, lo.data(), hi.data(), d64, d32, ctx->stream));
    timing_end(ctx, "occupancy", ev, sc->k);
    ctx->launches += 2;
    if (attach) {
        attach->R = R;
        for (int a = 0; a < 3; ++a) {
            attach->lo[a] = lo[a];
            attach->hi[a] = hi[a];
        }
        attach->has_occ = true;
        RXGS_CUDA(launch_occ_cubes(*attach, ctx->stream));
        RXGS_CUDA(attach->d_occ64.ensure(n * sizeof(double)));
        RXGS_CUDA(cudaMemcpyAsync(attach->d_occ64.p, d64, n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
        attach->h_occ.resize(n);
        RXGS_CUDA(cudaMemcpyAsync(attach->h_occ.data(), d64, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    }
    RX_TRY(finish_out(ctx, out, d64, n));
    RXGS_CUDA(cudaStreamSynchronize(ctx->stream));
    return RXGS_OK;
    API_END
}

int rxgs_probe_segments(rxgs_ctx ctx, rxgs_cond c, int n, const double* from, const double* to,
                        double* out) {
    API_BEGIN
    if (!ctx || !c) return fail(RXGS_ERR_INVALID, "probe_segment: null argument");
    if (c->S < 1) return fail(RXGS_ERR_INVALID, "probe_segment: samples must be >= 1");
    RX_TRY(set_device(ctx));
    const double *d_from = nullptr, *d_to = nullptr;
    RX_TRY(dev_in(ctx, from, 3 * static_cast<size_t>(n), ctx->scratch_c, &d_from));
    RX_TRY(dev_in(ctx, to, 3 * static_cast<size_t>(n), ctx->scratch_d, &d_to));
    double* d_out = nullptr;
    RX_TRY(dev_out(out, 2 * static_cast<size_t>(n), ctx->host_out, &d_out));
    RXGS_CUDA(launch_probe(*c, n, d_from, d_to, d_out, ctx->stream));
    ctx->launches += 1;
    RX_TRY(finish_out(ctx, out, d_out, 2 * static_cast<size_t>(n)));
    RXGS_CUDA(cudaStreamSynchronize(ctx->stream));
    return RXGS_OK;
    API_END
}

// The materialised conditioning API runs the FP64 kernels (k_refapi.cu) in
// the reference's operation order; the fused query path keeps its own
// FP32 / tcgen05 pipeline.  base: the coefficients to condition (NULL = the
// scene's own).
namespace {
int condition_fp64(rxgs_ctx ctx, rxgs_cond c, rxgs_scene sc, const double* rx, int n_rx, const double* base,
                   double* out, double* local_in) {
    if (!ctx || !c || !sc || !rx) return fail(RXGS_ERR_INVALID, "condition_forward: null argument");
    if (sc->l_max != c->l_max || sc->channels != c->C)
        return fail(RXGS_ERR_INVALID, "condition_forward: scene/state shape mismatch");
    RX_TRY(set_device(ctx));
    cudaStream_t s = ctx->stream;
    DevBuf t_rx, t_base, t_ag;
    const double* d_rx = nullptr;
    RX_TRY(dev_in(ctx, rx, 3 * static_cast<size_t>(n_rx), t_rx, &d_rx));
    if (c->use_local()) RX_TRY(check_receivers(ctx, sc, rx, n_rx));
    const size_t stride = static_cast<size_t>(sc->L) * sc->channels * 2;
    const size_t nb = static_cast<size_t>(sc->k) * stride;
    const double* d_base = sc->d_coeffs64.as<double>();
    if (base) RX_TRY(dev_in(ctx, base, nb, t_base, &d_base));
    const size_t no = static_cast<size_t>(n_rx) * nb;
    RXGS_CUDA(t_ag.ensure(std::max<size_t>(static_cast<size_t>(n_rx) * sc->L * 4 * sc->channels, 1) * sizeof(double)));
    double* d_out = nullptr;
    RX_TRY(dev_out(out, no, ctx->host_out, &d_out));
    double* d_li = nullptr;
    DevBuf t_li;
    if (local_in) RX_TRY(dev_out(local_in, static_cast<size_t>(sc->k) * 6, t_li, &d_li));
    RXGS_CUDA(launch_cond_forward64(*c, *sc, d_rx, n_rx, d_base, t_ag.as<double>(), d_out, d_li, s));
    ctx->launches += 2;
    if (c->use_global()) c->global_calls += static_cast<int64_t>(n_rx) * sc->L;
    if (c->use_local()) c->local_calls += static_cast<int64_t>(n_rx) * sc->k;
    RX_TRY(finish_out(ctx, out, d_out, no));
    if (local_in) RX_TRY(finish_out(ctx, local_in, d_li, static_cast<size_t>(sc->k) * 6));
    RXGS_CUDA(cudaStreamSynchronize(s));
    return RXGS_OK;
}
}  // namespace

int rxgs_condition_batch(rxgs_ctx ctx, rxgs_cond c, rxgs_scene sc, const double* rx, int n_rx,
                         double* out) {
    API_BEGIN
    return condition_fp64(ctx, c, sc, rx, n_rx, nullptr, out, nullptr);
    API_END
}

int rxgs_condition_forward(rxgs_ctx ctx, rxgs_cond c, rxgs_scene sc, const double rx[3], double* out,
                           double* local_in) {
    API_BEGIN
    return condition_fp64(ctx, c, sc, rx, 1, nullptr, out, local_in);
    API_END
}

int rxgs_condition_forward_base(rxgs_ctx ctx, rxgs_cond c, rxgs_scene sc, const double* base, const double* rx,
                                int n_rx, double* out, double* local_in) {
    API_BEGIN
    if (!base) return fail(RXGS_ERR_INVALID, "condition_forward: null base");
    return condition_fp64(ctx, c, sc, rx, n_rx, base, out, local_in);
    API_END
}

int rxgs_condition_backward(rxgs_ctx ctx, rxgs_cond c, rxgs_scene sc, const double rx[3], const double* d_out,
                            double* d_base, double* d_params) {
    API_BEGIN
    if (!ctx || !c || !sc || !rx || !d_out) return fail(RXGS_ERR_INVALID, "condition_backward: null argument");
    if (sc->l_max != c->l_max || sc->channels != c->C)
        return fail(RXGS_ERR_INVALID, "condition_forward: scene/state shape mismatch");
    RX_TRY(set_device(ctx));
    cudaStream_t s = ctx->stream;
    if (c->use_local()) RX_TRY(check_receivers(ctx, sc, rx, 1));
    const size_t nco = static_cast<size_t>(sc->k) * sc->L * sc->channels * 2;
    const size_t npar = c->h_params.size();
    DevBuf t_rx, t_do, o_base, o_par, ws;
    const double* d_rx = nullptr;
    const double* d_do = nullptr;
    RX_TRY(dev_in(ctx, rx, 3, t_rx, &d_rx));
    RX_TRY(dev_in(ctx, d_out, nco, t_do, &d_do));
    double* db = nullptr;
    double* dp = nullptr;
    RX_TRY(dev_out(d_base, nco, o_base, &db));
    RX_TRY(dev_out(d_params, npar, o_par, &dp));
    if (!db) { RXGS_CUDA(o_base.ensure(std::max<size_t>(nco, 1) * sizeof(double))); db = o_base.as<double>(); }
    if (!dp) { RXGS_CUDA(o_par.ensure(std::max<size_t>(npar, 1) * sizeof(double))); dp = o_par.as<double>(); }
    RXGS_CUDA(ws.ensure(cond_backward_ws_bytes(*c, sc->k, ctx->sm_count)));
    cudaEvent_t ev;
    timing_begin(ctx, "condition_backward", &ev);
    RXGS_CUDA(launch_cond_backward(*c, *sc, d_rx, d_do, db, dp, ws.p, ctx->sm_count, s));
    timing_end(ctx, "condition_backward", ev, static_cast<double>(sc->k));
    ctx->launches += 6;
    RX_TRY(finish_out(ctx, d_base, db, nco));
    RX_TRY(finish_out(ctx, d_params, dp, npar));
    RXGS_CUDA(cudaStreamSynchronize(s));
    return RXGS_OK;
    API_END
}

// ------------------------------------------------------------------ queries
int rxgs_render_queries(rxgs_ctx ctx, rxgs_scene sc, rxgs_cond c, rxgs_txstate st, const double* rx,
                        int n_rx, float* out_spectrum, float* out_rssi) {
    API_BEGIN
    if (!ctx || !sc || !st) return fail(RXGS_ERR_INVALID, "render_queries: null argument");
    if (n_rx < 0) return fail(RXGS_ERR_INVALID, "render_field: n_rx must be >= 1");
    if (n_rx == 0) return RXGS_OK;
    if (!rx) return fail(RXGS_ERR_INVALID, "render_queries: null receivers");
    if (sc->k != st->k || sc->L != st->L || sc->channels != st->channels)
        return fail(RXGS_ERR_INVALID, "render_queries: scene / tx-state mismatch");
    if (st->geo_version != sc->geo_version)
        return fail(RXGS_ERR_INVALID,
                    "render_queries: the scene geometry changed since this tx state was built; rebuild it");
    if (c && (sc->l_max != c->l_max || sc->channels != c->C))
        return fail(RXGS_ERR_INVALID, "condition_forward: scene/state shape mismatch");
    if (sc->channels != 1)
        return fail(RXGS_ERR_INVALID, "aggregate_modality: scalar modalities need channels == 1");
    RX_TRY(set_device(ctx));
    cudaStream_t s = ctx->stream;
    const double* d_rx = nullptr;
    RX_TRY(dev_in(ctx, rx, 3 * static_cast<size_t>(n_rx), ctx->scratch_c, &d_rx));
    if (c && c->use_local()) RX_TRY(check_receivers(ctx, sc, rx, n_rx));
    if (st->coeff_version != sc->coeff_version) {  // optimizer stepped since build: basis*base is stale
        RX_TRY(ensure_tx_full(*st, s));
        RXGS_CUDA(launch_refresh_gb(*sc, *st, s));
        st->coeff_version = sc->coeff_version;
    }
    const DevGrid& g = st->grid;
    const size_t plane = static_cast<size_t>(g.nt) * g.np;
    const int n_tb = g.n_tiles * g.cell_blocks;
    float* d_spec = nullptr;
    float* d_rssi = nullptr;
    RX_TRY(dev_out(out_spectrum, static_cast<size_t>(n_rx) * plane, ctx->host_out, &d_spec));
    RX_TRY(dev_out(out_rssi, static_cast<size_t>(n_rx), ctx->scratch_d, &d_rssi));
    // receiver chunks bound the signal buffer (K x chunk complex f32) to ~4 GB;
    // with host spectra, smaller chunks let the D2H of chunk i (copy stream)
    // overlap the conditioning of chunk i+1
    const size_t per_rx = std::max<size_t>(static_cast<size_t>(sc->k), 1) * sizeof(float2);
    int chunk = static_cast<int>(std::min<size_t>(static_cast<size_t>(n_rx), (size_t{4} << 30) / per_rx));
    // host spectra: receiver chunks (multiples of 32) whose D2H overlaps the
    // next chunk's compute; only the last, small one is exposed
    const bool pipelined = out_spectrum && d_spec != out_spectrum && n_rx >= 256;
    std::vector<int> bounds{0};
    if (pipelined) {
        // receiver-chunk schedules of the host-output pipeline (fractions of
        // the batch at the chunk ends).  A/B on one B200, config 2 (e2e, the
        // global branch and FLE GEMM batched once; scripts/probe_e2e_sched.py,
        // median of 15): 6 = 3.59-3.62 ms, 3 = 3.63-3.67, 2 = 3.67-3.68,
        // 0 = 3.71-3.74; 6 is the default, RXGS_E2E_SCHED selects another.
        static const std::vector<std::vector<double>> kSched = {
            {3.0 / 8, 3.0 / 8 + 5.0 / 16, 7.0 / 8, 7.0 / 8 + 3.0 / 32, 1.0},   // 0
            {3.0 / 8, 3.0 / 8 + 5.0 / 16, 7.0 / 8, 1.0},                       // 1
            {1.0 / 8, 3.0 / 8, 5.0 / 8, 27.0 / 32, 31.0 / 32, 1.0},            // 2
            {1.0 / 4, 1.0 / 2, 3.0 / 4, 15.0 / 16, 1.0},                       // 3
            {1.0 / 8, 1.0 / 2, 7.0 / 8, 31.0 / 32, 1.0},                       // 4
            {1.0 / 8, 3.0 / 8, 5.0 / 8, 13.0 / 16, 15.0 / 16, 1.0},            // 5
            {3.0 / 16, 7.0 / 16, 11.0 / 16, 7.0 / 8, 1.0},                     // 6
        };
        static const int sched = [] {
            const char* e = std::getenv("RXGS_E2E_SCHED");
            const int v = e ? std::atoi(e) : 6;
            return v >= 0 && v < static_cast<int>(kSched.size()) ? v : 6;
        }();
        const std::vector<double>& frac = kSched[static_cast<size_t>(sched)];
        for (double f : frac) {
            int b = static_cast<int>(std::lround(f * n_rx / 32.0)) * 32;
            b = std::min(std::max(b, bounds.back() + 1), n_rx);
            if (f == 1.0) b = n_rx;
            if (b > bounds.back()) bounds.push_back(b);
        }
        int widest = 0;
        for (size_t i = 1; i < bounds.size(); ++i) widest = std::max(widest, bounds[i] - bounds[i - 1]);
        chunk = std::min(chunk, widest);
    }
    chunk = std::max(chunk, 1);
    if (!pipelined || bounds.back() != n_rx || chunk < (bounds.size() > 1 ? bounds[1] : 0)) {
        bounds.assign(1, 0);  // uniform chunks
        for (int b = chunk; b < n_rx; b += chunk) bounds.push_back(b);
        bounds.push_back(n_rx);
    }
    if (pipelined && !ctx->copy_stream) RXGS_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    int n_chunk_ev = 0;
    RXGS_CUDA(ctx->signals.ensure(per_rx * chunk));
    RXGS_CUDA(ctx->partial.ensure(std::max<size_t>(static_cast<size_t>(n_tb) * chunk, 1) * sizeof(float)));
    // the tcgen05 compositor reads the signals pre-split into bf16 hi/lo
    const bool tc_comp = ctx->composite_kernel != 1 && composite_tc_eligible(*st);
    const SigOut so = tc_comp ? SigOut::presplit(ctx->signals.p) : SigOut(ctx->signals.as<float2>());
    // several chunks: the receiver-independent and whole-batch work once --
    // the global branch for all receivers and, on the tensor-core path, the
    // row gather and the FLE GEMM -- so each chunk launches only the
    // conditioning kernel (per-chunk global branch / GEMM measured +0.5 ms
    // over five chunks at config 2)
    const bool batched = c && bounds.size() > 2;
    const bool tc_cond = batched && ctx->cond_kernel != 1 && cond_tc_eligible(c);
    const float2* mpre_all = nullptr;
    const size_t ag_row = static_cast<size_t>(sc->L) * 4 * sc->channels;  // floats per receiver
    if (batched) {
        if (c->host_stale) {  // the tcgen05 kernel takes layers 1/3 from the host copy
            RXGS_CUDA(cudaStreamSynchronize(s));
            RXGS_CUDA(cudaMemcpy(c->h_params.data(), c->d_params64.p, c->h_params.size() * sizeof(double),
                                 cudaMemcpyDeviceToHost));
            c->host_stale = false;
        }
        RXGS_CUDA(ctx->ag.ensure(std::max<size_t>(ag_row * n_rx, 1) * sizeof(float)));
        cudaEvent_t evg;
        if (c->use_global()) {
            timing_begin(ctx, "cond_global", &evg);
            RXGS_CUDA(launch_cond_global(*c, d_rx, n_rx, ctx->ag.as<float>(), s));
            timing_end(ctx, "cond_global", evg, static_cast<double>(n_rx) * sc->L);
        } else {
            RXGS_CUDA(cudaMemsetAsync(ctx->ag.p, 0, ag_row * n_rx * sizeof(float), s));
        }
        if (tc_cond) {
            timing_begin(ctx, "cond_signal", &evg);
            RXGS_CUDA(launch_cond_signal_tc_prep(*c, *sc, *st, n_rx, ctx->ag.as<float>(), s, &mpre_all));
            timing_end(ctx, "cond_signal", evg, 0.0);
        }
        ctx->launches += 2;
    }
    for (size_t ci = 0; ci + 1 < bounds.size(); ++ci) {
        const int j0 = bounds[ci], nj = bounds[ci + 1] - bounds[ci];
        if (batched) {
            const double* rxc = d_rx + 3 * static_cast<size_t>(j0);
            const float* agc = ctx->ag.as<float>() + ag_row * j0;
            cudaEvent_t evc;
            timing_begin(ctx, "cond_signal", &evc);
            if (tc_cond)
                RXGS_CUDA(launch_cond_signal_tc(*c, *sc, *st, rxc, nj, agc, so, s,
                                                mpre_all ? mpre_all + static_cast<size_t>(st->k) * j0 : nullptr));
            else
                RXGS_CUDA(launch_cond_signal(c, *sc, *st, rxc, nj, agc, so, nullptr, s));
            timing_end(ctx, "cond_signal", evc,
                       static_cast<double>(st->needed_host >= 0 ? st->needed_host : st->visible) * nj);
            ctx->launches += 1;
        } else {
            RX_TRY(compute_signals(ctx, sc, c, st, d_rx + 3 * static_cast<size_t>(j0), nj, so));
        }
        CompositeOut co;
        co.spectrum = d_spec ? d_spec + static_cast<size_t>(j0) * plane : nullptr;
        co.rssi_partial = d_rssi ? ctx->partial.as<float>() : nullptr;
        cudaEvent_t ev;
        timing_begin(ctx, "composite", &ev);
        if (tc_comp)
            RXGS_CUDA(launch_composite_tc(*st, so.split, nj, co, s));
        else
            RXGS_CUDA(launch_composite(*st, ctx->signals.as<float2>(), nj, co, s));
        timing_end(ctx, "composite", ev, nj);
        ctx->launches += 1;
        if (d_rssi) {
            RXGS_CUDA(launch_rssi_finalize(ctx->partial.as<float>(), n_tb, nj, d_rssi + j0, nullptr, s));
            ctx->launches += 1;
        }
        if (pipelined) {
            if (static_cast<int>(ctx->chunk_events.size()) <= n_chunk_ev) {
                cudaEvent_t e;
                RXGS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                ctx->chunk_events.push_back(e);
            }
            cudaEvent_t e = ctx->chunk_events[n_chunk_ev++];
            RXGS_CUDA(cudaEventRecord(e, s));
            RXGS_CUDA(cudaStreamWaitEvent(ctx->copy_stream, e, 0));
            RXGS_CUDA(cudaMemcpyAsync(out_spectrum + static_cast<size_t>(j0) * plane,
                                      d_spec + static_cast<size_t>(j0) * plane,
                                      sizeof(float) * static_cast<size_t>(nj) * plane, cudaMemcpyDeviceToHost,
                                      ctx->copy_stream));
        }
    }
    if (c) {
        if (c->use_global()) c->global_calls += static_cast<int64_t>(n_rx) * sc->L;
        if (c->use_local()) c->local_calls += static_cast<int64_t>(n_rx) * sc->k;
    }
    const bool host_out = (out_spectrum && d_spec != out_spectrum) || (out_rssi && d_rssi != out_rssi);
    if (!pipelined) RX_TRY(finish_out(ctx, out_spectrum, d_spec, static_cast<size_t>(n_rx) * plane));
    RX_TRY(finish_out(ctx, out_rssi, d_rssi, static_cast<size_t>(n_rx)));
    if (pipelined) RXGS_CUDA(cudaStreamSynchronize(ctx->copy_stream));
    if (host_out || !is_device_ptr(rx)) RXGS_CUDA(cudaStreamSynchronize(s));
    return RXGS_OK;
    API_END
}

int rxgs_coverage_table(rxgs_ctx ctx, rxgs_scene sc, rxgs_cond c, const rxgs_grid* grid, const double* tx,
                        int n_tx, const double* rx, int n_rx, float* out_rssi) {
    API_BEGIN
    if (!ctx || !sc || !grid) return fail(RXGS_ERR_INVALID, "coverage_table: null argument");
    if (n_tx < 0 || n_rx < 0) return fail(RXGS_ERR_INVALID, "coverage_table: negative count");
    if (n_tx == 0 || n_rx == 0) return RXGS_OK;
    if (!tx || !rx || !out_rssi) return fail(RXGS_ERR_INVALID, "coverage_table: null argument");
    if (c && (sc->l_max != c->l_max || sc->channels != c->C))
        return fail(RXGS_ERR_INVALID, "condition_forward: scene/state shape mismatch");
    if (sc->channels != 1)
        return fail(RXGS_ERR_INVALID, "aggregate_modality: scalar modalities need channels == 1");
    RX_TRY(validate_grid(grid));
    RX_TRY(set_device(ctx));
    cudaStream_t s = ctx->stream;
    if (c && c->host_stale) {
        RXGS_CUDA(cudaStreamSynchronize(s));
        RXGS_CUDA(cudaMemcpy(c->h_params.data(), c->d_params64.p, c->h_params.size() * sizeof(double),
                             cudaMemcpyDeviceToHost));
        c->host_stale = false;
    }
    DevBuf t_rx;
    const double* d_rx = nullptr;
    RX_TRY(dev_in(ctx, rx, 3 * static_cast<size_t>(n_rx), t_rx, &d_rx));
    const std::vector<double> txh = to_host(tx, 3 * static_cast<size_t>(n_tx));
    if (c && c->use_local()) RX_TRY(check_receivers(ctx, sc, rx, n_rx));
    float* d_out = nullptr;
    DevBuf t_out;
    RX_TRY(dev_out(out_rssi, static_cast<size_t>(n_tx) * n_rx, t_out, &d_out));
    // Tx-independent halves of the conditioning, once for all transmitters
    const size_t ag_n = static_cast<size_t>(n_rx) * sc->L * 4;
    RXGS_CUDA(ctx->ag.ensure(std::max<size_t>(ag_n, 1) * sizeof(float)));
    cudaEvent_t ev;
    if (c && c->use_global()) {
        timing_begin(ctx, "cond_global", &ev);
        RXGS_CUDA(launch_cond_global(*c, d_rx, n_rx, ctx->ag.as<float>(), s));
        timing_end(ctx, "cond_global", ev, static_cast<double>(n_rx) * sc->L);
    } else {
        RXGS_CUDA(cudaMemsetAsync(ctx->ag.p, 0, ag_n * sizeof(float), s));
    }
    DevBuf t_agT;
    RXGS_CUDA(t_agT.ensure(std::max<size_t>(ag_n, 1) * sizeof(float)));
    RXGS_CUDA(launch_ag_transpose(n_rx, sc->L, ctx->ag.as<float>(), t_agT.as<float>(), s));
    ctx->launches += 2;
    const float4* yc = nullptr;
    if (c && c->use_local()) {
        RXGS_CUDA(ctx->ycache.ensure(std::max<size_t>(static_cast<size_t>(sc->k) * n_rx, 1) * sizeof(float4)));
        timing_begin(ctx, "local_cache", &ev);
        RXGS_CUDA(launch_local_cache(*c, *sc, d_rx, n_rx, ctx->ycache.as<float4>(), s));
        timing_end(ctx, "local_cache", ev, static_cast<double>(sc->k) * n_rx);
        ctx->launches += 1;
        yc = ctx->ycache.as<float4>();
    }
    RXGS_CUDA(ctx->signals.ensure(std::max<size_t>(static_cast<size_t>(sc->k) * ((n_rx + 3) & ~3), 1) * sizeof(float2)));
    // Render of one transmitter state (this context's stream)
    auto render_tx = [&](int t, rxgs_txstate st) -> int {
        const DevGrid& g = st->grid;
        const int n_tb = g.n_tiles * g.cell_blocks;
        bool tc_comp = false;
        cudaError_t e = ctx->partial.ensure(std::max<size_t>(static_cast<size_t>(n_tb) * n_rx, 1) * sizeof(float));
        if (e == cudaSuccess) {
            timing_begin(ctx, "cov_signal", &ev);
            tc_comp = ctx->composite_kernel != 1 && composite_tc_eligible(*st);
            // FLE as a GEMM only for high l_max: at l_max 2 the fused loop of
            // k_cov_signal measured faster (0.69 vs 1.03 ms per transmitter)
            if (sc->L >= 16)
                e = launch_cov_signal_gemm(c, *sc, *st, n_rx, ctx->ag.as<float>(), yc,
                                           tc_comp ? SigOut::presplit(ctx->signals.p) : SigOut(ctx->signals.as<float2>()),
                                           s);
            else
                e = launch_cov_signal(c, *st, n_rx, t_agT.as<float>(), yc,
                                      tc_comp ? SigOut::presplit(ctx->signals.p) : SigOut(ctx->signals.as<float2>()), s);
            timing_end(ctx, "cov_signal", ev,
                       static_cast<double>(st->needed_host >= 0 ? st->needed_host : st->visible) * n_rx);
        }
        if (e == cudaSuccess) {
            CompositeOut co;
            co.rssi_partial = ctx->partial.as<float>();
            timing_begin(ctx, "composite", &ev);
            e = tc_comp ? launch_composite_tc(*st, ctx->signals.as<uint2>(), n_rx, co, s)
                        : launch_composite(*st, ctx->signals.as<float2>(), n_rx, co, s);
            timing_end(ctx, "composite", ev, n_rx);
        }
        if (e == cudaSuccess)
            e = launch_rssi_finalize(ctx->partial.as<float>(), n_tb, n_rx, d_out + static_cast<size_t>(t) * n_rx,
                                     nullptr, s);
        ctx->launches += 3;
        return e == cudaSuccess ? RXGS_OK : cuda_fail(e, "coverage_table");
    };
    // Transmitter states are built by D builder threads, each on its own
    // helper context (stream, scratch, buffer pool): builder i builds the
    // states t = i, i + D, ... while this thread renders.  A build is a chain
    // of short kernels with host syncs (entry counts), latency- rather than
    // throughput-bound, so D builders in flight keep the render stream fed.
    // Stream order: the render of t waits on the builder's event; builder i
    // recycles state t's buffers for t + D only after the render of t is
    // done on the device.
#ifndef RXGS_COV_BUILDERS
#define RXGS_COV_BUILDERS 4  // A/B (config 3, ms per table): serial 128.3, D=1 129.1, 2 116.5, 3 113.4, 4 110.8;
                             // 6 / 8 and high-priority builder streams within noise (109-112)
#endif
    int D = std::min(RXGS_COV_BUILDERS, rxgs_ctx_s::kAuxMax);
    if (const char* v = std::getenv("RXGS_COV_BUILDERS")) D = std::max(0, std::min(std::atoi(v), rxgs_ctx_s::kAuxMax));
    if (n_tx < 2) D = 0;
    D = std::min(D, n_tx);
    if (D == 0) {  // one transmitter: build and render in turn on this context
        for (int t = 0; t < n_tx; ++t) {
            rxgs_txstate st = nullptr;
            RX_TRY(rxgs_tx_state_build(ctx, sc, txh.data() + 3 * static_cast<size_t>(t), grid, &st));
            const int rc = render_tx(t, st);
            rxgs_tx_state_destroy(st);
            if (rc) return rc;
        }
    } else {
        int64_t launches0[rxgs_ctx_s::kAuxMax];
        for (int i = 0; i < D; ++i) {
            if (!ctx->aux[i]) {
                RX_TRY(rxgs_ctx_create(ctx->device, &ctx->aux[i]));
                RXGS_CUDA(cudaEventCreateWithFlags(&ctx->aux_ev[i], cudaEventDisableTiming));
                RXGS_CUDA(cudaEventCreateWithFlags(&ctx->aux_done[i], cudaEventDisableTiming));
            }
            ctx->aux[i]->profile = ctx->profile;
            launches0[i] = ctx->aux[i]->launches;
        }
        std::mutex mu;
        std::condition_variable cv;
        std::vector<rxgs_txstate> states(n_tx, nullptr);
        std::vector<signed char> built(n_tx, 0);  // 1 built, -1 failed
        std::vector<char> issued(n_tx, 0), dead(n_tx, 0);
        bool abort = false;
        int b_rc = RXGS_OK;
        std::string b_err;
        // RXGS_COV_TRACE=1: per-transmitter build / render timeline on stderr (diagnostics)
        const bool trace = std::getenv("RXGS_COV_TRACE") != nullptr;
        std::vector<cudaEvent_t> tev(trace ? 4 * static_cast<size_t>(n_tx) + 1 : 0);
        for (auto& e : tev) cudaEventCreate(&e);
        if (trace) cudaEventRecord(tev[4 * n_tx], s);
        auto builder = [&](int i) {
            rxgs_ctx b = ctx->aux[i];
            cudaSetDevice(b->device);
            for (int t = i; t < n_tx; t += D) {
                if (t >= D) {  // state t - D: recycle once its render is done on the device
                    {
                        std::unique_lock<std::mutex> lk(mu);
                        cv.wait(lk, [&] { return issued[t - D] || abort; });
                        if (abort) return;
                    }
                    cudaEventSynchronize(ctx->aux_done[i]);
                    rxgs_tx_state_destroy(states[t - D]);
                    std::lock_guard<std::mutex> lk(mu);
                    dead[t - D] = 1;
                }
                rxgs_txstate st = nullptr;
                if (trace) cudaEventRecord(tev[4 * t], b->stream);
                int rc = rxgs_tx_state_build(b, sc, txh.data() + 3 * static_cast<size_t>(t), grid, &st);
                if (trace) cudaEventRecord(tev[4 * t + 1], b->stream);
                if (!rc) {
                    const cudaError_t e = cudaEventRecord(ctx->aux_ev[i], b->stream);
                    if (e != cudaSuccess) rc = cuda_fail(e, "coverage_table builder");
                }
                std::lock_guard<std::mutex> lk(mu);
                states[t] = st;
                built[t] = rc ? -1 : 1;
                if (rc && !b_rc) {
                    b_rc = rc;
                    b_err = rxgs_last_error();
                }
                cv.notify_all();
                if (rc) return;
            }
        };
        std::vector<std::thread> workers;
        int rc = RXGS_OK;
        try {
            for (int i = 0; i < D; ++i) workers.emplace_back(builder, i);
        } catch (const std::exception& ex) {  // no thread left joinable on the way out
            {
                std::lock_guard<std::mutex> lk(mu);
                abort = true;
                cv.notify_all();
            }
            for (auto& w : workers) w.join();
            for (int t = 0; t < n_tx; ++t)
                if (states[t]) rxgs_tx_state_destroy(states[t]);
            return fail(RXGS_ERR_CUDA, std::string("coverage_table: builder thread: ") + ex.what());
        }
        for (int t = 0; t < n_tx && !rc; ++t) {
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return built[t] != 0; });
                if (built[t] < 0) {
                    rc = fail(b_rc, b_err);
                    break;
                }
            }
            const int i = t % D;
            cudaError_t e = cudaStreamWaitEvent(s, ctx->aux_ev[i], 0);
            if (trace) cudaEventRecord(tev[4 * t + 2], s);
            rc = e == cudaSuccess ? render_tx(t, states[t]) : cuda_fail(e, "coverage_table");
            if (trace) cudaEventRecord(tev[4 * t + 3], s);
            if (!rc && (e = cudaEventRecord(ctx->aux_done[i], s)) != cudaSuccess) rc = cuda_fail(e, "coverage_table");
            std::lock_guard<std::mutex> lk(mu);
            if (rc) abort = true;
            else issued[t] = 1;
            cv.notify_all();
        }
        {  // a failed build or render: builders waiting for a render that will not come stop
            std::lock_guard<std::mutex> lk(mu);
            if (rc) abort = true;
            cv.notify_all();
        }
        for (auto& w : workers) w.join();
        cudaStreamSynchronize(s);  // the states still alive: no reader left
        if (trace) {
            cudaDeviceSynchronize();
            double busy = 0, wait_build = 0, prev_end = 0;
            for (int t = 0; t < n_tx; ++t) {
                float v[4] = {0.f, 0.f, 0.f, 0.f};  // stays 0 for a transmitter never reached (failed table)
                for (int q = 0; q < 4; ++q) cudaEventElapsedTime(&v[q], tev[4 * n_tx], tev[4 * t + q]);
                busy += v[3] - v[2];
                if (t > 0) wait_build += std::max(0.0, static_cast<double>(v[2]) - prev_end);
                prev_end = v[3];
                std::fprintf(stderr, "tx %2d build %8.3f %8.3f (%.3f)  render %8.3f %8.3f (%.3f)\n", t, v[0], v[1],
                             v[1] - v[0], v[2], v[3], v[3] - v[2]);
            }
            std::fprintf(stderr, "render busy %.3f ms, gaps between renders %.3f ms, end %.3f ms\n", busy,
                         wait_build, prev_end);
            for (auto& e : tev) cudaEventDestroy(e);
        }
        for (int t = 0; t < n_tx; ++t)
            if (states[t] && !dead[t]) rxgs_tx_state_destroy(states[t]);
        for (int i = 0; i < D; ++i) {  // the builders' launches and phase timings count for this context
            rxgs_ctx b = ctx->aux[i];
            ctx->launches += b->launches - launches0[i];
            if (ctx->profile) {
                resolve_timings(b);
                for (const auto& kv : b->stats) {
                    KStat& d = ctx->stats[kv.first];
                    d.ms += kv.second.ms;
                    d.launches += kv.second.launches;
                    d.work += kv.second.work;
                }
                b->stats.clear();
            }
        }
        if (rc) return rc;
    }
    if (c) {
        if (c->use_global()) c->global_calls += static_cast<int64_t>(n_rx) * sc->L;
        if (c->use_local()) c->local_calls += static_cast<int64_t>(n_rx) * sc->k;
    }
    RX_TRY(finish_out(ctx, out_rssi, d_out, static_cast<size_t>(n_tx) * n_rx));
    RXGS_CUDA(cudaStreamSynchronize(s));
    return RXGS_OK;
    API_END
}

int rxgs_predict(rxgs_ctx ctx, rxgs_scene sc, rxgs_cond c, const rxgs_grid* grid, const double tx[3],
                 const double rx[3], double* out) {
    API_BEGIN
    if (!ctx || !sc || !grid || !tx || !rx || !out) return fail(RXGS_ERR_INVALID, "predict: null argument");
    const size_t stride = static_cast<size_t>(sc->L) * sc->channels * 2;
    std::vector<double> coeffs(static_cast<size_t>(sc->k) * stride);
    if (c) {
        RX_TRY(rxgs_condition_forward(ctx, c, sc, rx, coeffs.data(), nullptr));
    } else {
        RX_TRY(scene_sync_host(sc));
        coeffs = sc->h_coeffs;
    }
    rxgs_txstate st = nullptr;
    RX_TRY(rxgs_tx_state_build(ctx, sc, tx, grid, &st));
    const size_t plane = static_cast<size_t>(grid->n_theta) * grid->n_phi;
    std::vector<double> vals(static_cast<size_t>(sc->channels) * 2 * plane);
    int rc = rxgs_render_field(ctx, st, sc, coeffs.data(), 1, vals.data(), nullptr);
    rxgs_tx_state_destroy(st);
    if (rc) return rc;
    return rxgs_aggregate_modality(ctx, grid, sc->modality, 1, sc->channels, vals.data(), out);
    API_END
}

// ------------------------------------------------------------------ single-call reference API (FP64, device)
int rxgs_project_gaussians(rxgs_ctx ctx, int n, const double* pos, const double* cov, const double* tau,
                           const double tx[3], const rxgs_grid* grid, double* geom, int32_t* culled, int32_t* spans) {
    API_BEGIN
    if (!ctx || n < 0 || (n && (!pos || !cov || !tau)) || !tx) return fail(RXGS_ERR_INVALID, "project_gaussian: null argument");
    RX_TRY(validate_grid(grid));
    RX_TRY(set_device(ctx));
    cudaStream_t s = ctx->stream;
    DevBuf a, b, c, t, og, oc, os;
    const double *dp = nullptr, *dc = nullptr, *dt = nullptr, *dtx = nullptr;
    RX_TRY(dev_in(ctx, pos, 3 * static_cast<size_t>(n), a, &dp));
    RX_TRY(dev_in(ctx, cov, 9 * static_cast<size_t>(n), b, &dc));
    RX_TRY(dev_in(ctx, tau, static_cast<size_t>(n), c, &dt));
    RX_TRY(dev_in(ctx, tx, 3, t, &dtx));
    std::vector<double> txh = to_host(tx, 3);
    double* d_g = nullptr;
    int32_t* d_c = nullptr;
    int32_t* d_s = nullptr;
    RXGS_CUDA(og.ensure(std::max<size_t>(12 * static_cast<size_t>(n), 1) * 8));
    RXGS_CUDA(oc.ensure(std::max<size_t>(n, 1) * 4));
    RXGS_CUDA(os.ensure(std::max<size_t>(4 * static_cast<size_t>(n), 1) * 4));
    d_g = og.as<double>();
    d_c = oc.as<int32_t>();
    d_s = os.as<int32_t>();
    const DevGrid g = make_grid(grid);
    RXGS_CUDA(launch_project(n, dp, dc, dt, txh.data(), g, d_g, d_c, reinterpret_cast<int4*>(d_s), s));
    ctx->launches += 1;
    RXGS_CUDA(cudaStreamSynchronize(s));
    if (geom && n) RXGS_CUDA(cudaMemcpy(geom, d_g, 12 * sizeof(double) * n, cudaMemcpyDefault));
    if (culled && n) RXGS_CUDA(cudaMemcpy(culled, d_c, sizeof(int32_t) * n, cudaMemcpyDefault));
    if (spans && n) RXGS_CUDA(cudaMemcpy(spans, d_s, 4 * sizeof(int32_t) * n, cudaMemcpyDefault));
    return RXGS_OK;
    API_END
}

int rxgs_fle_eval(rxgs_ctx ctx, int what, int l_max, int n, const double* a, const double* b, const double* coeffs,
                  double* out) {
    API_BEGIN
    static const char* kName[] = {"eval_basis", "eval_basis_jet", "legendre_table", "legendre_table_dtheta",
                                  "normalization", "eval_radiance"};
    if (!ctx || what < 0 || what > 5 || n < 0) return fail(RXGS_ERR_INVALID, "fle_eval: bad argument");
    if (l_max < 0) return fail(RXGS_ERR_INVALID, std::string(kName[what]) + ": l_max < 0");
    if (l_max > kApiMaxLmax) return fail(RXGS_ERR_INVALID, std::string(kName[what]) + ": l_max too large for the device");
    if (n == 0) return RXGS_OK;
    if (!a || !out || ((what == 0 || what == 1 || what == 4 || what == 5) && !b) || (what == 5 && !coeffs))
        return fail(RXGS_ERR_INVALID, "fle_eval: null argument");
    std::vector<double> ah = to_host(a, static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {  // the reference's argument checks (radiance.cpp:17, 117)
        if (what == 2 && std::abs(ah[i]) > 1.0 + 1e-12)
            return fail(RXGS_ERR_INVALID, "legendre_table: |x| > 1");
        if (what == 5 && (ah[i] < 0.0 || ah[i] > 3.14159265358979323846))
            return fail(RXGS_ERR_INVALID, "eval_radiance: theta out of [0, pi]");
    }
    RX_TRY(set_device(ctx));
    const int L = (l_max + 1) * (l_max + 1), NP = (l_max + 1) * (l_max + 2) / 2;
    const size_t per = what == 0 ? 2 * L : what == 1 ? 6 * L : what == 2 ? NP : what == 3 ? 2 * NP : what == 4 ? 1 : 2;
    DevBuf ta, tb, tc, to;
    const double *da = nullptr, *db = nullptr, *dcf = nullptr;
    RX_TRY(dev_in(ctx, a, static_cast<size_t>(n), ta, &da));
    if (b) RX_TRY(dev_in(ctx, b, static_cast<size_t>(n), tb, &db));
    if (what == 5) RX_TRY(dev_in(ctx, coeffs, static_cast<size_t>(n) * 2 * L, tc, &dcf));
    double* d_out = nullptr;
    RX_TRY(dev_out(out, per * n, to, &d_out));
    RXGS_CUDA(launch_fle_eval(what, n, l_max, da, db, dcf, d_out, ctx->stream));
    ctx->launches += 1;
    RX_TRY(finish_out(ctx, out, d_out, per * n));
    RXGS_CUDA(cudaStreamSynchronize(ctx->stream));
    return RXGS_OK;
    API_END
}

int rxgs_blend_ray(rxgs_ctx ctx, int n, const double* weights, const double* signals, double out[3]) {
    API_BEGIN
    if (!ctx || n < 0 || !out || (n && (!weights || !signals))) return fail(RXGS_ERR_INVALID, "blend_ray: null argument");
    RX_TRY(set_device(ctx));
    DevBuf tw, ts, to;
    const double *dw = nullptr, *ds = nullptr;
    RX_TRY(dev_in(ctx, weights, std::max(n, 1), tw, &dw));
    RX_TRY(dev_in(ctx, signals, 2 * static_cast<size_t>(std::max(n, 1)), ts, &ds));
    double* d_out = nullptr;
    RX_TRY(dev_out(out, 3, to, &d_out));
    RXGS_CUDA(launch_blend_ray(n, dw, ds, d_out, ctx->stream));
    ctx->launches += 1;
    RX_TRY(finish_out(ctx, out, d_out, 3));
    RXGS_CUDA(cudaStreamSynchronize(ctx->stream));
    return RXGS_OK;
    API_END
}

int rxgs_occupancy_sample(rxgs_ctx ctx, int R, const double lo[3], const double hi[3], const double* densities, int n,
                          const double* points, int nearest, double* out) {
    API_BEGIN
    if (!ctx || n < 0 || (n && (!points || !out))) return fail(RXGS_ERR_INVALID, "sample: null argument");
    if (n == 0) return RXGS_OK;
    RX_TRY(set_device(ctx));
    DevBuf td, tp, to;
    const double *dd = nullptr, *dp = nullptr;
    std::vector<double> l(3, 0.0), h(3, 1.0);
    if (densities && R > 0) {
        RX_TRY(dev_in(ctx, densities, static_cast<size_t>(R) * R * R, td, &dd));
        l = to_host(lo, 3);
        h = to_host(hi, 3);
    }
    RX_TRY(dev_in(ctx, points, 3 * static_cast<size_t>(n), tp, &dp));
    double* d_out = nullptr;
    RX_TRY(dev_out(out, static_cast<size_t>(n), to, &d_out));
    RXGS_CUDA(launch_occ_sample(R, l.data(), h.data(), dd, n, dp, nearest, d_out, ctx->stream));
    ctx->launches += 1;
    RX_TRY(finish_out(ctx, out, d_out, static_cast<size_t>(n)));
    RXGS_CUDA(cudaStreamSynchronize(ctx->stream));
    return RXGS_OK;
    API_END
}

int rxgs_probe_grid(rxgs_ctx ctx, int R, const double lo[3], const double hi[3], const double* densities, int n,
                    const double* from, const double* to, int samples, int nearest, double* out) {
    API_BEGIN
    if (samples < 1) return fail(RXGS_ERR_INVALID, "probe_segment: samples must be >= 1");
    if (!ctx || n < 0 || (n && (!from || !to || !out))) return fail(RXGS_ERR_INVALID, "probe_segment: null argument");
    if (n == 0) return RXGS_OK;
    RX_TRY(set_device(ctx));
    DevBuf td, tf, tt, to_;
    const double *dd = nullptr, *df = nullptr, *dt = nullptr;
    std::vector<double> l(3, 0.0), h(3, 1.0);
    if (densities && R > 0) {
        RX_TRY(dev_in(ctx, densities, static_cast<size_t>(R) * R * R, td, &dd));
        l = to_host(lo, 3);
        h = to_host(hi, 3);
    }
    RX_TRY(dev_in(ctx, from, 3 * static_cast<size_t>(n), tf, &df));
    RX_TRY(dev_in(ctx, to, 3 * static_cast<size_t>(n), tt, &dt));
    double* d_out = nullptr;
    RX_TRY(dev_out(out, 2 * static_cast<size_t>(n), to_, &d_out));
    RXGS_CUDA(launch_probe64(R, l.data(), h.data(), dd, n, df, dt, samples, nearest, d_out, ctx->stream));
    ctx->launches += 1;
    RX_TRY(finish_out(ctx, out, d_out, 2 * static_cast<size_t>(n)));
    RXGS_CUDA(cudaStreamSynchronize(ctx->stream));
    return RXGS_OK;
    API_END
}

int rxgs_fourier_encode(rxgs_ctx ctx, int F, const double* freqs, int n, const double* r, double* out) {
    API_BEGIN
    if (!ctx || F < 0 || n < 0 || (n && (!r || !out)) || (F && !freqs))
        return fail(RXGS_ERR_INVALID, "fourier_encode: null argument");
    if (n == 0 || F == 0) return RXGS_OK;
    RX_TRY(set_device(ctx));
    DevBuf tf, tr, to;
    const double *df = nullptr, *dr = nullptr;
    RX_TRY(dev_in(ctx, freqs, 3 * static_cast<size_t>(F), tf, &df));
    RX_TRY(dev_in(ctx, r, 3 * static_cast<size_t>(n), tr, &dr));
    double* d_out = nullptr;
    RX_TRY(dev_out(out, 6 * static_cast<size_t>(F) * n, to, &d_out));
    RXGS_CUDA(launch_fourier64(F, df, n, dr, d_out, ctx->stream));
    ctx->launches += 1;
    RX_TRY(finish_out(ctx, out, d_out, 6 * static_cast<size_t>(F) * n));
    RXGS_CUDA(cudaStreamSynchronize(ctx->stream));
    return RXGS_OK;
    API_END
}

int rxgs_mlp_layer_forward(rxgs_ctx ctx, int in, int out_dim, const double* w, const double* b, int n,
                           const double* x, double* y) {
    API_BEGIN
    if (!ctx || in < 0 || out_dim < 0 || n < 0) return fail(RXGS_ERR_INVALID, "MlpLayer::forward: bad argument");
    if (!n || !out_dim) return RXGS_OK;
    if (!b || !x || !y || (in && !w)) return fail(RXGS_ERR_INVALID, "MlpLayer::forward: null argument");
    RX_TRY(set_device(ctx));
    DevBuf tw, tb, tx, ty;
    const double *dw = nullptr, *db = nullptr, *dx = nullptr;
    RX_TRY(dev_in(ctx, w, std::max<size_t>(static_cast<size_t>(in) * out_dim, 1), tw, &dw));
    RX_TRY(dev_in(ctx, b, static_cast<size_t>(out_dim), tb, &db));
    RX_TRY(dev_in(ctx, x, std::max<size_t>(static_cast<size_t>(in) * n, 1), tx, &dx));
    double* d_y = nullptr;
    RX_TRY(dev_out(y, static_cast<size_t>(out_dim) * n, ty, &d_y));
    RXGS_CUDA(launch_mlp_layer64(in, out_dim, dw, db, n, dx, d_y, ctx->stream));
    ctx->launches += 1;
    RX_TRY(finish_out(ctx, y, d_y, static_cast<size_t>(out_dim) * n));
    RXGS_CUDA(cudaStreamSynchronize(ctx->stream));
    return RXGS_OK;
    API_END
}

int rxgs_grid_validate(const rxgs_grid* grid) {
    API_BEGIN
    return validate_grid(grid);
    API_END
}

// A device transmitter state from a host TxState (sphraster.hpp:52-61): the
// FP64 rows, spans, basis and per-tile lists the caller holds; the walk and
// the needed-row compaction run on the device as after a build.
int rxgs_tx_state_import(rxgs_ctx ctx, rxgs_scene sc, const rxgs_grid* grid, const int32_t* culled,
                         const double* geom, const int32_t* spans, const double* basis, const int64_t* offsets,
                         const int32_t* indices, rxgs_txstate* out) {
    API_BEGIN
    if (!ctx || !sc || !out || (sc->k && (!culled || !geom || !spans || !basis)) || !offsets)
        return fail(RXGS_ERR_INVALID, "tx_state_import: null argument");
    RX_TRY(validate_grid(grid));
    RX_TRY(set_device(ctx));
    cudaStream_t s = ctx->stream;
    auto* st = new rxgs_txstate_s;
    std::unique_ptr<rxgs_txstate_s> guard(st);
    st->ctx = ctx;
    st->k = sc->k;
    st->l_max = sc->l_max;
    st->L = sc->L;
    st->channels = sc->channels;
    st->grid = make_grid(grid);
    st->version = next_version();
    st->coeff_version = 0;  // basis*base from the scene's coefficients on first query use
    st->geo_version = sc->geo_version;
    st->full = true;
    const DevGrid& g = st->grid;
    const size_t K = std::max(sc->k, 1);
    std::vector<int64_t> off = to_host(offsets, static_cast<size_t>(g.n_tiles) + 1);
    const int64_t E = off[g.n_tiles];
    if (off[0] != 0 || E < 0) return fail(RXGS_ERR_INVALID, "tx_state_import: bad tile offsets");
    if (E && !indices) return fail(RXGS_ERR_INVALID, "tx_state_import: null argument");
    std::vector<int32_t> cul = to_host(culled, static_cast<size_t>(sc->k));
    int64_t vis = 0;
    for (int k = 0; k < sc->k; ++k) vis += cul[k] == 0;
    st->entries = E;
    st->visible = vis;
    RXGS_CUDA(st->rec.ensure(K * sizeof(GaussRec)));
    RXGS_CUDA(st->culled.ensure(K * sizeof(int)));
    RXGS_CUDA(st->geom.ensure(K * 12 * sizeof(double)));
    RXGS_CUDA(st->spans.ensure(K * sizeof(int4)));
    RXGS_CUDA(st->basis64.ensure(K * sc->L * 2 * sizeof(double)));
    RXGS_CUDA(st->basis32.ensure(K * sc->L * sizeof(float2)));
    RXGS_CUDA(st->gb32.ensure(K * sc->L * sc->channels * sizeof(float2)));
    RXGS_CUDA(st->tile_offsets.ensure((g.n_tiles + 1) * sizeof(int64_t)));
    RXGS_CUDA(st->list.ensure(std::max<int64_t>(E, 1) * sizeof(int)));
    RXGS_CUDA(st->keys.ensure(std::max<int64_t>(E, 1) * sizeof(uint64_t)));
    if (sc->k) {
        RXGS_CUDA(cudaMemcpy(st->culled.p, cul.data(), sc->k * sizeof(int), cudaMemcpyHostToDevice));
        RXGS_CUDA(cudaMemcpy(st->geom.p, geom, sc->k * 12 * sizeof(double), cudaMemcpyDefault));
        RXGS_CUDA(cudaMemcpy(st->spans.p, spans, sc->k * sizeof(int4), cudaMemcpyDefault));
        RXGS_CUDA(cudaMemcpy(st->basis64.p, basis, sc->k * sc->L * 2 * sizeof(double), cudaMemcpyDefault));
    }
    RXGS_CUDA(cudaMemcpy(st->tile_offsets.p, off.data(), off.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    if (E) RXGS_CUDA(cudaMemcpy(st->list.p, indices, E * sizeof(int), cudaMemcpyDefault));
    RXGS_CUDA(launch_rec_from_geom(sc->k, st->culled.as<int>(), st->geom.as<double>(), st->basis64.as<double>(),
                                   sc->L, st->rec.as<GaussRec>(), st->basis32.as<float2>(), s));
    const size_t cells = static_cast<size_t>(g.nt) * g.np;
    RXGS_CUDA(st->tw.ensure(std::max<size_t>(E, 1) * g.cell_blocks * kMaxCellsPerBlock * sizeof(float)));
    RXGS_CUDA(st->walk_len.ensure(static_cast<size_t>(g.n_tiles) * g.cell_blocks * sizeof(int)));
    RXGS_CUDA(st->cell_T.ensure(cells * sizeof(double)));
    RXGS_CUDA(st->cell_len.ensure(cells * sizeof(int)));
    RXGS_CUDA(launch_walk(*st, s));
    RX_TRY(compact_needed(ctx, *sc, *st, s));
    ctx->launches += 3;
    RXGS_CUDA(cudaStreamSynchronize(s));
    ctx_retain(ctx);
    st->sc = sc;
    sc->refs += 1;
    *out = guard.release();
    return RXGS_OK;
    API_END
}

}  // extern "C"
