// C-ABI of the training step (config 4): gradient of the Stage-II chain
// (trainer.cpp:429-449) summed over a batch of receivers of one
// transmitter, an exposed flat f64 gradient buffer for the data-parallel
// all-reduce (NCCL, done by the caller), and the fused Adam update
// (trainer.cpp:451-462 / diffengine.cpp:10-58).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <string>
#include <vector>

#include "rxgs_internal.cuh"

using namespace rxgs_b200;

struct rxgs_trainer_s {
    rxgs_ctx ctx = nullptr;
    rxgs_scene sc = nullptr;
    rxgs_cond c = nullptr;
    double feature_lr = 5e-3, rest_ratio = 0.2, cond_lr = 1e-3, lambda_ssim = 0.0, lambda_fft = 0.0;
    double b1 = 0.9, b2 = 0.999, eps = 1e-8;
    int64_t step = 0;
    int64_t n_base = 0, n_par = 0;
    DevBuf grad, m, v, field32, target, G, loss_part, loss, d_entry, d_s, u, part, red_part, row_part, gslice, rx,
        flag, loss_ws;
    int n_parts = 0, n_red = 592;  // k_global_red blocks (fixed-order partials)
};

namespace {

bool is_dev(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

#define TRY(expr)                          \
    do {                                   \
        const int rc__ = (expr);           \
        if (rc__ != RXGS_OK) return rc__;  \
    } while (0)

}  // namespace

extern "C" {

int rxgs_trainer_create(rxgs_ctx ctx, rxgs_scene sc, rxgs_cond c, const double hyper[8], rxgs_trainer* out) {
    if (!ctx || !sc || !c || !out) return fail(RXGS_ERR_INVALID, "rxgs_trainer_create: null argument");
    if (sc->modality != 2 || sc->channels != 1)
        return fail(RXGS_ERR_INVALID, "train: the B200 training step supports the spectrum modality with C == 1");
    if (c->hidden != 64 || c->C != 1 || c->l_max != sc->l_max)
        return fail(RXGS_ERR_INVALID, "train: conditioning must have hidden == 64, C == 1 and the scene's l_max");
    RXGS_CUDA(cudaSetDevice(ctx->device));
    auto* t = new rxgs_trainer_s;
    t->ctx = ctx;
    t->sc = sc;
    t->c = c;
    if (hyper) {
        t->feature_lr = hyper[0];
        t->rest_ratio = hyper[1];
        t->cond_lr = hyper[2];
        t->lambda_ssim = hyper[3];
        t->lambda_fft = hyper[4];
        t->b1 = hyper[5];
        t->b2 = hyper[6];
        t->eps = hyper[7];
    }
    if (t->lambda_ssim < 0.0 || t->lambda_fft < 0.0) {
        delete t;
        return fail(RXGS_ERR_INVALID, "train: loss weights must be non-negative");
    }
    t->n_base = static_cast<int64_t>(sc->k) * sc->L * sc->channels * 2;
    t->n_par = c->n_params;
    const size_t n = static_cast<size_t>(t->n_base + t->n_par);
    if (t->grad.ensure(n * 8) != cudaSuccess || t->m.ensure(n * 8) != cudaSuccess || t->v.ensure(n * 8) != cudaSuccess) {
        delete t;
        return fail(RXGS_ERR_CUDA, "train: allocation failed");
    }
    cudaMemset(t->grad.p, 0, n * 8);
    cudaMemset(t->m.p, 0, n * 8);
    cudaMemset(t->v.p, 0, n * 8);
    t->n_parts = cond_bwd_parts(ctx->sm_count);
    ctx_retain(ctx);
    *out = t;
    return RXGS_OK;
}

int rxgs_trainer_destroy(rxgs_trainer t) {
    if (!t) return RXGS_OK;
    rxgs_ctx ctx = t->ctx;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    delete t;
    ctx_release(ctx);
    return RXGS_OK;
}

int rxgs_train_grads(rxgs_trainer t, rxgs_txstate st, const double* rx, int n_rx, const float* targets,
                     double* losses, int accumulate) {
    if (!t || !st || !rx || !targets || n_rx < 1) return fail(RXGS_ERR_INVALID, "train: bad argument");
    rxgs_ctx ctx = t->ctx;
    rxgs_scene sc = t->sc;
    rxgs_cond c = t->c;
    if (st->k != sc->k) return fail(RXGS_ERR_INVALID, "train: tx state / scene mismatch");
    RXGS_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const DevGrid& g = st->grid;
    const int P = g.nt * g.np;
    const size_t n = static_cast<size_t>(t->n_base + t->n_par);
    // inputs
    const double* d_rx = rx;
    if (!is_dev(rx)) {
        RXGS_CUDA(t->rx.ensure(sizeof(double) * 3 * n_rx));
        RXGS_CUDA(cudaMemcpyAsync(t->rx.p, rx, sizeof(double) * 3 * n_rx, cudaMemcpyHostToDevice, s));
        d_rx = t->rx.as<double>();
    }
    const float* d_tg = targets;
    if (!is_dev(targets)) {
        RXGS_CUDA(t->target.ensure(sizeof(float) * static_cast<size_t>(n_rx) * P));
        RXGS_CUDA(cudaMemcpyAsync(t->target.p, targets, sizeof(float) * static_cast<size_t>(n_rx) * P,
                                  cudaMemcpyHostToDevice, s));
        d_tg = t->target.as<float>();
    }
    if (c->use_local()) {
        RXGS_CUDA(ctx->err_flag.ensure(16));
        const int big = INT_MAX;
        RXGS_CUDA(cudaMemcpyAsync(ctx->err_flag.p, &big, sizeof(int), cudaMemcpyHostToDevice, s));
        RXGS_CUDA(launch_check_coincide(*sc, d_rx, n_rx, ctx->err_flag.as<int>(), s));
        int err = INT_MAX;
        RXGS_CUDA(cudaMemcpyAsync(&err, ctx->err_flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        RXGS_CUDA(cudaStreamSynchronize(s));
        if (err != INT_MAX)
            return fail(RXGS_ERR_INVALID, "condition_forward: receiver coincides with gaussian " +
                                              std::to_string(err % std::max(sc->k, 1)));
    }
    if (!st->regrouped) TRY(train_regroup(ctx, *st, s));
    // ---- forward (coefficients may have changed since the state was built)
    RXGS_CUDA(launch_refresh_gb(*sc, *st, s));
    const size_t ag_n = static_cast<size_t>(n_rx) * sc->L * 4;
    RXGS_CUDA(ctx->ag.ensure(ag_n * sizeof(float)));
    RXGS_CUDA(launch_cond_global(*c, d_rx, n_rx, ctx->ag.as<float>(), s));
    RXGS_CUDA(ctx->signals.ensure(std::max<size_t>(static_cast<size_t>(sc->k) * n_rx, 1) * sizeof(float2)));
    // FP32 SIMT forward (conditioning + compositing): its field is ~10x closer
    // to the FP64 reference than the bf16x3 tensor-core path, which the
    // gradient parity of the SSIM term needs (measured: 2.6e-4 vs < 1e-4)
    const int saved = ctx->cond_kernel;
    ctx->cond_kernel = 1;
    const cudaError_t ef = launch_cond_signal(c, *sc, *st, d_rx, n_rx, ctx->ag.as<float>(),
                                              ctx->signals.as<float2>(), nullptr, s);
    ctx->cond_kernel = saved;
    RXGS_CUDA(ef);
    RXGS_CUDA(t->field32.ensure(sizeof(float) * 2 * static_cast<size_t>(n_rx) * P));
    CompositeOut co;
    co.field32 = t->field32.as<float>();
    RXGS_CUDA(launch_composite(*st, ctx->signals.as<float2>(), n_rx, co, s));
    // ---- loss + aggregate adjoint
    RXGS_CUDA(t->G.ensure(sizeof(float2) * static_cast<size_t>(n_rx) * P));
    RXGS_CUDA(t->loss_part.ensure(sizeof(double) * 16 * n_rx));
    RXGS_CUDA(t->loss.ensure(sizeof(double) * n_rx));
    const double l_weight = 1.0 - t->lambda_ssim - t->lambda_fft;
    if (t->lambda_ssim == 0.0 && t->lambda_fft == 0.0) {
        RXGS_CUDA(launch_loss_spectrum(n_rx, P, t->field32.as<float>(), d_tg, l_weight, t->G.as<float2>(),
                                       t->loss_part.as<double>(), t->loss.as<double>(), s));
    } else {  // composite_loss with SSIM and DFT terms (trainer.cpp:113-139)
        const DevGrid& gg = st->grid;
        if (t->lambda_ssim > 0.0 && (gg.nt < 11 || gg.np < 11))
            return fail(RXGS_ERR_INVALID, "ssim: image smaller than the window");
        RXGS_CUDA(t->loss_ws.ensure(loss_full_ws_bytes(n_rx, gg.nt, gg.np)));
        RXGS_CUDA(launch_loss_full(n_rx, gg.nt, gg.np, t->field32.as<float>(), d_tg, l_weight, t->lambda_ssim,
                                   t->lambda_fft, 1.0, t->G.as<float2>(), t->loss_ws.p, t->loss.as<double>(), s));
    }
    // ---- render adjoint -> d_s
    RXGS_CUDA(t->d_entry.ensure(sizeof(float2) * std::max<size_t>(static_cast<size_t>(st->entries) * n_rx, 1)));
    RXGS_CUDA(t->d_s.ensure(sizeof(float2) * std::max<size_t>(static_cast<size_t>(sc->k) * n_rx, 1)));
    RXGS_CUDA(t->u.ensure(sizeof(float2) * std::max<size_t>(static_cast<size_t>(sc->k) * n_rx, 1)));
    RXGS_CUDA(launch_render_adjoint(*st, t->G.as<float2>(), n_rx, t->d_entry.as<float2>(), t->d_s.as<float2>(), s));
    // ---- conditioning adjoint
    if (!accumulate) RXGS_CUDA(cudaMemsetAsync(t->grad.p, 0, n * 8, s));
    double* gbase = t->grad.as<double>();
    double* gpar = gbase + t->n_base;
    const int nl = local_grad_n();
    RXGS_CUDA(t->part.ensure(sizeof(float) * static_cast<size_t>(t->n_parts) * nl));
    RXGS_CUDA(launch_cond_bwd(*c, *sc, *st, d_rx, n_rx, ctx->ag.as<float>(), t->d_s.as<float2>(), t->u.as<float2>(),
                              t->part.as<float>(), t->n_parts, s));
    if (c->use_local()) RXGS_CUDA(launch_reduce_parts(t->n_parts, nl, t->part.as<float>(), gpar + c->o_lw1, s));
    RXGS_CUDA(launch_dbase(c, *sc, *st, n_rx, ctx->ag.as<float>(), t->u.as<float2>(), gbase, s));
    if (c->use_global()) {
        const int npair = n_rx * c->L;
        const size_t n_gpar = static_cast<size_t>(c->F * 3) + (c->o_emb - c->o_gw1) + static_cast<size_t>(c->L) * c->dc;
        RXGS_CUDA(t->red_part.ensure(sizeof(double) * 4 * static_cast<size_t>(t->n_red) * npair));
        RXGS_CUDA(t->row_part.ensure(sizeof(double) * static_cast<size_t>(npair) * n_gpar));
        RXGS_CUDA(t->gslice.ensure(sizeof(double) * n_gpar));
        RXGS_CUDA(launch_global_bwd(*c, *sc, *st, n_rx, d_rx, t->u.as<float2>(), t->red_part.as<double>(), t->n_red,
                                    t->row_part.as<double>(), t->gslice.as<double>(), gpar, s));
    }
    ctx->launches += 12;
    // ---- losses out + non-finite check (trainer.cpp:436-438)
    std::vector<double> lh(n_rx);
    RXGS_CUDA(cudaMemcpyAsync(lh.data(), t->loss.p, sizeof(double) * n_rx, cudaMemcpyDeviceToHost, s));
    RXGS_CUDA(cudaStreamSynchronize(s));
    for (int j = 0; j < n_rx; ++j)
        if (!std::isfinite(lh[j]))
            return fail(RXGS_ERR_RUNTIME, "train: non-finite loss at sample " + std::to_string(j));
    if (losses) {
        if (is_dev(losses))
            RXGS_CUDA(cudaMemcpy(losses, t->loss.p, sizeof(double) * n_rx, cudaMemcpyDeviceToDevice));
        else
            std::copy(lh.begin(), lh.end(), losses);
    }
    return RXGS_OK;
}

int rxgs_train_grad_buffer(rxgs_trainer t, double** dev_ptr, int64_t* n, int64_t* n_base) {
    if (!t) return fail(RXGS_ERR_INVALID, "null trainer");
    if (dev_ptr) *dev_ptr = t->grad.as<double>();
    if (n) *n = t->n_base + t->n_par;
    if (n_base) *n_base = t->n_base;
    return RXGS_OK;
}

int rxgs_train_get_grads(rxgs_trainer t, double* d_base, double* d_params) {
    if (!t) return fail(RXGS_ERR_INVALID, "null trainer");
    RXGS_CUDA(cudaSetDevice(t->ctx->device));
    RXGS_CUDA(cudaStreamSynchronize(t->ctx->stream));
    if (d_base) RXGS_CUDA(cudaMemcpy(d_base, t->grad.p, sizeof(double) * t->n_base, cudaMemcpyDefault));
    if (d_params)
        RXGS_CUDA(cudaMemcpy(d_params, t->grad.as<double>() + t->n_base, sizeof(double) * t->n_par, cudaMemcpyDefault));
    return RXGS_OK;
}

// Optimizer::step for "features" (lr_scale) and every conditioning group
// (diffengine.cpp:50-58, trainer.cpp:451-462): non-finite check per group,
// then Adam; the scene / conditioning device copies are updated in place.
int rxgs_train_apply(rxgs_trainer t) {
    if (!t) return fail(RXGS_ERR_INVALID, "null trainer");
    rxgs_ctx ctx = t->ctx;
    RXGS_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    RXGS_CUDA(t->flag.ensure(16));
    const int big = INT_MAX;
    int bad[2] = {INT_MAX, INT_MAX};
    RXGS_CUDA(cudaMemcpyAsync(t->flag.p, &big, sizeof(int), cudaMemcpyHostToDevice, s));
    RXGS_CUDA(cudaMemcpyAsync(t->flag.as<int>() + 1, &big, sizeof(int), cudaMemcpyHostToDevice, s));
    RXGS_CUDA(launch_check_finite64(t->n_base, t->grad.as<double>(), t->flag.as<int>(), s));
    RXGS_CUDA(launch_check_finite64(t->n_par, t->grad.as<double>() + t->n_base, t->flag.as<int>() + 1, s));
    RXGS_CUDA(cudaMemcpyAsync(bad, t->flag.p, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
    RXGS_CUDA(cudaStreamSynchronize(s));
    if (bad[0] != INT_MAX) return fail(RXGS_ERR_RUNTIME, "optimizer: non-finite gradient in group 'features'");
    if (bad[1] != INT_MAX) return fail(RXGS_ERR_RUNTIME, "optimizer: non-finite gradient in group 'cond'");
    t->step += 1;
    rxgs_scene sc = t->sc;
    rxgs_cond c = t->c;
    RXGS_CUDA(launch_adam(t->n_base, sc->d_coeffs64.as<double>(), t->grad.as<double>(), t->m.as<double>(),
                          t->v.as<double>(), t->feature_lr, t->step, t->b1, t->b2, t->eps, sc->L, sc->channels * 2,
                          t->rest_ratio, nullptr, s));
    RXGS_CUDA(launch_adam(t->n_par, c->d_params64.as<double>(), t->grad.as<double>() + t->n_base,
                          t->m.as<double>() + t->n_base, t->v.as<double>() + t->n_base, t->cond_lr, t->step, t->b1,
                          t->b2, t->eps, 0, 1, 1.0, c->d_params32.as<float>(), s));
    ctx->launches += 4;
    sc->host_stale = true;
    c->host_stale = true;
    return RXGS_OK;
}

int64_t rxgs_train_step_count(rxgs_trainer t) { return t ? t->step : -1; }

int rxgs_scene_get_coeffs(rxgs_scene sc, double* out) {
    if (!sc || !out) return fail(RXGS_ERR_INVALID, "null argument");
    RXGS_CUDA(cudaSetDevice(sc->ctx->device));
    RXGS_CUDA(cudaStreamSynchronize(sc->ctx->stream));
    const size_t n = static_cast<size_t>(sc->k) * sc->L * sc->channels * 2;
    if (n) RXGS_CUDA(cudaMemcpy(out, sc->d_coeffs64.p, n * sizeof(double), cudaMemcpyDefault));
    return RXGS_OK;
}

int rxgs_cond_get_params(rxgs_cond c, double* out) {
    if (!c || !out) return fail(RXGS_ERR_INVALID, "null argument");
    RXGS_CUDA(cudaSetDevice(c->ctx->device));
    RXGS_CUDA(cudaStreamSynchronize(c->ctx->stream));
    RXGS_CUDA(cudaMemcpy(out, c->d_params64.p, c->n_params * sizeof(double), cudaMemcpyDefault));
    return RXGS_OK;
}

}  // extern "C"
