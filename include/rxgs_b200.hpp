// include/rxgs_b200.hpp -- header-only C++ shim: the reference's C++ API for
// the render path (rxgs::raster / rxgs::cond / rxgs::train, same struct
// fields, same exception types and messages) implemented on top of the
// C-ABI in rxgs_b200.h, i.e. on the B200 kernels.
//
// Reference headers replaced (paths under /root/reference/proj/include/rxgs):
//   scene.hpp:19-48        GaussianScene
//   sphraster.hpp:15-133   SphericalGrid, ProjectedGaussian, TxState,
//                          build_tx_state, bin_and_sort, RenderedField,
//                          render_field (x2), Measurement, aggregate_modality
//   sphraster.hpp:46,60,82 project_gaussian, TxState::hash, blend_ray
//   conditioning.hpp:13-123 MlpLayer, Mlp, OccupancyGrid, ConditioningConfig,
//                          ConditioningState, init_conditioning,
//                          probe_segment, fourier_encode, build_occupancy,
//                          condition_forward, condition_batch
//   radiance.hpp:66        fle::eval_basis (+ normalization, eval_radiance)
// For a link-level drop-in that keeps the reference's own headers, see
// paper_2605_24290_b200/refapi (librxgs_refapi.so).
//   trainer.hpp:42-50      Model, predict
// Usage: include this header instead of the reference headers and link
// librxgs_b200.so.  Define RXGS_B200_AS_RXGS to expose everything as
// namespace rxgs (source-compatible with reference callers).
#pragma once

#include <array>
#include <cmath>
#include <complex>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "rxgs_b200.h"

namespace rxgs_b200 {
namespace api {

using cplx = std::complex<double>;
inline constexpr double kPi = 3.14159265358979323846;
inline constexpr double kTwoPi = 2.0 * kPi;

struct Vec3 {
    double x = 0.0, y = 0.0, z = 0.0;
};

enum class Modality { Rssi, Csi, Spectrum };  // channelsim.hpp:79

namespace detail {
inline void check(int rc) {
    if (rc == RXGS_OK) return;
    const std::string msg = rxgs_last_error();
    if (rc == RXGS_ERR_INVALID) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}
struct Ctx {
    rxgs_ctx h = nullptr;
    Ctx() { check(rxgs_ctx_create(0, &h)); }
    ~Ctx() { rxgs_ctx_destroy(h); }
};
inline rxgs_ctx ctx() {
    thread_local Ctx c;
    return c.h;
}
struct SceneHandle {
    rxgs_scene h = nullptr;
    ~SceneHandle() { rxgs_scene_destroy(h); }
};
struct TxHandle {
    rxgs_txstate h = nullptr;
    std::shared_ptr<SceneHandle> scene;
    ~TxHandle() { rxgs_tx_state_destroy(h); }
};
}  // namespace detail

inline int component_count(int l_max) { return (l_max + 1) * (l_max + 1); }

// GaussianScene (scene.hpp:19-48)
struct GaussianScene {
    int l_max = 0;
    int channels = 1;
    Modality modality = Modality::Rssi;
    std::vector<double> positions, log_scales, quaternions, tau_logits, fle_coeffs;
    int count() const { return static_cast<int>(tau_logits.size()); }
    int n_components() const { return component_count(l_max); }
    std::size_t coeff_stride() const { return static_cast<std::size_t>(n_components()) * channels * 2; }
    Vec3 position(int k) const { return {positions[3 * k], positions[3 * k + 1], positions[3 * k + 2]}; }
};

namespace detail {
inline std::shared_ptr<SceneHandle> upload(const GaussianScene& s) {
    auto h = std::make_shared<SceneHandle>();
    check(rxgs_scene_create(ctx(), s.count(), s.l_max, s.channels, static_cast<int>(s.modality),
                            s.positions.data(), s.log_scales.data(), s.quaternions.data(),
                            s.tau_logits.data(), s.fle_coeffs.data(), &h->h));
    return h;
}
}  // namespace detail

// ---- Stage-I densification (scene.hpp:69-99) on the device
struct DensifyState {
    std::vector<double> grad_accum;  // sum of ||dL/dp_k||_2 per Gaussian
    std::vector<int> accum_count;
    double scene_extent = 0.0;
    void resize(int k) {
        grad_accum.assign(static_cast<std::size_t>(k), 0.0);
        accum_count.assign(static_cast<std::size_t>(k), 0);
    }
    void accumulate(const std::vector<double>& d_positions) {  // scene.cpp:141-151
        const std::size_t k = grad_accum.size();
        if (d_positions.size() != 3 * k)
            throw std::invalid_argument("DensifyState::accumulate: gradient size mismatch");
        for (std::size_t i = 0; i < k; ++i) {
            const double gx = d_positions[3 * i], gy = d_positions[3 * i + 1], gz = d_positions[3 * i + 2];
            grad_accum[i] += std::sqrt(gx * gx + gy * gy + gz * gz);
            accum_count[i] += 1;
        }
    }
};
struct DensifyThresholds {
    double grad_threshold = 2e-4;
    double size_frac = 0.01;
    double prune_extent_frac = 0.1;
    double split_scale_factor = 0.8;
};
struct DensifyReport {
    int cloned = 0, split = 0, pruned = 0;
    std::vector<int> source_row;
};

inline DensifyReport densify_and_prune(GaussianScene& scene, DensifyState& state, const DensifyThresholds& t,
                                       uint64_t seed, uint64_t pass_index) {
    const int k = scene.count();
    if (static_cast<int>(state.grad_accum.size()) != k || static_cast<int>(state.accum_count.size()) != k)
        throw std::invalid_argument("densify_and_prune: state size mismatch");
    auto h = detail::upload(scene);
    const double thr[4] = {t.grad_threshold, t.size_frac, t.prune_extent_frac, t.split_scale_factor};
    int32_t rep[3] = {0, 0, 0}, nk = 0;
    std::vector<int32_t> src(2 * static_cast<std::size_t>(k) + 1);
    detail::check(rxgs_densify_and_prune(detail::ctx(), h->h, state.grad_accum.data(), state.accum_count.data(),
                                         state.scene_extent, thr, seed, pass_index, rep, src.data(), &nk));
    scene.positions.resize(3 * static_cast<std::size_t>(nk));
    scene.log_scales.resize(3 * static_cast<std::size_t>(nk));
    scene.quaternions.resize(4 * static_cast<std::size_t>(nk));
    scene.tau_logits.resize(static_cast<std::size_t>(nk));
    scene.fle_coeffs.resize(static_cast<std::size_t>(nk) * scene.coeff_stride());
    detail::check(rxgs_scene_get_arrays(h->h, scene.positions.data(), scene.log_scales.data(), scene.quaternions.data(),
                                        scene.tau_logits.data(), scene.fle_coeffs.data()));
    DensifyReport r;
    r.cloned = rep[0];
    r.split = rep[1];
    r.pruned = rep[2];
    r.source_row.assign(src.begin(), src.begin() + nk);
    state.resize(nk);
    return r;
}

inline void reset_transmittance(GaussianScene& scene) {  // scene.cpp:276-279
    auto h = detail::upload(scene);
    detail::check(rxgs_reset_transmittance(h->h));
    detail::check(rxgs_scene_get_arrays(h->h, nullptr, nullptr, nullptr, scene.tau_logits.data(), nullptr));
}

// ---- evaluation metrics (metrics.hpp:10-34) on the device
namespace met {
inline constexpr double kDbSentinel = 300.0;
struct SsimOptions {
    int window = 11;
    double sigma = 1.5;
    double dynamic_range = 1.0;
};
namespace detail_m {
inline std::array<double, 4> all(const std::vector<double>& pred, const std::vector<double>& gt, int h, int w,
                                 double max_val, const double* opts, const char* who) {
    if (pred.size() != gt.size() || pred.empty())
        throw std::invalid_argument(std::string(who) + ": need equal non-empty inputs");
    std::array<double, 4> out{};
    detail::check(rxgs_image_metrics(detail::ctx(), pred.data(), 0, gt.data(), 1, h, w, max_val, opts, out.data()));
    return out;
}
}  // namespace detail_m
inline double mae(const std::vector<double>& pred, const std::vector<double>& gt) {
    const double o[3] = {0, 1.5, 1.0};
    return detail_m::all(pred, gt, 1, static_cast<int>(pred.size()), 1.0, o, "mae")[0];
}
inline double mse(const std::vector<double>& pred, const std::vector<double>& gt) {
    const double o[3] = {0, 1.5, 1.0};
    return detail_m::all(pred, gt, 1, static_cast<int>(pred.size()), 1.0, o, "mse")[1];
}
inline double psnr(const std::vector<double>& pred, const std::vector<double>& gt, double max_val) {
    const double o[3] = {0, 1.5, 1.0};
    return detail_m::all(pred, gt, 1, static_cast<int>(pred.size()), max_val, o, "mse")[2];
}
// the value only (the reference's optional d_pred output is the training
// loss's business here: rxgs_train_grads with lambda_ssim > 0)
inline double ssim(const std::vector<double>& pred, const std::vector<double>& gt, int h, int w,
                   const SsimOptions& options = {}) {
    if (h < options.window || w < options.window) throw std::invalid_argument("ssim: image smaller than the window");
    if (pred.size() != static_cast<std::size_t>(h) * w || gt.size() != pred.size())
        throw std::invalid_argument("ssim: shape mismatch");
    const double o[3] = {static_cast<double>(options.window), options.sigma, options.dynamic_range};
    return detail_m::all(pred, gt, h, w, 1.0, o, "ssim")[3];
}
}  // namespace met

namespace fle {  // radiance.hpp:36-70, evaluated on the device in FP64

struct BasisValues {
    int l_max = 0;
    std::vector<cplx> b;
    const cplx& at(int comp) const { return b[static_cast<std::size_t>(comp)]; }
};

// eval_basis (radiance.hpp:66, radiance.cpp:79-92)
inline BasisValues eval_basis(double theta, double phi, int l_max) {
    const int L = component_count(l_max);
    std::vector<double> o(2 * static_cast<std::size_t>(L));
    detail::check(rxgs_fle_eval(detail::ctx(), 0, l_max, 1, &theta, &phi, nullptr, o.data()));
    BasisValues r;
    r.l_max = l_max;
    for (int i = 0; i < L; ++i) r.b.push_back(cplx{o[2 * i], o[2 * i + 1]});
    return r;
}

// normalization (radiance.cpp:9-14)
inline double normalization(int l, int m) {
    const double a = l, b = m;
    double o = 0.0;
    detail::check(rxgs_fle_eval(detail::ctx(), 4, 0, 1, &a, &b, nullptr, &o));
    return o;
}

// eval_radiance (radiance.cpp:116-125): coeffs L complex
inline cplx eval_radiance(const double* coeffs, double theta, double phi, int l_max) {
    double o[2];
    detail::check(rxgs_fle_eval(detail::ctx(), 5, l_max, 1, &theta, &phi, coeffs, o));
    return cplx{o[0], o[1]};
}

}  // namespace fle

namespace raster {

inline constexpr double kWeightClamp = 0.999;
inline constexpr double kEarlyExitT = 1e-4;

struct SphericalGrid {  // sphraster.hpp:15-32
    int n_theta = 1, n_phi = 1, tile_size = 8;
    double radius = 1.0, theta_min = 0.0, theta_max = kPi;
    double dtheta() const { return (theta_max - theta_min) / n_theta; }
    double dphi() const { return kTwoPi / n_phi; }
    double theta_at(int i) const { return theta_min + (i + 0.5) * dtheta(); }
    double phi_at(int j) const { return (j + 0.5) * dphi(); }
    int tiles_theta() const { return (n_theta + tile_size - 1) / tile_size; }
    int tiles_phi() const { return (n_phi + tile_size - 1) / tile_size; }
    std::size_t cells() const { return static_cast<std::size_t>(n_theta) * n_phi; }
    rxgs_grid c() const { return {n_theta, n_phi, tile_size, 0, radius, theta_min, theta_max}; }
};

struct Mat2 {
    double a = 0.0, b = 0.0, c = 0.0, d = 0.0;
};

struct ProjectedGaussian {  // sphraster.hpp:34-44
    bool culled = true;
    double theta = 0.0, phi = 0.0, depth = 0.0;
    Mat2 angular_cov, angular_prec;
    double weight_scale = 0.0;
    int t0 = 0, t1 = -1, p0 = 0, p1 = -1;
};

struct TxState {  // sphraster.hpp:52-61 (materialised from the device)
    SphericalGrid grid;
    int k = 0, l_max = 0;
    std::vector<ProjectedGaussian> proj;
    std::vector<std::vector<int>> tile_lists;
    std::vector<cplx> basis;
    std::shared_ptr<detail::TxHandle> device;  // B200 state (lists, blend weights)
    // TxState::hash (sphraster.hpp:60, sphraster.cpp:121-148): FNV-1a over the
    // same fields in the same order and byte widths as the reference
    uint64_t hash() const {
        uint64_t h = 0xcbf29ce484222325ull;
        auto bytes = [&h](const void* d, std::size_t n) {
            const auto* p = static_cast<const unsigned char*>(d);
            for (std::size_t i = 0; i < n; ++i) {
                h ^= p[i];
                h *= 0x100000001b3ull;
            }
        };
        auto val = [&bytes](const auto& v) { bytes(&v, sizeof(v)); };
        val(grid.n_theta);
        val(grid.n_phi);
        val(grid.tile_size);
        val(grid.radius);
        val(k);
        val(l_max);
        for (const auto& pg : proj) {
            val(pg.culled);
            if (pg.culled) continue;
            val(pg.theta);
            val(pg.phi);
            val(pg.depth);
            val(pg.angular_cov);
            val(pg.weight_scale);
            val(pg.t0);
            val(pg.t1);
            val(pg.p0);
            val(pg.p1);
        }
        for (const auto& list : tile_lists) {
            val(list.size());
            for (const int idx : list) val(idx);
        }
        bytes(basis.data(), basis.size() * sizeof(cplx));
        return h;
    }
};

// project_gaussian (sphraster.hpp:46, sphraster.cpp:22-83) on the device
// (FP64, the k_tx_prep arithmetic).  cov3: row-major 3x3.
inline ProjectedGaussian project_gaussian(const Vec3& position, const std::array<double, 9>& cov3, double tau,
                                          const Vec3& tx, const SphericalGrid& grid) {
    const double p[3] = {position.x, position.y, position.z}, t[3] = {tx.x, tx.y, tx.z};
    double g[12];
    int32_t culled = 1, sp[4];
    const rxgs_grid gc = grid.c();
    detail::check(rxgs_project_gaussians(detail::ctx(), 1, p, cov3.data(), &tau, t, &gc, g, &culled, sp));
    ProjectedGaussian o;
    o.culled = culled != 0;
    o.theta = g[0];
    o.phi = g[1];
    o.depth = g[2];
    o.angular_cov = {g[3], g[4], g[5], g[6]};
    o.angular_prec = {g[7], g[8], g[9], g[10]};
    o.weight_scale = g[11];
    o.t0 = sp[0];
    o.t1 = sp[1];
    o.p0 = sp[2];
    o.p1 = sp[3];
    return o;
}

struct BlendResult {  // sphraster.hpp:77-80
    cplx c{0.0, 0.0};
    double transmittance = 1.0;
};

// blend_ray (sphraster.hpp:82, sphraster.cpp:174-185) on the device
inline BlendResult blend_ray(const std::vector<double>& weights, const std::vector<cplx>& signals) {
    if (weights.size() != signals.size()) throw std::invalid_argument("blend_ray: weights/signals size mismatch");
    std::vector<double> sg(2 * signals.size());
    for (std::size_t i = 0; i < signals.size(); ++i) {
        sg[2 * i] = signals[i].real();
        sg[2 * i + 1] = signals[i].imag();
    }
    double o[3];
    detail::check(rxgs_blend_ray(detail::ctx(), static_cast<int>(weights.size()), weights.data(), sg.data(), o));
    BlendResult r;
    r.c = cplx{o[0], o[1]};
    r.transmittance = o[2];
    return r;
}

inline TxState build_tx_state(const GaussianScene& scene, const Vec3& tx, const SphericalGrid& grid) {
    auto th = std::make_shared<detail::TxHandle>();
    th->scene = detail::upload(scene);
    const double t[3] = {tx.x, tx.y, tx.z};
    const rxgs_grid g = grid.c();
    detail::check(rxgs_tx_state_build(detail::ctx(), th->scene->h, t, &g, &th->h));
    TxState st;
    st.grid = grid;
    st.k = scene.count();
    st.l_max = scene.l_max;
    st.device = th;
    const int K = st.k, L = scene.n_components();
    const int64_t E = rxgs_tx_state_entries(th->h);
    std::vector<int32_t> culled(K), spans(4 * static_cast<std::size_t>(K)), idx(E > 0 ? E : 1);
    std::vector<double> geom(12 * static_cast<std::size_t>(K)), basis(2 * static_cast<std::size_t>(K) * L);
    std::vector<int64_t> offs(static_cast<std::size_t>(grid.tiles_theta()) * grid.tiles_phi() + 1);
    detail::check(rxgs_tx_state_get(th->h, culled.data(), geom.data(), spans.data(), basis.data(), offs.data(),
                                    idx.data()));
    st.proj.resize(K);
    for (int k = 0; k < K; ++k) {
        ProjectedGaussian& p = st.proj[k];
        const double* g12 = geom.data() + 12 * static_cast<std::size_t>(k);
        p.culled = culled[k] != 0;
        p.theta = g12[0]; p.phi = g12[1]; p.depth = g12[2];
        p.angular_cov = {g12[3], g12[4], g12[5], g12[6]};
        p.angular_prec = {g12[7], g12[8], g12[9], g12[10]};
        p.weight_scale = g12[11];
        p.t0 = spans[4 * k]; p.t1 = spans[4 * k + 1]; p.p0 = spans[4 * k + 2]; p.p1 = spans[4 * k + 3];
    }
    st.basis.resize(static_cast<std::size_t>(K) * L);
    for (std::size_t i = 0; i < st.basis.size(); ++i) st.basis[i] = {basis[2 * i], basis[2 * i + 1]};
    st.tile_lists.resize(offs.size() - 1);
    for (std::size_t t = 0; t + 1 < offs.size(); ++t)
        st.tile_lists[t].assign(idx.begin() + offs[t], idx.begin() + offs[t + 1]);
    return st;
}

inline std::vector<std::vector<int>> bin_and_sort(const std::vector<ProjectedGaussian>& projected,
                                                  const SphericalGrid& grid) {
    const int K = static_cast<int>(projected.size());
    std::vector<int32_t> culled(K), spans(4 * static_cast<std::size_t>(K));
    std::vector<double> depth(K);
    for (int k = 0; k < K; ++k) {
        const auto& p = projected[k];
        culled[k] = p.culled ? 1 : 0;
        depth[k] = p.depth;
        spans[4 * k] = p.t0; spans[4 * k + 1] = p.t1; spans[4 * k + 2] = p.p0; spans[4 * k + 3] = p.p1;
    }
    const rxgs_grid g = grid.c();
    std::vector<int64_t> offs(static_cast<std::size_t>(grid.tiles_theta()) * grid.tiles_phi() + 1);
    int64_t n = 0;
    detail::check(rxgs_bin_and_sort(detail::ctx(), K, culled.data(), depth.data(), spans.data(), &g, offs.data(),
                                    nullptr, 0, &n));
    std::vector<int32_t> idx(n > 0 ? n : 1);
    detail::check(rxgs_bin_and_sort(detail::ctx(), K, culled.data(), depth.data(), spans.data(), &g, offs.data(),
                                    idx.data(), n, &n));
    std::vector<std::vector<int>> lists(offs.size() - 1);
    for (std::size_t t = 0; t + 1 < offs.size(); ++t) lists[t].assign(idx.begin() + offs[t], idx.begin() + offs[t + 1]);
    return lists;
}

struct RenderedField {  // sphraster.hpp:75-86
    int n_rx = 0, channels = 1, h = 0, w = 0;
    std::vector<double> values;
    std::vector<double> transmittance;
    std::size_t plane() const { return static_cast<std::size_t>(h) * w; }
    double value(int j, int c, int reim, std::size_t cell) const {
        return values[((static_cast<std::size_t>(j) * channels + c) * 2 + reim) * plane() + cell];
    }
};

inline RenderedField render_field(const TxState& st, const GaussianScene& scene, const std::vector<double>& coeffs,
                                  int n_rx, int /*threads*/ = 1) {
    if (n_rx < 1) throw std::invalid_argument("render_field: n_rx must be >= 1");
    if (coeffs.size() != static_cast<std::size_t>(n_rx) * scene.count() * scene.coeff_stride())
        throw std::invalid_argument("render_field: coefficient tensor has wrong size");
    RenderedField f;
    f.n_rx = n_rx;
    f.channels = scene.channels;
    f.h = st.grid.n_theta;
    f.w = st.grid.n_phi;
    f.values.assign(static_cast<std::size_t>(n_rx) * f.channels * 2 * f.plane(), 0.0);
    f.transmittance.assign(static_cast<std::size_t>(n_rx) * f.plane(), 1.0);
    detail::check(rxgs_render_field(detail::ctx(), st.device->h, st.device->scene->h,
                                    coeffs.empty() ? nullptr : coeffs.data(), n_rx, f.values.data(),
                                    f.transmittance.data()));
    return f;
}

inline RenderedField render_field(const GaussianScene& scene, const Vec3& tx, const SphericalGrid& grid,
                                  const std::vector<double>& coeffs, int n_rx, int threads = 1) {
    return render_field(build_tx_state(scene, tx, grid), scene, coeffs, n_rx, threads);
}

struct Measurement {  // sphraster.hpp:100-105
    Modality modality = Modality::Rssi;
    double scalar = 0.0;
    std::vector<cplx> csi;
    std::vector<double> image;
};

inline std::vector<Measurement> aggregate_modality(const RenderedField& field, Modality modality,
                                                   const SphericalGrid& grid) {
    const rxgs_grid g = grid.c();
    const int m = static_cast<int>(modality);
    const std::size_t n = m == 0 ? field.n_rx
                                 : (m == 1 ? static_cast<std::size_t>(field.n_rx) * field.channels * 2
                                           : static_cast<std::size_t>(field.n_rx) * field.plane());
    std::vector<double> out(n > 0 ? n : 1);
    detail::check(rxgs_aggregate_modality(detail::ctx(), &g, m, field.n_rx, field.channels, field.values.data(),
                                          out.data()));
    std::vector<Measurement> ms(field.n_rx);
    for (int j = 0; j < field.n_rx; ++j) {
        Measurement& r = ms[j];
        r.modality = modality;
        if (m == 0) {
            r.scalar = out[j];
        } else if (m == 1) {
            for (int c = 0; c < field.channels; ++c)
                r.csi.push_back({out[(static_cast<std::size_t>(j) * field.channels + c) * 2],
                                 out[(static_cast<std::size_t>(j) * field.channels + c) * 2 + 1]});
        } else {
            r.image.assign(out.begin() + static_cast<std::ptrdiff_t>(j * field.plane()),
                           out.begin() + static_cast<std::ptrdiff_t>((j + 1) * field.plane()));
        }
    }
    return ms;
}

// sphraster.hpp:110-113: upstream Measurements (forward shapes) -> d field values
inline std::vector<double> aggregate_modality_backward(const RenderedField& field, Modality modality,
                                                       const SphericalGrid& grid,
                                                       const std::vector<Measurement>& upstream) {
    if (upstream.size() != static_cast<std::size_t>(field.n_rx))
        throw std::invalid_argument("aggregate_modality_backward: upstream count mismatch");
    const rxgs_grid g = grid.c();
    const int m = static_cast<int>(modality);
    std::vector<double> up;
    for (const Measurement& u : upstream) {
        if (m == 0) {
            up.push_back(u.scalar);
        } else if (m == 1) {
            for (int c = 0; c < field.channels; ++c) {
                const cplx v = c < static_cast<int>(u.csi.size()) ? u.csi[c] : cplx{0, 0};
                up.push_back(v.real());
                up.push_back(v.imag());
            }
        } else {
            if (u.image.size() != field.plane())
                throw std::invalid_argument("aggregate_modality_backward: image size mismatch");
            up.insert(up.end(), u.image.begin(), u.image.end());
        }
    }
    std::vector<double> dv(field.values.size());
    detail::check(rxgs_aggregate_modality_backward(detail::ctx(), &g, m, field.n_rx, field.channels,
                                                   field.values.data(), up.empty() ? nullptr : up.data(),
                                                   dv.data()));
    return dv;
}

struct GradientBundle {  // sphraster.hpp:118-128
    std::vector<double> d_positions, d_log_scales, d_quaternions, d_tau_logits, d_coeffs;
    void resize(int k, int n_rx, std::size_t coeff_stride) {
        d_positions.assign(3 * static_cast<std::size_t>(k), 0.0);
        d_log_scales.assign(3 * static_cast<std::size_t>(k), 0.0);
        d_quaternions.assign(4 * static_cast<std::size_t>(k), 0.0);
        d_tau_logits.assign(k, 0.0);
        d_coeffs.assign(static_cast<std::size_t>(n_rx) * k * coeff_stride, 0.0);
    }
    void add(const GradientBundle& o) {
        auto acc = [](std::vector<double>& a, const std::vector<double>& b) {
            for (std::size_t i = 0; i < a.size() && i < b.size(); ++i) a[i] += b[i];
        };
        acc(d_positions, o.d_positions);
        acc(d_log_scales, o.d_log_scales);
        acc(d_quaternions, o.d_quaternions);
        acc(d_tau_logits, o.d_tau_logits);
        acc(d_coeffs, o.d_coeffs);
    }
};

// sphraster.hpp:130-133: exact adjoint of render_field (FP64, on the B200)
inline GradientBundle backward_render(const TxState& st, const GaussianScene& scene, const std::vector<double>& coeffs,
                                      int n_rx, const std::vector<double>& d_values, int /*threads*/ = 1) {
    GradientBundle b;
    b.resize(scene.count(), n_rx, scene.coeff_stride());
    auto sh = detail::upload(scene);
    detail::check(rxgs_backward_render(detail::ctx(), st.device->h, sh->h, coeffs.empty() ? nullptr : coeffs.data(),
                                       n_rx, d_values.data(), b.d_positions.data(), b.d_log_scales.data(),
                                       b.d_quaternions.data(), b.d_tau_logits.data(), b.d_coeffs.data()));
    return b;
}

}  // namespace raster

namespace cond {

struct MlpLayer {  // conditioning.hpp:13-19
    int in = 0, out = 0;
    std::vector<double> w, b;
};
struct Mlp {
    MlpLayer l1, l2, l3;
};
struct Aabb {
    Vec3 lo, hi;
};
struct OccupancyGrid {  // conditioning.hpp:29-37
    int resolution = 0;
    Aabb bounds;
    std::vector<double> densities;
    bool empty() const { return densities.empty(); }
};
enum class ConditioningMode { Full, GlobalOnly, LocalOnly, AdditiveOnly, NoOcclusion };
struct ConditioningConfig {  // conditioning.hpp:58-66
    int fourier_bands = 6, hidden = 64, embed_dim = 16, probe_samples = 16, occupancy_resolution = 32;
    bool nearest_lookup = false;
    ConditioningMode mode = ConditioningMode::Full;
};
struct ConditioningState {  // conditioning.hpp:72-92
    ConditioningConfig config;
    int l_max = 0, channels = 1;
    std::vector<double> fourier_freqs;
    Mlp global_mlp;
    std::vector<double> component_embed;
    Mlp local_mlp;
    OccupancyGrid occupancy;
    mutable std::int64_t global_calls = 0;
    mutable std::int64_t local_calls = 0;
};

namespace detail_c {
struct CondHandle {
    rxgs_cond h = nullptr;
    ~CondHandle() { rxgs_cond_destroy(h); }
};
inline std::unique_ptr<CondHandle> upload(const ConditioningState& s) {
    const ConditioningConfig& c = s.config;
    const int32_t cfg[9] = {c.fourier_bands, c.hidden, c.embed_dim, c.probe_samples,
                            s.occupancy.empty() ? c.occupancy_resolution : s.occupancy.resolution,
                            c.nearest_lookup ? 1 : 0, static_cast<int32_t>(c.mode), s.l_max, s.channels};
    std::vector<double> p;
    auto put = [&p](const std::vector<double>& v) { p.insert(p.end(), v.begin(), v.end()); };
    put(s.fourier_freqs);
    for (const MlpLayer* l : {&s.global_mlp.l1, &s.global_mlp.l2, &s.global_mlp.l3}) {
        put(l->w);
        put(l->b);
    }
    put(s.component_embed);
    for (const MlpLayer* l : {&s.local_mlp.l1, &s.local_mlp.l2, &s.local_mlp.l3}) {
        put(l->w);
        put(l->b);
    }
    auto h = std::make_unique<CondHandle>();
    const double lo[3] = {s.occupancy.bounds.lo.x, s.occupancy.bounds.lo.y, s.occupancy.bounds.lo.z};
    const double hi[3] = {s.occupancy.bounds.hi.x, s.occupancy.bounds.hi.y, s.occupancy.bounds.hi.z};
    api::detail::check(rxgs_cond_create(api::detail::ctx(), cfg, p.data(),
                                        s.occupancy.empty() ? nullptr : s.occupancy.densities.data(), lo, hi, &h->h));
    return h;
}
}  // namespace detail_c

struct ProbeResult {  // conditioning.hpp:44-47
    double transmittance = 1.0;
    double mean_density = 0.0;
};

// probe_segment (conditioning.hpp:50, conditioning.cpp:163-178) on the device, FP64
inline ProbeResult probe_segment(const OccupancyGrid& grid, const Vec3& from, const Vec3& to, int samples,
                                 bool nearest_lookup = false) {
    if (samples < 1) throw std::invalid_argument("probe_segment: samples must be >= 1");
    const double lo[3] = {grid.bounds.lo.x, grid.bounds.lo.y, grid.bounds.lo.z};
    const double hi[3] = {grid.bounds.hi.x, grid.bounds.hi.y, grid.bounds.hi.z};
    const double f[3] = {from.x, from.y, from.z}, t[3] = {to.x, to.y, to.z};
    double o[2];
    api::detail::check(rxgs_probe_grid(api::detail::ctx(), grid.resolution, lo, hi,
                                       grid.empty() ? nullptr : grid.densities.data(), 1, f, t, samples,
                                       nearest_lookup ? 1 : 0, o));
    return {o[0], o[1]};
}

// init_conditioning (conditioning.hpp:93, conditioning.cpp:217-253): the
// reference's derive_stream initialisation (rxgs_synth_cond, randomize = 0)
inline ConditioningState init_conditioning(const ConditioningConfig& config, int l_max, int channels,
                                           const Aabb& scene_bounds, uint64_t seed) {
    if (config.fourier_bands < 1 || config.hidden < 1 || config.embed_dim < 1)
        throw std::invalid_argument("init_conditioning: bad dimensions");
    const int32_t cfg[9] = {config.fourier_bands, config.hidden, config.embed_dim, config.probe_samples,
                            config.occupancy_resolution, config.nearest_lookup ? 1 : 0,
                            static_cast<int32_t>(config.mode), l_max, channels};
    const double lo[3] = {scene_bounds.lo.x, scene_bounds.lo.y, scene_bounds.lo.z};
    const double hi[3] = {scene_bounds.hi.x, scene_bounds.hi.y, scene_bounds.hi.z};
    std::vector<double> p(static_cast<std::size_t>(rxgs_synth_cond(cfg, l_max, channels, lo, hi, seed, 0, nullptr)));
    rxgs_synth_cond(cfg, l_max, channels, lo, hi, seed, 0, p.data());
    ConditioningState s;
    s.config = config;
    s.l_max = l_max;
    s.channels = channels;
    const int F = config.fourier_bands, d = config.hidden, dc = config.embed_dim;
    const double* q = p.data();
    auto take = [&q](std::vector<double>& v, std::size_t n) {
        v.assign(q, q + n);
        q += n;
    };
    auto layer = [&take](MlpLayer& l, int in, int out) {
        l.in = in;
        l.out = out;
        take(l.w, static_cast<std::size_t>(in) * out);
        take(l.b, static_cast<std::size_t>(out));
    };
    take(s.fourier_freqs, 3 * static_cast<std::size_t>(F));
    layer(s.global_mlp.l1, 6 * F + 2 + dc, d);
    layer(s.global_mlp.l2, d, d);
    layer(s.global_mlp.l3, d, 4 * channels);
    take(s.component_embed, static_cast<std::size_t>(api::component_count(l_max)) * dc);
    layer(s.local_mlp.l1, 6, d);
    layer(s.local_mlp.l2, d, d);
    layer(s.local_mlp.l3, d, 4 * channels);
    return s;
}

// fourier_encode (conditioning.cpp:255-265) on the device
inline std::vector<double> fourier_encode(const Vec3& r, const std::vector<double>& freqs) {
    const int F = static_cast<int>(freqs.size() / 3);
    std::vector<double> out(6 * static_cast<std::size_t>(F));
    const double rv[3] = {r.x, r.y, r.z};
    api::detail::check(rxgs_fourier_encode(api::detail::ctx(), F, freqs.data(), 1, rv, out.data()));
    return out;
}

inline OccupancyGrid build_occupancy(const GaussianScene& scene, int resolution, const Aabb& bounds) {
    auto sh = api::detail::upload(scene);
    OccupancyGrid g;
    g.resolution = resolution;
    g.bounds = bounds;
    const double lo[3] = {bounds.lo.x, bounds.lo.y, bounds.lo.z};
    const double hi[3] = {bounds.hi.x, bounds.hi.y, bounds.hi.z};
    g.densities.resize(resolution > 0 ? static_cast<std::size_t>(resolution) * resolution * resolution : 0);
    api::detail::check(rxgs_build_occupancy(api::detail::ctx(), sh->h, resolution, lo, hi,
                                            g.densities.empty() ? nullptr : g.densities.data(), nullptr));
    return g;
}

inline std::vector<double> condition_batch(const ConditioningState& state, const std::vector<double>& base,
                                           const GaussianScene& scene, const std::vector<Vec3>& rx_list) {
    if (base.size() != static_cast<std::size_t>(scene.count()) * scene.coeff_stride())
        throw std::invalid_argument("condition_forward: base coefficient size mismatch");
    GaussianScene s2 = scene;
    s2.fle_coeffs = base;
    auto sh = api::detail::upload(s2);
    auto ch = detail_c::upload(state);
    std::vector<double> rx;
    for (const Vec3& r : rx_list) rx.insert(rx.end(), {r.x, r.y, r.z});
    std::vector<double> out(base.size() * rx_list.size());
    if (!rx_list.empty())
        api::detail::check(rxgs_condition_batch(api::detail::ctx(), ch->h, sh->h, rx.data(),
                                                static_cast<int>(rx_list.size()), out.data()));
    if (state.config.mode != ConditioningMode::LocalOnly)
        state.global_calls += static_cast<std::int64_t>(rx_list.size()) * scene.n_components();
    if (state.config.mode != ConditioningMode::GlobalOnly)
        state.local_calls += static_cast<std::int64_t>(rx_list.size()) * scene.count();
    return out;
}

// conditioning.hpp:97-110.  The B200 adjoint recomputes the MLP activations on
// the device, so only rx and local_in are materialised; scene keeps the
// uploaded scene for condition_backward.
struct ConditionWorkspace {
    Vec3 rx;
    std::vector<double> gamma, global_in, global_h1, global_h2, global_out, mid;
    std::vector<double> local_in, local_h1, local_h2, local_out;
    std::shared_ptr<api::detail::SceneHandle> scene;
};

inline std::vector<double> condition_forward(const ConditioningState& state, const std::vector<double>& base,
                                             const GaussianScene& scene, const Vec3& rx,
                                             ConditionWorkspace* workspace = nullptr) {
    if (!workspace) return condition_batch(state, base, scene, {rx});
    if (base.size() != static_cast<std::size_t>(scene.count()) * scene.coeff_stride())
        throw std::invalid_argument("condition_forward: base coefficient size mismatch");
    GaussianScene s2 = scene;
    s2.fle_coeffs = base;
    workspace->scene = api::detail::upload(s2);
    workspace->rx = rx;
    workspace->local_in.assign(6 * static_cast<std::size_t>(scene.count()), 0.0);
    auto ch = detail_c::upload(state);
    std::vector<double> out(base.size());
    const double r[3] = {rx.x, rx.y, rx.z};
    api::detail::check(rxgs_condition_forward(api::detail::ctx(), ch->h, workspace->scene->h, r, out.data(),
                                              workspace->local_in.data()));
    if (state.config.mode != ConditioningMode::LocalOnly) state.global_calls += scene.n_components();
    if (state.config.mode != ConditioningMode::GlobalOnly) state.local_calls += scene.count();
    return out;
}

struct MlpGrads {  // conditioning.hpp:113-118
    std::vector<double> w1, b1, w2, b2, w3, b3;
    void resize(const Mlp& m) {
        w1.assign(m.l1.w.size(), 0.0); b1.assign(m.l1.b.size(), 0.0);
        w2.assign(m.l2.w.size(), 0.0); b2.assign(m.l2.b.size(), 0.0);
        w3.assign(m.l3.w.size(), 0.0); b3.assign(m.l3.b.size(), 0.0);
    }
};
struct ConditioningGrads {  // conditioning.hpp:120-128
    std::vector<double> d_freqs;
    MlpGrads d_global;
    std::vector<double> d_embed;
    MlpGrads d_local;
    void resize(const ConditioningState& s) {
        d_freqs.assign(s.fourier_freqs.size(), 0.0);
        d_global.resize(s.global_mlp);
        d_embed.assign(s.component_embed.size(), 0.0);
        d_local.resize(s.local_mlp);
    }
};

// conditioning.hpp:131-133: accumulates into d_base and grads (the packed
// parameter order of rxgs_cond_create)
inline void condition_backward(const ConditioningState& state, const ConditionWorkspace& ws,
                               const std::vector<double>& base, const std::vector<double>& d_out,
                               std::vector<double>& d_base, ConditioningGrads& grads) {
    if (!ws.scene) throw std::invalid_argument("condition_backward: workspace not filled by condition_forward");
    if (d_out.size() != base.size() || d_base.size() != base.size())
        throw std::invalid_argument("condition_backward: gradient size mismatch");
    auto ch = detail_c::upload(state);
    std::vector<double> db(base.size()), dp(static_cast<std::size_t>(rxgs_cond_param_count(ch->h)));
    const double r[3] = {ws.rx.x, ws.rx.y, ws.rx.z};
    api::detail::check(rxgs_condition_backward(api::detail::ctx(), ch->h, ws.scene->h, r, d_out.data(), db.data(),
                                               dp.data()));
    for (std::size_t i = 0; i < db.size(); ++i) d_base[i] += db[i];
    if (grads.d_freqs.empty()) grads.resize(state);
    std::size_t o = 0;
    auto take = [&](std::vector<double>& v) {
        for (double& x : v) x += dp[o++];
    };
    take(grads.d_freqs);
    for (auto* v : {&grads.d_global.w1, &grads.d_global.b1, &grads.d_global.w2, &grads.d_global.b2,
                    &grads.d_global.w3, &grads.d_global.b3})
        take(*v);
    take(grads.d_embed);
    for (auto* v : {&grads.d_local.w1, &grads.d_local.b1, &grads.d_local.w2, &grads.d_local.b2,
                    &grads.d_local.w3, &grads.d_local.b3})
        take(*v);
}

}  // namespace cond

namespace train {

struct Model {  // trainer.hpp:42-47
    GaussianScene scene;
    raster::SphericalGrid grid;
    bool has_conditioning = false;
    cond::ConditioningState conditioning;
};

// trainer.cpp:147-154
inline raster::Measurement predict(const Model& model, const Vec3& tx, const Vec3& rx, int threads = 1) {
    const std::vector<double> coeffs =
        model.has_conditioning ? cond::condition_forward(model.conditioning, model.scene.fle_coeffs, model.scene, rx)
                               : model.scene.fle_coeffs;
    const auto field = raster::render_field(model.scene, tx, model.grid, coeffs, 1, threads);
    return raster::aggregate_modality(field, model.scene.modality, model.grid)[0];
}

}  // namespace train

namespace io {  // checkpoint.hpp / dataset.hpp

struct IoError : std::runtime_error {  // dataset.hpp:16
    using std::runtime_error::runtime_error;
};

namespace detail_io {
inline void check(int rc) {
    if (rc == RXGS_ERR_IO) throw IoError(rxgs_last_error());
    api::detail::check(rc);
}
}  // namespace detail_io

// checkpoint.cpp:93-155: the RXGS container, written by the B200 library
inline void save_checkpoint(const std::string& path, const train::Model& model) {
    auto sh = api::detail::upload(model.scene);
    std::unique_ptr<cond::detail_c::CondHandle> ch;
    if (model.has_conditioning) ch = cond::detail_c::upload(model.conditioning);
    const rxgs_grid g = model.grid.c();
    detail_io::check(rxgs_checkpoint_save(path.c_str(), sh->h, &g, ch ? ch->h : nullptr));
}

// checkpoint.cpp:157-231: read by the library, materialised as host structs
inline train::Model load_checkpoint(const std::string& path) {
    auto sh = std::make_shared<api::detail::SceneHandle>();
    rxgs_grid g{};
    rxgs_cond c = nullptr;
    detail_io::check(rxgs_checkpoint_load(api::detail::ctx(), path.c_str(), &sh->h, &g, &c));
    cond::detail_c::CondHandle ch;
    ch.h = c;
    train::Model m;
    int32_t k = 0, l_max = 0, channels = 1, modality = 0;
    api::detail::check(rxgs_scene_info(sh->h, &k, &l_max, &channels, &modality));
    GaussianScene& s = m.scene;
    s.l_max = l_max;
    s.channels = channels;
    s.modality = static_cast<Modality>(modality);
    s.positions.resize(3 * static_cast<std::size_t>(k));
    s.log_scales.resize(3 * static_cast<std::size_t>(k));
    s.quaternions.resize(4 * static_cast<std::size_t>(k));
    s.tau_logits.resize(k);
    s.fle_coeffs.resize(static_cast<std::size_t>(k) * s.coeff_stride());
    api::detail::check(rxgs_scene_get_arrays(sh->h, s.positions.data(), s.log_scales.data(), s.quaternions.data(),
                                             s.tau_logits.data(), s.fle_coeffs.data()));
    m.grid.n_theta = g.n_theta;
    m.grid.n_phi = g.n_phi;
    m.grid.tile_size = g.tile_size;
    m.grid.radius = g.radius;
    m.grid.theta_min = g.theta_min;
    m.grid.theta_max = g.theta_max;
    m.has_conditioning = c != nullptr;
    if (c) {
        int32_t cfg[9];
        api::detail::check(rxgs_cond_config(c, cfg));
        cond::ConditioningState& st = m.conditioning;
        st.config = {cfg[0], cfg[1], cfg[2], cfg[3], cfg[4], cfg[5] != 0, static_cast<cond::ConditioningMode>(cfg[6])};
        st.l_max = cfg[7];
        st.channels = cfg[8];
        std::vector<double> p(static_cast<std::size_t>(rxgs_cond_param_count(c)));
        api::detail::check(rxgs_cond_get_params(c, p.data()));
        std::size_t o = 0;
        auto take = [&](std::vector<double>& v, std::size_t n) {
            v.assign(p.begin() + static_cast<std::ptrdiff_t>(o), p.begin() + static_cast<std::ptrdiff_t>(o + n));
            o += n;
        };
        const std::size_t F = cfg[0], d = cfg[1], dc = cfg[2], C4 = 4 * static_cast<std::size_t>(cfg[8]);
        const std::size_t L = static_cast<std::size_t>(component_count(cfg[7]));
        auto mlp = [&](cond::Mlp& net, int in) {
            net.l1 = {in, static_cast<int>(d), {}, {}};
            net.l2 = {static_cast<int>(d), static_cast<int>(d), {}, {}};
            net.l3 = {static_cast<int>(d), static_cast<int>(C4), {}, {}};
            take(net.l1.w, d * in);
            take(net.l1.b, d);
            take(net.l2.w, d * d);
            take(net.l2.b, d);
            take(net.l3.w, C4 * d);
            take(net.l3.b, C4);
        };
        take(st.fourier_freqs, 3 * F);
        mlp(st.global_mlp, static_cast<int>(6 * F + 2 + dc));
        take(st.component_embed, L * dc);
        mlp(st.local_mlp, 6);
        int32_t has = 0;
        double lo[3], hi[3];
        const std::size_t R = cfg[4];
        std::vector<double> dens(R * R * R);
        api::detail::check(rxgs_cond_get_occupancy(c, &has, dens.data(), lo, hi));
        st.occupancy.resolution = cfg[4];
        st.occupancy.bounds = {{lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]}};
        if (has) st.occupancy.densities = std::move(dens);
    }
    return m;
}

}  // namespace io

}  // namespace api
}  // namespace rxgs_b200

#ifdef RXGS_B200_AS_RXGS
namespace rxgs = rxgs_b200::api;
#endif
