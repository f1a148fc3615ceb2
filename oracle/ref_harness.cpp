// oracle/ref_harness.cpp -- TEST INFRASTRUCTURE ONLY (never the product path).
//
// A thin extern "C" shim over the UNMODIFIED reference library compiled from
// /root/reference/proj/src (see oracle/Makefile).  It lets the pytest suite
// and bench.py's cpu_baseline / --impl reference leg call the reference's own
// C++ functions through ctypes:
//   * rxgs::raster::{build_tx_state, bin_and_sort, render_field,
//     aggregate_modality(_backward), backward_render}   (sphraster.hpp:63-133)
//   * rxgs::cond::{init_conditioning, build_occupancy, probe_segment,
//     condition_forward, condition_backward}           (conditioning.hpp:41-146)
//   * rxgs::train::{predict, composite_loss}            (trainer.hpp:38-50)
// plus the synthetic-input generators defined in DESIGN.md section 5, written
// with the reference's own derive_stream (rng.hpp:67-72) so the GPU product
// and the reference see bit-identical inputs.
//
// Packed conditioning parameter order (shared with include/rxgs_b200.h):
//   freqs[F*3] | g.w1 g.b1 g.w2 g.b2 g.w3 g.b3 | embed[L*dc] |
//   l.w1 l.b1 l.w2 l.b2 l.w3 l.b3
// Integer config: {F, hidden, dc, S, R, nearest_lookup, mode, l_max, C}.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "rxgs/apps.hpp"
#include "rxgs/conditioning.hpp"
#include "rxgs/metrics.hpp"
#include "rxgs/radiance.hpp"
#include "rxgs/rng.hpp"
#include "rxgs/scene.hpp"
#include "rxgs/sphraster.hpp"
#include "rxgs/trainer.hpp"
#ifdef RXGS_REF_CHECKPOINT
#include "rxgs/checkpoint.hpp"
#endif

using namespace rxgs;

namespace {

void set_err(char* err, int errlen, const char* msg) {
    if (!err || errlen <= 0) return;
    std::snprintf(err, static_cast<std::size_t>(errlen), "%s", msg);
}

raster::SphericalGrid make_grid(const int* gi, const double* gd) {
    raster::SphericalGrid g;
    g.n_theta = gi[0];
    g.n_phi = gi[1];
    g.tile_size = gi[2];
    g.radius = gd[0];
    g.theta_min = gd[1];
    g.theta_max = gd[2];
    return g;
}

struct Handle {
    GaussianScene scene;
};

std::size_t cond_param_count(const cond::ConditioningState& s) {
    return s.fourier_freqs.size() + s.global_mlp.param_count() + s.component_embed.size() +
           s.local_mlp.param_count();
}

template <typename F>
void for_each_param(cond::ConditioningState& s, F&& f) {
    f(s.fourier_freqs);
    for (auto* l : {&s.global_mlp.l1, &s.global_mlp.l2, &s.global_mlp.l3}) {
        f(l->w);
        f(l->b);
    }
    f(s.component_embed);
    for (auto* l : {&s.local_mlp.l1, &s.local_mlp.l2, &s.local_mlp.l3}) {
        f(l->w);
        f(l->b);
    }
}

template <typename F>
void for_each_grad(cond::ConditioningGrads& g, F&& f) {
    f(g.d_freqs);
    for (auto* m : {&g.d_global}) {
        f(m->w1); f(m->b1); f(m->w2); f(m->b2); f(m->w3); f(m->b3);
    }
    f(g.d_embed);
    for (auto* m : {&g.d_local}) {
        f(m->w1); f(m->b1); f(m->w2); f(m->b2); f(m->w3); f(m->b3);
    }
}

cond::ConditioningConfig make_cfg(const int* cfg) {
    cond::ConditioningConfig c;
    c.fourier_bands = cfg[0];
    c.hidden = cfg[1];
    c.embed_dim = cfg[2];
    c.probe_samples = cfg[3];
    c.occupancy_resolution = cfg[4];
    c.nearest_lookup = cfg[5] != 0;
    c.mode = static_cast<cond::ConditioningMode>(cfg[6]);
    return c;
}

}  // namespace

extern "C" {

int ref_abi_version() { return 3; }

// ---------------------------------------------------------------- generators
// bench scene.  Draw order per Gaussian k: pos x,y,z
// U(box); log_scale x3 = ln(0.554 (144/K)^(1/3)) + U(-0.3,0.3); quaternion
// 4 x N(0,1) normalised; tau_logit U(-2,1).  Then all K*L*C*2 coefficients
// N(0,1) in storage order from a second stream.
void ref_synth_scene(int k, int l_max, int channels, uint64_t seed, double* pos, double* ls,
                     double* q, double* tau, double* coeffs) {
    Rng rng = derive_stream(seed, "bench.scene");
    const double base = std::log(0.554 * std::cbrt(144.0 / static_cast<double>(k)));
    for (int i = 0; i < k; ++i) {
        pos[3 * i + 0] = rng.uniform(-4.0, 4.0);
        pos[3 * i + 1] = rng.uniform(-3.0, 3.0);
        pos[3 * i + 2] = rng.uniform(-1.5, 1.5);
        for (int a = 0; a < 3; ++a) ls[3 * i + a] = base + rng.uniform(-0.3, 0.3);
        double qq[4];
        for (int a = 0; a < 4; ++a) qq[a] = rng.normal();
        const double n = std::sqrt(qq[0] * qq[0] + qq[1] * qq[1] + qq[2] * qq[2] + qq[3] * qq[3]);
        for (int a = 0; a < 4; ++a) q[4 * i + a] = qq[a] / n;
        tau[i] = rng.uniform(-2.0, 1.0);
    }
    Rng crng = derive_stream(seed, "bench.scene.coeffs");
    const std::size_t n = static_cast<std::size_t>(k) * fle::component_count(l_max) * channels * 2;
    for (std::size_t i = 0; i < n; ++i) coeffs[i] = crng.normal();
}

// Uniform points in [lo + m*ext, hi - m*ext]; x, y, z per point.
void ref_synth_points(int n, uint64_t seed, const char* tag, const double* lo, const double* hi,
                      double margin, double* out) {
    Rng rng = derive_stream(seed, tag);
    double a[3], b[3];
    for (int d = 0; d < 3; ++d) {
        const double ext = hi[d] - lo[d];
        a[d] = lo[d] + margin * ext;
        b[d] = hi[d] - margin * ext;
    }
    for (int i = 0; i < n; ++i)
        for (int d = 0; d < 3; ++d) out[3 * i + d] = rng.uniform(a[d], b[d]);
}

// init_conditioning (conditioning.cpp:217-253) then, if randomize, the bench
// overwrite: weights U(-1,1)/sqrt(fan_in), l1/l2 biases 0.1 N(0,1), l3 bias 0,
// streams "bench.cond.<global|local>.<w1|b1|w2|b2|w3|b3>".
long ref_synth_cond(const int* cfg, int l_max, int channels, const double* blo, const double* bhi,
                    uint64_t seed, int randomize, double* params_out) {
    const Aabb bounds{{blo[0], blo[1], blo[2]}, {bhi[0], bhi[1], bhi[2]}};
    cond::ConditioningState s =
        cond::init_conditioning(make_cfg(cfg), l_max, channels, bounds, seed);
    if (randomize) {
        auto fill = [&](cond::Mlp& mlp, const char* name) {
            cond::MlpLayer* layers[3] = {&mlp.l1, &mlp.l2, &mlp.l3};
            for (int li = 0; li < 3; ++li) {
                cond::MlpLayer& L = *layers[li];
                const std::string p = std::string("bench.cond.") + name + ".";
                Rng rw = derive_stream(seed, p + "w" + std::to_string(li + 1));
                Rng rb = derive_stream(seed, p + "b" + std::to_string(li + 1));
                const double sc = 1.0 / std::sqrt(static_cast<double>(L.in));
                for (auto& w : L.w) w = rw.uniform(-1.0, 1.0) * sc;
                for (auto& b : L.b) b = li < 2 ? 0.1 * rb.normal() : 0.0;
            }
        };
        fill(s.global_mlp, "global");
        fill(s.local_mlp, "local");
    }
    std::size_t off = 0;
    for_each_param(s, [&](std::vector<double>& v) {
        if (params_out) std::memcpy(params_out + off, v.data(), v.size() * sizeof(double));
        off += v.size();
    });
    return static_cast<long>(off);
}

// ---------------------------------------------------------------- scene
void* ref_scene_new(int k, int l_max, int channels, int modality, const double* pos,
                    const double* ls, const double* q, const double* tau, const double* coeffs) {
    auto* h = new Handle;
    GaussianScene& s = h->scene;
    s.l_max = l_max;
    s.channels = channels;
    s.modality = static_cast<Modality>(modality);
    s.positions.assign(pos, pos + 3 * static_cast<std::size_t>(k));
    s.log_scales.assign(ls, ls + 3 * static_cast<std::size_t>(k));
    s.quaternions.assign(q, q + 4 * static_cast<std::size_t>(k));
    s.tau_logits.assign(tau, tau + static_cast<std::size_t>(k));
    s.fle_coeffs.assign(coeffs, coeffs + static_cast<std::size_t>(k) * s.coeff_stride());
    return h;
}
void ref_scene_free(void* h) { delete static_cast<Handle*>(h); }
void ref_scene_bounds(void* h, double inflate, double* lo, double* hi) {
    const Aabb b = static_cast<Handle*>(h)->scene.position_bounds().inflated(inflate);
    for (int a = 0; a < 3; ++a) {
        lo[a] = b.lo[a];
        hi[a] = b.hi[a];
    }
}
int ref_scene_count(void* h) { return static_cast<Handle*>(h)->scene.count(); }
void ref_scene_get(void* h, double* pos, double* ls, double* q, double* tau, double* coeffs) {
    const GaussianScene& s = static_cast<Handle*>(h)->scene;
    std::memcpy(pos, s.positions.data(), s.positions.size() * sizeof(double));
    std::memcpy(ls, s.log_scales.data(), s.log_scales.size() * sizeof(double));
    std::memcpy(q, s.quaternions.data(), s.quaternions.size() * sizeof(double));
    std::memcpy(tau, s.tau_logits.data(), s.tau_logits.size() * sizeof(double));
    std::memcpy(coeffs, s.fle_coeffs.data(), s.fle_coeffs.size() * sizeof(double));
}
// densify_and_prune (scene.cpp:178-274) in place on the handle's scene, from
// a DensifyState built with accumulate() calls of the given d_positions
// (n_acc of them, K*3 each); report = {cloned, split, pruned}; source_row has
// room for 2K entries.  reset_transmittance (scene.cpp:276-279) if reset_tau.
int ref_densify(void* h, const double* d_pos_list, int n_acc, double extent, const double* thr, unsigned long seed,
                unsigned long pass, int* report, int* source_row, char* err, int errlen) {
    try {
        GaussianScene& s = static_cast<Handle*>(h)->scene;
        DensifyState st;
        st.resize(s.count());
        st.scene_extent = extent;
        const std::size_t n3 = 3 * static_cast<std::size_t>(s.count());
        for (int a = 0; a < n_acc; ++a)
            st.accumulate(std::vector<double>(d_pos_list + a * n3, d_pos_list + (a + 1) * n3));
        DensifyThresholds t;
        t.grad_threshold = thr[0];
        t.size_frac = thr[1];
        t.prune_extent_frac = thr[2];
        t.split_scale_factor = thr[3];
        const DensifyReport r = densify_and_prune(s, st, t, seed, pass);
        report[0] = r.cloned;
        report[1] = r.split;
        report[2] = r.pruned;
        std::copy(r.source_row.begin(), r.source_row.end(), source_row);
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}
void ref_reset_transmittance(void* h) { reset_transmittance(static_cast<Handle*>(h)->scene); }

void ref_covariance(void* h, double* out) {
    const GaussianScene& s = static_cast<Handle*>(h)->scene;
    for (int k = 0; k < s.count(); ++k) {
        const Mat3 c = s.covariance(k);
        std::memcpy(out + 9 * static_cast<std::size_t>(k), c.m.data(), 9 * sizeof(double));
    }
}

// ---------------------------------------------------------------- tx state
void* ref_tx_new(void* scene, const double* tx, const int* gi, const double* gd, char* err,
                 int errlen) {
    try {
        auto* st = new raster::TxState(raster::build_tx_state(
            static_cast<Handle*>(scene)->scene, {tx[0], tx[1], tx[2]}, make_grid(gi, gd)));
        return st;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return nullptr;
    }
}
void ref_tx_free(void* h) { delete static_cast<raster::TxState*>(h); }
long ref_tx_entries(void* h) {
    long n = 0;
    for (const auto& l : static_cast<raster::TxState*>(h)->tile_lists) n += static_cast<long>(l.size());
    return n;
}
// geom per Gaussian: theta, phi, depth, cov a b c d, prec a b c d, weight_scale (12 f64)
void ref_tx_get(void* h, int* culled, double* geom, int* spans, double* basis, long* offsets,
                int* indices, uint64_t* hash) {
    const auto& st = *static_cast<raster::TxState*>(h);
    for (int k = 0; k < st.k; ++k) {
        const auto& p = st.proj[static_cast<std::size_t>(k)];
        culled[k] = p.culled ? 1 : 0;
        double* g = geom + 12 * static_cast<std::size_t>(k);
        g[0] = p.theta; g[1] = p.phi; g[2] = p.depth;
        g[3] = p.angular_cov.a; g[4] = p.angular_cov.b; g[5] = p.angular_cov.c; g[6] = p.angular_cov.d;
        g[7] = p.angular_prec.a; g[8] = p.angular_prec.b; g[9] = p.angular_prec.c; g[10] = p.angular_prec.d;
        g[11] = p.weight_scale;
        spans[4 * k + 0] = p.t0; spans[4 * k + 1] = p.t1;
        spans[4 * k + 2] = p.p0; spans[4 * k + 3] = p.p1;
    }
    for (std::size_t i = 0; i < st.basis.size(); ++i) {
        basis[2 * i] = st.basis[i].real();
        basis[2 * i + 1] = st.basis[i].imag();
    }
    long off = 0;
    for (std::size_t t = 0; t < st.tile_lists.size(); ++t) {
        offsets[t] = off;
        for (const int idx : st.tile_lists[t]) indices[off++] = idx;
    }
    offsets[st.tile_lists.size()] = off;
    if (hash) *hash = st.hash();
}

// bin_and_sort on caller-supplied projections (sphraster.cpp:85-102).
long ref_bin_and_sort(int k, const int* culled, const double* depth, const int* spans,
                      const int* gi, const double* gd, long* offsets, int* indices, long cap) {
    std::vector<raster::ProjectedGaussian> proj(static_cast<std::size_t>(k));
    for (int i = 0; i < k; ++i) {
        auto& p = proj[static_cast<std::size_t>(i)];
        p.culled = culled[i] != 0;
        p.depth = depth[i];
        p.t0 = spans[4 * i]; p.t1 = spans[4 * i + 1]; p.p0 = spans[4 * i + 2]; p.p1 = spans[4 * i + 3];
    }
    const auto lists = raster::bin_and_sort(proj, make_grid(gi, gd));
    long off = 0;
    for (std::size_t t = 0; t < lists.size(); ++t) {
        offsets[t] = off;
        for (const int idx : lists[t]) {
            if (off < cap) indices[off] = idx;
            ++off;
        }
    }
    offsets[lists.size()] = off;
    return off;
}

// ---------------------------------------------------------------- render
int ref_render(void* tx, void* scene, const double* coeffs, long n_coeffs, int n_rx, int threads,
               double* values, double* transmittance, char* err, int errlen) {
    try {
        const std::vector<double> c(coeffs, coeffs + n_coeffs);
        const auto f = raster::render_field(*static_cast<raster::TxState*>(tx),
                                            static_cast<Handle*>(scene)->scene, c, n_rx, threads);
        std::memcpy(values, f.values.data(), f.values.size() * sizeof(double));
        std::memcpy(transmittance, f.transmittance.data(), f.transmittance.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

// out: spectrum n_rx*h*w; rssi n_rx; csi n_rx*C*2
int ref_aggregate(int n_rx, int channels, const int* gi, const double* gd, const double* values,
                  int modality, double* out, char* err, int errlen) {
    try {
        const auto grid = make_grid(gi, gd);
        raster::RenderedField f;
        f.n_rx = n_rx;
        f.channels = channels;
        f.h = grid.n_theta;
        f.w = grid.n_phi;
        f.values.assign(values, values + static_cast<std::size_t>(n_rx) * channels * 2 * f.plane());
        const auto ms = raster::aggregate_modality(f, static_cast<Modality>(modality), grid);
        for (int j = 0; j < n_rx; ++j) {
            const auto& m = ms[static_cast<std::size_t>(j)];
            if (modality == 0) out[j] = m.scalar;
            else if (modality == 1)
                for (int c = 0; c < channels; ++c) {
                    out[(static_cast<std::size_t>(j) * channels + c) * 2] = m.csi[c].real();
                    out[(static_cast<std::size_t>(j) * channels + c) * 2 + 1] = m.csi[c].imag();
                }
            else
                std::memcpy(out + static_cast<std::size_t>(j) * f.plane(), m.image.data(),
                            f.plane() * sizeof(double));
        }
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

// upstream has the same layout as ref_aggregate's out.
int ref_aggregate_backward(int n_rx, int channels, const int* gi, const double* gd,
                           const double* values, int modality, const double* upstream,
                           double* d_values) {
    const auto grid = make_grid(gi, gd);
    raster::RenderedField f;
    f.n_rx = n_rx;
    f.channels = channels;
    f.h = grid.n_theta;
    f.w = grid.n_phi;
    f.values.assign(values, values + static_cast<std::size_t>(n_rx) * channels * 2 * f.plane());
    std::vector<raster::Measurement> up(static_cast<std::size_t>(n_rx));
    for (int j = 0; j < n_rx; ++j) {
        auto& m = up[static_cast<std::size_t>(j)];
        m.modality = static_cast<Modality>(modality);
        if (modality == 0) m.scalar = upstream[j];
        else if (modality == 1) {
            m.csi.resize(static_cast<std::size_t>(channels));
            for (int c = 0; c < channels; ++c)
                m.csi[c] = {upstream[(static_cast<std::size_t>(j) * channels + c) * 2],
                            upstream[(static_cast<std::size_t>(j) * channels + c) * 2 + 1]};
        } else
            m.image.assign(upstream + static_cast<std::size_t>(j) * f.plane(),
                           upstream + static_cast<std::size_t>(j + 1) * f.plane());
    }
    const auto d = raster::aggregate_modality_backward(f, static_cast<Modality>(modality), grid, up);
    std::memcpy(d_values, d.data(), d.size() * sizeof(double));
    return 0;
}

int ref_backward_render(void* tx, void* scene, const double* coeffs, long n_coeffs, int n_rx,
                        const double* d_values, long n_dv, int threads, double* d_pos,
                        double* d_ls, double* d_q, double* d_tau, double* d_coeffs, char* err,
                        int errlen) {
    try {
        const std::vector<double> c(coeffs, coeffs + n_coeffs);
        const std::vector<double> dv(d_values, d_values + n_dv);
        const auto b = raster::backward_render(*static_cast<raster::TxState*>(tx),
                                               static_cast<Handle*>(scene)->scene, c, n_rx, dv,
                                               threads);
        std::memcpy(d_pos, b.d_positions.data(), b.d_positions.size() * sizeof(double));
        std::memcpy(d_ls, b.d_log_scales.data(), b.d_log_scales.size() * sizeof(double));
        std::memcpy(d_q, b.d_quaternions.data(), b.d_quaternions.size() * sizeof(double));
        std::memcpy(d_tau, b.d_tau_logits.data(), b.d_tau_logits.size() * sizeof(double));
        std::memcpy(d_coeffs, b.d_coeffs.data(), b.d_coeffs.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

// ---------------------------------------------------------------- conditioning
void* ref_cond_new(const int* cfg, const double* params, const double* occ, const double* occ_lo,
                   const double* occ_hi) {
    auto* s = new cond::ConditioningState;
    s->config = make_cfg(cfg);
    s->l_max = cfg[7];
    s->channels = cfg[8];
    const int F = cfg[0], d = cfg[1], dc = cfg[2], C = cfg[8];
    const int L = fle::component_count(cfg[7]);
    const int gin = 6 * F + 2 + dc;
    s->fourier_freqs.resize(static_cast<std::size_t>(F) * 3);
    auto set_layer = [](cond::MlpLayer& l, int in, int out) {
        l.in = in;
        l.out = out;
        l.w.resize(static_cast<std::size_t>(in) * out);
        l.b.resize(static_cast<std::size_t>(out));
    };
    set_layer(s->global_mlp.l1, gin, d);
    set_layer(s->global_mlp.l2, d, d);
    set_layer(s->global_mlp.l3, d, 4 * C);
    s->component_embed.resize(static_cast<std::size_t>(L) * dc);
    set_layer(s->local_mlp.l1, 6, d);
    set_layer(s->local_mlp.l2, d, d);
    set_layer(s->local_mlp.l3, d, 4 * C);
    std::size_t off = 0;
    for_each_param(*s, [&](std::vector<double>& v) {
        std::memcpy(v.data(), params + off, v.size() * sizeof(double));
        off += v.size();
    });
    if (occ) {
        const int R = cfg[4];
        s->occupancy.resolution = R;
        s->occupancy.bounds = {{occ_lo[0], occ_lo[1], occ_lo[2]}, {occ_hi[0], occ_hi[1], occ_hi[2]}};
        s->occupancy.densities.assign(occ, occ + static_cast<std::size_t>(R) * R * R);
    }
    return s;
}
void ref_cond_free(void* h) { delete static_cast<cond::ConditioningState*>(h); }
long ref_cond_param_count(void* h) {
    return static_cast<long>(cond_param_count(*static_cast<cond::ConditioningState*>(h)));
}
void ref_cond_calls(void* h, long* g, long* l) {
    const auto* s = static_cast<cond::ConditioningState*>(h);
    *g = static_cast<long>(s->global_calls);
    *l = static_cast<long>(s->local_calls);
}

void ref_build_occupancy(void* scene, int resolution, const double* lo, const double* hi,
                         double* out) {
    const auto g = cond::build_occupancy(static_cast<Handle*>(scene)->scene, resolution,
                                         {{lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]}});
    std::memcpy(out, g.densities.data(), g.densities.size() * sizeof(double));
}

void ref_probe(int resolution, const double* lo, const double* hi, const double* dens,
               const double* from, const double* to, int samples, int nearest, double* out2) {
    cond::OccupancyGrid g;
    if (dens) {
        g.resolution = resolution;
        g.bounds = {{lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]}};
        g.densities.assign(dens, dens + static_cast<std::size_t>(resolution) * resolution * resolution);
    }
    const auto r = cond::probe_segment(g, {from[0], from[1], from[2]}, {to[0], to[1], to[2]},
                                       samples, nearest != 0);
    out2[0] = r.transmittance;
    out2[1] = r.mean_density;
}

// ws_local_in (K*6) / ws_local_out (K*4C) / ws_global_out (L*4C) are optional.
int ref_cond_forward(void* cond, void* scene, const double* rx, double* out, double* ws_local_in,
                     double* ws_local_out, double* ws_global_out, char* err, int errlen) {
    try {
        cond::ConditionWorkspace ws;
        const auto& sc = static_cast<Handle*>(scene)->scene;
        const auto o = cond::condition_forward(*static_cast<cond::ConditioningState*>(cond),
                                               sc.fle_coeffs, sc, {rx[0], rx[1], rx[2]}, &ws);
        std::memcpy(out, o.data(), o.size() * sizeof(double));
        if (ws_local_in && !ws.local_in.empty())
            std::memcpy(ws_local_in, ws.local_in.data(), ws.local_in.size() * sizeof(double));
        if (ws_local_out && !ws.local_out.empty())
            std::memcpy(ws_local_out, ws.local_out.data(), ws.local_out.size() * sizeof(double));
        if (ws_global_out && !ws.global_out.empty())
            std::memcpy(ws_global_out, ws.global_out.data(), ws.global_out.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

int ref_cond_backward(void* cond, void* scene, const double* rx, const double* d_out,
                      double* d_base, double* d_params) {
    auto& st = *static_cast<cond::ConditioningState*>(cond);
    const auto& sc = static_cast<Handle*>(scene)->scene;
    cond::ConditionWorkspace ws;
    (void)cond::condition_forward(st, sc.fle_coeffs, sc, {rx[0], rx[1], rx[2]}, &ws);
    std::vector<double> db(sc.fle_coeffs.size(), 0.0);
    cond::ConditioningGrads g;
    g.resize(st);
    const std::vector<double> dout(d_out, d_out + sc.fle_coeffs.size());
    cond::condition_backward(st, ws, sc.fle_coeffs, dout, db, g);
    std::memcpy(d_base, db.data(), db.size() * sizeof(double));
    std::size_t off = 0;
    for_each_grad(g, [&](std::vector<double>& v) {
        std::memcpy(d_params + off, v.data(), v.size() * sizeof(double));
        off += v.size();
    });
    return 0;
}

// ---------------------------------------------------------------- query API
// train::predict (trainer.cpp:147-154) for one (tx, rx); out = image or scalar.
int ref_predict(void* scene, void* cond, const int* gi, const double* gd, const double* tx,
                const double* rx, int threads, double* out, char* err, int errlen) {
    try {
        train::Model m;
        m.scene = static_cast<Handle*>(scene)->scene;
        m.grid = make_grid(gi, gd);
        if (cond) {
            m.has_conditioning = true;
            m.conditioning = *static_cast<cond::ConditioningState*>(cond);
        }
        const auto r = train::predict(m, {tx[0], tx[1], tx[2]}, {rx[0], rx[1], rx[2]}, threads);
        if (m.scene.modality == Modality::Spectrum)
            std::memcpy(out, r.image.data(), r.image.size() * sizeof(double));
        else if (m.scene.modality == Modality::Rssi)
            out[0] = r.scalar;
        else
            for (std::size_t c = 0; c < r.csi.size(); ++c) {
                out[2 * c] = r.csi[c].real();
                out[2 * c + 1] = r.csi[c].imag();
            }
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

// The reference CPU path for the batched query workload:
// build_tx_state once; condition_forward per receiver fanned over `threads`
// host threads (harness-level parallelism, one ConditioningState copy per
// thread); render_field over receiver chunks of 16 with `threads`; then
// spectrum + RSSI aggregation.  Returns wall seconds.  Outputs optional.
double ref_bench_queries(void* scene, void* cond, const int* gi, const double* gd,
                         const double* tx, const double* rx, int n_rx, int threads,
                         float* out_spec, double* out_rssi) {
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    const GaussianScene& sc = static_cast<Handle*>(scene)->scene;
    const auto grid = make_grid(gi, gd);
    const raster::TxState st = raster::build_tx_state(sc, {tx[0], tx[1], tx[2]}, grid);
    const std::size_t per = sc.fle_coeffs.size();
    const std::size_t plane = grid.cells();
    const int chunk = 16;
    for (int j0 = 0; j0 < n_rx; j0 += chunk) {
        const int nj = std::min(chunk, n_rx - j0);
        std::vector<double> coeffs(per * static_cast<std::size_t>(nj));
        if (cond) {
            const int nt = std::max(1, std::min(threads, nj));
            std::vector<std::thread> pool;
            for (int t = 0; t < nt; ++t)
                pool.emplace_back([&, t] {
                    cond::ConditioningState local = *static_cast<cond::ConditioningState*>(cond);
                    for (int j = t; j < nj; j += nt) {
                        const int r = j0 + j;
                        const auto o = cond::condition_forward(
                            local, sc.fle_coeffs, sc, {rx[3 * r], rx[3 * r + 1], rx[3 * r + 2]});
                        std::memcpy(coeffs.data() + per * static_cast<std::size_t>(j), o.data(),
                                    per * sizeof(double));
                    }
                });
            for (auto& th : pool) th.join();
        } else {
            for (int j = 0; j < nj; ++j)
                std::memcpy(coeffs.data() + per * static_cast<std::size_t>(j), sc.fle_coeffs.data(),
                            per * sizeof(double));
        }
        const auto f = raster::render_field(st, sc, coeffs, nj, threads);
        const auto spec = raster::aggregate_modality(f, Modality::Spectrum, grid);
        const auto rssi = raster::aggregate_modality(f, Modality::Rssi, grid);
        for (int j = 0; j < nj; ++j) {
            if (out_spec)
                for (std::size_t c = 0; c < plane; ++c)
                    out_spec[static_cast<std::size_t>(j0 + j) * plane + c] =
                        static_cast<float>(spec[static_cast<std::size_t>(j)].image[c]);
            if (out_rssi) out_rssi[j0 + j] = rssi[static_cast<std::size_t>(j)].scalar;
        }
    }
    return std::chrono::duration<double>(clk::now() - t0).count();
}

// Coverage-table CPU baseline (BASELINE config 3 timing rules, BASELINE.md
// "Coverage per config"): condition every receiver once (fanned over
// threads, one ConditioningState copy each), then per Tx build_tx_state +
// render_field (chunks of 16, `threads`) + RSSI aggregation, reusing the
// conditioned coefficients.  out_rssi[t*n_rx + j]; phase[0..2] = seconds in
// conditioning, build_tx_state, render+aggregate.
double ref_bench_coverage(void* scene, void* cond, const int* gi, const double* gd, const double* tx,
                          int n_tx, const double* rx, int n_rx, int threads, double* out_rssi,
                          double* phase) {
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    const GaussianScene& sc = static_cast<Handle*>(scene)->scene;
    const auto grid = make_grid(gi, gd);
    const std::size_t per = sc.fle_coeffs.size();
    std::vector<double> coeffs(per * static_cast<std::size_t>(n_rx));
    if (cond) {
        const int nt = std::max(1, std::min(threads, n_rx));
        std::vector<std::thread> pool;
        for (int t = 0; t < nt; ++t)
            pool.emplace_back([&, t] {
                cond::ConditioningState local = *static_cast<cond::ConditioningState*>(cond);
                for (int j = t; j < n_rx; j += nt) {
                    const auto o = cond::condition_forward(local, sc.fle_coeffs, sc,
                                                           {rx[3 * j], rx[3 * j + 1], rx[3 * j + 2]});
                    std::memcpy(coeffs.data() + per * static_cast<std::size_t>(j), o.data(),
                                per * sizeof(double));
                }
            });
        for (auto& th : pool) th.join();
    } else {
        for (int j = 0; j < n_rx; ++j)
            std::memcpy(coeffs.data() + per * static_cast<std::size_t>(j), sc.fle_coeffs.data(),
                        per * sizeof(double));
    }
    const auto t1 = clk::now();
    double t_build = 0.0, t_render = 0.0;
    const int chunk = 16;
    for (int t = 0; t < n_tx; ++t) {
        const auto a = clk::now();
        const raster::TxState st =
            raster::build_tx_state(sc, {tx[3 * t], tx[3 * t + 1], tx[3 * t + 2]}, grid);
        const auto b = clk::now();
        for (int j0 = 0; j0 < n_rx; j0 += chunk) {
            const int nj = std::min(chunk, n_rx - j0);
            const std::vector<double> part(coeffs.begin() + per * static_cast<std::size_t>(j0),
                                           coeffs.begin() + per * static_cast<std::size_t>(j0 + nj));
            const auto f = raster::render_field(st, sc, part, nj, threads);
            const auto rssi = raster::aggregate_modality(f, Modality::Rssi, grid);
            for (int j = 0; j < nj; ++j)
                if (out_rssi) out_rssi[static_cast<std::size_t>(t) * n_rx + j0 + j] = rssi[j].scalar;
        }
        t_build += std::chrono::duration<double>(b - a).count();
        t_render += std::chrono::duration<double>(clk::now() - b).count();
    }
    if (phase) {
        phase[0] = std::chrono::duration<double>(t1 - t0).count();
        phase[1] = t_build;
        phase[2] = t_render;
    }
    return std::chrono::duration<double>(clk::now() - t0).count();
}

// One conditioned training sample (trainer.cpp:429-449): condition -> render
// (N=1) -> aggregate(spectrum) -> composite_loss vs target -> adjoints.
// Outputs loss, d_base (K*L*C*2), d_params (packed cond order), and the
// geometry gradients (d_pos K*3, d_ls K*3, d_q K*4, d_tau K) if non-null.
int ref_train_sample(void* scene, void* cond, const int* gi, const double* gd, const double* tx,
                     const double* rx, const double* target, double lambda_ssim,
                     double lambda_fft, int threads, double* loss, double* d_base,
                     double* d_params, double* d_pos, double* d_ls, double* d_q, double* d_tau,
                     char* err, int errlen) {
    try {
        const GaussianScene& sc = static_cast<Handle*>(scene)->scene;
        // cond == NULL: the unconditioned Stage-I chain (trainer.cpp:317-340)
        auto* stp = static_cast<cond::ConditioningState*>(cond);
        const auto grid = make_grid(gi, gd);
        const raster::TxState ts = raster::build_tx_state(sc, {tx[0], tx[1], tx[2]}, grid);
        cond::ConditionWorkspace ws;
        const auto coeffs = stp ? cond::condition_forward(*stp, sc.fle_coeffs, sc, {rx[0], rx[1], rx[2]}, &ws)
                                : sc.fle_coeffs;
        const auto field = raster::render_field(ts, sc, coeffs, 1, threads);
        const auto pred = raster::aggregate_modality(field, Modality::Spectrum, grid)[0];
        raster::Measurement gt;
        gt.modality = Modality::Spectrum;
        gt.image.assign(target, target + grid.cells());
        train::LossWeights lw;
        lw.lambda_ssim = lambda_ssim;
        lw.lambda_fft = lambda_fft;
        const auto lr = train::composite_loss(pred, gt, Modality::Spectrum, lw, grid.n_theta,
                                              grid.n_phi);
        *loss = lr.value;
        const auto dv = raster::aggregate_modality_backward(field, Modality::Spectrum, grid,
                                                            {lr.d_pred});
        const auto b = raster::backward_render(ts, sc, coeffs, 1, dv, threads);
        if (stp) {
            std::vector<double> db(sc.fle_coeffs.size(), 0.0);
            cond::ConditioningGrads g;
            g.resize(*stp);
            cond::condition_backward(*stp, ws, sc.fle_coeffs, b.d_coeffs, db, g);
            std::memcpy(d_base, db.data(), db.size() * sizeof(double));
            std::size_t off = 0;
            for_each_grad(g, [&](std::vector<double>& v) {
                std::memcpy(d_params + off, v.data(), v.size() * sizeof(double));
                off += v.size();
            });
        } else {
            std::memcpy(d_base, b.d_coeffs.data(), b.d_coeffs.size() * sizeof(double));
        }
        if (d_pos) std::memcpy(d_pos, b.d_positions.data(), b.d_positions.size() * sizeof(double));
        if (d_ls) std::memcpy(d_ls, b.d_log_scales.data(), b.d_log_scales.size() * sizeof(double));
        if (d_q) std::memcpy(d_q, b.d_quaternions.data(), b.d_quaternions.size() * sizeof(double));
        if (d_tau) std::memcpy(d_tau, b.d_tau_logits.data(), b.d_tau_logits.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

// apps::coverage_fraction / greedy_plan (apps.cpp:69-116) on a tx-major table.
int ref_coverage_fraction(const double* table, long tx, long cand, const int* sel, int n_sel, double thr, double* out,
                          char* err, int errlen) {
    try {
        *out = apps::coverage_fraction(std::vector<double>(table, table + tx * cand), static_cast<std::size_t>(tx),
                                       static_cast<std::size_t>(cand), std::vector<int>(sel, sel + n_sel), thr);
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

int ref_greedy_plan(const double* table, long tx, long cand, int k, double thr, int* order, char* err, int errlen) {
    try {
        const auto o = apps::greedy_plan(std::vector<double>(table, table + tx * cand), static_cast<std::size_t>(tx),
                                         static_cast<std::size_t>(cand), k, thr);
        std::copy(o.begin(), o.end(), order);
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

// met::mae / mse / psnr / ssim (metrics.cpp:11-112) of one image;
// out = {mae, mse, psnr, ssim}; ssim skipped (NaN) when window == 0.
int ref_image_metrics(const double* pred, const double* gt, int h, int w, double max_val, int window, double sigma,
                      double dyn, double* out, char* err, int errlen) {
    try {
        const std::size_t n = static_cast<std::size_t>(h) * w;
        const std::span<const double> p(pred, n), g(gt, n);
        out[0] = met::mae(p, g);
        out[1] = met::mse(p, g);
        out[2] = met::psnr(p, g, max_val);
        out[3] = std::nan("");
        if (window > 0) {
            met::SsimOptions o;
            o.window = window;
            o.sigma = sigma;
            o.dynamic_range = dyn;
            out[3] = met::ssim(p, g, h, w, o);
        }
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

// met::snr_csi (metrics.cpp:114-125) of one (pred, gt) pair of n complex.
int ref_snr_csi(const double* pred, const double* gt, long n, double* out, char* err, int errlen) {
    try {
        std::vector<cplx> p(static_cast<std::size_t>(n)), g(static_cast<std::size_t>(n));
        for (long i = 0; i < n; ++i) {
            p[i] = cplx{pred[2 * i], pred[2 * i + 1]};
            g[i] = cplx{gt[2 * i], gt[2 * i + 1]};
        }
        *out = met::snr_csi(p, g);
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

// met::per_receiver_aggregate (metrics.cpp:127-149): per receiver (ascending
// rx) the mean and count; *n_unique, *mean, *stddev.
int ref_per_receiver_aggregate(const int* rx, const double* values, long n, int* out_rx, double* out_mean,
                               long* out_count, int* n_unique, double* mean, double* stddev, char* err,
                               int errlen) {
    try {
        std::vector<std::pair<int, double>> rec;
        for (long i = 0; i < n; ++i) rec.emplace_back(rx[i], values[i]);
        const auto a = met::per_receiver_aggregate(rec);
        *n_unique = static_cast<int>(a.per_receiver.size());
        for (std::size_t i = 0; i < a.per_receiver.size(); ++i) {
            out_rx[i] = std::get<0>(a.per_receiver[i]);
            out_mean[i] = std::get<1>(a.per_receiver[i]);
            out_count[i] = static_cast<long>(std::get<2>(a.per_receiver[i]));
        }
        *mean = a.mean;
        *stddev = a.stddev;
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

// FLE basis (radiance.cpp:79-92) at one direction, out L complex (2L f64).
void ref_eval_basis(double theta, double phi, int l_max, double* out) {
    const auto b = fle::eval_basis(theta, phi, l_max);
    for (std::size_t i = 0; i < b.b.size(); ++i) {
        out[2 * i] = b.b[i].real();
        out[2 * i + 1] = b.b[i].imag();
    }
}

// ---------------------------------------------------------------- checkpoint (io::save/load_checkpoint)
#ifdef RXGS_REF_CHECKPOINT
int ref_has_checkpoint() { return 1; }
int ref_checkpoint_save(const char* path, void* scene, void* cond, const int* gi, const double* gd, char* err,
                        int errlen) {
    try {
        train::Model m;
        m.scene = static_cast<Handle*>(scene)->scene;
        m.grid = make_grid(gi, gd);
        if (cond) {
            m.has_conditioning = true;
            m.conditioning = *static_cast<cond::ConditioningState*>(cond);
        }
        io::save_checkpoint(path, m);
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}
// Returns the scene handle (NULL on error); *cond_out = conditioning or NULL;
// gi = {n_theta, n_phi, tile_size}, gd = {radius, theta_min, theta_max}.
void* ref_checkpoint_load(const char* path, void** cond_out, int* gi, double* gd, char* err, int errlen) {
    try {
        train::Model m = io::load_checkpoint(path);
        auto* h = new Handle;
        h->scene = std::move(m.scene);
        *cond_out = m.has_conditioning ? new cond::ConditioningState(std::move(m.conditioning)) : nullptr;
        gi[0] = m.grid.n_theta;
        gi[1] = m.grid.n_phi;
        gi[2] = m.grid.tile_size;
        gd[0] = m.grid.radius;
        gd[1] = m.grid.theta_min;
        gd[2] = m.grid.theta_max;
        return h;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return nullptr;
    }
}
int ref_scene_modality(void* scene) { return static_cast<int>(static_cast<Handle*>(scene)->scene.modality); }
void ref_scene_shape(void* scene, int* out) {
    const GaussianScene& sc = static_cast<Handle*>(scene)->scene;
    out[0] = sc.count();
    out[1] = sc.l_max;
    out[2] = sc.channels;
}
void ref_cond_export(void* cond, int* cfg, double* params, double* occ, double* lo, double* hi) {
    auto* s = static_cast<cond::ConditioningState*>(cond);
    const auto& c = s->config;
    const int v[9] = {c.fourier_bands, c.hidden, c.embed_dim, c.probe_samples, s->occupancy.resolution,
                      c.nearest_lookup ? 1 : 0, static_cast<int>(c.mode), s->l_max, s->channels};
    std::memcpy(cfg, v, sizeof v);
    std::size_t off = 0;
    for_each_param(*s, [&](std::vector<double>& x) {
        if (params) std::memcpy(params + off, x.data(), x.size() * sizeof(double));
        off += x.size();
    });
    if (occ && !s->occupancy.densities.empty())
        std::memcpy(occ, s->occupancy.densities.data(), s->occupancy.densities.size() * sizeof(double));
    const auto& b = s->occupancy.bounds;
    lo[0] = b.lo.x; lo[1] = b.lo.y; lo[2] = b.lo.z;
    hi[0] = b.hi.x; hi[1] = b.hi.y; hi[2] = b.hi.z;
}
#else
int ref_has_checkpoint() { return 0; }
#endif

}  // extern "C"
