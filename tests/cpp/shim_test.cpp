// Reference-style tests written against the reference's C++ API, compiled
// against include/rxgs_b200.hpp (RXGS_B200_AS_RXGS) and run on the B200.
// Cases restate test_sphraster.cpp / test_conditioning.cpp known answers.
#define RXGS_B200_AS_RXGS
#include "rxgs_b200.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>

using namespace rxgs;
using namespace rxgs::raster;

#ifndef RXGS_SHIM_TS
#define RXGS_SHIM_TS 4
#endif
static int g_fail = 0, g_checks = 0;
#define CHECK(x)                                                            \
    do {                                                                    \
        ++g_checks;                                                         \
        if (!(x)) {                                                         \
            ++g_fail;                                                       \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #x);        \
        }                                                                   \
    } while (0)

static double rel_err(double a, double b) {
    return std::abs(a - b) / std::max({1.0, std::abs(a), std::abs(b)});
}

static GaussianScene random_scene(unsigned seed, int k, int l_max, int channels) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(0.0, 1.0);
    std::normal_distribution<double> nrm(0.0, 1.0);
    GaussianScene s;
    s.l_max = l_max;
    s.channels = channels;
    for (int i = 0; i < k; ++i) {
        double x = 1.0 + 3.0 * u(rng);
        if (u(rng) < 0.5) x = -x;
        s.positions.insert(s.positions.end(), {x, -3.0 + 6.0 * u(rng), -2.0 + 4.0 * u(rng)});
        for (int a = 0; a < 3; ++a) s.log_scales.push_back(-1.8 + 1.2 * u(rng));
        double q[4], n = 0;
        for (double& v : q) { v = nrm(rng); n += v * v; }
        for (double v : q) s.quaternions.push_back(v / std::sqrt(n));
        s.tau_logits.push_back(-2.0 + 3.0 * u(rng));
    }
    s.fle_coeffs.resize(static_cast<std::size_t>(k) * s.coeff_stride());
    for (double& c : s.fle_coeffs) c = nrm(rng);
    return s;
}

static SphericalGrid small_grid() {
    SphericalGrid g;
    g.n_theta = 6;
    g.n_phi = 12;
    g.tile_size = 4;
    g.radius = 0.25;
    return g;
}

int main() {
    {  // projection: axis direction (test_sphraster.cpp:59-66) + culling (:88-94)
        GaussianScene s;
        s.positions = {1, 0, 0, 0.1, 0, 0};
        s.log_scales = {std::log(0.1), std::log(0.1), std::log(0.1), 0, 0, 0};
        s.quaternions = {1, 0, 0, 0, 1, 0, 0, 0};
        s.tau_logits = {0, 0};
        s.fle_coeffs = {0, 0, 0, 0};
        const auto st = build_tx_state(s, {0, 0, 0}, small_grid());
        CHECK(!st.proj[0].culled);
        CHECK(rel_err(st.proj[0].theta, kPi / 2) < 1e-14);
        CHECK(std::abs(st.proj[0].phi) < 1e-14);
        CHECK(st.proj[1].culled);
    }
    {  // bin_and_sort: coverage, depth order, index tiebreak (test_sphraster.cpp:96-119)
        std::vector<ProjectedGaussian> proj(3);
        for (auto& p : proj) p.culled = false;
        proj[0].depth = 2.0; proj[0].t0 = 0; proj[0].t1 = 1; proj[0].p0 = 0; proj[0].p1 = 2;
        proj[1].depth = 1.0; proj[1].t0 = 0; proj[1].t1 = 0; proj[1].p0 = 1; proj[1].p1 = 1;
        proj[2].depth = 2.0; proj[2].t0 = 0; proj[2].t1 = 0; proj[2].p0 = 1; proj[2].p1 = 1;
        const auto lists = bin_and_sort(proj, small_grid());
        CHECK(lists.size() == 6);
        CHECK((lists[1] == std::vector<int>{1, 0, 2}));
        std::vector<ProjectedGaussian> seam(1);
        seam[0].culled = false; seam[0].depth = 1.0; seam[0].t0 = 0; seam[0].t1 = 0; seam[0].p0 = 2; seam[0].p1 = 3;
        const auto l2 = bin_and_sort(seam, small_grid());
        CHECK((l2[0] == std::vector<int>{0}) && l2[1].empty() && (l2[2] == std::vector<int>{0}));
    }
    {  // render: batched == sequential bitwise (test_sphraster.cpp:180-199)
        const auto scene = random_scene(41, 6, 2, 2);
        const int n_rx = 3;
        std::vector<double> coeffs(n_rx * scene.count() * scene.coeff_stride());
        std::mt19937_64 rng(42);
        std::normal_distribution<double> nrm(0.0, 1.0);
        for (double& c : coeffs) c = nrm(rng);
        const auto batched = render_field(scene, {0, 0, 0}, small_grid(), coeffs, n_rx);
        const std::size_t stride = scene.coeff_stride() * scene.count();
        for (int j = 0; j < n_rx; ++j) {
            const std::vector<double> slice(coeffs.begin() + j * stride, coeffs.begin() + (j + 1) * stride);
            const auto single = render_field(scene, {0, 0, 0}, small_grid(), slice, 1);
            const std::size_t per_rx = static_cast<std::size_t>(scene.channels) * 2 * batched.plane();
            bool same = true;
            for (std::size_t i = 0; i < per_rx; ++i) same &= batched.values[j * per_rx + i] == single.values[i];
            CHECK(same);
        }
    }
    {  // located non-finite error (test_sphraster.cpp:211-223)
        const auto scene = random_scene(45, 3, 1, 1);
        std::vector<double> coeffs(2 * scene.count() * scene.coeff_stride(), 0.5);
        coeffs[scene.coeff_stride() * scene.count() + 5] = std::nan("");
        bool threw = false;
        try {
            render_field(scene, {0, 0, 0}, small_grid(), coeffs, 2);
        } catch (const std::invalid_argument& e) {
            threw = std::string(e.what()).find("rx 1") != std::string::npos &&
                    std::string(e.what()).find("gaussian 0") != std::string::npos;
        }
        CHECK(threw);
    }
    {  // empty scene (test_sphraster.cpp:170-178)
        GaussianScene s;
        s.l_max = 1;
        const auto f = render_field(s, {0, 0, 0}, small_grid(), {}, 2);
        bool ok = true;
        for (double v : f.values) ok &= v == 0.0;
        for (double t : f.transmittance) ok &= t == 1.0;
        CHECK(ok);
    }
    {  // spectrum stabiliser (test_sphraster.cpp:289-303)
        RenderedField f;
        f.n_rx = 1; f.channels = 1; f.h = 1; f.w = 1;
        f.values = {3.0, 4.0};
        f.transmittance = {1.0};
        SphericalGrid g;
        const auto ms = aggregate_modality(f, Modality::Spectrum, g);
        CHECK(rel_err(ms[0].image[0], std::sqrt(25.0 + 1e-8)) < 1e-15);
    }
    {  // conditioning: zero final layers = identity, bitwise (test_conditioning.cpp:157-169)
        auto scene = random_scene(101, 5, 1, 2);
        cond::ConditioningState st;
        st.config.fourier_bands = 2; st.config.hidden = 8; st.config.embed_dim = 3; st.config.probe_samples = 4;
        st.l_max = 1; st.channels = 2;
        st.fourier_freqs.assign(6, 1.0);
        auto layer = [](int in, int out, double v) { cond::MlpLayer l; l.in = in; l.out = out; l.w.assign(in * out, v); l.b.assign(out, 0.1); return l; };
        st.global_mlp = {layer(6 * 2 + 2 + 3, 8, 0.05), layer(8, 8, 0.05), layer(8, 8, 0.0)};
        st.global_mlp.l3.b.assign(8, 0.0);
        st.component_embed.assign(4 * 3, 0.01);
        st.local_mlp = {layer(6, 8, 0.05), layer(8, 8, 0.05), layer(8, 8, 0.0)};
        st.local_mlp.l3.b.assign(8, 0.0);
        st.occupancy = cond::build_occupancy(scene, 8, {{-4, -4, -4}, {4, 4, 4}});
        const auto out = cond::condition_forward(st, scene.fle_coeffs, scene, {0.3, 0.2, -1.0});
        CHECK(out == scene.fle_coeffs);
        CHECK(st.global_calls == 4 && st.local_calls == 5);
        bool threw = false;
        try {
            cond::condition_forward(st, scene.fle_coeffs, scene, scene.position(1));
        } catch (const std::invalid_argument& e) {
            threw = std::string(e.what()).find("gaussian 1") != std::string::npos;
        }
        CHECK(threw);
        // io::save_checkpoint / load_checkpoint round trip (checkpoint.cpp:93-231)
        train::Model m;
        m.scene = scene;
        m.grid = small_grid();
        m.has_conditioning = true;
        m.conditioning = st;
        const std::string path = "/tmp/rxgs_shim_ckpt.rxgs";
        io::save_checkpoint(path, m);
        const train::Model back = io::load_checkpoint(path);
        CHECK(back.scene.positions == m.scene.positions && back.scene.fle_coeffs == m.scene.fle_coeffs);
        CHECK(back.scene.tau_logits == m.scene.tau_logits && back.scene.l_max == 1 && back.scene.channels == 2);
        CHECK(back.grid.n_theta == m.grid.n_theta && back.grid.theta_max == m.grid.theta_max);
        CHECK(back.has_conditioning && back.conditioning.local_mlp.l2.w == st.local_mlp.l2.w);
        CHECK(back.conditioning.occupancy.densities == st.occupancy.densities);
        CHECK(back.conditioning.occupancy.bounds.hi.z == 4.0 && back.conditioning.config.hidden == 8);
        bool io_threw = false;
        try {
            io::load_checkpoint("/tmp/rxgs_shim_no_such_file.rxgs");
        } catch (const io::IoError& e) {
            io_threw = std::string(e.what()).find("load_checkpoint: cannot open") != std::string::npos;
        }
        CHECK(io_threw);
    }
    {  // adjoints through the shim (test_sphraster_grad.cpp:116-250 style): FD of
       // L = sum(spectrum) w.r.t. a tau logit, a position and a coefficient
        GaussianScene s = random_scene(11, 25, 1, 1);
        s.modality = Modality::Spectrum;
        SphericalGrid g;
        g.n_theta = 12;
        g.n_phi = 24;
        g.tile_size = RXGS_SHIM_TS;
        g.radius = 0.25;
        const Vec3 tx{0.2, -0.1, 0.05};
        auto loss = [&](const GaussianScene& sc) {
            const auto f = render_field(sc, tx, g, sc.fle_coeffs, 1);
            const auto m = aggregate_modality(f, Modality::Spectrum, g)[0];
            double a = 0;
            for (double v : m.image) a += v;
            return a;
        };
        const auto st = build_tx_state(s, tx, g);
        const auto f = render_field(st, s, s.fle_coeffs, 1);
        Measurement up;
        up.modality = Modality::Spectrum;
        up.image.assign(f.plane(), 1.0);
        const auto dv = aggregate_modality_backward(f, Modality::Spectrum, g, {up});
        const auto gb = backward_render(st, s, s.fle_coeffs, 1, dv);
        // the B200 render carries signals in FP32, so the FD step is 1e-3
        // (FP32 quantisation of a 1e-6 step alone is ~10%)
        const double h = 1e-3;
        int k = 0;
        while (k < s.count() && st.proj[k].culled) ++k;
        {
            GaussianScene p = s, m = s;
            p.tau_logits[k] += h;
            m.tau_logits[k] -= h;
            CHECK(rel_err((loss(p) - loss(m)) / (2 * h), gb.d_tau_logits[k]) < 2e-3);
        }
        {
            GaussianScene p = s, m = s;
            p.fle_coeffs[k * s.coeff_stride() + 2] += h;
            m.fle_coeffs[k * s.coeff_stride() + 2] -= h;
            CHECK(rel_err((loss(p) - loss(m)) / (2 * h), gb.d_coeffs[k * s.coeff_stride() + 2]) < 2e-3);
        }
        // condition_backward: FD of sum(out * w) w.r.t. a base coefficient
        cond::ConditioningState cs;
        cs.config.fourier_bands = 2; cs.config.hidden = 8; cs.config.embed_dim = 3; cs.config.probe_samples = 4;
        cs.l_max = 1; cs.channels = 1;
        cs.fourier_freqs.assign(6, 0.7);
        auto layer = [](int in, int out, double v) { cond::MlpLayer l; l.in = in; l.out = out; l.w.assign(in * out, v); l.b.assign(out, 0.05); return l; };
        cs.global_mlp = {layer(6 * 2 + 2 + 3, 8, 0.04), layer(8, 8, -0.03), layer(8, 4, 0.02)};
        cs.component_embed.assign(4 * 3, 0.01);
        cs.local_mlp = {layer(6, 8, 0.05), layer(8, 8, 0.04), layer(8, 4, -0.03)};
        cs.occupancy = cond::build_occupancy(s, 8, {{-4, -4, -4}, {4, 4, 4}});
        const Vec3 rx{0.3, 0.2, -0.9};
        cond::ConditionWorkspace ws;
        const auto out = cond::condition_forward(cs, s.fle_coeffs, s, rx, &ws);
        CHECK(ws.local_in.size() == 6 * static_cast<std::size_t>(s.count()));
        std::vector<double> w(out.size());
        for (std::size_t i = 0; i < w.size(); ++i) w[i] = std::sin(0.37 * i);
        std::vector<double> d_base(out.size(), 0.0);
        cond::ConditioningGrads grads;
        cond::condition_backward(cs, ws, s.fle_coeffs, w, d_base, grads);
        auto obj = [&](const std::vector<double>& base) {
            const auto o = cond::condition_forward(cs, base, s, rx);
            double a = 0;
            for (std::size_t i = 0; i < o.size(); ++i) a += o[i] * w[i];
            return a;
        };
        std::vector<double> bp = s.fle_coeffs, bm = s.fle_coeffs;
        const double hc = 1e-6;  // the materialised conditioning path is FP64
        bp[5] += hc;
        bm[5] -= hc;
        CHECK(rel_err((obj(bp) - obj(bm)) / (2 * hc), d_base[5]) < 1e-4);
        CHECK(grads.d_local.w2.size() == 64 && grads.d_global.b3.size() == 4);
    }
    {  // Stage-I densification: test_scene.cpp:175-245 restated on the shim
        auto cloud = [](std::vector<Vec3> pts, double ls) {
            GaussianScene s;
            s.l_max = 0;
            for (const Vec3& p : pts) {
                s.positions.insert(s.positions.end(), {p.x, p.y, p.z});
                s.log_scales.insert(s.log_scales.end(), {ls, ls, ls});
                s.quaternions.insert(s.quaternions.end(), {1.0, 0.0, 0.0, 0.0});
                s.tau_logits.push_back(std::log(0.1 / 0.9));
            }
            s.fle_coeffs.assign(static_cast<std::size_t>(s.count()) * s.coeff_stride(), 0.0);
            return s;
        };
        {  // below threshold: no-op
            auto s = cloud({{0, 0, 0}, {1, 0, 0}, {0, 1, 0}}, 0.0);
            DensifyState st;
            st.resize(3);
            st.scene_extent = 10.0;
            st.accumulate(std::vector<double>(9, 1e-9));
            const auto before = s.positions;
            const auto r = densify_and_prune(s, st, {}, 1, 0);
            CHECK(s.count() == 3 && s.positions == before && r.cloned == 0 && r.split == 0 && r.pruned == 0);
            CHECK((r.source_row == std::vector<int>{0, 1, 2}));
        }
        {  // small Gaussian cloned
            auto s = cloud({{0, 0, 0}, {1, 0, 0}}, 0.0);
            DensifyState st;
            st.resize(2);
            st.scene_extent = 1000.0;
            st.accumulate({1.0, 0, 0, 0, 0, 0});
            const auto r = densify_and_prune(s, st, {}, 1, 0);
            CHECK(r.cloned == 1 && s.count() == 3);
            CHECK(s.positions[6] == s.positions[0] && s.positions[7] == s.positions[1] && s.positions[8] == s.positions[2]);
            CHECK((r.source_row == std::vector<int>{0, 1, -1}));
            CHECK(st.grad_accum.size() == 3);
        }
        {  // large Gaussian splits: children 2 sigma apart, scales shrunk by 0.8
            auto s = cloud({{0, 0, 0}, {1, 0, 0}}, 0.0);
            s.log_scales[0] = s.log_scales[1] = s.log_scales[2] = std::log(0.5);
            DensifyState st;
            st.resize(2);
            st.scene_extent = 10.0;
            st.accumulate({1.0, 0, 0, 0, 0, 0});
            const auto r = densify_and_prune(s, st, {}, 1, 0);
            CHECK(r.split == 1 && s.count() == 3);
            CHECK(rel_err(s.log_scales[0], std::log(0.5) + std::log(0.8)) < 1e-12);
            const double dx = s.positions[0] - s.positions[6], dy = s.positions[1] - s.positions[7],
                         dz = s.positions[2] - s.positions[8];
            CHECK(rel_err(std::sqrt(dx * dx + dy * dy + dz * dz), 1.0) < 1e-12);
        }
        {  // oversized pruned
            auto s = cloud({{0, 0, 0}, {1, 0, 0}, {0, 1, 0}}, std::log(5.0));
            DensifyState st;
            st.resize(3);
            st.scene_extent = 10.0;
            st.accumulate(std::vector<double>(9, 0.0));
            const auto r = densify_and_prune(s, st, {}, 1, 0);
            CHECK(r.pruned == 3 && s.count() == 0 && st.grad_accum.empty());
        }
        {  // reset_transmittance: tau = 0.01, idempotent (test_scene.cpp:164-173)
            auto s = cloud({{0, 0, 0}, {1, 0, 0}, {0, 2, 0}}, 0.0);
            reset_transmittance(s);
            for (double v : s.tau_logits) CHECK(rel_err(1.0 / (1.0 + std::exp(-v)), 0.01) < 1e-12);
            const auto once = s.tau_logits;
            reset_transmittance(s);
            CHECK(s.tau_logits == once);
        }
        bool threw = false;
        try {
            auto s = cloud({{0, 0, 0}, {1, 0, 0}}, 0.0);
            DensifyState st;
            st.resize(3);
            densify_and_prune(s, st, {}, 1, 0);
        } catch (const std::invalid_argument& e) {
            threw = std::string(e.what()) == "densify_and_prune: state size mismatch";
        }
        CHECK(threw);
    }
    {  // metrics (test_metrics.cpp-style known answers)
        std::vector<double> a = {1, 2, 3, 4}, b = {1, 2, 3, 6};
        CHECK(rel_err(met::mae(a, b), 0.5) < 1e-15);
        CHECK(rel_err(met::mse(a, b), 1.0) < 1e-15);
        CHECK(rel_err(met::psnr(a, b, 2.0), 10.0 * std::log10(4.0)) < 1e-14);
        CHECK(met::psnr(a, a, 1.0) == met::kDbSentinel);
        std::vector<double> img(16 * 16), img2(16 * 16);
        for (std::size_t i = 0; i < img.size(); ++i) {
            img[i] = std::sin(0.1 * i);
            img2[i] = img[i] + 0.05 * std::cos(0.7 * i);
        }
        CHECK(rel_err(met::ssim(img, img, 16, 16), 1.0) < 1e-14);
        const double s1 = met::ssim(img, img2, 16, 16);
        CHECK(s1 < 1.0 && s1 > 0.5);
        bool threw = false;
        try {
            met::ssim(std::vector<double>(100, 0.0), std::vector<double>(100, 0.0), 10, 10);
        } catch (const std::invalid_argument& e) {
            threw = std::string(e.what()) == "ssim: image smaller than the window";
        }
        CHECK(threw);
    }
    {  // project_gaussian: isotropic sigma^2/d^2 (test_sphraster.cpp:68-77), culling (:88-94)
        const std::array<double, 9> cov = {0.04, 0, 0, 0, 0.04, 0, 0, 0, 0.04};
        const auto pg = project_gaussian({0, 2, 0}, cov, 0.5, {0, 0, 0}, small_grid());
        CHECK(!pg.culled);
        CHECK(rel_err(pg.angular_cov.a, 0.04 / 4.0) < 1e-12);
        CHECK(rel_err(pg.angular_cov.d, 0.04 / 4.0) < 1e-12);
        CHECK(std::abs(pg.angular_cov.b) < 1e-15);
        CHECK(project_gaussian({0.1, 0, 0}, cov, 0.5, {0, 0, 0}, small_grid()).culled);
    }
    {  // blend_ray closed forms (test_sphraster.cpp:134-142)
        const auto one = blend_ray({0.5}, {cplx{1, 0}});
        CHECK(one.c == cplx(0.5, 0.0) && one.transmittance == 0.5);
        const auto two = blend_ray({0.5, 0.25}, {cplx{1, 0}, cplx{2, 0}});
        CHECK(rel_err(two.c.real(), 0.75) < 1e-15 && rel_err(two.transmittance, 0.375) < 1e-15);
    }
    {  // TxState::hash is receiver-invariant (test_sphraster.cpp:225-237)
        const auto scene = random_scene(47, 5, 2, 1);
        const auto s1 = build_tx_state(scene, {0, 0, 0}, small_grid());
        const auto s2 = build_tx_state(scene, {0, 0, 0}, small_grid());
        CHECK(s1.hash() == s2.hash());
        const auto s3 = build_tx_state(scene, {0.1, 0, 0}, small_grid());
        CHECK(s1.hash() != s3.hash());
    }
    {  // probe_segment 0.9^16 (test_conditioning.cpp:114-133), init_conditioning ladder (:67-76)
        cond::OccupancyGrid u;
        u.resolution = 4;
        u.bounds = {{-10, -10, -10}, {10, 10, 10}};
        u.densities.assign(64, 0.1);
        const auto pr = cond::probe_segment(u, {-5, 0, 0}, {5, 0, 0}, 16);
        CHECK(rel_err(pr.transmittance, std::pow(0.9, 16)) < 1e-12);
        CHECK(rel_err(pr.mean_density, 0.1) < 1e-12);
        cond::ConditioningConfig cfg;
        cfg.fourier_bands = 2;
        cfg.hidden = 8;
        cfg.embed_dim = 3;
        const auto st = cond::init_conditioning(cfg, 1, 1, {{0, 0, 0}, {4, 2, 1}}, 5);
        CHECK(rel_err(st.fourier_freqs[0], kTwoPi / 4.0) < 1e-15);
        CHECK(rel_err(st.fourier_freqs[1], kTwoPi / 2.0) < 1e-15);
        bool zero = true;
        for (double w : st.local_mlp.l3.w) zero = zero && w == 0.0;
        CHECK(zero);
        const auto enc = cond::fourier_encode({0, 0, 0}, std::vector<double>(18, 1.7));
        CHECK(enc.size() == 36 && enc[0] == 0.0 && enc[1] == 1.0);
    }
    {  // fle::eval_basis closed forms (test_radiance.cpp:99-126)
        const auto b = fle::eval_basis(0.3, 1.1, 1);
        CHECK(rel_err(b.at(0).real(), 0.2820947917738781) < 1e-15 && b.at(0).imag() == 0.0);
        CHECK(rel_err(b.at(2).real(), 0.4886025119029199 * std::cos(0.3)) < 1e-14);
        CHECK(rel_err(fle::normalization(1, 0), 0.4886025119029199) < 1e-15);
    }
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
