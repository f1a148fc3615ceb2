/* oracle/rxgs_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, not the product).
 *
 * Plain-C restatement of the RxGS reference render path.  See rxgs_oracle.h.
 * Reference citations are relative to /root/reference/proj.
 * Parity pinning: tests/test_oracle.py compares every entry point here with
 * the reference itself (oracle/_ref/librxgs_ref.so, built from the reference
 * sources by oracle/Makefile) and with the committed fixtures in
 * tests/golden/ (generated from the reference by tests/golden/make_golden.py).
 */
#include "rxgs_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define K_PI 3.14159265358979323846
#define K_TWO_PI (2.0 * K_PI)
#define K_WEIGHT_CLAMP 0.999 /* sphraster.hpp:72 */
#define K_EARLY_EXIT_T 1e-4  /* sphraster.hpp:73 */
#define K_RSSI_FLOOR 1e-12   /* channelsim.hpp:115 */
#define K_AMP_EPS 1e-8       /* radiance.hpp:80 */

int or_abi_version(void) { return 3; }

static void set_err(char* err, int errlen, const char* msg) {
    if (err && errlen > 0) snprintf(err, (size_t)errlen, "%s", msg);
}

/* ------------------------------------------------------------------ rng
 * SplitMix64 stream + FNV-1a tag hashing: rng.hpp:17-72. */
typedef struct { uint64_t s; } rng_t;

static uint64_t rng_next(rng_t* r) {
    r->s += 0x9e3779b97f4a7c15ull;
    uint64_t z = r->s;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
static double rng_u01(rng_t* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }
static double rng_uniform(rng_t* r, double lo, double hi) { return lo + (hi - lo) * rng_u01(r); }
static double rng_normal(rng_t* r) { /* rng.hpp:39-44 (Box-Muller, u1 > 0) */
    double u1 = rng_u01(r);
    while (u1 <= 0.0) u1 = rng_u01(r);
    const double u2 = rng_u01(r);
    return sqrt(-2.0 * log(u1)) * cos(6.28318530717958647692 * u2);
}
static uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
static rng_t derive_stream(uint64_t seed, const char* tag, uint64_t counter) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (const unsigned char* p = (const unsigned char*)tag; *p; ++p) {
        h ^= *p;
        h *= 0x100000001b3ull;
    }
    h = mix64(h ^ mix64(seed));
    h = mix64(h ^ mix64(counter ^ 0xa5a5a5a5a5a5a5a5ull));
    rng_t r = {h};
    return r;
}

/* ------------------------------------------------------------------ small helpers */
static double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); } /* linalg.hpp:157 */
static double wrap_pm_pi(double a) {                                 /* linalg.hpp:152-157 */
    a = fmod(a, K_TWO_PI);
    if (a > K_PI) a -= K_TWO_PI;
    if (a <= -K_PI) a += K_TWO_PI;
    return a;
}
static double wrap_two_pi(double a) { /* linalg.hpp:160-164 */
    a = fmod(a, K_TWO_PI);
    if (a < 0.0) a += K_TWO_PI;
    return a;
}
static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }
static double dmax(double a, double b) { return a < b ? b : a; } /* std::max(a, b) */
static int n_comp(int l_max) { return (l_max + 1) * (l_max + 1); }

/* 3x3 row-major helpers with the reference's operation order (linalg.hpp:46-104). */
static void mat3_vec(const double* m, const double* v, double* o) {
    o[0] = m[0] * v[0] + m[1] * v[1] + m[2] * v[2];
    o[1] = m[3] * v[0] + m[4] * v[1] + m[5] * v[2];
    o[2] = m[6] * v[0] + m[7] * v[1] + m[8] * v[2];
}
static double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

/* quat_to_rotation: linalg.hpp:122-131 */
static void quat_to_rotation(const double* q, double* r) {
    const double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    const double w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
    r[0] = 1 - 2 * (y * y + z * z); r[1] = 2 * (x * y - w * z);     r[2] = 2 * (x * z + w * y);
    r[3] = 2 * (x * y + w * z);     r[4] = 1 - 2 * (x * x + z * z); r[5] = 2 * (y * z - w * x);
    r[6] = 2 * (x * z - w * y);     r[7] = 2 * (y * z + w * x);     r[8] = 1 - 2 * (x * x + y * y);
}

/* covariance_from: scene.cpp:42-51, Sigma = (R diag(e^s)) (R diag(e^s))^T */
static void covariance_from(const double* ls, const double* q, double* sig) {
    double m[9];
    quat_to_rotation(q, m);
    for (int row = 0; row < 3; ++row)
        for (int col = 0; col < 3; ++col) m[row * 3 + col] *= exp(ls[col]);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0.0;
            for (int k = 0; k < 3; ++k) s += m[i * 3 + k] * m[j * 3 + k];
            sig[i * 3 + j] = s;
        }
}

static void mat3_inverse(const double* m, double* r) { /* linalg.hpp:88-100 */
    const double d = m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
                     m[2] * (m[3] * m[7] - m[4] * m[6]);
    r[0] = (m[4] * m[8] - m[5] * m[7]) / d; r[1] = (m[2] * m[7] - m[1] * m[8]) / d;
    r[2] = (m[1] * m[5] - m[2] * m[4]) / d; r[3] = (m[5] * m[6] - m[3] * m[8]) / d;
    r[4] = (m[0] * m[8] - m[2] * m[6]) / d; r[5] = (m[2] * m[3] - m[0] * m[5]) / d;
    r[6] = (m[3] * m[7] - m[4] * m[6]) / d; r[7] = (m[1] * m[6] - m[0] * m[7]) / d;
    r[8] = (m[0] * m[4] - m[1] * m[3]) / d;
}

/* ------------------------------------------------------------------ generators
 * DESIGN.md section 5 (identical to oracle/ref_harness.cpp). */
void or_synth_scene(int k, int l_max, int channels, uint64_t seed, double* pos, double* ls,
                    double* q, double* tau, double* coeffs) {
    rng_t rng = derive_stream(seed, "bench.scene", 0);
    const double base = log(0.554 * cbrt(144.0 / (double)k));
    for (int i = 0; i < k; ++i) {
        pos[3 * i + 0] = rng_uniform(&rng, -4.0, 4.0);
        pos[3 * i + 1] = rng_uniform(&rng, -3.0, 3.0);
        pos[3 * i + 2] = rng_uniform(&rng, -1.5, 1.5);
        for (int a = 0; a < 3; ++a) ls[3 * i + a] = base + rng_uniform(&rng, -0.3, 0.3);
        double qq[4];
        for (int a = 0; a < 4; ++a) qq[a] = rng_normal(&rng);
        const double n = sqrt(qq[0] * qq[0] + qq[1] * qq[1] + qq[2] * qq[2] + qq[3] * qq[3]);
        for (int a = 0; a < 4; ++a) q[4 * i + a] = qq[a] / n;
        tau[i] = rng_uniform(&rng, -2.0, 1.0);
    }
    rng_t crng = derive_stream(seed, "bench.scene.coeffs", 0);
    const size_t n = (size_t)k * n_comp(l_max) * channels * 2;
    for (size_t i = 0; i < n; ++i) coeffs[i] = rng_normal(&crng);
}

void or_synth_points(int n, uint64_t seed, const char* tag, const double* lo, const double* hi,
                     double margin, double* out) {
    rng_t rng = derive_stream(seed, tag, 0);
    double a[3], b[3];
    for (int d = 0; d < 3; ++d) {
        const double ext = hi[d] - lo[d];
        a[d] = lo[d] + margin * ext;
        b[d] = hi[d] - margin * ext;
    }
    for (int i = 0; i < n; ++i)
        for (int d = 0; d < 3; ++d) out[3 * i + d] = rng_uniform(&rng, a[d], b[d]);
}

/* Packed conditioning layout (see ref_harness.cpp header). */
typedef struct {
    int F, d, dc, S, R, nearest, mode, l_max, C, L, gin;
    size_t o_freq, o_gw1, o_gb1, o_gw2, o_gb2, o_gw3, o_gb3, o_emb, o_lw1, o_lb1, o_lw2, o_lb2,
        o_lw3, o_lb3, total;
} cond_layout;

static cond_layout make_layout(const int* cfg, int l_max, int channels) {
    cond_layout c;
    c.F = cfg[0]; c.d = cfg[1]; c.dc = cfg[2]; c.S = cfg[3]; c.R = cfg[4];
    c.nearest = cfg[5]; c.mode = cfg[6]; c.l_max = l_max; c.C = channels;
    c.L = n_comp(l_max);
    c.gin = 6 * c.F + 2 + c.dc;
    size_t o = 0;
    c.o_freq = o; o += (size_t)c.F * 3;
    c.o_gw1 = o; o += (size_t)c.d * c.gin;
    c.o_gb1 = o; o += (size_t)c.d;
    c.o_gw2 = o; o += (size_t)c.d * c.d;
    c.o_gb2 = o; o += (size_t)c.d;
    c.o_gw3 = o; o += (size_t)4 * c.C * c.d;
    c.o_gb3 = o; o += (size_t)4 * c.C;
    c.o_emb = o; o += (size_t)c.L * c.dc;
    c.o_lw1 = o; o += (size_t)c.d * 6;
    c.o_lb1 = o; o += (size_t)c.d;
    c.o_lw2 = o; o += (size_t)c.d * c.d;
    c.o_lb2 = o; o += (size_t)c.d;
    c.o_lw3 = o; o += (size_t)4 * c.C * c.d;
    c.o_lb3 = o; o += (size_t)4 * c.C;
    c.total = o;
    return c;
}

/* init_conditioning: conditioning.cpp:217-253 (+ bench overwrite). */
long or_synth_cond(const int* cfg, int l_max, int channels, const double* blo, const double* bhi,
                   uint64_t seed, int randomize, double* p) {
    const cond_layout c = make_layout(cfg, l_max, channels);
    if (!p) return (long)c.total;
    memset(p, 0, c.total * sizeof(double));
    for (int band = 0; band < c.F; ++band)
        for (int a = 0; a < 3; ++a) {
            const double ext = bhi[a] - blo[a];
            const double e = ext > 0.0 ? ext : 1.0;
            p[c.o_freq + (size_t)band * 3 + a] = pow(2.0, band) * K_TWO_PI / e;
        }
    /* make_layer: conditioning.cpp:202-213; w1 and w3 share a stream, w3 zeroed */
    struct { const char* tag; size_t off; int in, out; } init[4] = {
        {"cond.global.w1", c.o_gw1, c.gin, c.d}, {"cond.global.w2", c.o_gw2, c.d, c.d},
        {"cond.local.w1", c.o_lw1, 6, c.d}, {"cond.local.w2", c.o_lw2, c.d, c.d}};
    for (int i = 0; i < 4; ++i) {
        rng_t r = derive_stream(seed, init[i].tag, 0);
        const double sc = 1.0 / sqrt((double)init[i].in);
        for (int e = 0; e < init[i].in * init[i].out; ++e)
            p[init[i].off + (size_t)e] = rng_uniform(&r, -sc, sc);
    }
    rng_t er = derive_stream(seed, "cond.embed", 0);
    for (int e = 0; e < c.L * c.dc; ++e) p[c.o_emb + (size_t)e] = 0.1 * rng_normal(&er);
    if (randomize) {
        const char* names[2] = {"global", "local"};
        const size_t ow[2][3] = {{c.o_gw1, c.o_gw2, c.o_gw3}, {c.o_lw1, c.o_lw2, c.o_lw3}};
        const size_t ob[2][3] = {{c.o_gb1, c.o_gb2, c.o_gb3}, {c.o_lb1, c.o_lb2, c.o_lb3}};
        const int fin[2][3] = {{c.gin, c.d, c.d}, {6, c.d, c.d}};
        const int fout[3] = {c.d, c.d, 4 * c.C};
        char tag[64];
        for (int m = 0; m < 2; ++m)
            for (int li = 0; li < 3; ++li) {
                snprintf(tag, sizeof tag, "bench.cond.%s.w%d", names[m], li + 1);
                rng_t rw = derive_stream(seed, tag, 0);
                snprintf(tag, sizeof tag, "bench.cond.%s.b%d", names[m], li + 1);
                rng_t rb = derive_stream(seed, tag, 0);
                const double sc = 1.0 / sqrt((double)fin[m][li]);
                for (int e = 0; e < fin[m][li] * fout[li]; ++e)
                    p[ow[m][li] + (size_t)e] = rng_uniform(&rw, -1.0, 1.0) * sc;
                for (int e = 0; e < fout[li]; ++e)
                    p[ob[m][li] + (size_t)e] = li < 2 ? 0.1 * rng_normal(&rb) : 0.0;
            }
    }
    return (long)c.total;
}

/* ------------------------------------------------------------------ scene */
typedef struct {
    int k, l_max, C, modality;
    double *pos, *ls, *q, *tau, *coeffs;
} scene_t;

static double* dup(const double* src, size_t n) {
    double* d = (double*)malloc((n ? n : 1) * sizeof(double));
    if (n) memcpy(d, src, n * sizeof(double));
    return d;
}

void* or_scene_new(int k, int l_max, int channels, int modality, const double* pos,
                   const double* ls, const double* q, const double* tau, const double* coeffs) {
    scene_t* s = (scene_t*)calloc(1, sizeof(scene_t));
    s->k = k; s->l_max = l_max; s->C = channels; s->modality = modality;
    s->pos = dup(pos, 3 * (size_t)k);
    s->ls = dup(ls, 3 * (size_t)k);
    s->q = dup(q, 4 * (size_t)k);
    s->tau = dup(tau, (size_t)k);
    s->coeffs = dup(coeffs, (size_t)k * n_comp(l_max) * channels * 2);
    return s;
}
void or_scene_free(void* h) {
    scene_t* s = (scene_t*)h;
    if (!s) return;
    free(s->pos); free(s->ls); free(s->q); free(s->tau); free(s->coeffs);
    free(s);
}
/* position_bounds().inflated(f): scene.cpp:18-30, linalg.hpp:143-147 */
void or_scene_bounds(void* h, double inflate, double* lo, double* hi) {
    const scene_t* s = (const scene_t*)h;
    for (int a = 0; a < 3; ++a) { lo[a] = 1.7976931348623157e308; hi[a] = -1.7976931348623157e308; }
    for (int k = 0; k < s->k; ++k)
        for (int a = 0; a < 3; ++a) {
            const double v = s->pos[3 * k + a];
            lo[a] = lo[a] < v ? lo[a] : v;
            hi[a] = hi[a] < v ? v : hi[a];
        }
    for (int a = 0; a < 3; ++a) {
        const double pad = (hi[a] - lo[a]) * (0.5 * inflate);
        lo[a] = lo[a] - pad;
        hi[a] = hi[a] + pad;
    }
}
void or_covariance(void* h, double* out) {
    const scene_t* s = (const scene_t*)h;
    for (int k = 0; k < s->k; ++k) covariance_from(s->ls + 3 * k, s->q + 4 * k, out + 9 * (size_t)k);
}

/* ------------------------------------------------------------------ projection
 * project_gaussian: sphraster.cpp:22-83.  geom[12] = theta, phi, depth,
 * cov a b c d, prec a b c d, weight_scale.  spans = t0 t1 p0 p1. */
typedef struct { int nt, np, ts; double radius, tmin, tmax; } grid_t;
static grid_t mkgrid(const int* gi, const double* gd) {
    grid_t g = {gi[0], gi[1], gi[2], gd[0], gd[1], gd[2]};
    return g;
}
static double g_dtheta(const grid_t* g) { return (g->tmax - g->tmin) / g->nt; }
static double g_dphi(const grid_t* g) { return K_TWO_PI / g->np; }
static int g_tiles_t(const grid_t* g) { return (g->nt + g->ts - 1) / g->ts; }
static int g_tiles_p(const grid_t* g) { return (g->np + g->ts - 1) / g->ts; }

static int project_one(const double* p, const double* cov, double tau, const double* tx,
                       const grid_t* g, double* geom, int* span) {
    memset(geom, 0, 12 * sizeof(double));
    span[0] = 0; span[1] = -1; span[2] = 0; span[3] = -1;
    const double u[3] = {p[0] - tx[0], p[1] - tx[1], p[2] - tx[2]};
    const double d = sqrt(dot3(u, u));
    if (!(d >= g->radius) || d == 0.0) return 1;
    const double rho = sqrt(u[0] * u[0] + u[1] * u[1]);
    const double theta = atan2(rho, u[2]);
    const double phi = wrap_two_pi(atan2(u[1], u[0]));
    geom[0] = theta; geom[1] = phi; geom[2] = d; geom[11] = tau;
    const double st = sin(theta), ct = cos(theta), sp = sin(phi), cp = cos(phi);
    const double et[3] = {ct * cp, ct * sp, -st};
    const double ep[3] = {-sp, cp, 0.0};
    const double inv_d2 = 1.0 / (d * d);
    double tmp[3];
    mat3_vec(cov, et, tmp);
    const double a = dot3(et, tmp) * inv_d2;
    mat3_vec(cov, ep, tmp);
    const double b = dot3(et, tmp) * inv_d2;
    const double dd = dot3(ep, tmp) * inv_d2;
    geom[3] = a; geom[4] = b; geom[5] = b; geom[6] = dd;
    const double det = a * dd - b * b; /* Mat2::inverse, linalg.hpp:112-115 */
    geom[7] = dd / det; geom[8] = -b / det; geom[9] = -b / det; geom[10] = a / det;

    const double r_theta = 3.0 * sqrt(dmax(a, 0.0));
    const double r_phi_scaled = 3.0 * sqrt(dmax(dd, 0.0));
    const double theta_lo = theta - r_theta, theta_hi = theta + r_theta;
    if (theta_hi < g->tmin || theta_lo > g->tmax) return 1;
    const double cell_t = g_dtheta(g), cell_p = g_dphi(g);
    const int i0 = clampi((int)floor((theta_lo - g->tmin) / cell_t), 0, g->nt - 1);
    const int i1 = clampi((int)floor((theta_hi - g->tmin) / cell_t), 0, g->nt - 1);
    span[0] = i0 / g->ts;
    span[1] = i1 / g->ts;
    const int tiles_p = g_tiles_p(g);
    const double w_phi = st > 1e-12 ? r_phi_scaled / st : K_PI;
    if (w_phi >= K_PI) {
        span[2] = 0; span[3] = tiles_p - 1;
    } else {
        const int j0 = clampi((int)floor(wrap_two_pi(phi - w_phi) / cell_p), 0, g->np - 1);
        const int j1 = clampi((int)floor(wrap_two_pi(phi + w_phi) / cell_p), 0, g->np - 1);
        span[2] = j0 / g->ts;
        span[3] = j1 / g->ts;
        if (j0 > j1) span[3] += tiles_p;
        if (span[3] - span[2] + 1 > tiles_p) { span[2] = 0; span[3] = tiles_p - 1; }
    }
    return 0;
}

/* ------------------------------------------------------------------ FLE basis
 * normalization radiance.cpp:9-14; legendre_table :16-37; eval_basis :79-92 */
static double normalization(int l, int m) {
    const int am = m < 0 ? -m : m;
    double ratio = 1.0;
    for (int i = l - am + 1; i <= l + am; ++i) ratio /= (double)i;
    return sqrt((2.0 * l + 1.0) / (4.0 * K_PI) * ratio);
}
static void eval_basis(double theta, double phi, int l_max, double* out /* 2L */) {
    double x = cos(theta);
    if (x < -1.0) x = -1.0;
    if (x > 1.0) x = 1.0;
    const int nt = (l_max + 1) * (l_max + 2) / 2;
    double* P = (double*)calloc((size_t)nt, sizeof(double));
#define AT(l, m) P[(l) * ((l) + 1) / 2 + (m)]
    const double s = sqrt(dmax(0.0, (1.0 - x) * (1.0 + x)));
    AT(0, 0) = 1.0;
    for (int m = 1; m <= l_max; ++m) AT(m, m) = AT(m - 1, m - 1) * (2.0 * m - 1.0) * s;
    for (int m = 0; m < l_max; ++m) AT(m + 1, m) = x * (2.0 * m + 1.0) * AT(m, m);
    for (int m = 0; m <= l_max; ++m)
        for (int l = m + 2; l <= l_max; ++l)
            AT(l, m) = (x * (2.0 * l - 1.0) * AT(l - 1, m) - (l + m - 1.0) * AT(l - 2, m)) /
                       (double)(l - m);
    for (int l = 0; l <= l_max; ++l)
        for (int m = -l; m <= l; ++m) {
            const int am = m < 0 ? -m : m;
            const double np = normalization(l, am) * AT(l, am);
            const int idx = l * l + m + l;
            out[2 * idx] = np * cos(m * phi);
            out[2 * idx + 1] = np * sin(m * phi);
        }
#undef AT
    free(P);
}
void or_eval_basis(double theta, double phi, int l_max, double* out) { eval_basis(theta, phi, l_max, out); }

/* ------------------------------------------------------------------ binning
 * bin_and_sort: sphraster.cpp:85-102 (std::stable_sort by depth == sort by
 * (depth, index) because lists are filled in index order). */
static const double* g_sort_depth;
static int cmp_depth_index(const void* a, const void* b) {
    const int ia = *(const int*)a, ib = *(const int*)b;
    const double da = g_sort_depth[ia], db = g_sort_depth[ib];
    if (da < db) return -1;
    if (db < da) return 1;
    return ia < ib ? -1 : (ia > ib);
}

long or_bin_and_sort(int k, const int* culled, const double* depth, const int* spans,
                     const int* gi, const double* gd, long* offsets, int* indices, long cap) {
    const grid_t g = mkgrid(gi, gd);
    const int tp = g_tiles_p(&g), n_tiles = g_tiles_t(&g) * tp;
    long* count = (long*)calloc((size_t)n_tiles + 1, sizeof(long));
    for (int i = 0; i < k; ++i) {
        if (culled[i]) continue;
        for (int tt = spans[4 * i]; tt <= spans[4 * i + 1]; ++tt)
            for (int pp = spans[4 * i + 2]; pp <= spans[4 * i + 3]; ++pp) count[tt * tp + pp % tp]++;
    }
    long total = 0;
    for (int t = 0; t < n_tiles; ++t) {
        offsets[t] = total;
        total += count[t];
        count[t] = offsets[t];
    }
    offsets[n_tiles] = total;
    if (total > cap) { free(count); return total; }
    for (int i = 0; i < k; ++i) {
        if (culled[i]) continue;
        for (int tt = spans[4 * i]; tt <= spans[4 * i + 1]; ++tt)
            for (int pp = spans[4 * i + 2]; pp <= spans[4 * i + 3]; ++pp)
                indices[count[tt * tp + pp % tp]++] = i;
    }
    g_sort_depth = depth;
    for (int t = 0; t < n_tiles; ++t)
        qsort(indices + offsets[t], (size_t)(offsets[t + 1] - offsets[t]), sizeof(int), cmp_depth_index);
    free(count);
    return total;
}

/* ------------------------------------------------------------------ tx state
 * build_tx_state: sphraster.cpp:150-172; hash: :121-148 */
typedef struct {
    grid_t g;
    int k, l_max;
    int* culled;
    double* geom;
    int* spans;
    double* basis; /* K*L*2 */
    long* offsets;
    int* indices;
    long entries;
} tx_t;

void* or_tx_new(void* scene, const double* tx, const int* gi, const double* gd, char* err,
                int errlen) {
    const scene_t* s = (const scene_t*)scene;
    const grid_t g = mkgrid(gi, gd);
    /* SphericalGrid::validate: sphraster.cpp:14-20 */
    if (g.nt < 1 || g.np < 1) { set_err(err, errlen, "grid: n_theta * n_phi must be >= 1"); return NULL; }
    if (g.ts < 1) { set_err(err, errlen, "grid: tile_size must be >= 1"); return NULL; }
    if (!(g.radius > 0.0)) { set_err(err, errlen, "grid: radius must be > 0"); return NULL; }
    if (!(g.tmin >= 0.0 && g.tmax <= K_PI && g.tmin < g.tmax)) {
        set_err(err, errlen, "grid: elevation span must satisfy 0 <= min < max <= pi");
        return NULL;
    }
    tx_t* t = (tx_t*)calloc(1, sizeof(tx_t));
    t->g = g; t->k = s->k; t->l_max = s->l_max;
    const int L = n_comp(s->l_max);
    t->culled = (int*)calloc((size_t)s->k + 1, sizeof(int));
    t->geom = (double*)calloc((size_t)s->k * 12 + 1, sizeof(double));
    t->spans = (int*)calloc((size_t)s->k * 4 + 1, sizeof(int));
    t->basis = (double*)calloc((size_t)s->k * L * 2 + 1, sizeof(double));
    double* depth = (double*)calloc((size_t)s->k + 1, sizeof(double));
    for (int k = 0; k < s->k; ++k) {
        double cov[9];
        covariance_from(s->ls + 3 * k, s->q + 4 * k, cov);
        t->culled[k] = project_one(s->pos + 3 * k, cov, sigmoid(s->tau[k]), tx, &g, t->geom + 12 * (size_t)k,
                                   t->spans + 4 * k);
        depth[k] = t->geom[12 * (size_t)k + 2];
        if (!t->culled[k]) eval_basis(t->geom[12 * (size_t)k], t->geom[12 * (size_t)k + 1], s->l_max,
                                      t->basis + (size_t)k * L * 2);
    }
    const int n_tiles = g_tiles_t(&g) * g_tiles_p(&g);
    t->offsets = (long*)calloc((size_t)n_tiles + 1, sizeof(long));
    long total = or_bin_and_sort(s->k, t->culled, depth, t->spans, gi, gd, t->offsets, NULL, 0);
    t->indices = (int*)calloc((size_t)total + 1, sizeof(int));
    or_bin_and_sort(s->k, t->culled, depth, t->spans, gi, gd, t->offsets, t->indices, total);
    t->entries = total;
    free(depth);
    return t;
}
void or_tx_free(void* h) {
    tx_t* t = (tx_t*)h;
    if (!t) return;
    free(t->culled); free(t->geom); free(t->spans); free(t->basis); free(t->offsets); free(t->indices);
    free(t);
}
long or_tx_entries(void* h) { return ((tx_t*)h)->entries; }

static void fnv(uint64_t* h, const void* data, size_t n) {
    const unsigned char* p = (const unsigned char*)data;
    for (size_t i = 0; i < n; ++i) { *h ^= p[i]; *h *= 0x100000001b3ull; }
}

void or_tx_get(void* h, int* culled, double* geom, int* spans, double* basis, long* offsets,
               int* indices, uint64_t* hash) {
    const tx_t* t = (const tx_t*)h;
    const int L = n_comp(t->l_max);
    const int n_tiles = g_tiles_t(&t->g) * g_tiles_p(&t->g);
    memcpy(culled, t->culled, (size_t)t->k * sizeof(int));
    memcpy(geom, t->geom, (size_t)t->k * 12 * sizeof(double));
    memcpy(spans, t->spans, (size_t)t->k * 4 * sizeof(int));
    memcpy(basis, t->basis, (size_t)t->k * L * 2 * sizeof(double));
    memcpy(offsets, t->offsets, ((size_t)n_tiles + 1) * sizeof(long));
    memcpy(indices, t->indices, (size_t)t->entries * sizeof(int));
    if (hash) {
        uint64_t x = 0xcbf29ce484222325ull;
        fnv(&x, &t->g.nt, 4); fnv(&x, &t->g.np, 4); fnv(&x, &t->g.ts, 4);
        fnv(&x, &t->g.radius, 8); fnv(&x, &t->k, 4); fnv(&x, &t->l_max, 4);
        for (int k = 0; k < t->k; ++k) {
            const unsigned char c = (unsigned char)(t->culled[k] != 0);
            fnv(&x, &c, 1);
            if (c) continue;
            const double* gm = t->geom + 12 * (size_t)k;
            fnv(&x, gm + 0, 8); fnv(&x, gm + 1, 8); fnv(&x, gm + 2, 8);
            fnv(&x, gm + 3, 32); fnv(&x, gm + 11, 8);
            fnv(&x, t->spans + 4 * k, 16);
        }
        for (int tt = 0; tt < n_tiles; ++tt) {
            const uint64_t n = (uint64_t)(t->offsets[tt + 1] - t->offsets[tt]);
            fnv(&x, &n, 8);
            fnv(&x, t->indices + t->offsets[tt], (size_t)n * 4);
        }
        fnv(&x, t->basis, (size_t)t->k * L * 16);
        *hash = x;
    }
}

/* ------------------------------------------------------------------ render
 * reduce_signals sphraster.cpp:190-226; gaussian_weight :239-251;
 * render_field :255-315.  values [j][c][re/im][row][col]; T [j][row][col]. */
int or_render(void* txh, void* scene, const double* coeffs, long n_coeffs, int n_rx, int threads,
              double* values, double* transmittance, char* err, int errlen) {
    (void)threads;
    const tx_t* t = (const tx_t*)txh;
    const scene_t* s = (const scene_t*)scene;
    if (n_rx < 1) { set_err(err, errlen, "render_field: n_rx must be >= 1"); return 1; }
    const int L = n_comp(s->l_max), C = s->C, K = t->k;
    const size_t stride = (size_t)L * C * 2;
    if ((size_t)n_coeffs != (size_t)n_rx * K * stride) {
        set_err(err, errlen, "render_field: coefficient tensor has wrong size");
        return 1;
    }
    for (int j = 0; j < n_rx; ++j)
        for (int k = 0; k < K; ++k)
            for (size_t i = 0; i < stride; ++i)
                if (!isfinite(coeffs[((size_t)j * K + k) * stride + i])) {
                    char msg[160];
                    snprintf(msg, sizeof msg, "render_field: non-finite coefficient at rx %d, gaussian %d", j, k);
                    set_err(err, errlen, msg);
                    return 1;
                }
    double* sig = (double*)calloc((size_t)K * n_rx * C * 2 + 1, sizeof(double));
    for (int k = 0; k < K; ++k) {
        if (t->culled[k]) continue;
        const double* B = t->basis + (size_t)k * L * 2;
        for (int j = 0; j < n_rx; ++j) {
            const double* cb = coeffs + ((size_t)j * K + k) * stride;
            double* o = sig + ((size_t)k * n_rx + j) * C * 2;
            for (int comp = 0; comp < L; ++comp)
                for (int c = 0; c < C; ++c) {
                    const double a = cb[((size_t)comp * C + c) * 2], b = cb[((size_t)comp * C + c) * 2 + 1];
                    const double br = B[2 * comp], bi = B[2 * comp + 1];
                    o[2 * c] += a * br - b * bi;
                    o[2 * c + 1] += a * bi + b * br;
                }
        }
    }
    const grid_t* g = &t->g;
    const size_t plane = (size_t)g->nt * g->np;
    for (size_t i = 0; i < (size_t)n_rx * C * 2 * plane; ++i) values[i] = 0.0;
    for (size_t i = 0; i < (size_t)n_rx * plane; ++i) transmittance[i] = 1.0;
    const int tp = g_tiles_p(g), n_tiles = g_tiles_t(g) * tp;
    double* acc = (double*)malloc((size_t)n_rx * C * 2 * sizeof(double));
    const double dth = g_dtheta(g), dph = g_dphi(g);
    for (int tile = 0; tile < n_tiles; ++tile) {
        const int tt = tile / tp, tq = tile % tp;
        const int r0 = tt * g->ts, r1 = (tt + 1) * g->ts < g->nt ? (tt + 1) * g->ts : g->nt;
        const int c0 = tq * g->ts, c1 = (tq + 1) * g->ts < g->np ? (tq + 1) * g->ts : g->np;
        for (int row = r0; row < r1; ++row) {
            const double theta_r = g->tmin + (row + 0.5) * dth;
            for (int col = c0; col < c1; ++col) {
                const double phi_r = (col + 0.5) * dph;
                const size_t cell = (size_t)row * g->np + col;
                memset(acc, 0, (size_t)n_rx * C * 2 * sizeof(double));
                double T = 1.0;
                for (long e = t->offsets[tile]; e < t->offsets[tile + 1]; ++e) {
                    const int k = t->indices[e];
                    const double* gm = t->geom + 12 * (size_t)k;
                    const double dt = theta_r - gm[0];
                    const double dpraw = wrap_pm_pi(phi_r - gm[1]);
                    const double dp = sin(gm[0]) * dpraw;
                    const double m2 = gm[7] * dt * dt + (gm[8] + gm[9]) * dt * dp + gm[10] * dp * dp;
                    double w = gm[11] * exp(-0.5 * m2);
                    if (w > K_WEIGHT_CLAMP) w = K_WEIGHT_CLAMP; /* std::min(w, clamp) */
                    const double tw = T * w;
                    const double* sk = sig + (size_t)k * n_rx * C * 2;
                    for (int jc = 0; jc < n_rx * C; ++jc) {
                        acc[2 * jc] += tw * sk[2 * jc];
                        acc[2 * jc + 1] += tw * sk[2 * jc + 1];
                    }
                    T *= 1.0 - w;
                    if (T < K_EARLY_EXIT_T) break;
                }
                for (int j = 0; j < n_rx; ++j) {
                    for (int c = 0; c < C; ++c) {
                        const size_t base = (((size_t)j * C + c) * 2) * plane;
                        values[base + cell] = acc[2 * ((size_t)j * C + c)];
                        values[base + plane + cell] = acc[2 * ((size_t)j * C + c) + 1];
                    }
                    transmittance[(size_t)j * plane + cell] = T;
                }
            }
        }
    }
    free(acc);
    free(sig);
    return 0;
}

/* aggregate_modality: sphraster.cpp:323-381.  modality 0 rssi, 1 csi, 2 spectrum */
int or_aggregate(int n_rx, int channels, const int* gi, const double* gd, const double* values,
                 int modality, double* out, char* err, int errlen) {
    const grid_t g = mkgrid(gi, gd);
    const size_t plane = (size_t)g.nt * g.np;
    for (size_t i = 0; i < (size_t)n_rx * channels * 2 * plane; ++i)
        if (!isfinite(values[i])) { set_err(err, errlen, "aggregate_modality: non-finite field"); return 1; }
    if (modality != 1 && channels != 1) {
        set_err(err, errlen, "aggregate_modality: scalar modalities need channels == 1");
        return 1;
    }
    const double dth = g_dtheta(&g), dph = g_dphi(&g);
    for (int j = 0; j < n_rx; ++j) {
        if (modality == 0) {
            const size_t base = ((size_t)j * 2) * plane;
            double power = 0.0;
            for (int row = 0; row < g.nt; ++row) {
                const double dom = sin(g.tmin + (row + 0.5) * dth) * dth * dph;
                for (int col = 0; col < g.np; ++col) {
                    const size_t cell = (size_t)row * g.np + col;
                    const double re = values[base + cell], im = values[base + plane + cell];
                    power += (re * re + im * im) * dom;
                }
            }
            out[j] = 10.0 * log10(power + K_RSSI_FLOOR);
        } else if (modality == 1) {
            for (int c = 0; c < channels; ++c) {
                const size_t base = (((size_t)j * channels + c) * 2) * plane;
                double sr = 0.0, si = 0.0;
                for (int row = 0; row < g.nt; ++row) {
                    const double dom = sin(g.tmin + (row + 0.5) * dth) * dth * dph;
                    for (int col = 0; col < g.np; ++col) {
                        const size_t cell = (size_t)row * g.np + col;
                        sr += values[base + cell] * dom;
                        si += values[base + plane + cell] * dom;
                    }
                }
                out[((size_t)j * channels + c) * 2] = sr;
                out[((size_t)j * channels + c) * 2 + 1] = si;
            }
        } else {
            const size_t base = ((size_t)j * 2) * plane;
            for (size_t cell = 0; cell < plane; ++cell) {
                const double re = values[base + cell], im = values[base + plane + cell];
                out[(size_t)j * plane + cell] = sqrt(re * re + im * im + K_AMP_EPS);
            }
        }
    }
    return 0;
}

/* ------------------------------------------------------------------ conditioning */
typedef struct {
    cond_layout c;
    double* p;
    double* occ; /* NULL = empty grid */
    double lo[3], hi[3];
} cond_t;

void* or_cond_new(const int* cfg, const double* params, const double* occ, const double* occ_lo,
                  const double* occ_hi) {
    cond_t* s = (cond_t*)calloc(1, sizeof(cond_t));
    s->c = make_layout(cfg, cfg[7], cfg[8]);
    s->p = dup(params, s->c.total);
    if (occ) {
        s->occ = dup(occ, (size_t)s->c.R * s->c.R * s->c.R);
        for (int a = 0; a < 3; ++a) { s->lo[a] = occ_lo[a]; s->hi[a] = occ_hi[a]; }
    }
    return s;
}
void or_cond_free(void* h) {
    cond_t* s = (cond_t*)h;
    if (!s) return;
    free(s->p); free(s->occ); free(s);
}
long or_cond_param_count(void* h) { return (long)((cond_t*)h)->c.total; }

/* build_occupancy: conditioning.cpp:114-161 */
void or_build_occupancy(void* scene, int R, const double* lo, const double* hi, double* out) {
    const scene_t* s = (const scene_t*)scene;
    const double ext[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
    for (size_t i = 0; i < (size_t)R * R * R; ++i) out[i] = 0.0;
    const double cell[3] = {ext[0] / R, ext[1] / R, ext[2] / R};
    for (int k = 0; k < s->k; ++k) {
        const double* p = s->pos + 3 * k;
        double sig[9], prec[9];
        covariance_from(s->ls + 3 * k, s->q + 4 * k, sig);
        mat3_inverse(sig, prec);
        const double tau = sigmoid(s->tau[k]);
        int a0[3], a1[3];
        for (int a = 0; a < 3; ++a) {
            const double half = 2.0 * sqrt(sig[a * 4]);
            const int l = (int)floor((p[a] - half - lo[a]) / cell[a] - 0.5);
            const int h = (int)ceil((p[a] + half - lo[a]) / cell[a] - 0.5);
            a0[a] = l > 0 ? l : 0;
            a1[a] = h < R - 1 ? h : R - 1;
        }
        for (int ix = a0[0]; ix <= a1[0]; ++ix)
            for (int iy = a0[1]; iy <= a1[1]; ++iy)
                for (int iz = a0[2]; iz <= a1[2]; ++iz) {
                    const double ctr[3] = {lo[0] + (ix + 0.5) * cell[0], lo[1] + (iy + 0.5) * cell[1],
                                           lo[2] + (iz + 0.5) * cell[2]};
                    const double d[3] = {ctr[0] - p[0], ctr[1] - p[1], ctr[2] - p[2]};
                    double pd[3];
                    mat3_vec(prec, d, pd);
                    const double m2 = dot3(d, pd);
                    if (m2 > 4.0) continue;
                    const double v = tau * exp(-0.5 * m2);
                    double* slot = out + ((size_t)ix * R + iy) * R + iz;
                    *slot = dmax(*slot, v);
                }
    }
    for (size_t i = 0; i < (size_t)R * R * R; ++i) {
        const double v = out[i];
        out[i] = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    }
}

/* sample_trilinear :74-98, sample_nearest :100-112 */
static double sample_trilinear(int R, const double* lo, const double* hi, const double* dens,
                               const double* p) {
    if (!dens) return 0.0;
    double f[3];
    int i0[3];
    for (int a = 0; a < 3; ++a) {
        const double cell = (hi[a] - lo[a]) / R;
        const double u = (p[a] - lo[a]) / cell - 0.5;
        i0[a] = (int)floor(u);
        f[a] = u - i0[a];
    }
    double acc = 0.0;
    for (int dx = 0; dx < 2; ++dx)
        for (int dy = 0; dy < 2; ++dy)
            for (int dz = 0; dz < 2; ++dz) {
                const int ix = i0[0] + dx, iy = i0[1] + dy, iz = i0[2] + dz;
                if (ix < 0 || iy < 0 || iz < 0 || ix >= R || iy >= R || iz >= R) continue;
                const double w = (dx ? f[0] : 1 - f[0]) * (dy ? f[1] : 1 - f[1]) * (dz ? f[2] : 1 - f[2]);
                acc += w * dens[((size_t)ix * R + iy) * R + iz];
            }
    return acc;
}
static double sample_nearest(int R, const double* lo, const double* hi, const double* dens,
                             const double* p) {
    if (!dens) return 0.0;
    int idx[3];
    for (int a = 0; a < 3; ++a) {
        const double cell = (hi[a] - lo[a]) / R;
        const int i = (int)floor((p[a] - lo[a]) / cell);
        if (i < 0 || i >= R) return 0.0;
        idx[a] = i;
    }
    return dens[((size_t)idx[0] * R + idx[1]) * R + idx[2]];
}
/* probe_segment :163-178 */
static void probe(int R, const double* lo, const double* hi, const double* dens, const double* from,
                  const double* to, int S, int nearest, double* T, double* mean) {
    double tr = 1.0, sum = 0.0;
    for (int s = 0; s < S; ++s) {
        const double t = S == 1 ? 0.5 : 0.05 + 0.9 * (double)s / (S - 1);
        const double q[3] = {from[0] + (to[0] - from[0]) * t, from[1] + (to[1] - from[1]) * t,
                             from[2] + (to[2] - from[2]) * t};
        const double v = nearest ? sample_nearest(R, lo, hi, dens, q) : sample_trilinear(R, lo, hi, dens, q);
        tr *= 1.0 - v;
        sum += v;
    }
    *T = tr;
    *mean = sum / S;
}
void or_probe(int R, const double* lo, const double* hi, const double* dens, const double* from,
              const double* to, int S, int nearest, double* out2) {
    probe(R, lo, hi, dens, from, to, S, nearest, out2, out2 + 1);
}

/* MlpLayer::forward :12-19 and mlp_forward :23-29 (ReLU = std::max(0.0, h)) */
static void layer_fwd(const double* w, const double* b, int in, int out, const double* x, double* y) {
    for (int o = 0; o < out; ++o) {
        double acc = b[o];
        const double* row = w + (size_t)o * in;
        for (int i = 0; i < in; ++i) acc += row[i] * x[i];
        y[o] = acc;
    }
}
static void mlp_fwd(const double* p, size_t w1, size_t b1, size_t w2, size_t b2, size_t w3, size_t b3,
                    int in, int d, int out, const double* x, double* h1, double* h2, double* y) {
    layer_fwd(p + w1, p + b1, in, d, x, h1);
    for (int i = 0; i < d; ++i) h1[i] = dmax(0.0, h1[i]);
    layer_fwd(p + w2, p + b2, d, d, h1, h2);
    for (int i = 0; i < d; ++i) h2[i] = dmax(0.0, h2[i]);
    layer_fwd(p + w3, p + b3, d, out, h2, y);
}

/* condition_forward: conditioning.cpp:284-423 (fourier_encode :255-265,
 * affine_apply :271-275).  mode: 0 full 1 global_only 2 local_only
 * 3 additive_only 4 no_occlusion. */
int or_cond_forward(void* condh, void* sceneh, const double* rx, double* out, double* ws_local_in,
                    double* ws_local_out, double* ws_global_out, char* err, int errlen) {
    const cond_t* st = (const cond_t*)condh;
    const scene_t* s = (const scene_t*)sceneh;
    const cond_layout* c = &st->c;
    const double* p = st->p;
    if (s->l_max != c->l_max || s->C != c->C) {
        set_err(err, errlen, "condition_forward: scene/state shape mismatch");
        return 1;
    }
    const int K = s->k, L = c->L, C = c->C, d = c->d;
    const size_t stride = (size_t)L * C * 2, n = (size_t)K * stride;
    const int use_global = c->mode != 2, use_local = c->mode != 1, additive = c->mode == 3;
    double* mid = (double*)malloc((n ? n : 1) * sizeof(double));
    double* in = (double*)malloc(((size_t)c->gin + 6) * sizeof(double));
    double* h1 = (double*)malloc((size_t)d * sizeof(double));
    double* h2 = (double*)malloc((size_t)d * sizeof(double));
    double* y = (double*)malloc((size_t)4 * C * sizeof(double));
    if (use_global) {
        const int F = c->F;
        for (int a = 0; a < 3; ++a)
            for (int band = 0; band < F; ++band) {
                const double arg = p[c->o_freq + (size_t)band * 3 + a] * rx[a];
                in[(a * F + band) * 2] = sin(arg);
                in[(a * F + band) * 2 + 1] = cos(arg);
            }
        const double denom = c->l_max > 0 ? (double)c->l_max : 1.0;
        for (int comp = 0; comp < L; ++comp) {
            int l = 0;
            while ((l + 1) * (l + 1) <= comp) ++l;
            const int m = comp - l * l - l;
            in[6 * F] = l / denom;
            in[6 * F + 1] = m / denom;
            for (int e = 0; e < c->dc; ++e) in[6 * F + 2 + e] = p[c->o_emb + (size_t)comp * c->dc + e];
            mlp_fwd(p, c->o_gw1, c->o_gb1, c->o_gw2, c->o_gb2, c->o_gw3, c->o_gb3, c->gin, d, 4 * C, in, h1, h2, y);
            if (ws_global_out) memcpy(ws_global_out + (size_t)comp * 4 * C, y, (size_t)4 * C * sizeof(double));
            for (int ch = 0; ch < C; ++ch) {
                const double ar = additive ? 0.0 : y[4 * ch], ai = additive ? 0.0 : y[4 * ch + 1];
                const double br = y[4 * ch + 2], bi = y[4 * ch + 3];
                for (int k = 0; k < K; ++k) {
                    const size_t idx = ((size_t)k * L + comp) * C * 2 + (size_t)ch * 2;
                    const double zr = s->coeffs[idx], zi = s->coeffs[idx + 1];
                    mid[idx] = zr + (ar * zr - ai * zi + br);
                    mid[idx + 1] = zi + (ai * zr + ar * zi + bi);
                }
            }
        }
    } else {
        memcpy(mid, s->coeffs, n * sizeof(double));
    }
    int rc = 0;
    if (!use_local) {
        memcpy(out, mid, n * sizeof(double));
    } else {
        const int no_occ = c->mode == 4 || st->occ == NULL;
        for (int k = 0; k < K; ++k) {
            const double* pk = s->pos + 3 * k;
            const double diff[3] = {rx[0] - pk[0], rx[1] - pk[1], rx[2] - pk[2]};
            const double dist = sqrt(dot3(diff, diff));
            if (dist == 0.0) {
                char msg[128];
                snprintf(msg, sizeof msg, "condition_forward: receiver coincides with gaussian %d", k);
                set_err(err, errlen, msg);
                rc = 1;
                break;
            }
            in[0] = diff[0] / dist; in[1] = diff[1] / dist; in[2] = diff[2] / dist; in[3] = dist;
            if (no_occ) {
                in[4] = 1.0; in[5] = 0.0;
            } else {
                probe(c->R, st->lo, st->hi, st->occ, pk, rx, c->S, c->nearest, &in[4], &in[5]);
            }
            mlp_fwd(p, c->o_lw1, c->o_lb1, c->o_lw2, c->o_lb2, c->o_lw3, c->o_lb3, 6, d, 4 * C, in, h1, h2, y);
            if (ws_local_in) memcpy(ws_local_in + (size_t)k * 6, in, 6 * sizeof(double));
            if (ws_local_out) memcpy(ws_local_out + (size_t)k * 4 * C, y, (size_t)4 * C * sizeof(double));
            for (int ch = 0; ch < C; ++ch) {
                const double ar = additive ? 0.0 : y[4 * ch], ai = additive ? 0.0 : y[4 * ch + 1];
                const double br = y[4 * ch + 2], bi = y[4 * ch + 3];
                for (int comp = 0; comp < L; ++comp) {
                    const size_t idx = ((size_t)k * L + comp) * C * 2 + (size_t)ch * 2;
                    const double zr = mid[idx], zi = mid[idx + 1];
                    out[idx] = zr + (ar * zr - ai * zi + br);
                    out[idx + 1] = zi + (ai * zr + ar * zi + bi);
                }
            }
        }
    }
    free(mid); free(in); free(h1); free(h2); free(y);
    return rc;
}

/* train::predict: trainer.cpp:147-154 */
int or_predict(void* scene, void* cond, const int* gi, const double* gd, const double* tx,
               const double* rx, int threads, double* out, char* err, int errlen) {
    const scene_t* s = (const scene_t*)scene;
    const size_t n = (size_t)s->k * n_comp(s->l_max) * s->C * 2;
    double* coeffs = (double*)malloc((n ? n : 1) * sizeof(double));
    int rc = 0;
    if (cond) {
        rc = or_cond_forward(cond, scene, rx, coeffs, NULL, NULL, NULL, err, errlen);
    } else {
        memcpy(coeffs, s->coeffs, n * sizeof(double));
    }
    void* t = rc ? NULL : or_tx_new(scene, tx, gi, gd, err, errlen);
    if (!rc && !t) rc = 1;
    if (!rc) {
        const size_t plane = (size_t)gi[0] * gi[1];
        double* vals = (double*)malloc((size_t)s->C * 2 * plane * sizeof(double));
        double* T = (double*)malloc(plane * sizeof(double));
        rc = or_render(t, scene, coeffs, (long)n, 1, threads, vals, T, err, errlen);
        if (!rc) rc = or_aggregate(1, s->C, gi, gd, vals, s->modality, out, err, errlen);
        free(vals); free(T);
    }
    or_tx_free(t);
    free(coeffs);
    return rc;
}
