// Transmitter-side geometry in FP64 on sm_100a.
//
// Compiled with -fmad=false: the reference is built without FMA contraction
// (x86-64 baseline), and the per-tile lists must match
// it bit for bit, so every FP64 expression here keeps the reference's
// operation order and rounding steps.
//
//   k_tx_prep   = covariance_from (scene.cpp:42-51) + project_gaussian
//                 (sphraster.cpp:22-83) + eval_basis (radiance.cpp:79-92),
//                 one thread per Gaussian.
//   k_occupancy = build_occupancy (conditioning.cpp:114-161): scatter-max of
//                 tau*exp(-m2/2) with atomicMax on the IEEE bits of the
//                 non-negative doubles (order independent, hence exact).
#include "rxgs_internal.cuh"

namespace rxgs_b200 {
namespace {

__device__ __forceinline__ double wrap_two_pi(double a) {  // linalg.hpp:160-164
    // fmod(a, 2 pi) is exact and returns a itself when |a| < 2 pi (an atan2
    // result always): the software FP64 fmod is skipped there
    if (!(fabs(a) < kTwoPi)) a = fmod(a, kTwoPi);
    if (a < 0.0) a += kTwoPi;
    return a;
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

__device__ __forceinline__ double dmax(double a, double b) { return a < b ? b : a; }

// quat_to_rotation (linalg.hpp:122-131) then M = R diag(e^s), Sigma = M M^T.
__device__ void covariance(const double* ls, const double* q, double* sig) {
    const double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    const double w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
    double m[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z),     2 * (x * z + w * y),
                   2 * (x * y + w * z),     1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                   2 * (x * z - w * y),     2 * (y * z + w * x),     1 - 2 * (x * x + y * y)};
    const double e[3] = {exp(ls[0]), exp(ls[1]), exp(ls[2])};
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) m[r * 3 + c] *= e[c];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < 3; ++k) s += m[i * 3 + k] * m[j * 3 + k];
            sig[i * 3 + j] = s;
        }
}

__device__ __forceinline__ double normalization(int l, int am) {  // radiance.cpp:9-14
    double ratio = 1.0;
    for (int i = l - am + 1; i <= l + am; ++i) ratio /= static_cast<double>(i);
    return sqrt((2.0 * l + 1.0) / (4.0 * kPi) * ratio);
}

// project_gaussian (sphraster.cpp:22-83) of one Gaussian at u = p - tx with
// covariance sig and activated tau: gm = [theta, phi, depth, A (a, b, c, d),
// A^-1 (4), tau], the inclusive tile span, the culled flag and the walk's
// record.  Shared by k_tx_prep and the single-Gaussian API (k_project).
__device__ __forceinline__ void project_core(double u0, double u1, double u2, const double* sig, double tau,
                                             const DevGrid& g, double* gm, int4& sp, int& is_culled,
                                             GaussRec& r) {
    const double d = sqrt(u0 * u0 + u1 * u1 + u2 * u2);
    double theta = 0.0, phi = 0.0;
    if ((d >= g.radius) && d != 0.0) {
        const double rho = sqrt(u0 * u0 + u1 * u1);
        theta = atan2(rho, u2);
        phi = wrap_two_pi(atan2(u1, u0));
        gm[0] = theta;
        gm[1] = phi;
        gm[2] = d;
        gm[11] = tau;
        const double st = sin(theta), ct = cos(theta), sp_ = sin(phi), cp = cos(phi);
        const double et[3] = {ct * cp, ct * sp_, -st};
        const double ep[3] = {-sp_, cp, 0.0};
        const double inv_d2 = 1.0 / (d * d);
        double t[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) t[i] = sig[3 * i] * et[0] + sig[3 * i + 1] * et[1] + sig[3 * i + 2] * et[2];
        const double a = (et[0] * t[0] + et[1] * t[1] + et[2] * t[2]) * inv_d2;
#pragma unroll
        for (int i = 0; i < 3; ++i) t[i] = sig[3 * i] * ep[0] + sig[3 * i + 1] * ep[1] + sig[3 * i + 2] * ep[2];
        const double b = (et[0] * t[0] + et[1] * t[1] + et[2] * t[2]) * inv_d2;
        const double dd = (ep[0] * t[0] + ep[1] * t[1] + ep[2] * t[2]) * inv_d2;
        const double det = a * dd - b * b;
        const double pa = dd / det, pb = -b / det, pc = -b / det, pd = a / det;
        gm[3] = a; gm[4] = b; gm[5] = b; gm[6] = dd;
        gm[7] = pa; gm[8] = pb; gm[9] = pc; gm[10] = pd;

        const double r_theta = 3.0 * sqrt(dmax(a, 0.0));
        const double r_phi_scaled = 3.0 * sqrt(dmax(dd, 0.0));
        const double theta_lo = theta - r_theta, theta_hi = theta + r_theta;
        if (!(theta_hi < g.tmin || theta_lo > g.tmax)) {
            const int i0 = clampi(static_cast<int>(floor((theta_lo - g.tmin) / g.dth)), 0, g.nt - 1);
            const int i1 = clampi(static_cast<int>(floor((theta_hi - g.tmin) / g.dth)), 0, g.nt - 1);
            sp.x = i0 / g.ts;
            sp.y = i1 / g.ts;
            const double w_phi = st > 1e-12 ? r_phi_scaled / st : kPi;
            if (w_phi >= kPi) {
                sp.z = 0;
                sp.w = g.tiles_p - 1;
            } else {
                const int j0 = clampi(static_cast<int>(floor(wrap_two_pi(phi - w_phi) / g.dph)), 0, g.np - 1);
                const int j1 = clampi(static_cast<int>(floor(wrap_two_pi(phi + w_phi) / g.dph)), 0, g.np - 1);
                sp.z = j0 / g.ts;
                sp.w = j1 / g.ts;
                if (j0 > j1) sp.w += g.tiles_p;
                if (sp.w - sp.z + 1 > g.tiles_p) {
                    sp.z = 0;
                    sp.w = g.tiles_p - 1;
                }
            }
            is_culled = 0;
            r.theta = theta;
            r.phi = phi;
            r.sin_theta = st;
            r.cos_theta = ct;
            r.pa = pa;
            r.pbc = pb + pc;
            r.pd = pd;
            r.tau = tau;
        }
    }
}

// FULL: also the FP64 per-Gaussian geometry (geom) and basis (basis64) that
// only the adjoint, the materialised render API and the state accessors
// read; the query path builds lean states and completes them on demand
// (ensure_tx_full, capi.cu) with the identical arithmetic.
// FLE basis of Gaussian k at the centre direction (theta, phi) into the
// FP64 / f32 basis rows and the f32 basis*base rows (eval_basis,
// radiance.cpp:79-92); zeros for a culled Gaussian.
template <int LMT, bool FULL>
__device__ __forceinline__ void fle_basis_row(int k, int l_max, int C, int is_culled, double theta, double phi,
                                              const double* __restrict__ coeffs64, double* __restrict__ basis64,
                                              float2* __restrict__ basis32, float2* __restrict__ gb32) {
    const int L = (l_max + 1) * (l_max + 1);
    double* b64 = basis64 + static_cast<size_t>(k) * L * 2;
    float2* b32 = basis32 + static_cast<size_t>(k) * L;
    float2* g32 = gb32 + static_cast<size_t>(k) * L * C;
    const double* cb = coeffs64 + static_cast<size_t>(k) * L * C * 2;
    if (is_culled) {
        for (int i = 0; i < L; ++i) {
            if (FULL) {
                b64[2 * i] = 0.0;
                b64[2 * i + 1] = 0.0;
            }
            b32[i] = make_float2(0.f, 0.f);
            for (int c = 0; c < C; ++c) g32[i * C + c] = make_float2(0.f, 0.f);
        }
        return;
    }
    // legendre_table (radiance.cpp:16-37) on x = cos(theta), without the
    // Condon-Shortley phase; entries packed l*(l+1)/2 + m.
    constexpr int LM = LMT > 0 ? LMT : kMaxLmax;  // array bound
    const int LB = LMT > 0 ? LMT : l_max;         // loop bound (constant when specialised)
    double P[(LM + 1) * (LM + 2) / 2];
    double x = cos(theta);
    x = x < -1.0 ? -1.0 : (x > 1.0 ? 1.0 : x);
    const double s = sqrt(dmax(0.0, (1.0 - x) * (1.0 + x)));
#define AT(l, m) P[(l) * ((l) + 1) / 2 + (m)]
    AT(0, 0) = 1.0;
#pragma unroll
    for (int m = 1; m <= LB; ++m) AT(m, m) = AT(m - 1, m - 1) * (2.0 * m - 1.0) * s;
#pragma unroll
    for (int m = 0; m < LB; ++m) AT(m + 1, m) = x * (2.0 * m + 1.0) * AT(m, m);
#pragma unroll
    for (int m = 0; m <= LB; ++m)
#pragma unroll
        for (int l = m + 2; l <= LB; ++l)
            AT(l, m) = (x * (2.0 * l - 1.0) * AT(l - 1, m) - (l + m - 1.0) * AT(l - 2, m)) /
                       static_cast<double>(l - m);
    // cos(m phi), sin(m phi) once per distinct m (eval_basis evaluates them
    // per (l, m); the same argument m * phi gives the same values)
    double cm[2 * LM + 1], sn[2 * LM + 1];
#pragma unroll
    for (int m = -LB; m <= LB; ++m) sincos(m * phi, &sn[m + LM], &cm[m + LM]);
#pragma unroll
    for (int l = 0; l <= LB; ++l) {
#pragma unroll
        for (int m = -l; m <= l; ++m) {
            const int am = m < 0 ? -m : m;
            const double np = normalization(l, am) * AT(l, am);
            const int idx = l * l + m + l;
            const double br = np * cm[m + LM], bi = np * sn[m + LM];
            if (FULL) reinterpret_cast<double2*>(b64)[idx] = make_double2(br, bi);
            b32[idx] = make_float2(static_cast<float>(br), static_cast<float>(bi));
            for (int c = 0; c < C; ++c) {
                const double a_ = cb[(idx * C + c) * 2], b_ = cb[(idx * C + c) * 2 + 1];
                g32[idx * C + c] = make_float2(static_cast<float>(a_ * br - b_ * bi),
                                               static_cast<float>(a_ * bi + b_ * br));
            }
        }
    }
#undef AT
}


template <int LMT, bool FULL, bool BASIS>  // LMT > 0: l_max known at compile time (tables in registers)
__global__ void k_tx_prep(int K, int l_max_rt, int C, const double* __restrict__ pos,
                          const double* __restrict__ ls, const double* __restrict__ q,
                          const double* __restrict__ tau_logit,
                          const double* __restrict__ coeffs64, double tx0, double tx1, double tx2,
                          DevGrid g, GaussRec* __restrict__ rec, int* __restrict__ culled,
                          double* __restrict__ geom, int4* __restrict__ spans,
                          double* __restrict__ basis64, float2* __restrict__ basis32,
                          float2* __restrict__ gb32, uint64_t* __restrict__ depth_key,
                          int* __restrict__ tile_count) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    const int l_max = LMT > 0 ? LMT : l_max_rt;
    double gm[12];
#pragma unroll
    for (int i = 0; i < 12; ++i) gm[i] = 0.0;
    int4 sp = make_int4(0, -1, 0, -1);
    int is_culled = 1;
    GaussRec r{};

    double sig[9];
    covariance(ls + 3 * static_cast<size_t>(k), q + 4 * static_cast<size_t>(k), sig);
    const double tau = 1.0 / (1.0 + exp(-tau_logit[k]));  // linalg.hpp:157

    const double u0 = pos[3 * static_cast<size_t>(k)] - tx0;
    const double u1 = pos[3 * static_cast<size_t>(k) + 1] - tx1;
    const double u2 = pos[3 * static_cast<size_t>(k) + 2] - tx2;
    project_core(u0, u1, u2, sig, tau, g, gm, sp, is_culled, r);
    const double d = gm[2], theta = gm[0], phi = gm[1];
    if (FULL) {
        double* gout = geom + 12 * static_cast<size_t>(k);
#pragma unroll
        for (int i = 0; i < 12; ++i) gout[i] = gm[i];
    }
    rec[k] = r;
    culled[k] = is_culled;
    spans[k] = sp;
    tile_count[k] = is_culled ? 0 : (sp.y - sp.x + 1) * (sp.w - sp.z + 1);
    depth_key[k] = is_culled ? ~0ull : static_cast<uint64_t>(__double_as_longlong(d));

    // FLE basis at the centre direction (zero for culled Gaussians).  A lean
    // build (BASIS = false) defers it to k_basis_rows for the Gaussians the
    // walk reaches (compact_needed): the only rows the query path reads.
    if (BASIS) fle_basis_row<LMT, FULL>(k, l_max, C, is_culled, theta, phi, coeffs64, basis64, basis32, gb32);
}

// The needed rows' f32 basis and basis*base of a lean build, from the walk
// records' theta / phi: the same arithmetic as k_tx_prep's basis.
template <int LMT>
__global__ void k_basis_rows(const int* __restrict__ n_rows, const int* __restrict__ rows, int l_max_rt, int C,
                             const GaussRec* __restrict__ rec, const double* __restrict__ coeffs64,
                             float2* __restrict__ basis32, float2* __restrict__ gb32) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= *n_rows) return;
    const int k = rows[r];
    const int l_max = LMT > 0 ? LMT : l_max_rt;
    fle_basis_row<LMT, false>(k, l_max, C, 0, rec[k].theta, rec[k].phi, coeffs64, nullptr, basis32, gb32);
}

// ---------------------------------------------------------------- single-call API kernels
// project_gaussian (sphraster.cpp:22-83) of n Gaussians given their
// covariances and activated tau: the arithmetic of k_tx_prep (project_core).
__global__ void k_project(int n, const double* __restrict__ pos, const double* __restrict__ cov,
                          const double* __restrict__ tau, double tx0, double tx1, double tx2, DevGrid g,
                          double* __restrict__ geom, int* __restrict__ culled, int4* __restrict__ spans) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double gm[12];
#pragma unroll
    for (int a = 0; a < 12; ++a) gm[a] = 0.0;
    int4 sp = make_int4(0, -1, 0, -1);
    int c = 1;
    GaussRec r{};
    project_core(pos[3 * static_cast<size_t>(i)] - tx0, pos[3 * static_cast<size_t>(i) + 1] - tx1,
                 pos[3 * static_cast<size_t>(i) + 2] - tx2, cov + 9 * static_cast<size_t>(i), tau[i], g, gm, sp, c,
                 r);
    for (int a = 0; a < 12; ++a) geom[12 * static_cast<size_t>(i) + a] = gm[a];
    culled[i] = c;
    spans[i] = sp;
}

// The walk record of an imported state (rxgs_tx_state_import) from its FP64
// geometry rows: the same values k_tx_prep writes (sin / cos of theta on the
// device, p_b + p_c summed once), and the f32 basis.
__global__ void k_rec_from_geom(int K, const int* __restrict__ culled, const double* __restrict__ geom,
                                const double* __restrict__ basis64, int L, GaussRec* __restrict__ rec,
                                float2* __restrict__ basis32) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    GaussRec r{};
    if (!culled[k]) {
        const double* gm = geom + 12 * static_cast<size_t>(k);
        r.theta = gm[0];
        r.phi = gm[1];
        r.sin_theta = sin(gm[0]);
        r.cos_theta = cos(gm[0]);
        r.pa = gm[7];
        r.pbc = gm[8] + gm[9];
        r.pd = gm[10];
        r.tau = gm[11];
    }
    rec[k] = r;
    for (int l = 0; l < L; ++l) {
        const double* b = basis64 + (static_cast<size_t>(k) * L + l) * 2;
        basis32[static_cast<size_t>(k) * L + l] = make_float2(static_cast<float>(b[0]), static_cast<float>(b[1]));
    }
}

constexpr int kApiLmax = 24;
constexpr int kApiNP = (kApiLmax + 1) * (kApiLmax + 2) / 2;

// legendre_table (radiance.cpp:16-37) after the |x| check / clamp
__device__ void legendre_rt(double x, int l_max, double* P) {
    x = x < -1.0 ? -1.0 : (x > 1.0 ? 1.0 : x);
    const double s = sqrt(dmax(0.0, (1.0 - x) * (1.0 + x)));
    for (int i = 0; i < (l_max + 1) * (l_max + 2) / 2; ++i) P[i] = 0.0;
#define AT(l, m) P[(l) * ((l) + 1) / 2 + (m)]
    AT(0, 0) = 1.0;
    for (int m = 1; m <= l_max; ++m) AT(m, m) = AT(m - 1, m - 1) * (2.0 * m - 1.0) * s;
    for (int m = 0; m < l_max; ++m) AT(m + 1, m) = x * (2.0 * m + 1.0) * AT(m, m);
    for (int m = 0; m <= l_max; ++m)
        for (int l = m + 2; l <= l_max; ++l)
            AT(l, m) = (x * (2.0 * l - 1.0) * AT(l - 1, m) - (l + m - 1.0) * AT(l - 2, m)) / static_cast<double>(l - m);
#undef AT
}

// legendre_table_dtheta (radiance.cpp:39-77)
__device__ void legendre_dtheta_rt(double theta, int l_max, double* P, double* D) {
    const double x = cos(theta), s = sin(theta);
    for (int i = 0; i < (l_max + 1) * (l_max + 2) / 2; ++i) P[i] = D[i] = 0.0;
#define AT(l, m) P[(l) * ((l) + 1) / 2 + (m)]
#define DAT(l, m) D[(l) * ((l) + 1) / 2 + (m)]
    AT(0, 0) = 1.0;
    DAT(0, 0) = 0.0;
    for (int m = 1; m <= l_max; ++m) {
        const double c = 2.0 * m - 1.0;
        AT(m, m) = AT(m - 1, m - 1) * c * s;
        DAT(m, m) = c * (DAT(m - 1, m - 1) * s + AT(m - 1, m - 1) * x);
    }
    for (int m = 0; m < l_max; ++m) {
        const double c = 2.0 * m + 1.0;
        AT(m + 1, m) = x * c * AT(m, m);
        DAT(m + 1, m) = c * (-s * AT(m, m) + x * DAT(m, m));
    }
    for (int m = 0; m <= l_max; ++m)
        for (int l = m + 2; l <= l_max; ++l) {
            const double a = 2.0 * l - 1.0, b = l + m - 1.0, inv = 1.0 / (l - m);
            AT(l, m) = (x * a * AT(l - 1, m) - b * AT(l - 2, m)) * inv;
            DAT(l, m) = (a * (-s * AT(l - 1, m) + x * DAT(l - 1, m)) - b * DAT(l - 2, m)) * inv;
        }
#undef AT
#undef DAT
}

// The FLE basis API (radiance.hpp:36-70), one item per thread:
//   0 eval_basis(theta, phi)            -> L complex
//   1 eval_basis_jet(theta, phi)        -> b, db/dtheta, db/dphi (3 L complex)
//   2 legendre_table(x)                 -> NP
//   3 legendre_table_dtheta(theta)      -> P (NP), dP/dtheta (NP)
//   4 normalization(l, m)               -> 1
//   5 eval_radiance(coeffs, theta, phi) -> 1 complex
__global__ void k_fle_eval(int what, int n, int l_max, const double* __restrict__ a, const double* __restrict__ b,
                           const double* __restrict__ coeffs, double* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int L = (l_max + 1) * (l_max + 1), NP = (l_max + 1) * (l_max + 2) / 2;
    double P[kApiNP], D[kApiNP];
    if (what == 4) {
        const int l = static_cast<int>(a[i]), m = static_cast<int>(b[i]);
        out[i] = normalization(l, m < 0 ? -m : m);
        return;
    }
    if (what == 2) {
        legendre_rt(a[i], l_max, P);
        for (int q = 0; q < NP; ++q) out[static_cast<size_t>(i) * NP + q] = P[q];
        return;
    }
    if (what == 3) {
        legendre_dtheta_rt(a[i], l_max, P, D);
        for (int q = 0; q < NP; ++q) {
            out[static_cast<size_t>(i) * 2 * NP + q] = P[q];
            out[static_cast<size_t>(i) * 2 * NP + NP + q] = D[q];
        }
        return;
    }
    const double theta = a[i], phi = b[i];
    if (what == 1) legendre_dtheta_rt(theta, l_max, P, D);
    else legendre_rt(cos(theta), l_max, P);
    double rr = 0.0, ri = 0.0;
    for (int l = 0; l <= l_max; ++l)
        for (int m = -l; m <= l; ++m) {
            const int am = m < 0 ? -m : m;
            const int idx = l * l + m + l;
            const double c = cos(m * phi), sn = sin(m * phi);
            if (what == 1) {
                const double nrm = normalization(l, am);
                const double pb = nrm * P[l * (l + 1) / 2 + am], pd = nrm * D[l * (l + 1) / 2 + am];
                const double br = pb * c, bi = pb * sn;
                double* o = out + static_cast<size_t>(i) * 6 * L;
                o[2 * idx] = br;
                o[2 * idx + 1] = bi;
                o[2 * L + 2 * idx] = pd * c;
                o[2 * L + 2 * idx + 1] = pd * sn;
                o[4 * L + 2 * idx] = 0.0 * br - static_cast<double>(m) * bi;  // cplx{0, m} * b
                o[4 * L + 2 * idx + 1] = 0.0 * bi + static_cast<double>(m) * br;
            } else {
                const double np = normalization(l, am) * P[l * (l + 1) / 2 + am];
                const double br = np * c, bi = np * sn;
                if (what == 0) {
                    out[static_cast<size_t>(i) * 2 * L + 2 * idx] = br;
                    out[static_cast<size_t>(i) * 2 * L + 2 * idx + 1] = bi;
                } else {  // eval_radiance: r += cplx{coef} * basis, component order
                    (void)0;
                }
            }
        }
    if (what == 5) {  // accumulate in component order (radiance.cpp:116-125)
        for (int comp = 0; comp < L; ++comp) {
            int l = 0;
            while ((l + 1) * (l + 1) <= comp) ++l;
            const int m = comp - l * l - l, am = m < 0 ? -m : m;
            const double np = normalization(l, am) * P[l * (l + 1) / 2 + am];
            const double br = np * cos(m * phi), bi = np * sin(m * phi);
            const double cr = coeffs[static_cast<size_t>(i) * 2 * L + 2 * comp],
                         ci = coeffs[static_cast<size_t>(i) * 2 * L + 2 * comp + 1];
            rr += cr * br - ci * bi;
            ri += cr * bi + ci * br;
        }
        out[2 * static_cast<size_t>(i)] = rr;
        out[2 * static_cast<size_t>(i) + 1] = ri;
    }
}

__global__ void k_occupancy(int K, int R, const double* __restrict__ pos,
                            const double* __restrict__ ls, const double* __restrict__ q,
                            const double* __restrict__ tau_logit, double lo0, double lo1,
                            double lo2, double hi0, double hi1, double hi2,
                            unsigned long long* __restrict__ out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    const double lo[3] = {lo0, lo1, lo2};
    const double ext[3] = {hi0 - lo0, hi1 - lo1, hi2 - lo2};
    const double cell[3] = {ext[0] / R, ext[1] / R, ext[2] / R};
    const double* p = pos + 3 * static_cast<size_t>(k);
    double m[9], r[9];
    covariance(ls + 3 * static_cast<size_t>(k), q + 4 * static_cast<size_t>(k), m);
    // Mat3::inverse (linalg.hpp:88-100)
    const double det = m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
                       m[2] * (m[3] * m[7] - m[4] * m[6]);
    r[0] = (m[4] * m[8] - m[5] * m[7]) / det; r[1] = (m[2] * m[7] - m[1] * m[8]) / det;
    r[2] = (m[1] * m[5] - m[2] * m[4]) / det; r[3] = (m[5] * m[6] - m[3] * m[8]) / det;
    r[4] = (m[0] * m[8] - m[2] * m[6]) / det; r[5] = (m[2] * m[3] - m[0] * m[5]) / det;
    r[6] = (m[3] * m[7] - m[4] * m[6]) / det; r[7] = (m[1] * m[6] - m[0] * m[7]) / det;
    r[8] = (m[0] * m[4] - m[1] * m[3]) / det;
    const double tau = 1.0 / (1.0 + exp(-tau_logit[k]));
    int a0[3], a1[3];
    for (int a = 0; a < 3; ++a) {
        const double half = 2.0 * sqrt(m[a * 4]);
        const int l = static_cast<int>(floor((p[a] - half - lo[a]) / cell[a] - 0.5));
        const int h = static_cast<int>(ceil((p[a] + half - lo[a]) / cell[a] - 0.5));
        a0[a] = l > 0 ? l : 0;
        a1[a] = h < R - 1 ? h : R - 1;
    }
    for (int ix = a0[0]; ix <= a1[0]; ++ix)
        for (int iy = a0[1]; iy <= a1[1]; ++iy)
            for (int iz = a0[2]; iz <= a1[2]; ++iz) {
                const double d0 = (lo[0] + (ix + 0.5) * cell[0]) - p[0];
                const double d1 = (lo[1] + (iy + 0.5) * cell[1]) - p[1];
                const double d2 = (lo[2] + (iz + 0.5) * cell[2]) - p[2];
                const double q0 = r[0] * d0 + r[1] * d1 + r[2] * d2;
                const double q1 = r[3] * d0 + r[4] * d1 + r[5] * d2;
                const double q2 = r[6] * d0 + r[7] * d1 + r[8] * d2;
                const double m2 = d0 * q0 + d1 * q1 + d2 * q2;
                if (m2 > 4.0) continue;
                const double v = tau * exp(-0.5 * m2);
                atomicMax(out + (static_cast<size_t>(ix) * R + iy) * R + iz,
                          static_cast<unsigned long long>(__double_as_longlong(v)));
            }
}

__global__ void k_occ_finish(size_t n, const unsigned long long* __restrict__ bits,
                             double* __restrict__ out64, float* __restrict__ out32) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    double v = __longlong_as_double(static_cast<long long>(bits[i]));
    v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    if (out64) out64[i] = v;
    if (out32) out32[i] = static_cast<float>(v);
}

}  // namespace

cudaError_t launch_tx_prep(const rxgs_scene_s& sc, rxgs_txstate_s& st, cudaStream_t s, bool full) {
    if (sc.k == 0) return cudaSuccess;
    const int threads = 128;
    const int blocks = (sc.k + threads - 1) / threads;
    auto kern = full ? (sc.l_max == 2 ? k_tx_prep<2, true, true>
                                      : (sc.l_max == 9 ? k_tx_prep<9, true, true> : k_tx_prep<0, true, true>))
                     : (sc.l_max == 2 ? k_tx_prep<2, false, false>
                                      : (sc.l_max == 9 ? k_tx_prep<9, false, false> : k_tx_prep<0, false, false>));
    kern<<<blocks, threads, 0, s>>>(
        sc.k, sc.l_max, sc.channels, sc.d_pos.as<double>(), sc.d_ls.as<double>(),
        sc.d_q.as<double>(), sc.d_tau.as<double>(), sc.d_coeffs64.as<double>(), st.tx[0], st.tx[1],
        st.tx[2], st.grid, st.rec.as<GaussRec>(), st.culled.as<int>(), st.geom.as<double>(),
        st.spans.as<int4>(), st.basis64.as<double>(), st.basis32.as<float2>(),
        st.gb32.as<float2>(), st.depth_key.as<uint64_t>(), st.tile_count.as<int>());
    return cudaGetLastError();
}

cudaError_t launch_basis_rows(const rxgs_scene_s& sc, rxgs_txstate_s& st, cudaStream_t s) {
    if (st.visible <= 0) return cudaSuccess;
    const int threads = 128;
    const unsigned blocks = static_cast<unsigned>((st.visible + threads - 1) / threads);
    auto kern = sc.l_max == 2 ? k_basis_rows<2> : (sc.l_max == 9 ? k_basis_rows<9> : k_basis_rows<0>);
    kern<<<blocks, threads, 0, s>>>(st.needed_count.as<int>(), st.needed_order.as<int>(), sc.l_max, sc.channels,
                                    st.rec.as<GaussRec>(), sc.d_coeffs64.as<double>(), st.basis32.as<float2>(),
                                    st.gb32.as<float2>());
    return cudaGetLastError();
}

cudaError_t launch_project(int n, const double* pos, const double* cov, const double* tau, const double* tx,
                           const DevGrid& g, double* geom, int* culled, int4* spans, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_project<<<(n + 127) / 128, 128, 0, s>>>(n, pos, cov, tau, tx[0], tx[1], tx[2], g, geom, culled, spans);
    return cudaGetLastError();
}

cudaError_t launch_fle_eval(int what, int n, int l_max, const double* a, const double* b, const double* coeffs,
                            double* out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    if (l_max > kApiLmax) return cudaErrorInvalidValue;
    k_fle_eval<<<(n + 63) / 64, 64, 0, s>>>(what, n, l_max, a, b, coeffs, out);
    return cudaGetLastError();
}

cudaError_t launch_rec_from_geom(int K, const int* culled, const double* geom, const double* basis64, int L,
                                 GaussRec* rec, float2* basis32, cudaStream_t s) {
    if (K == 0) return cudaSuccess;
    k_rec_from_geom<<<(K + 127) / 128, 128, 0, s>>>(K, culled, geom, basis64, L, rec, basis32);
    return cudaGetLastError();
}

cudaError_t launch_occupancy(const rxgs_scene_s& sc, int R, const double* lo, const double* hi,
                             double* d_out64, float* d_out32, cudaStream_t s) {
    const size_t n = static_cast<size_t>(R) * R * R;
    unsigned long long* bits = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&bits), n * 8, s);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(bits, 0, n * 8, s);
    if (e != cudaSuccess) return e;
    if (sc.k > 0) {
        k_occupancy<<<(sc.k + 127) / 128, 128, 0, s>>>(
            sc.k, R, sc.d_pos.as<double>(), sc.d_ls.as<double>(), sc.d_q.as<double>(),
            sc.d_tau.as<double>(), lo[0], lo[1], lo[2], hi[0], hi[1], hi[2], bits);
    }
    k_occ_finish<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(n, bits, d_out64, d_out32);
    e = cudaGetLastError();
    cudaFreeAsync(bits, s);
    return e;
}

}  // namespace rxgs_b200
