// Internal types shared by the C-ABI layer (capi.cu) and the kernels.
// Device-side data layout is documented in DESIGN.md section 3.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <map>
#include <string>
#include <unordered_map>
#include <vector>

#include "rxgs_b200.h"

namespace rxgs_b200 {

constexpr double kPi = 3.14159265358979323846;
constexpr double kTwoPi = 2.0 * kPi;
constexpr double kWeightClamp = 0.999;  // sphraster.hpp:72
constexpr double kEarlyExitT = 1e-4;    // sphraster.hpp:73
constexpr double kRssiFloor = 1e-12;    // channelsim.hpp:115
constexpr double kAmpEps = 1e-8;        // radiance.hpp:80
constexpr int kMaxLmax = 15;            // basis recurrences kept in registers/local memory
constexpr int kMaxCellsPerBlock = 64;   // composite cell block (one 8x8 tile)

struct DevGrid {
    int nt, np, ts, tiles_t, tiles_p, n_tiles, cpt, cell_blocks;
    double radius, tmin, tmax, dth, dph;
};

// Receiver-independent per-Gaussian record read by the FP64 blend walk.
struct alignas(64) GaussRec {
    double theta, phi, sin_theta, pa, pbc, pd, tau, cos_theta;  // cos_theta: for the adjoint re-walk
};

// Error capture: thread-local message + status.
struct Status {
    int code = RXGS_OK;
    std::string msg;
};
int fail(int code, const std::string& msg);
uint64_t next_version();  // process-wide, never 0
int cuda_fail(cudaError_t e, const char* what);

#define RXGS_CUDA(call)                                              \
    do {                                                             \
        cudaError_t e__ = (call);                                    \
        if (e__ != cudaSuccess) return ::rxgs_b200::cuda_fail(e__, #call); \
    } while (0)

#define TRY_RC(expr)                      \
    do {                                  \
        const int rc__ = (expr);          \
        if (rc__ != RXGS_OK) return rc__; \
    } while (0)

// initial SplitMix64 state of the reference's derive_stream (synth.cpp)
uint64_t derive_stream_state(uint64_t seed, const char* tag, uint64_t counter);

// Grow-only device buffer.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) {
        o.p = nullptr;
        o.bytes = 0;
    }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            if (p) cudaFree(p);
            p = o.p;
            bytes = o.bytes;
            o.p = nullptr;
            o.bytes = 0;
        }
        return *this;
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    cudaError_t ensure(size_t n) {
        if (n <= bytes && p) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        cudaError_t e = cudaMalloc(&p, n ? n : 16);
        if (e == cudaSuccess) bytes = n;
        return e;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// Destination of the per-(Gaussian, receiver) signals s[k][j][c]: either
// complex f32 (f2), or -- for the tcgen05 compositor, C == 1 -- the same 8
// bytes pre-split for its bf16x3 product: split[k][j] = {hi, lo} with hi =
// bf16x2(re, im) rounded to nearest and lo = bf16x2 of the remainders.
struct SigOut {
    float2* f2 = nullptr;
    uint2* split = nullptr;
    SigOut() = default;
    SigOut(float2* p) : f2(p) {}  // NOLINT: implicit on purpose
    static SigOut presplit(void* p) {
        SigOut o;
        o.split = static_cast<uint2*>(p);
        return o;
    }
};

struct KStat {
    double ms = 0.0;
    int64_t launches = 0;
    double work = 0.0;
};

struct PendingTiming {
    std::string name;
    cudaEvent_t a, b;
    double work;
};

}  // namespace rxgs_b200

struct rxgs_txstate_s;

struct rxgs_ctx_s {
    std::vector<rxgs_txstate_s*> spare_tx;  // recycled transmitter-state buffers (<= 2)
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    bool profile = false;
    int64_t launches = 0;
    std::map<std::string, rxgs_b200::KStat> stats;
    std::vector<rxgs_b200::PendingTiming> pending;
    std::vector<cudaEvent_t> event_pool;
    // scratch
    rxgs_b200::DevBuf sort_tmp, scratch_a, scratch_b, scratch_c, scratch_d, signals, ag, partial,
        err_flag, host_in, host_out, ycache;
    // conditioning rows gathered into row order (k_cond_tc.cu): positions,
    // (basis*base, basis) transposed to [l][row], their sums over l
    rxgs_b200::DevBuf row_pos, row_GB, row_S;
    // FLE GEMM operands / result for high l_max (k_fle_gemm.cu)
    rxgs_b200::DevBuf fle_a, fle_b, fle_m;
    rxgs_b200::DevBuf probe_tr;  // (T, rho) per (receiver, needed row) from k_probe_rows
    // version of the transmitter state whose receiver-independent row data
    // (row_pos / row_GB / row_S and the GEMM's A operand) the buffers hold,
    // so receiver chunks of one query batch gather and pack it once
    uint64_t rows_version = 0, fle_a_version = 0;
    int sm_count = 148;
    int cond_kernel = 0;  // 0 auto (tcgen05 when eligible), 1 force SIMT
    int composite_kernel = 0;  // 0 auto (tcgen05 when eligible), 1 force SIMT
    std::atomic<int> refs{0};  // live handles on this context (builder threads retain / release)
    cudaStream_t copy_stream = nullptr;  // D2H of finished receiver chunks (host outputs)
    std::vector<cudaEvent_t> chunk_events;
    bool closed = false;  // rxgs_ctx_destroy called while handles were alive
    // helper context (own stream and scratch) that builds the next
    // transmitter's state while this one's stream renders the current one
    // (rxgs_coverage_table); created on first use
    static constexpr int kAuxMax = 8;
    rxgs_ctx_s* aux[kAuxMax] = {};
    cudaEvent_t aux_ev[kAuxMax] = {}, aux_done[kAuxMax] = {};
};

struct rxgs_scene_s {
    rxgs_ctx ctx = nullptr;
    int k = 0, l_max = 0, channels = 1, L = 1, modality = 0;
    std::vector<double> h_pos, h_ls, h_q, h_tau, h_coeffs;
    rxgs_b200::DevBuf d_pos, d_ls, d_q, d_tau, d_coeffs64, d_coeffs32, d_pos32;
    // Morton (Z-order) permutation of the Gaussians and their f32 positions
    // in that order (build_scene_order, k_sort.cu)
    rxgs_b200::DevBuf d_morton, d_mpos32;
    bool host_stale = false;  // device coefficients updated by the optimizer
    bool geo_stale = false;   // device geometry updated by the joint optimizer
    // bumped whenever the device FLE coefficients / geometry change (optimizer
    // steps, densify): transmitter states remember the values they were built
    // or refreshed at, so a reused state never renders stale basis*base rows
    uint64_t coeff_version = 1, geo_version = 1;
    // transmitter states built from this scene keep it alive (lean states are
    // completed from it on demand); rxgs_scene_destroy drops the caller's ref
    std::atomic<int> refs{1};
    // exact position -> lowest Gaussian index (receiver-on-Gaussian check,
    // conditioning.cpp:380-382), built lazily on the host
    std::unordered_map<std::string, int> pos_index;
    bool pos_index_built = false;
};

struct rxgs_txstate_s {
    rxgs_ctx ctx = nullptr;
    int k = 0, l_max = 0, L = 1, channels = 1;
    rxgs_b200::DevGrid grid{};
    double tx[3] = {0, 0, 0};
    int64_t entries = 0, visible = 0;
    double walk_sum = 0.0, tile_walk_sum = 0.0;
    rxgs_b200::DevBuf rec, culled, geom, spans, basis64, basis32, gb32, depth_key, tile_count,
        order, rank, scan, tile_offsets, list, keys, tw, walk_len, cell_T, cell_len, needed,
        needed_order, needed_count;
    // Gaussians reached by at least one cell's walk (list position < the
    // tile's longest walk), in the scene's Morton order: the only rows whose
    // conditioned signal is ever read by the compositor.  needed_count is
    // device-side.
    int64_t needed_host = -1;
    // changes whenever the state's per-Gaussian data does (build, refresh_gb)
    uint64_t version = 0;
    // the scene's coeff_version / geo_version this state's basis*base rows
    // and geometry were computed from
    uint64_t coeff_version = 0, geo_version = 0;
    // the scene it was built from (retained), and whether geom / basis64 are
    // filled (false after a lean build: the query path never reads them)
    rxgs_scene_s* sc = nullptr;
    bool full = false;
    // walked list entries regrouped by Gaussian (training adjoint), built lazily
    rxgs_b200::DevBuf gauss_off, gauss_ent;
    bool regrouped = false;
};

struct rxgs_cond_s {
    rxgs_ctx ctx = nullptr;
    int F = 6, hidden = 64, dc = 16, S = 16, R = 32, nearest = 0, mode = 0, l_max = 0, C = 1;
    int L = 1, gin = 0;
    int64_t n_params = 0;
    size_t o_freq, o_gw1, o_gb1, o_gw2, o_gb2, o_gw3, o_gb3, o_emb, o_lw1, o_lb1, o_lw2, o_lb2,
        o_lw3, o_lb3;
    std::vector<double> h_params;
    bool has_occ = false;
    std::vector<double> h_occ;  // host f64 copy of the occupancy densities (checkpoint save)
    double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    int64_t global_calls = 0, local_calls = 0;
    rxgs_b200::DevBuf d_params32, d_params64, d_occ32, d_occ64;  // d_occ64: the FP64 API kernels (k_refapi.cu)
    // trilinear cell table: per cell c in [-1, R]^3 the 8 polynomial
    // coefficients of its trilinear patch (k_occ_cubes, k_cond.cu)
    rxgs_b200::DevBuf d_occ_cube;
    bool host_stale = false;  // device parameters updated by the optimizer
    bool use_global() const { return mode != 2; }
    bool use_local() const { return mode != 1; }
    bool additive() const { return mode == 3; }
    bool no_occ() const { return mode == 4 || !has_occ; }
};

namespace rxgs_b200 {

// ---- context lifetime (capi.cu)
void ctx_retain(rxgs_ctx ctx);
void ctx_release(rxgs_ctx ctx);
void scene_release(rxgs_scene_s* sc);  // drops one reference, frees at zero

// ---- timing helpers (capi.cu)
void timing_begin(rxgs_ctx ctx, const char* name, cudaEvent_t* a);
void timing_end(rxgs_ctx ctx, const char* name, cudaEvent_t a, double work);

// ---- k_geometry.cu (FP64, compiled with -fmad=false)
cudaError_t launch_tx_prep(const rxgs_scene_s& sc, rxgs_txstate_s& st, cudaStream_t s, bool full);
// the lean build's basis rows for the needed Gaussians (after compact_needed)
cudaError_t launch_basis_rows(const rxgs_scene_s& sc, rxgs_txstate_s& st, cudaStream_t s);
// Completes a lean state with its FP64 geometry / basis (capi.cu): the scene
// must still have the geometry the state was built from.
int ensure_tx_full(rxgs_txstate_s& st, cudaStream_t s);
cudaError_t launch_project(int n, const double* pos, const double* cov, const double* tau, const double* tx,
                           const DevGrid& g, double* geom, int* culled, int4* spans, cudaStream_t s);
cudaError_t launch_fle_eval(int what, int n, int l_max, const double* a, const double* b, const double* coeffs,
                            double* out, cudaStream_t s);
constexpr int kApiMaxLmax = 24;
// ---- k_sort.cu helpers: stable LSD radix sort of (u32 key, int) pairs on the
// low `bits` bits (work: radix_sort_work_ints(n) ints, zeroed), exclusive
// int64 scan (bsum: n / 2048 + 2 int64)
size_t radix_sort_work_ints(int n);
cudaError_t radix_sort_pairs(int n, int bits, uint32_t* kin, int* vin, uint32_t* ktmp, int* vtmp, int* work,
                             bool hist_ready, cudaStream_t s);
cudaError_t scan_i64(int64_t n, const int64_t* in, int64_t* out, int64_t* bsum, cudaStream_t s);
cudaError_t scan_i32(int64_t n, const int* in, int* out, int64_t* bsum, cudaStream_t s);
size_t scan_bsum_count(int64_t n);
// ---- k_refapi.cu (FP64 single-call API kernels)
// located non-finite check of n coefficients, rows of per_row (k_cond.cu)
cudaError_t launch_check_finite(long long n, long long per_row, const double* d_coeffs, int* d_err, cudaStream_t s);
// materialised render_field, FP64 signals and walk (k_refapi.cu)
cudaError_t launch_render64(const rxgs_txstate_s& st, const double* d_co, int n_rx, double2* d_sig, double* values,
                            double* tout, cudaStream_t s);
cudaError_t launch_blend_ray(int n, const double* w, const double* sig, double* out, cudaStream_t s);
cudaError_t launch_occ_sample(int R, const double* lo, const double* hi, const double* dens, int n, const double* pts,
                              int nearest, double* out, cudaStream_t s);
cudaError_t launch_probe64(int R, const double* lo, const double* hi, const double* dens, int n, const double* from,
                           const double* to, int samples, int nearest, double* out, cudaStream_t s);
cudaError_t launch_fourier64(int F, const double* freqs, int n, const double* r, double* out, cudaStream_t s);
cudaError_t launch_mlp_layer64(int in, int nout, const double* w, const double* b, int n, const double* x, double* y,
                               cudaStream_t s);
cudaError_t launch_cond_forward64(const rxgs_cond_s& c, const rxgs_scene_s& sc, const double* d_rx, int n_rx,
                                  const double* base, double* ag64, double* out, double* local_in, cudaStream_t s);
cudaError_t launch_rec_from_geom(int K, const int* culled, const double* geom, const double* basis64, int L,
                                 GaussRec* rec, float2* basis32, cudaStream_t s);
cudaError_t launch_occupancy(const rxgs_scene_s& sc, int R, const double* lo, const double* hi,
                             double* d_out64, float* d_out32, cudaStream_t s);

// ---- k_sort.cu
// Bins culled/spans/depth_key already in st; fills tile_offsets, list, keys.
int bin_tiles(rxgs_ctx ctx, rxgs_txstate_s& st, cudaStream_t s);

// ---- k_walk.cu (FP64, -fmad=false)
cudaError_t launch_walk(rxgs_txstate_s& st, cudaStream_t s);
// Marks and compacts the Gaussians the walk reaches (st.needed_order/count).
int compact_needed(rxgs_ctx ctx, const rxgs_scene_s& sc, rxgs_txstate_s& st, cudaStream_t s);
// Morton order of the scene (sc.d_morton, sc.d_mpos32), once at scene creation.
int build_scene_order(rxgs_ctx ctx, rxgs_scene_s& sc, cudaStream_t s);

// ---- k_cond.cu
cudaError_t launch_cond_global(const rxgs_cond_s& c, const double* d_rx, int n_rx, float* d_ag,
                               cudaStream_t s);
// Fused local branch + FLE reduction: signals[k][j][c] complex f32.
cudaError_t launch_cond_signal(const rxgs_cond_s* c, const rxgs_scene_s& sc,
                               const rxgs_txstate_s& st, const double* d_rx, int n_rx,
                               const float* d_ag, SigOut d_sig, int* d_err, cudaStream_t s);
// Materialised conditioned coefficients (condition_forward API).
cudaError_t launch_cond_materialize(const rxgs_cond_s& c, const rxgs_scene_s& sc,
                                    const double* d_rx, int n_rx, const float* d_ag, double* d_out,
                                    double* d_local_in, int* d_err, cudaStream_t s);
// the same, only for the TxState's needed Gaussians (other rows untouched)
// the joint step's materialised conditioning on tcgen05: y = (alpha_L, beta_L)
// of the needed rows, then both affines in FP64 (C == 1)
cudaError_t launch_local_y_rows(const rxgs_cond_s& cs, const rxgs_scene_s& sc, const rxgs_txstate_s& st,
                                const double* d_rx, int n_rx, float4* y, cudaStream_t s);
cudaError_t launch_materialize_y(const rxgs_cond_s& c, const rxgs_scene_s& sc, const rxgs_txstate_s& st, int n_rx,
                                 const float* d_ag, const float4* y, double* d_out, cudaStream_t s);
cudaError_t launch_cond_materialize_needed(const rxgs_cond_s& c, const rxgs_scene_s& sc, const rxgs_txstate_s& st,
                                           const double* d_rx, int n_rx, const float* d_ag, double* d_out,
                                           cudaStream_t s);
// (re)build rxgs_cond_s::d_occ_cube from d_occ32
cudaError_t launch_occ_cubes(rxgs_cond_s& c, cudaStream_t s);
cudaError_t launch_probe(const rxgs_cond_s& c, int n, const double* d_from, const double* d_to,
                         double* d_out, cudaStream_t s);
cudaError_t launch_check_coincide(const rxgs_scene_s& sc, const double* d_rx, int n_rx, int* d_err,
                                  cudaStream_t s);
// tcgen05 variant of the hot kernel (k_cond_tc.cu): hidden 64, C == 1.
bool cond_tc_eligible(const rxgs_cond_s* c);
bool cond_ws_enabled();
cudaError_t launch_cond_signal_tc(const rxgs_cond_s& c, const rxgs_scene_s& sc, const rxgs_txstate_s& st,
                                  const double* d_rx, int n_rx, const float* d_ag, SigOut d_sig,
                                  cudaStream_t s, const float2* mpre_given = nullptr);
cudaError_t launch_cond_signal_tc_prep(const rxgs_cond_s& cs, const rxgs_scene_s& sc, const rxgs_txstate_s& st,
                                       int n_rx, const float* d_ag, cudaStream_t s, const float2** mpre);
cudaError_t launch_tc_selftest(float* d_err, cudaStream_t s);
// FLE reduction of the query path as a tensor-core GEMM: Mout[j][row] (k_fle_gemm.cu)
int fle_gemm_kpad(int L);
cudaError_t launch_fle_gemm(rxgs_ctx ctx, const int* n_rows_dev, long long rows_bound, int cap, int L, int n_rx,
                            const float4* rGB, const float4* rS, const float* d_ag, float2* Mout, cudaStream_t s,
                            uint64_t a_version, bool row_major = false);
// Per-row Tx data of the needed rows into ctx->row_* (k_cond_tc.cu), once per state version.
cudaError_t gather_rows(const rxgs_scene_s& sc, const rxgs_txstate_s& st, cudaStream_t s);
cudaError_t launch_tc_selftest_mn(float* d_err, cudaStream_t s);
// reduce_signals from materialised f64 coefficients.
cudaError_t launch_reduce_signals(const rxgs_txstate_s& st, const double* d_coeffs, int n_rx,
                                  float2* d_sig, int* d_err, cudaStream_t s);

// ---- k_composite.cu
struct CompositeOut {
    float* spectrum = nullptr;    // [j][cell] (C == 1)
    float* rssi_partial = nullptr;  // [tile][j] power partials (C == 1)
    double* values = nullptr;     // [j][c][re/im][cell] f64 (materialised field)
    float* csi_partial = nullptr; // [tile][j][c][2]
    float* field32 = nullptr;     // [j][c][re/im][cell] f32 (training forward)
};
cudaError_t launch_composite(const rxgs_txstate_s& st, const float2* d_sig, int n_rx,
                             const CompositeOut& out, cudaStream_t s);
// tcgen05 compositing (k_composite_tc.cu): 8x8 tiles, C == 1.
bool composite_tc_eligible(const rxgs_txstate_s& st);
// reads the pre-split signals (SigOut::presplit)
cudaError_t launch_composite_tc(const rxgs_txstate_s& st, const uint2* d_sig, int n_rx, const CompositeOut& out,
                                cudaStream_t s);
cudaError_t launch_rssi_finalize(const float* d_partial, int n_tiles, int n_rx, float* d_rssi,
                                 double* d_rssi64, cudaStream_t s);
cudaError_t launch_aggregate(const DevGrid& g, int modality, int n_rx, int channels,
                             const double* d_values, double* d_out, int* d_err, bool reduce,
                             cudaStream_t s);
cudaError_t launch_fill_transmittance(const rxgs_txstate_s& st, int n_rx, double* d_T,
                                      cudaStream_t s);

// ---- k_train.cu
int train_regroup(rxgs_ctx ctx, rxgs_txstate_s& st, cudaStream_t s);
// ---- k_coverage.cu (config-3 coverage table)
cudaError_t launch_local_cache_tc(const rxgs_cond_s& cs, const rxgs_scene_s& sc, const double* d_rx, int n_rx,
                                  float4* ycache, cudaStream_t s);
cudaError_t launch_local_cache(const rxgs_cond_s& cs, const rxgs_scene_s& sc, const double* d_rx, int n_rx,
                               float4* ycache, cudaStream_t s);
cudaError_t launch_ag_transpose(int n_rx, int L, const float* d_ag, float* d_agT, cudaStream_t s);
cudaError_t launch_cov_signal(const rxgs_cond_s* cs, const rxgs_txstate_s& st, int n_rx, const float* d_agT,
                              const float4* ycache, SigOut d_sig, cudaStream_t s);
// the same signals from the FLE GEMM's M[row][j] (k_coverage.cu)
cudaError_t launch_cov_signal_gemm(const rxgs_cond_s* cs, const rxgs_scene_s& sc, const rxgs_txstate_s& st, int n_rx,
                                   const float* d_ag, const float4* ycache, SigOut d_sig, cudaStream_t s);
// ---- k_cond_bwd.cu (FP64 materialised conditioning adjoint)
size_t cond_backward_ws_bytes(const rxgs_cond_s& cs, int K, int sms);
cudaError_t launch_cond_backward(const rxgs_cond_s& cs, const rxgs_scene_s& sc, const double* d_rx,
                                 const double* d_out, double* d_base, double* d_params, void* ws, int sms,
                                 cudaStream_t s);
// ---- k_backward.cu (FP64 adjoints of the materialised API)
cudaError_t launch_aggregate_bwd(const DevGrid& g, int modality, int n_rx, int channels, const double* values,
                                 const double* up, double* dv, cudaStream_t s);
// bytes of the ent_geo scratch of launch_backward_render (per receiver chunk)
size_t bwd_geo_bytes(int64_t entries, int n_jc);
cudaError_t launch_backward_render(const rxgs_txstate_s& st, const rxgs_scene_s& sc, const double* d_coeffs_in,
                                   int n_rx, const double* d_values, double2* sig64, double* ent_geo,
                                   double2* ent_ds, double* raw_geo, double2* raw_ds, double* d_pos, double* d_ls,
                                   double* d_q, double* d_tau, double* d_coeffs, cudaStream_t s,
                                   bool needed_only = false);  // coefficients valid for the needed rows only

cudaError_t launch_refresh_gb(const rxgs_scene_s& sc, rxgs_txstate_s& st, cudaStream_t s);
cudaError_t launch_loss_spectrum(int n_rx, int P, const float* field, const float* target, double l_weight,
                                 float2* G, double* loss_part, double* loss, cudaStream_t s);
// composite_loss (spectrum) with the SSIM and DFT terms; ws of loss_full_ws_bytes
size_t loss_full_ws_bytes(int n_rx, int h, int w);
cudaError_t launch_loss_full(int n_rx, int h, int w, const float* field, const float* target, double l_w,
                             double lambda_ssim, double lambda_fft, double dyn_range, float2* G, void* ws, double* loss,
                             cudaStream_t s);
cudaError_t launch_render_adjoint(const rxgs_txstate_s& st, const float2* G, int n_rx, float2* d_entry, float2* d_s,
                                  cudaStream_t s);
size_t cond_bwd_smem();
int cond_bwd_parts(int sms);
int local_grad_n();
cudaError_t launch_cond_bwd(const rxgs_cond_s& cs, const rxgs_scene_s& sc, const rxgs_txstate_s& st,
                            const double* d_rx, int n_rx, const float* d_ag, const float2* d_s, float2* u,
                            float* part, int n_parts, cudaStream_t s, float* act = nullptr, bool tc_rows = false);
// the per-row half of the split backward on tcgen05 (spectrum-L1 training)
cudaError_t launch_cond_bwd_tc(const rxgs_cond_s& cs, const rxgs_scene_s& sc, const rxgs_txstate_s& st,
                               const double* d_rx, int n_rx, const float* d_ag, const float2* d_s, float2* u,
                               uint16_t* act, long long rpad, cudaStream_t s);
// scratch of the split backward (0 when the fused kernel is used)
size_t cond_bwd_act_bytes(long long rows);
cudaError_t launch_reduce_parts(int n_parts, int n, const float* part, double* out, cudaStream_t s);
cudaError_t launch_dbase(const rxgs_cond_s* cs, const rxgs_scene_s& sc, const rxgs_txstate_s& st, int n_rx,
                         const float* d_ag, const float2* u, double* d_base, cudaStream_t s);
cudaError_t launch_global_bwd(const rxgs_cond_s& cs, const rxgs_scene_s& sc, const rxgs_txstate_s& st, int n_rx,
                              const double* d_rx, const float2* u, double* red_part, int n_red, double* row_part,
                              double* gslice, double* grad, cudaStream_t s);
cudaError_t launch_check_finite64(int64_t n, const double* v, int* bad, cudaStream_t s);
// joint (geometry) training step helpers (k_train.cu)
struct GroupBounds {
    int n;
    int64_t start[24];
};
cudaError_t launch_dv_from_G(int n_rx, int P, const float2* G, double* dv, cudaStream_t s);
cudaError_t launch_degree_mask(int64_t n, int L, int per_comp, int active, double* g, cudaStream_t s);
cudaError_t launch_add64(int64_t n, const double* a, double* out, cudaStream_t s);
cudaError_t launch_check_groups(int64_t n, const GroupBounds& b, const double* g, int* bad, cudaStream_t s);
cudaError_t launch_geo_post(rxgs_scene_s& sc, cudaStream_t s);
// met::{mae, mse, psnr, ssim} of a batch of images (k_train.cu)
size_t image_metrics_ws_bytes(int n_img, int h, int w, int win);
cudaError_t launch_image_metrics(int n_img, int h, int w, const void* pred, bool pred_f32, const double* gt,
                                 double max_val, int win, double sigma, double dyn, void* ws, double* out,
                                 cudaStream_t s);
// Stage-I densification (k_densify.cu)
cudaError_t launch_dens_accumulate(int K, const double* dpos, double* accum, int* count, cudaStream_t s);
cudaError_t launch_remap_rows(int n_rows, int width, const int* source, const double* in, double* out,
                              cudaStream_t s);
cudaError_t launch_fill64(int64_t n, double v, double* x, cudaStream_t s);
// densify_and_prune on the scene's device arrays (replaced in place, then
// scene_resized); source_out[new K] = source row or -1
int densify_scene(rxgs_ctx ctx, rxgs_scene_s* sc, const double* d_accum, const int* d_count, double extent,
                  const double thr[4], uint64_t stream_state, int report[3], DevBuf& source_out);
// host copies + f32 mirrors + Morton order after the scene's row set changed
int scene_resized(rxgs_scene_s* sc);
// host copies of a scene whose device arrays the optimizer updated
int scene_sync_host(rxgs_scene_s* sc);
cudaError_t launch_adam(int64_t n, double* w, const double* g, double* m, double* v, double lr, int64_t step,
                        double b1, double b2, double eps, int lr_scale_L, int per_comp, double rest_ratio, float* w32,
                        cudaStream_t s);

}  // namespace rxgs_b200
