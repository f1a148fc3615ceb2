/* include/rxgs_b200.h -- C-ABI of the B200-native RxGS render path.
 *
 * This is the drop-in boundary: plain pointers and sizes, int status codes,
 * thread-local error text, no C++ or torch types.  Each entry point names the
 * reference interface it replaces (paths relative to /root/reference/proj).
 * The reference is a static C++ library with no FFI; the header-only C++
 * shim include/rxgs_b200.hpp re-exposes these calls under the reference's
 * own rxgs::raster / rxgs::cond / rxgs::train names and exception types.
 *
 * Pointers: every array argument may be HOST or DEVICE memory (detected with
 * cudaPointerGetAttributes).  Host outputs are written before the call
 * returns; device outputs are written in stream order on the context stream.
 * Layouts follow the reference exactly:
 *   scene coefficients   ((k*L + l)*C + c)*2 + {re,im}          scene.hpp:16-18
 *   per-rx coefficients  (((j*K + k)*L + l)*C + c)*2 + {re,im}   sphraster.hpp:92-93
 *   field values         [j][c][re/im][row][col]                 sphraster.hpp:83
 *   transmittance        [j][row][col]                           sphraster.hpp:84
 * Modality: 0 rssi, 1 csi, 2 spectrum (channelsim.hpp:79).
 * Conditioning mode: 0 full, 1 global_only, 2 local_only, 3 additive_only,
 * 4 no_occlusion (conditioning.hpp:55).
 */
#ifndef RXGS_B200_H
#define RXGS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RXGS_OK 0
#define RXGS_ERR_INVALID 1 /* reference: std::invalid_argument */
#define RXGS_ERR_RUNTIME 2 /* reference: std::runtime_error    */
#define RXGS_ERR_CUDA 3    /* device / driver failure          */
#define RXGS_ERR_IO 4      /* reference: io::IoError (dataset.hpp:16) */

typedef struct rxgs_ctx_s* rxgs_ctx;
typedef struct rxgs_scene_s* rxgs_scene;
typedef struct rxgs_txstate_s* rxgs_txstate;
typedef struct rxgs_cond_s* rxgs_cond;
typedef struct rxgs_trainer_s* rxgs_trainer;

/* raster::SphericalGrid (sphraster.hpp:15-32). */
typedef struct rxgs_grid {
    int32_t n_theta, n_phi, tile_size, reserved;
    double radius, theta_min, theta_max;
} rxgs_grid;

/* Thread-local text of the last failing call on this thread ("" if none).
 * Messages match the reference's exception text, e.g.
 * "render_field: non-finite coefficient at rx 1, gaussian 0". */
const char* rxgs_last_error(void);
int rxgs_version(void);

/* ------------------------------------------------------------ context */
int rxgs_ctx_create(int device, rxgs_ctx* out);
int rxgs_ctx_destroy(rxgs_ctx ctx);
/* Use an external cudaStream_t (e.g. torch's current stream); NULL = own. */
int rxgs_ctx_set_stream(rxgs_ctx ctx, void* cuda_stream);
int rxgs_ctx_synchronize(rxgs_ctx ctx);
/* Per-kernel CUDA-event timing of the hot kernels (off by default). */
int rxgs_ctx_profile(rxgs_ctx ctx, int enable);
/* Totals since the last reset for one kernel name ("cond_local", "composite",
 * "walk", "tx_prep", "cond_global", "signal", ...).  Synchronizes. */
int rxgs_ctx_kernel_stats(rxgs_ctx ctx, const char* name, double* total_ms, int64_t* launches,
                          double* work_units);
int rxgs_ctx_reset_stats(rxgs_ctx ctx);
/* Free the context's grow-only work buffers and recycled Tx-state buffers
 * (e.g. between workloads of very different sizes). */
int rxgs_ctx_release_cache(rxgs_ctx ctx);
/* Number of kernels of this library launched since the last reset. */
int64_t rxgs_ctx_launch_count(rxgs_ctx ctx);
/* Conditioning kernel selection: 0 = auto (tcgen05 when hidden == 64 and
 * C == 1, else FP32 SIMT), 1 = force the FP32 SIMT kernel (A/B checks). */
int rxgs_ctx_set_cond_kernel(rxgs_ctx ctx, int which);
/* Query-path compositing: 0 = auto (tcgen05 for 8x8 tiles, C == 1), 1 = FP32 SIMT. */
int rxgs_ctx_set_composite_kernel(rxgs_ctx ctx, int which);
/* Diagnostic: a 128x64x64 bf16 tcgen05 GEMM with A in TMEM and with A in
 * shared memory, max |error| vs FP32 FMA of the same values; err[5] =
 * {smooth: A-in-TMEM, A-in-smem; small integers (exact): TMEM, smem;
 * small integers, both operands MN-major (the compositor's layout)}. */
int rxgs_selftest_tcgen05(rxgs_ctx ctx, double* err);

/* ------------------------------------------------------------ synthetic inputs
 * DESIGN.md section 5 (bit-identical to oracle/ and to the reference-side
 * harness; built on the reference RNG, rng.hpp:17-72). */
int rxgs_synth_scene(int k, int l_max, int channels, uint64_t seed, double* positions,
                     double* log_scales, double* quaternions, double* tau_logits,
                     double* fle_coeffs);
int rxgs_synth_points(int n, uint64_t seed, const char* tag, const double lo[3],
                      const double hi[3], double margin, double* out);
/* Returns the packed parameter count; params may be NULL to query it. */
int64_t rxgs_synth_cond(const int32_t cfg[9], int l_max, int channels, const double lo[3],
                        const double hi[3], uint64_t seed, int randomize, double* params);

/* ------------------------------------------------------------ scene
 * GaussianScene (scene.hpp:19-48) upload. */
int rxgs_scene_create(rxgs_ctx ctx, int k, int l_max, int channels, int modality,
                      const double* positions, const double* log_scales,
                      const double* quaternions, const double* tau_logits,
                      const double* fle_coeffs, rxgs_scene* out);
int rxgs_scene_destroy(rxgs_scene scene);
/* GaussianScene::position_bounds().inflated(f) (scene.cpp:18-30). */
int rxgs_scene_bounds(rxgs_scene scene, double inflate, double lo[3], double hi[3]);

/* ------------------------------------------------------------ transmitter state
 * raster::build_tx_state (sphraster.cpp:150-172): projection
 * (project_gaussian :22-83, FP64), FLE basis (radiance.cpp:79-92), per-tile
 * depth-sorted lists (bin_and_sort :85-102) and the receiver-independent
 * front-to-back blend weights of every cell (render_field :285-298). */
int rxgs_tx_state_build(rxgs_ctx ctx, rxgs_scene scene, const double tx[3],
                        const rxgs_grid* grid, rxgs_txstate* out);
int rxgs_tx_state_destroy(rxgs_txstate st);
int64_t rxgs_tx_state_entries(rxgs_txstate st);
/* Materialise TxState fields (sphraster.hpp:52-61).  Any pointer may be NULL.
 * geom per Gaussian = theta, phi, depth, cov a b c d, prec a b c d,
 * weight_scale (12 f64); spans = t0 t1 p0 p1; basis K*L complex (2 f64);
 * offsets n_tiles+1 (int64); indices = concatenated tile lists (int32). */
int rxgs_tx_state_get(rxgs_txstate st, int32_t* culled, double* geom, int32_t* spans,
                      double* basis, int64_t* offsets, int32_t* indices);
/* Sort keys in list order: (tile << 32) | depth_rank, depth_rank = position
 * of the Gaussian in the (depth, index) order of all Gaussians. */
int rxgs_tx_state_keys(rxgs_txstate st, uint64_t* keys);
/* Receiver-independent statistics: visible Gaussians, list entries,
 * mean walk per cell, mean tile-walk per cell (roofline inputs). */
int rxgs_tx_state_stats(rxgs_txstate st, int64_t* visible, int64_t* entries, double* walk_per_cell,
                        double* tile_walk_per_cell);
/* Gaussians reached by at least one cell's front-to-back walk (list position
 * below the tile's longest walk): the rows the batched query conditions. */
int rxgs_tx_state_needed(rxgs_txstate st, int64_t* needed);
/* Per-cell final transmittance (cells f64); identical for every receiver. */
int rxgs_tx_state_transmittance(rxgs_txstate st, double* out);

/* raster::bin_and_sort on caller-supplied projections (sphraster.cpp:85-102):
 * culled[k], depth[k], spans[k*4].  Writes offsets (n_tiles+1) and, when
 * cap >= entries, indices; *entries receives the total. */
int rxgs_bin_and_sort(rxgs_ctx ctx, int k, const int32_t* culled, const double* depth,
                      const int32_t* spans, const rxgs_grid* grid, int64_t* offsets,
                      int32_t* indices, int64_t cap, int64_t* entries);

/* ------------------------------------------------------------ render
 * raster::render_field(TxState, scene, coeffs, n_rx) (sphraster.cpp:255-315)
 * with the reference's materialised per-receiver coefficient tensor
 * (n_rx*K*L*C*2 f64).  values / transmittance in the reference layouts. */
int rxgs_render_field(rxgs_ctx ctx, rxgs_txstate st, rxgs_scene scene, const double* coeffs,
                      int n_rx, double* values, double* transmittance);

/* raster::aggregate_modality (sphraster.cpp:323-381).  out: rssi n_rx f64;
 * csi n_rx*C*2; spectrum n_rx*H*W. */
int rxgs_aggregate_modality(rxgs_ctx ctx, const rxgs_grid* grid, int modality, int n_rx,
                            int channels, const double* values, double* out);

/* raster::aggregate_modality_backward (sphraster.cpp:383-449).  upstream has
 * rxgs_aggregate_modality's out layout; d_values the field layout
 * (n_rx*C*2*H*W f64).  Scalar modalities need channels == 1. */
int rxgs_aggregate_modality_backward(rxgs_ctx ctx, const rxgs_grid* grid, int modality, int n_rx,
                                     int channels, const double* values, const double* upstream,
                                     double* d_values);

/* raster::backward_render (sphraster.cpp:509-733): exact FP64 adjoint of
 * rxgs_render_field.  d_values: n_rx*C*2*H*W; outputs (GradientBundle,
 * sphraster.hpp): d_positions K*3, d_log_scales K*3, d_quaternions K*4,
 * d_tau_logits K, d_coeffs n_rx*K*L*C*2.  Any output may be NULL. */
int rxgs_backward_render(rxgs_ctx ctx, rxgs_txstate st, rxgs_scene scene, const double* coeffs,
                         int n_rx, const double* d_values, double* d_positions,
                         double* d_log_scales, double* d_quaternions, double* d_tau_logits,
                         double* d_coeffs);

/* ------------------------------------------------------------ coverage consumers
 * apps::coverage_fraction / apps::greedy_plan (apps.hpp:34-43, apps.cpp:69-116)
 * over a tx-major RSSI table (tx_count x cand_count f64 dBm, host or
 * device; e.g. rxgs_coverage_table's output widened to f64).  Exact:
 * threshold tests and counts; greedy ties break on the lower candidate.
 * greedy_plan writes k candidate indices in selection order. */
/* ------------------------------------------------------------ Stage-I densification
 * densify_and_prune (scene.cpp:178-274, scene.hpp:69-97) on the device, in
 * place: the scene's row set becomes the reference's (in-place rows, then
 * clones / second split children in source order, then the prune), with
 * the split signs drawn from derive_stream(seed, "scene.densify",
 * pass_index).  grad_accum / accum_count: the DensifyState (K each, host or
 * device); thresholds = {grad_threshold, size_frac, prune_extent_frac,
 * split_scale_factor} (NULL: DensifyThresholds defaults).  report =
 * {cloned, split, pruned}; source_row (new K entries, caller-sized for 2K)
 * maps each row to its source row or -1.  TxStates built before the call
 * are stale. */
int rxgs_densify_and_prune(rxgs_ctx ctx, rxgs_scene scene, const double* grad_accum, const int32_t* accum_count,
                           double scene_extent, const double thresholds[4], uint64_t seed, uint64_t pass_index,
                           int32_t report[3], int32_t* source_row, int32_t* new_count);
/* reset_transmittance (scene.cpp:276-279): every tau logit = logit(0.01). */
int rxgs_reset_transmittance(rxgs_scene scene);

/* met::mae / mse / psnr / ssim (metrics.hpp:14-28, metrics.cpp:11-112) of a
 * batch of n_img images (h x w row-major; pred f32 if pred_f32 else f64, gt
 * f64; host or device): out[4*i..] = {mae, mse, psnr(max_val), ssim}.
 * ssim_opts = {window, sigma, dynamic_range} (NULL: SsimOptions defaults
 * 11, 1.5, 1.0; window 0 skips SSIM and writes NaN).  Identical images give
 * the 300 dB sentinel (kDbSentinel); errors carry the reference texts. */
int rxgs_image_metrics(rxgs_ctx ctx, const void* pred, int pred_f32, const double* gt, int n_img, int h, int w,
                       double max_val, const double ssim_opts[3], double* out);
/* met::snr_csi (metrics.hpp:33, metrics.cpp:114-125) for n_sets pairs of
 * len complex values (pred / gt n_sets*len*2 f64): out_db n_sets; identical
 * inputs give the 300 dB sentinel; the reference's errors. */
int rxgs_snr_csi(rxgs_ctx ctx, int n_sets, int64_t len, const double* pred, const double* gt, double* out_db);
/* met::per_receiver_aggregate (metrics.hpp:35-41, metrics.cpp:127-149) of n
 * (rx, value) records: per receiver in ascending rx order the mean and the
 * record count (outputs sized n, *n_unique filled), the mean of those means
 * and their population stddev. */
int rxgs_per_receiver_aggregate(rxgs_ctx ctx, int64_t n, const int32_t* rx, const double* values, int32_t* out_rx,
                                double* out_mean, int64_t* out_count, int32_t* n_unique, double* mean,
                                double* stddev);

int rxgs_coverage_fraction(rxgs_ctx ctx, const double* table, int64_t tx_count, int64_t cand_count,
                           const int32_t* selected, int n_selected, double threshold_dbm, double* out);
int rxgs_greedy_plan(rxgs_ctx ctx, const double* table, int64_t tx_count, int64_t cand_count, int k,
                     double threshold_dbm, int32_t* order);

/* ------------------------------------------------------------ scene / model load
 * io::save_checkpoint / io::load_checkpoint (checkpoint.hpp:17-18,
 * checkpoint.cpp:93-231): the RXGS container ("RXGS", u32 version 1, u64
 * header length, JSON header with a named f64 array manifest, the arrays).
 * save: the scene (device coefficients synced first), the grid and, when
 * cond is non-NULL, the conditioning state incl. its occupancy grid.
 * load: creates the scene on ctx, fills *grid, and creates *cond when the
 * file has a conditioning state (cond may be NULL to skip it).  Errors
 * carry the reference's IoError text (RXGS_ERR_IO). */
int rxgs_checkpoint_save(const char* path, rxgs_scene scene, const rxgs_grid* grid, rxgs_cond cond);
int rxgs_checkpoint_load(rxgs_ctx ctx, const char* path, rxgs_scene* scene, rxgs_grid* grid, rxgs_cond* cond);
/* Shape of a scene (GaussianScene::count / l_max / channels / modality) and
 * the configuration of a conditioning state (rxgs_cond_create's cfg). */
int rxgs_scene_info(rxgs_scene scene, int32_t* k, int32_t* l_max, int32_t* channels, int32_t* modality);
int rxgs_cond_config(rxgs_cond cond, int32_t cfg[9]);
/* Host copies of a scene's per-Gaussian arrays (any pointer may be NULL;
 * coefficients are the device's current values). */
int rxgs_scene_get_arrays(rxgs_scene scene, double* positions, double* log_scales, double* quaternions,
                          double* tau_logits, double* fle_coeffs);
/* A conditioning state's occupancy grid: *has = 0 for an empty grid;
 * densities (R^3, may be NULL) and bounds (may be NULL) otherwise. */
int rxgs_cond_get_occupancy(rxgs_cond cond, int32_t* has, double* densities, double lo[3], double hi[3]);

/* ------------------------------------------------------------ conditioning
 * cond::ConditioningState (conditioning.hpp:72-92).  cfg = {F, hidden, d_c,
 * S, R, nearest_lookup, mode, l_max, C}; params packed as
 * freqs | global l1.w l1.b l2.w l2.b l3.w l3.b | embed | local (same six).
 * occupancy: R^3 f64 (index (ix*R+iy)*R+iz) or NULL for an empty grid. */
int rxgs_cond_create(rxgs_ctx ctx, const int32_t cfg[9], const double* params,
                     const double* occupancy, const double occ_lo[3], const double occ_hi[3],
                     rxgs_cond* out);
int rxgs_cond_destroy(rxgs_cond c);
int64_t rxgs_cond_param_count(rxgs_cond c);
/* Per-branch MLP invocation counters (conditioning.hpp:81-82). */
int rxgs_cond_calls(rxgs_cond c, int64_t* global_calls, int64_t* local_calls);
/* cond::build_occupancy (conditioning.cpp:114-161) on device; out R^3 f64 may
 * be NULL.  If attach_to is non-NULL the grid becomes its occupancy. */
int rxgs_build_occupancy(rxgs_ctx ctx, rxgs_scene scene, int resolution, const double lo[3],
                         const double hi[3], double* out, rxgs_cond attach_to);
/* cond::probe_segment (conditioning.cpp:163-178) for n segments against the
 * conditioning state's occupancy (device FP32): out n*2 = (T, mean). */
int rxgs_probe_segments(rxgs_ctx ctx, rxgs_cond c, int n, const double* from, const double* to,
                        double* out);
/* cond::condition_forward (conditioning.cpp:284-423) for one receiver:
 * out K*L*C*2.  local_in (K*6) may be NULL (ConditionWorkspace::local_in). */
int rxgs_condition_forward(rxgs_ctx ctx, rxgs_cond c, rxgs_scene scene, const double rx[3],
                           double* out, double* local_in);

/* cond::condition_backward (conditioning.cpp:472-587) for one receiver, with
 * the workspace recomputed on device.  d_out: K*L*C*2 gradient w.r.t. the
 * conditioned coefficients; d_base: K*L*C*2 gradient w.r.t. the scene's
 * base coefficients; d_params: ConditioningGrads packed in the
 * rxgs_cond_create parameter order (freqs | global MLP | embed | local MLP),
 * rxgs_cond_param_count values.  d_base / d_params may be NULL. */
int rxgs_condition_backward(rxgs_ctx ctx, rxgs_cond cond, rxgs_scene scene, const double rx[3],
                            const double* d_out, double* d_base, double* d_params);
/* cond::condition_batch (conditioning.cpp:425-435): out n_rx*K*L*C*2. */
int rxgs_condition_batch(rxgs_ctx ctx, rxgs_cond c, rxgs_scene scene, const double* rx, int n_rx,
                         double* out);

/* ------------------------------------------------------------ batched queries
 * The hot path: train::predict (trainer.cpp:147-154) batched over receivers
 * (paper Algorithm 1) without materialising N*K*L*C*2 coefficients:
 * conditioning (global + local branch) fused with the FLE basis reduction,
 * then front-to-back compositing with the spectrum / RSSI epilogue.
 * rx: n_rx*3 f64.  out_spectrum: n_rx*H*W f32 (may be NULL); out_rssi: n_rx
 * f32 dB (may be NULL).  cond may be NULL (unconditioned model). */
int rxgs_render_queries(rxgs_ctx ctx, rxgs_scene scene, rxgs_cond c, rxgs_txstate st,
                        const double* rx, int n_rx, float* out_spectrum, float* out_rssi);

/* Coverage table (BASELINE config 3): out_rssi[t*n_rx + j] = RSSI (dB) of
 * train::predict(model, tx_t, rx_j) (trainer.cpp:147-154), the table
 * apps::coverage_fraction / greedy_plan consume (apps.cpp:70-116, layout
 * rssi_table[t*candidates + c]).  The Tx-independent conditioning (local
 * branch per (Gaussian, rx), global branch per rx) is computed once and
 * reused for every transmitter.  cond may be NULL (unconditioned scene).
 * Requires channels == 1.  With two or more transmitters the per-Tx states
 * are built by up to 4 host threads (RXGS_COV_BUILDERS, 0 = serial), each on
 * a helper context of ctx (own stream and buffer pool, created on first use
 * and freed with ctx) while the calling thread renders on ctx's stream; the
 * table is bitwise the same for any builder count.  The call returns after
 * ctx's stream has finished the table. */
int rxgs_coverage_table(rxgs_ctx ctx, rxgs_scene scene, rxgs_cond cond, const rxgs_grid* grid,
                        const double* tx, int n_tx, const double* rx, int n_rx, float* out_rssi);

/* train::predict for one (tx, rx): builds the TxState internally; out is the
 * scene modality's measurement (spectrum H*W, rssi 1, csi C*2) in f64. */
int rxgs_predict(rxgs_ctx ctx, rxgs_scene scene, rxgs_cond c, const rxgs_grid* grid,
                 const double tx[3], const double rx[3], double* out);

/* ------------------------------------------------------------ training (config 4)
 * One step of the Stage-II chain of conditioned_training_loop
 * (trainer.cpp:410-466): condition_forward -> render_field -> spectrum
 * aggregate -> composite_loss (L1 + SSIM + DFT2 terms) ->
 * aggregate_modality_backward -> backward_render (coefficient part) ->
 * condition_backward, for a batch of receivers sharing one transmitter.
 * hyper = {feature_lr, rest_lr_ratio, conditioning_lr, lambda_ssim,
 * lambda_fft, adam beta1, beta2, epsilon}; NULL = the reference defaults
 * 5e-3, 0.2, 1e-3 (TrainConfig, trainer.hpp:68-97), 0.2, 0.1 (LossWeights,
 * trainer.hpp:25-29), 0.9, 0.999, 1e-8. */
int rxgs_trainer_create(rxgs_ctx ctx, rxgs_scene scene, rxgs_cond c, const double hyper[8], rxgs_trainer* out);
int rxgs_trainer_destroy(rxgs_trainer t);
/* Sum over the n_rx samples of the per-sample gradients (the reference's
 * d_base and ConditioningGrads, packed like the parameters) into the
 * trainer's flat f64 gradient buffer [d_base | d_params] (added to it when
 * accumulate != 0).  targets: n_rx x H x W spectra (f32); losses: n_rx. */
int rxgs_train_grads(rxgs_trainer t, rxgs_txstate st, const double* rx, int n_rx, const float* targets,
                     double* losses, int accumulate);
/* Device pointer and sizes of the flat gradient buffer, for the caller's
 * data-parallel all-reduce (sum) before rxgs_train_apply. */
int rxgs_train_grad_buffer(rxgs_trainer t, double** dev_ptr, int64_t* n, int64_t* n_base);
int rxgs_train_get_grads(rxgs_trainer t, double* d_base, double* d_params);
/* Copy of the whole flat buffer (n values of rxgs_train_grad_buffer) into a
 * host or device array, after the trainer's stream has drained. */
int rxgs_train_get_grad_buffer(rxgs_trainer t, double* out);
/* In-place NCCL all-reduce (sum, ncclFloat64) of the flat gradient buffer
 * on the trainer's stream, over the caller's communicator (an ncclComm_t
 * passed as void*, one rank per GPU): the data-parallel exchange between
 * rxgs_train_grads and rxgs_train_apply, over the whole
 * buffer (n of rxgs_train_grad_buffer, geometry gradients included in joint
 * and Stage-I trainers). NCCL is resolved at run time from the library the
 * process already loaded (RXGS_NCCL_LIBRARY overrides the soname). */
int rxgs_train_allreduce(rxgs_trainer t, void* nccl_comm);
/* Optimizer::step on "features" (degree >= 1 scaled by rest_lr_ratio) and
 * every conditioning group (diffengine.cpp:50-58): throws the reference's
 * "optimizer: non-finite gradient in group ..." error, else Adam in place on
 * the device copies of the scene coefficients and conditioning parameters. */
int rxgs_train_apply(rxgs_trainer t);
/* Joint training (train_joint / the train_geometry branch of
 * conditioned_training_loop, trainer.cpp:417-463): call once before the
 * first step.  The flat gradient buffer grows by the geometry gradients of
 * backward_render, [d_positions 3K | d_tau_logits K | d_log_scales 3K |
 * d_quaternions 4K], summed over the batch; rxgs_train_apply then applies
 * the FLE degree mask (apply_degree_mask, trainer.cpp:233-248) and Adam on
 * position (opt::lr_at schedule, diffengine.cpp:36-48), transmittance,
 * scaling and rotation, and renormalises the quaternions
 * (scene.cpp:281-288).  The caller rebuilds the TxState every step, as the
 * reference does.  geo (NULL = TrainConfig defaults, trainer.hpp:78-92):
 * {position lr_init, lr_final, total_steps, delay_mult, delay_steps,
 *  transmittance_lr, scaling_lr, rotation_lr, fle_ramp_interval}. */
int rxgs_trainer_enable_geometry(rxgs_trainer t, const double geo[9]);
/* Stage I (train_stage1, trainer.cpp:294-380) is the joint step with
 * cond == NULL at rxgs_trainer_create: the scene's own coefficients render,
 * d_base is backward_render's d_coeffs, and rxgs_train_apply accumulates the
 * DensifyState (||d_position|| per Gaussian, scene.cpp:141-151).
 * rxgs_train_densify runs one densification tick on it (densify_and_prune +
 * Optimizer::remap_rows of every per-Gaussian group, trainer.cpp:359-372;
 * thresholds as rxgs_densify_and_prune); rxgs_train_reset_transmittance is
 * reset_transmittance + optimizer.reset("transmittance") (trainer.cpp:354-358).
 * Both need rxgs_trainer_enable_geometry; the flat gradient buffer is
 * reallocated by rxgs_train_densify (query rxgs_train_grad_buffer again). */
int rxgs_train_densify(rxgs_trainer t, double scene_extent, const double thresholds[4], uint64_t seed,
                       uint64_t pass_index, int32_t report[3]);
int rxgs_train_reset_transmittance(rxgs_trainer t);
int rxgs_train_get_geometry_grads(rxgs_trainer t, double* d_positions, double* d_log_scales,
                                  double* d_quaternions, double* d_tau_logits);
int64_t rxgs_train_step_count(rxgs_trainer t);
/* Current (possibly trained) device parameters. */
int rxgs_scene_get_coeffs(rxgs_scene scene, double* out);
int rxgs_cond_get_params(rxgs_cond c, double* out);

/* ------------------------------------------------------------ single-call reference API
 * The reference's per-call helpers on the device in FP64 with the
 * reference's operation order (k_geometry.cu / k_refapi.cu, -fmad=false);
 * they back the link-level drop-in paper_2605_24290_b200/refapi and the
 * header shim include/rxgs_b200.hpp.  Host or device buffers. */
/* raster::project_gaussian (sphraster.hpp:46, sphraster.cpp:22-83) for n
 * Gaussians: pos n*3, cov n*9 (row-major Mat3), tau n (activated); out geom
 * n*12 = {theta, phi, depth, A (a, b, c, d), A^-1 (a, b, c, d), tau},
 * culled n, spans n*4 = {t0, t1, p0, p1}. */
int rxgs_project_gaussians(rxgs_ctx ctx, int n, const double* pos, const double* cov, const double* tau,
                           const double tx[3], const rxgs_grid* grid, double* geom, int32_t* culled, int32_t* spans);
/* fle:: (radiance.hpp:36-70): what = 0 eval_basis (a=theta, b=phi; out n*L
 * complex), 1 eval_basis_jet (out n*3L complex: b, db/dtheta, db/dphi),
 * 2 legendre_table (a=x; out n*NP, NP=(l_max+1)(l_max+2)/2), 3
 * legendre_table_dtheta (a=theta; out n*2NP: P then dP), 4 normalization
 * (a=l, b=m; out n), 5 eval_radiance (a=theta, b=phi, coeffs n*L complex;
 * out n complex).  The reference's argument errors. */
int rxgs_fle_eval(rxgs_ctx ctx, int what, int l_max, int n, const double* a, const double* b, const double* coeffs,
                  double* out);
/* raster::blend_ray (sphraster.hpp:82, sphraster.cpp:174-185): weights n,
 * signals n complex; out = {re, im, transmittance}. */
int rxgs_blend_ray(rxgs_ctx ctx, int n, const double* weights, const double* signals, double out[3]);
/* OccupancyGrid::sample_trilinear / sample_nearest (conditioning.cpp:74-112)
 * at n points; densities R^3 or NULL (empty grid -> 0). */
int rxgs_occupancy_sample(rxgs_ctx ctx, int R, const double lo[3], const double hi[3], const double* densities, int n,
                          const double* points, int nearest, double* out);
/* cond::probe_segment (conditioning.hpp:50, conditioning.cpp:163-178) over an
 * explicit grid (FP64): out n*2 = {transmittance, mean_density}. */
int rxgs_probe_grid(rxgs_ctx ctx, int R, const double lo[3], const double hi[3], const double* densities, int n,
                    const double* from, const double* to, int samples, int nearest, double* out);
/* cond::fourier_encode (conditioning.cpp:255-265): freqs F*3, r n*3, out n*6F. */
int rxgs_fourier_encode(rxgs_ctx ctx, int F, const double* freqs, int n, const double* r, double* out);
/* cond::MlpLayer::forward (conditioning.cpp:12-19) on n input vectors. */
int rxgs_mlp_layer_forward(rxgs_ctx ctx, int in, int out_dim, const double* w, const double* b, int n,
                           const double* x, double* y);
/* raster::SphericalGrid::validate (sphraster.cpp:14-20): the reference's errors. */
int rxgs_grid_validate(const rxgs_grid* grid);
/* cond::condition_forward with an explicit base (conditioning.hpp:114-117):
 * base K*L*C*2 instead of the scene's coefficients; n_rx receivers, out
 * n_rx*K*L*C*2; local_in K*6 of the first receiver or NULL. */
int rxgs_condition_forward_base(rxgs_ctx ctx, rxgs_cond c, rxgs_scene scene, const double* base, const double* rx,
                                int n_rx, double* out, double* local_in);
/* A device transmitter state from a host raster::TxState (sphraster.hpp:52-61):
 * the rows of rxgs_tx_state_get (culled, geom, spans, basis) and the per-tile
 * lists as CSR (offsets n_tiles+1, indices); the blend walk and the needed-row
 * compaction run on the device.  render_field / backward_render /
 * render_queries accept it like a built state (no sort keys). */
int rxgs_tx_state_import(rxgs_ctx ctx, rxgs_scene scene, const rxgs_grid* grid, const int32_t* culled,
                         const double* geom, const int32_t* spans, const double* basis, const int64_t* offsets,
                         const int32_t* indices, rxgs_txstate* out);

#ifdef __cplusplus
}
#endif
#endif /* RXGS_B200_H */
