/* oracle/rxgs_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C CPU restatement of the RxGS reference render path, used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg as the CHECKER.
 * It is never linked into, called by, or measured as the product.  Every
 * function cites the reference file:line it restates (paths relative to
 * /root/reference/proj).  FP64 throughout, compiled with -ffp-contract=off
 * and the reference's operation order, so geometry matches the reference
 * build (oracle/_ref) bit for bit (pinned in tests/test_oracle.py).
 *
 * The entry points mirror oracle/ref_harness.cpp one-for-one (prefix or_
 * instead of ref_), so tests can run the same checks against either.
 */
#ifndef RXGS_ORACLE_H
#define RXGS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* grid: gi = {n_theta, n_phi, tile_size}, gd = {radius, theta_min, theta_max} */

int or_abi_version(void);
void or_synth_scene(int k, int l_max, int channels, uint64_t seed, double* pos, double* ls,
                    double* q, double* tau, double* coeffs);
void or_synth_points(int n, uint64_t seed, const char* tag, const double* lo, const double* hi,
                     double margin, double* out);
long or_synth_cond(const int* cfg, int l_max, int channels, const double* blo, const double* bhi,
                   uint64_t seed, int randomize, double* params_out);

void* or_scene_new(int k, int l_max, int channels, int modality, const double* pos,
                   const double* ls, const double* q, const double* tau, const double* coeffs);
void or_scene_free(void* h);
void or_scene_bounds(void* h, double inflate, double* lo, double* hi);
void or_covariance(void* h, double* out);

void* or_tx_new(void* scene, const double* tx, const int* gi, const double* gd, char* err,
                int errlen);
void or_tx_free(void* h);
long or_tx_entries(void* h);
void or_tx_get(void* h, int* culled, double* geom, int* spans, double* basis, long* offsets,
               int* indices, uint64_t* hash);
long or_bin_and_sort(int k, const int* culled, const double* depth, const int* spans,
                     const int* gi, const double* gd, long* offsets, int* indices, long cap);

int or_render(void* tx, void* scene, const double* coeffs, long n_coeffs, int n_rx, int threads,
              double* values, double* transmittance, char* err, int errlen);
int or_aggregate(int n_rx, int channels, const int* gi, const double* gd, const double* values,
                 int modality, double* out, char* err, int errlen);

void* or_cond_new(const int* cfg, const double* params, const double* occ, const double* occ_lo,
                  const double* occ_hi);
void or_cond_free(void* h);
long or_cond_param_count(void* h);
void or_build_occupancy(void* scene, int resolution, const double* lo, const double* hi,
                        double* out);
void or_probe(int resolution, const double* lo, const double* hi, const double* dens,
              const double* from, const double* to, int samples, int nearest, double* out2);
int or_cond_forward(void* cond, void* scene, const double* rx, double* out, double* ws_local_in,
                    double* ws_local_out, double* ws_global_out, char* err, int errlen);
void or_eval_basis(double theta, double phi, int l_max, double* out);
int or_predict(void* scene, void* cond, const int* gi, const double* gd, const double* tx,
               const double* rx, int threads, double* out, char* err, int errlen);

#ifdef __cplusplus
}
#endif
#endif
