/*
 * sgdt_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the SGD_Tucker reference algorithm (arXiv 2012.03550,
 * reference tree /root/reference/proj) used as the parity CHECKER for the
 * B200 path.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * / --impl reference legs may load it.  The product library (libsgdt.so) never
 * links or calls anything in this directory.
 *
 * Every routine follows the reference's own operation order in fp64 so that its
 * results are bit-identical to the reference compiled from source
 * (oracle/_ref, built by oracle/Makefile); tests/test_oracle_pin.py checks that.
 * Parity of this restatement is therefore PINNED against the reference itself.
 *
 * Conventions follow the reference: coordinates are 1-based u32, entry-major
 * (coords[e*order + k]); factors A^(n) are I_n x J_n row-major; Kruskal
 * matrices B^(n) are J_n x R row-major.
 */
#ifndef SGDT_ORACLE_H
#define SGDT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OR_MAX_ORDER 8

/* Error codes: the reference's exception taxonomy (common.hpp:13-43). */
enum {
  OR_OK = 0,
  OR_INTERNAL = 1,
  OR_CONFIG = 2,
  OR_DATA = 3,
  OR_NUMERIC = 4,
  OR_DOMAIN = 5
};

/* ---- RNG: std::mt19937_64 + Rng distributions (rng.hpp:13-49) ---------- */
typedef struct {
  uint64_t mt[312];
  uint32_t idx;
  int has_spare;
  double spare;
} or_rng;

void or_rng_seed(or_rng* r, uint64_t seed);
uint64_t or_rng_next(or_rng* r);
uint64_t or_next_below(or_rng* r, uint64_t bound);
double or_next_unit(or_rng* r);
double or_next_gaussian(or_rng* r, double mean, double stddev);
/* n raw engine outputs from seed (KAT helper). */
void or_mt_outputs(uint64_t seed, size_t n, uint64_t* out);

/* ---- sparse tensor (sptensor.hpp:66-107, sptensor.cpp:80-118) ----------- */
typedef struct {
  int order;
  uint32_t dims[OR_MAX_ORDER];
  size_t nnz;
  uint32_t* coords;                 /* nnz*order, 1-based */
  double* values;                   /* nnz */
  uint32_t* perm[OR_MAX_ORDER];     /* per-mode bucketed entry ids */
  uint64_t* offsets[OR_MAX_ORDER];  /* dims[n]+1 */
} or_tensor;

int or_tensor_init(or_tensor* t, int order, const uint32_t* dims, size_t nnz,
                   const uint32_t* coords, const double* values);
void or_tensor_free(or_tensor* t);

/* ---- model (model.hpp:40-91, model.cpp) --------------------------------- */
typedef struct {
  int order;
  uint32_t dims[OR_MAX_ORDER];
  uint32_t J[OR_MAX_ORDER];
  uint32_t R;
  double* A[OR_MAX_ORDER];        /* I_n x J_n */
  double* B[OR_MAX_ORDER];        /* J_n x R */
  uint64_t core_elems;
  double* core;                   /* prod J, mode-1 fastest */
  double* unfold[OR_MAX_ORDER];   /* J_n x prod_{k!=n} J_k */
} or_model;

int or_model_init(or_model* m, int order, const uint32_t* dims, const uint32_t* J, uint32_t R);
void or_model_free(or_model* m);
int or_model_copy(or_model* dst, const or_model* src);
int or_model_init_gaussian(or_model* m, double mean, double stddev, uint64_t seed);
void or_model_refresh_core(or_model* m);
double or_model_predict(const or_model* m, const uint32_t* coord);
int or_model_all_finite(const or_model* m);

/* ---- scheduling helpers (scheduler.cpp:34-46) --------------------------- */
void or_partition_even(size_t count, size_t workers, size_t* begins, size_t* ends);

/* ---- sampler (sptensor.cpp:256-270) ------------------------------------- */
/* pool is nnz long; if *pool_valid == 0 it is (re)initialised to iota. */
int or_sample_batch(size_t nnz, size_t m, or_rng* rng, uint32_t* pool, int* pool_valid,
                    uint32_t* out);

/* ---- optimizers (core_optimizer.cpp:112-257, factor_optimizer.cpp:101-273) */
typedef struct {
  double lr;
  double reg;
  size_t batch_m;            /* 0 = full training set */
  int resample_per_mode;
  int incremental_residual;
} or_core_hyper;

typedef struct {
  double lr;
  double reg;
  double row_fraction;
} or_factor_hyper;

typedef struct {
  uint32_t* pool;   /* nnz, persistent across epochs */
  int pool_valid;
  uint32_t* batch;  /* last Psi drawn (capacity nnz) */
  size_t batch_len;
} or_core_ws;

int or_core_ws_init(or_core_ws* ws, size_t nnz);
void or_core_ws_free(or_core_ws* ws);

/* Serial strategy.  If psi_log != NULL, every Psi drawn is appended there
 * (psi_log_len counts entries written). */
int or_update_core_epoch(or_model* m, const or_tensor* t, const or_core_hyper* h, or_rng* rng,
                         or_core_ws* ws);
int or_update_factor_epoch(or_model* m, const or_tensor* t, const or_factor_hyper* h,
                           or_rng* rng, size_t* rows_updated, size_t* rows_skipped);

/* ---- eval (eval.cpp:15-33) ---------------------------------------------- */
int or_rmse_mae(const or_model* m, const or_tensor* t, double* rmse, double* mae);

/* ---- trainer (trainer.cpp:66-139) --------------------------------------- */
typedef struct {
  double lr_a, lr_b, reg_a, reg_b;
  size_t batch_m;
  double row_fraction;
  size_t epochs;
  uint64_t seed;
  double init_mean, init_stddev;
  int resample_core_batch;
  int incremental_residual;
} or_hyper;

/* metrics: epochs x 4 doubles {train_rmse, train_mae, test_rmse, test_mae}. */
int or_train(or_model* m, const or_tensor* train, const or_tensor* test, const or_hyper* h,
             double* metrics);

/* ---- synthetic data + split (synth.cpp:16-67, sptensor.cpp:217-254) ----- */
/* coords_out: nnz*order, values_out: nnz. */
int or_synth_planted(int order, const uint32_t* dims, const uint32_t* tJ, uint32_t tR,
                     size_t nnz, double noise_stddev, double teacher_mean,
                     double teacher_stddev, uint64_t seed, uint32_t* coords_out,
                     double* values_out);
/* Writes the entry ids of the test half then the train half (each ascending)
 * into ids_out (nnz); returns ntest via *ntest_out. */
int or_train_test_split_ids(size_t nnz, double test_fraction, uint64_t seed, uint32_t* ids_out,
                            size_t* ntest_out);

#ifdef __cplusplus
}
#endif

#endif
