/*
 * sgdt.h -- C-ABI of the B200-native SGD_Tucker training hot path.
 *
 * This is the drop-in boundary: plain pointers, sizes and POD structs, no
 * exceptions and no torch types.  The C++ host API that mirrors the reference
 * (paper_2012_03550_b200/cpp/include/sptucker/ headers, namespace sptucker) sits on
 * top of it, exactly as the reference's per-epoch calls sit on top of its CPU
 * loops.  Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj).
 *
 * Error codes mirror the reference exception taxonomy
 * (include/sptucker/common.hpp:13-43) and the CLI exit codes
 * (tools/sptucker_main.cpp:430-445):
 *   0 OK, 1 internal / CUDA, 2 ConfigError, 3 DataError, 4 NumericError,
 *   5 DomainError.  sgdt_last_error() returns the message of the last failure
 *   on the calling thread.
 *
 * Conventions (same as the reference): modes are 0-based, coordinate VALUES
 * are 1-based u32 in entry-major order (CooTensor::coord, sptensor.hpp:80-82),
 * A^(n) is I_n x J_n row-major, B^(n) is J_n x R row-major, fp64 on the host.
 * On the device parameters are fp32; the sampler, permutations and shard
 * assignment are bit-exact with the reference.
 */
#ifndef SGDT_H
#define SGDT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SGDT_OK 0
#define SGDT_ERR_INTERNAL 1
#define SGDT_ERR_CONFIG 2
#define SGDT_ERR_DATA 3
#define SGDT_ERR_NUMERIC 4
#define SGDT_ERR_DOMAIN 5

#define SGDT_MAX_ORDER 8
#define SGDT_MAX_RCORE 32
#define SGDT_MAX_J 64

typedef struct sgdt_session sgdt_session;

/* A CooTensor as the reference holds it (sptensor.hpp:66-107). */
typedef struct {
  int order;                          /* N, 2..SGDT_MAX_ORDER */
  const uint32_t* dims;               /* N */
  uint64_t nnz;                       /* < 2^32 (sptensor.cpp:87-88) */
  const uint32_t* coords;             /* nnz*N, 1-based, entry-major */
  const double* values;               /* nnz */
  /* Optional: CooTensor::mode_perm(n) for n < N (entry ids bucketed by the
   * mode-n coordinate, ascending entry id inside a bucket,
   * sptensor.cpp:102-117).  NULL -> the library computes the same stable
   * counting sort on the host. */
  const uint32_t* const* mode_perm;
} sgdt_tensor_desc;

/* CoreHyper (core_optimizer.hpp:13-19). */
typedef struct {
  double lr;
  double reg;
  uint64_t batch_m; /* |Psi|; 0 = full training set (no RNG) */
  int resample_per_mode;
  int incremental_residual; /* accepted; the device V-identity is exact for both */
} sgdt_core_hyper;

/* FactorHyper (factor_optimizer.hpp:14-18). */
typedef struct {
  double lr;
  double reg;
  double row_fraction; /* (0,1]; < 1 draws per-row subsets from the session RNG */
} sgdt_factor_hyper;

/* CoreEpochStats (core_optimizer.hpp:51-54). */
typedef struct {
  uint64_t batch_size;
  uint64_t effective_workers;
} sgdt_core_stats;

/* FactorEpochStats (factor_optimizer.hpp:44-48).  max_imbalance: the
 * reference's improved-strategy slice imbalance with the ranks of a sharded
 * session as its workers (largest partition_even(nnz, world) slice / (nnz /
 * world) - 1); 0 for a single session, as the reference with one worker. */
typedef struct {
  uint64_t rows_updated;
  uint64_t rows_skipped;
  double max_imbalance;
} sgdt_factor_stats;

/* Per-phase device times from CUDA events on the session stream: the means
 * over the epochs of the last sgdt_run_epochs / sgdt_run_epochs_host /
 * sgdt_train call (its last 1024 epochs at most; `epochs` says how many). */
typedef struct {
  float sample_ms;
  float core_ms;
  float factor_ms;
  float factor_mode_ms[SGDT_MAX_ORDER];
  uint32_t epochs;
} sgdt_timing;

const char* sgdt_last_error(void);
const char* sgdt_version(void);
/* Number of CUDA devices visible (0 without a GPU or driver). */
int sgdt_device_count(void);

/* The CooTensor constructor's work on the device (sptensor.cpp:80-118): the
 * coordinate range and duplicate checks -- DataError "entry <e>: coordinate
 * out of range" / "entry <e>: duplicate coordinate" at the first failing
 * entry, range first, as the reference's entry-by-entry loop reports it --
 * and, for each mode n with a non-NULL perm_out[n] / offsets_out[n] (host
 * buffers of nnz / I_n + 1 entries), CooTensor::mode_perm(n) (entry ids
 * bucketed by i_n, ascending inside a bucket; a stable radix sort) and
 * mode_offsets(n) (offsets[0] = 0, offsets[i] = end of bucket i).
 * perm_out / offsets_out may be NULL (checks only). */
int sgdt_tensor_layout(const sgdt_tensor_desc* t, int device, uint32_t* const* perm_out,
                       uint64_t* const* offsets_out);

/* Upload a training tensor (and optional test tensor, may be NULL) and size
 * the device model for ranks J (N entries) and R.  Builds the entry-order
 * record copy, one mode-sorted record copy per mode (the layout of
 * CooTensor::mode_perm/mode_offsets) and the nnz-balanced chunk schedule.
 * Replaces the per-call setup inside update_core_epoch / update_factor_epoch
 * (core_optimizer.cpp:112-151, factor_optimizer.cpp:101-136).
 * device < 0 selects the current device. */
int sgdt_session_create(const sgdt_tensor_desc* train, const sgdt_tensor_desc* test,
                        const uint32_t* J, uint32_t R, int device, sgdt_session** out);
void sgdt_session_destroy(sgdt_session* s);

/* The session's CUDA stream (cudaStream_t) -- every kernel runs on it. */
void* sgdt_session_stream(sgdt_session* s);

/* Model state in/out, fp64 host <-> fp32 device.  A[n] is I_n x J_n, B[n] is
 * J_n x R (TuckerModel::factor/kruskal, model.hpp:54-58).  sgdt_get_model
 * skips A (or B) when that argument is NULL (a phase changed only the other). */
int sgdt_set_model(sgdt_session* s, const double* const* A, const double* const* B);
int sgdt_get_model(sgdt_session* s, double* const* A, double* const* B);

/* RNG state crossing the boundary: the 312-word std::mt19937_64 state plus
 * its position (rng.hpp:46).  The device consumes exactly the outputs the
 * host Rng would have consumed. */
int sgdt_set_rng(sgdt_session* s, const uint64_t* mt312, uint32_t pos);
int sgdt_get_rng(sgdt_session* s, uint64_t* mt312, uint32_t* pos);
/* Reset the persistent sample pool to iota (CoreBatchWorkspace::sample_pool
 * sized wrong, sptensor.cpp:260-263). */
int sgdt_reset_pool(sgdt_session* s);

/* The persistent sample pool (CoreBatchWorkspace::sample_pool,
 * core_optimizer.hpp:36): nnz entry ids, a permutation of 0..nnz-1. */
int sgdt_set_pool(sgdt_session* s, const uint32_t* pool);
int sgdt_get_pool(sgdt_session* s, uint32_t* pool);

/* sample_batch (sptensor.cpp:256-270) on the device pool; out (host, m
 * entries) may be NULL. */
int sgdt_sample_batch(sgdt_session* s, uint64_t m, uint32_t* out);
/* The last Psi drawn by the core phase or sgdt_sample_batch (host copy). */
int sgdt_last_batch(sgdt_session* s, uint32_t* out, uint64_t* len);

/* update_core_epoch (core_optimizer.cpp:112-257). */
int sgdt_core_epoch(sgdt_session* s, const sgdt_core_hyper* h, sgdt_core_stats* st);
/* update_factor_epoch (factor_optimizer.cpp:101-273). */
int sgdt_factor_epoch(sgdt_session* s, const sgdt_factor_hyper* h, sgdt_factor_stats* st);
/* update_factor_epoch on a host Model& (the drop-in's per-epoch call): the
 * factor passes, with A^(n) copied out to A_out[n] (fp64 host, pageable or
 * pinned) as soon as mode n is final -- the copy of mode n overlaps the
 * passes of the later modes.  B is not touched. */
int sgdt_factor_epoch_host(sgdt_session* s, const sgdt_factor_hyper* h, double* const* A_out,
                           sgdt_factor_stats* st);
/* The persistent pool's change from the last sgdt_core_epoch / sgdt_sample_batch
 * call (exactly one sampler run of m draws): pos[i] = j_i (the draw targets,
 * sample_batch's partial Fisher-Yates) and val[i] = pool[j_i] afterwards, for
 * i < m; with positions < m holding the batch, applying them to the previous
 * host pool gives the new one.  *n = m.  SGDT_ERR_CONFIG when the last call
 * made no or several sampler runs (resample_per_mode): use sgdt_get_pool. */
int sgdt_pool_delta(sgdt_session* s, uint32_t* pos, uint32_t* val, uint64_t* n);
/* Record, in every later sampler run, the pool values the run reads (off by
 * default; the drop-in's per-epoch calls turn it on). */
int sgdt_set_pool_capture(sgdt_session* s, int on);
/* sgdt_pool_delta plus the values the run read before it wrote:
 * pre_j[i] = pool[pos[i]] and pre_lo[i] = pool[i] as they were before the run
 * (i < m).  A host copy of the pool that agrees with these at every read
 * position is the pool the device ran on, and after pool[pos[i]] = val[i]
 * and pool[i] = batch[i] it is the pool the device holds -- every step an
 * independent per-position check or store (the drop-in does them on host
 * threads).  SGDT_ERR_CONFIG when capture was off for that run. */
int sgdt_pool_delta_pre(sgdt_session* s, uint32_t* pos, uint32_t* val, uint32_t* pre_j, uint32_t* pre_lo,
                        uint64_t* n);
/* The same four arrays without a copy: pointers into session-owned pinned
 * host memory, valid until the next sgdt_pool_delta_view / _pre call. */
int sgdt_pool_delta_view(sgdt_session* s, const uint32_t** pos, const uint32_t** val, const uint32_t** pre_j,
                         const uint32_t** pre_lo, uint64_t* n);
/* `epochs` x (core phase; factor phase) enqueued back to back, one host
 * synchronisation at the end (the timed part of train(), trainer.cpp:94-107).
 * A divergence anywhere returns SGDT_ERR_NUMERIC (trainer.cpp:101-103). */
int sgdt_run_epochs(sgdt_session* s, const sgdt_core_hyper* ch, const sgdt_factor_hyper* fh,
                    uint64_t epochs);

/* The host-model form of sgdt_run_epochs, for callers whose Model lives in
 * host memory (update_core_epoch / update_factor_epoch take a host Model&,
 * core_optimizer.cpp:112, factor_optimizer.cpp:101): loads A_in/B_in (fp64,
 * host), runs `epochs` epochs and writes the final model to A_out/B_out.
 * Same result as set_model + run_epochs + get_model; the copy-out of B^(k)
 * overlaps the last factor phase and that of A^(n) overlaps the factor
 * passes of the modes after n.  A_in/B_in may alias A_out/B_out.  Pinned
 * host buffers give full PCIe rate. */
int sgdt_run_epochs_host(sgdt_session* s, const sgdt_core_hyper* ch, const sgdt_factor_hyper* fh,
                         uint64_t epochs, const double* const* A_in, const double* const* B_in,
                         double* const* A_out, double* const* B_out);

/* rmse_mae (eval.cpp:15-33) over the training (which=0) or test (which=1)
 * entries of the session, fp64 accumulation, fixed summation order. */
int sgdt_eval(sgdt_session* s, int which, double* rmse, double* mae);

/* train() (trainer.cpp:66-125) with the model already set: per epoch core,
 * factor, finiteness check, train/test RMSE+MAE.  metrics: epochs x 6
 * {core_s, factor_s, train_rmse, train_mae, test_rmse, test_mae}, core_s and
 * factor_s measured with CUDA events (RMSE excluded, as in the reference). */
int sgdt_train(sgdt_session* s, const sgdt_core_hyper* ch, const sgdt_factor_hyper* fh,
               uint64_t epochs, double* metrics);

int sgdt_last_timing(sgdt_session* s, sgdt_timing* t);

/* Device bytes held by the session's per-epoch scratch (the analogue of the
 * workspace footprint the reference reports as peak_bytes, trainer.cpp:116-119). */
uint64_t sgdt_workspace_bytes(sgdt_session* s);

/* Number of kernels this session has launched so far (all sgdt_* kernels). */
uint64_t sgdt_launch_count(sgdt_session* s);

/* ---- multi-GPU: sharded factor phase -------------
 *
 * A sharded session holds the full entry-order records (the replicated core
 * phase draws and gathers the same Psi on every rank) but only this rank's
 * slice partition_even(nnz, world)[rank] of every mode-sorted order -- the
 * `improved` strategy's slices (factor_optimizer.cpp:209-210) with ranks in
 * place of workers.  Per mode, a rank finalises the rows inside its slice and
 * exports the <= 2 rows cut by the slice edges; the caller merges the exports
 * of all ranks in rank order (factor_optimizer.cpp:247-270), finishes those
 * rows, then publishes rows [row_lo, row_hi) of A^(n) to every rank and
 * refreshes Q^(n).  paper_2012_03550_b200/distributed.py drives this over
 * torch.distributed (NCCL on GPUs). */
typedef struct {
  int rank, world;
  uint64_t entry_begin, entry_end; /* this rank's slice of the mode-sorted order */
  uint32_t row_lo, row_hi;         /* rows this rank publishes after the mode */
  uint32_t n_export;               /* rows cut by the slice edges (0..2) */
  uint32_t export_rows[2];         /* 0-based row ids */
} sgdt_shard_info;

int sgdt_session_create_shard(const sgdt_tensor_desc* train, const sgdt_tensor_desc* test,
                              const uint32_t* J, uint32_t R, int device, int rank, int world,
                              sgdt_session** out);
int sgdt_get_shard_info(sgdt_session* s, int mode, sgdt_shard_info* out);
/* Factor step of `mode` over this rank's slice; export_g receives n_export x R
 * fp64 partial gradients g = sum (p - x) c of the cut rows. */
int sgdt_factor_mode_local(sgdt_session* s, int mode, const sgdt_factor_hyper* h, double* export_g);
/* Finalise k rows from merged gradients g (k x R fp64): F = B g, SGD step with
 * the full bucket size as the batch count, Q row rewrite. */
int sgdt_factor_mode_finish(sgdt_session* s, int mode, const sgdt_factor_hyper* h, uint32_t k,
                            const uint32_t* rows, const double* g);
/* Copy rows [row_lo, row_hi) of A^(mode) (fp32, J_mode per row) out of
 * (to_device = 0) or into (1) the session; buf is host memory, or device
 * memory when buf_on_device. */
int sgdt_factor_rows(sgdt_session* s, int mode, uint32_t row_lo, uint32_t row_hi, float* buf,
                     int to_device, int buf_on_device);
/* Device address of A^(mode) (fp32, I_mode x J_mode row-major). */
int sgdt_factor_device_ptr(sgdt_session* s, int mode, void** ptr);
/* Q^(mode) = A^(mode) B^(mode) for every row. */
int sgdt_refresh_q(sgdt_session* s, int mode);
/* Copy rows [row_lo, row_hi) of the device's Kruskal rows Q^(mode) = A^(mode)
 * B^(mode) (fp32, R_core per row) to host memory.  Diagnostic: the device
 * counterpart of the reference's core cache (model.cpp:116-122) has no host
 * mirror; the tests compare it with A B formed on the host. */
int sgdt_q_rows(sgdt_session* s, int mode, uint32_t row_lo, uint32_t row_hi, float* buf);
/* Wait for all work of the session (both of its streams). */
int sgdt_synchronize(sgdt_session* s);

/* ---- peer-memory publication of the sharded factor phase ----------------
 * Replaces the host round trip of the boundary merge and the row-block
 * broadcast (factor_optimizer.cpp:247-270 plus the all-gather of A^(n)):
 * after sgdt_set_peers, every row the factor kernels finalise is stored into
 * the local A^(n)/Q^(n) and into every peer's copy (NVLink P2P stores from
 * the finaliser), and the export record of the cut rows is stored into every
 * peer's record slot.  The caller orders the ranks with a barrier after
 * sgdt_factor_mode_p2p and after sgdt_factor_merge_p2p (a stream-ordered
 * collective or a host barrier after sgdt_synchronize). */

/* This session's peer-visible buffers, 2N+2 device pointers: A^(0..N-1),
 * Q^(0..N-1), the export-record slots, the core-phase exchange buffer
 * (sgdt_core_plan). */
int sgdt_peer_buffers(sgdt_session* s, void** ptrs);
/* The same buffers as CUDA IPC handles (2N+2 x 64 bytes), for peers in other
 * processes; sgdt_ipc_open maps one into the calling process. */
int sgdt_peer_ipc_handles(sgdt_session* s, void* handles);
int sgdt_ipc_open(const void* handle, int device, void** ptr);
/* Install every rank's buffers: ptrs is world x (2N+2) pointers valid in this
 * process, rank-major (this rank's own row is ignored). */
int sgdt_set_peers(sgdt_session* s, const void* const* ptrs);
/* ---- sharded core phase (update_core_epoch, core_optimizer.cpp:112-257,
 * with Psi sliced by partition_even(M, world) over the ranks as the
 * reference slices it over workers, scheduler.cpp:34-46, and the per-worker
 * partials merged in rank order, core_optimizer.cpp:225-243) -------------
 * The columns of B^(n) are taken in blocks of T.  Per block every rank
 * reduces, over its Psi slice, V0_r = sum_s c_{s,r} (xhat_s - x_s) a_s and
 * G_{r,r'} = sum_s c_{s,r} c_{s,r'} a_s a_s^T for the block's columns, and
 * stores that vector into slot `rank` of every rank's exchange buffer (P2P
 * stores); the next step sums the slots in rank order and replays the T
 * Gauss-Seidel column steps identically on every rank.  So the only
 * cross-GPU traffic of the core phase is these B^(n)-gradient vectors,
 * N * ceil(R/T) per epoch.  Usage:
 *   steps = sgdt_core_plan(...);
 *   for k < steps: sgdt_core_step(s, k); if k + 1 < steps: barrier over ranks
 * (the barrier: a stream-ordered collective, or sgdt_synchronize + a host
 * barrier).  With world = 1 no barrier is needed; sgdt_core_plan draws Psi
 * (or consumes a pending sgdt_sample_ahead) exactly as sgdt_core_epoch_async.
 * *steps = 0 for lr = 0 (a frozen phase, no RNG).  `block` = 0 picks T from
 * a cost model (SGDT_CORE_T overrides); *T_out receives it. */
int sgdt_core_plan(sgdt_session* s, const sgdt_core_hyper* h, uint32_t block, uint32_t* steps,
                   uint32_t* T_out);
int sgdt_core_step(sgdt_session* s, uint32_t k);

/* Replicated core phase without a host synchronisation (the numeric flag is
 * checked by sgdt_check). */
int sgdt_core_epoch_async(sgdt_session* s, const sgdt_core_hyper* h);
/* Draw the NEXT core phase's Psi now, on the side stream, overlapped with the
 * rest of this epoch (Psi does not depend on the model).  The RNG and pool
 * advance immediately, exactly as the next core phase would advance them;
 * the next sgdt_core_epoch_async (same hyper-parameters) consumes the draw.
 * Until then other RNG consumers are refused and RNG/pool setters discard it. */
int sgdt_sample_ahead(sgdt_session* s, const sgdt_core_hyper* h);
/* Factor pass of `mode` over this rank's slice with peer stores, then this
 * rank's export record {n_export, row0, row1, g0[RP], g1[RP]} into slot
 * `rank` of every rank's record buffer.  Asynchronous. */
int sgdt_factor_mode_p2p(sgdt_session* s, int mode, const sgdt_factor_hyper* h);
/* After every rank's sgdt_factor_mode_p2p: rank-ordered fp64 merge of the
 * records and the owner's finalisation of the cut row it publishes (peer
 * stores included).  Asynchronous. */
int sgdt_factor_merge_p2p(sgdt_session* s, int mode, const sgdt_factor_hyper* h);
/* Peer access between the devices of a group driven by one process
 * (cudaDeviceEnablePeerAccess for every ordered pair of distinct devices;
 * pairs already enabled are fine).  SGDT_ERR_CONFIG when a pair has no P2P. */
int sgdt_enable_peer_access(const int* devices, int n);
/* Stream-ordered barrier over sessions held by one process: each session's
 * stream waits (cudaStreamWaitEvent, across devices) for the work enqueued so
 * far on every other session's stream.  No host synchronisation, and no
 * kernel ever waits on another: the ordering is the streams'.  This is the
 * barrier of the C++ multi-GPU train() (one host thread enqueues every rank
 * in lockstep). */
int sgdt_stream_barrier(sgdt_session* const* sessions, int n);
/* Synchronise and check the numeric flag (SGDT_ERR_NUMERIC on divergence). */
int sgdt_check(sgdt_session* s);

/* train_test_split (sptensor.cpp:217-254) on the device: the Fisher-Yates
 * of the entry ids 0..nnz-1 with Rng(seed) (nnz-1 draws, bit-exact: the
 * sampler's parallel swap-chain resolution), then both halves sorted
 * ascending.  test_ids receives llround(fraction * nnz) ids, train_ids the
 * rest (host buffers).  DomainError for a fraction outside (0,1) or a
 * degenerate split, as the reference. */
int sgdt_split_ids(uint64_t nnz, double test_fraction, uint64_t seed, int device, uint32_t* test_ids,
                   uint32_t* train_ids);

/* Device next_below over an explicit MT state (test hook for the rejection
 * path, rng.hpp:20-25): draws n values with bounds[i] sequentially. */
int sgdt_rng_next_below(const uint64_t* mt312, uint32_t pos, const uint64_t* bounds,
                        uint64_t n, uint64_t* out, uint64_t* mt312_out, uint32_t* pos_out);

/* The BASELINE config 2-5 generator (extending
 * synth.cpp:16-103): nnz distinct positions drawn per mode from a
 * bounded-support Zipf(zipf[n]) (0 = uniform) with a Philox4x32-10 stream,
 * first draw wins, ascending linear position (mode 1 fastest, as
 * synth.cpp:40); values from a planted Kruskal teacher with J = teacher_j,
 * R = teacher_r, entries N(0, sigma^2), sigma = (J R^(1/N))^(-1/4): ratings
 * (round(3 + standardised xhat), clipped to [1, 5]) or xhat + noise N(0, 1).
 * coords (nnz*N, 1-based, entry-major) and values (nnz) are host buffers.
 * ConfigError when the device runs out of memory. */
typedef struct {
  int order;
  const uint32_t* dims;
  const double* zipf;
  uint64_t nnz;
  uint32_t teacher_j;
  uint32_t teacher_r;
  int ratings;
  double noise;
  uint64_t seed;
} sgdt_synth_spec;
int sgdt_synth(const sgdt_synth_spec* spec, int device, uint32_t* coords, double* values);

/* partition_even (scheduler.cpp:34-46): slice w of count over workers. */
void sgdt_partition_even(uint64_t count, uint64_t workers, uint64_t* begins, uint64_t* ends);

#ifdef __cplusplus
}
#endif

#endif /* SGDT_H */
