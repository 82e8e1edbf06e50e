// sgdt_internal.cuh -- device session layout shared by the sgdt_*.cu units.
//
// HBM layout:
//   * entry-order record copy: idx[k*nnz + e] (u32, 0-based) for k < N,
//     val[e] (fp32)  -- Psi gathers of the core phase and train RMSE.
//   * one mode-sorted copy per mode n, the reference's mode_perm(n) order
//     (sptensor.cpp:102-117): idx_n[k*nnz + q], val_n[q]; row_ptr[I_n+1];
//     an nnz-balanced chunk schedule for the factor kernel.
//   * A^(n) fp32 I_n x J (stride J), B^(n) fp32 J x R, Q^(n) = A^(n) B^(n)
//     fp32 I_n x RP (RP = R rounded up to a multiple of 4, zero padded, so a
//     row is float4-gatherable).
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/sgdt.h"

namespace sgdt {

constexpr int kMaxOrder = SGDT_MAX_ORDER;
constexpr uint32_t kNone = 0xFFFFFFFFu;

// Factor-phase work unit: entries [begin, end) of the mode-sorted copy.
// piece < 0: the chunk holds whole rows; otherwise it is piece `piece` of a
// row longer than the chunk size (finalised by the split-row kernel).
// pad = 1: whole rows that are all short -- one row per lane.
// Jump-ahead of the mt19937_64 engine for long draw runs (sgdt_sampler.cu):
// J = T^L (column-major, 19968 x 312 words) and the segment starts.
struct MtJump {
  uint64_t* J = nullptr;
  uint64_t* st = nullptr;
  uint64_t st_cap = 0;
  uint64_t* part = nullptr;
};

// Split rows with more pieces than this are reduced by a whole CTA.
constexpr uint32_t kSplitBig = 64;

struct Chunk {
  uint32_t begin;
  uint32_t end;
  int32_t piece;
  uint32_t pad;
};

// A row split over several chunks: pieces [first, first + count).
// pad = 0: finalised on this device; pad = 1 + slot: the row is cut by this
// rank's slice, its summed pieces go to export slot `slot` instead.
struct SplitRow {
  uint32_t row;
  uint32_t first;
  uint32_t count;
  uint32_t pad;
};

// This rank's share of one mode (single GPU: the whole order).
struct ShardPlan {
  uint64_t qb = 0, qe = 0;        // slice [qb, qe) of the mode-sorted order
  uint32_t row_lo = 0, row_hi = 0;  // rows this rank publishes after the mode
  uint32_t n_export = 0;          // rows cut by the slice edges (<= 2)
  uint32_t export_rows[2] = {0, 0};
};

// Peer-memory publication (sharded factor phase): the other ranks' copies of
// A^(n) and Q^(n), into which every finalised row is also stored, so the
// row all-gather rides on the finaliser's own stores (NVLink P2P).
constexpr int kMaxPeers = 7;
struct PeerTable {
  int n;
  int pad;
  float* A[kMaxPeers];
  float* Q[kMaxPeers];
};

struct RecordCopy {
  uint32_t* idx = nullptr;  // order x nnz
  float* val = nullptr;     // nnz
  uint64_t nnz = 0;
};

// row_fraction < 1: the per-epoch row subsets of one mode (draw scratch,
// subset records and their chunk schedule; rebuilt when the fraction changes).
struct RowSubset {
  double fraction = -1.0;
  uint64_t total = 0;           // draws = kept entries, sum_i keep_i
  uint32_t* sub_off = nullptr;  // I_n + 1 prefix sums of keep (the subset's row_ptr)
  uint32_t *target = nullptr, *pos = nullptr, *link = nullptr, *kprev = nullptr, *lprev = nullptr,
           *out = nullptr;      // per draw
  RecordCopy rec;               // kept records, row-grouped
  struct Chunk* chunks = nullptr;
  uint32_t n_chunks = 0;
  struct SplitRow* splits = nullptr;
  uint32_t n_splits = 0;
  uint32_t n_big_splits = 0;  // splits[0, n_big_splits) have > kSplitBig pieces
  uint32_t n_pieces = 0;
};

struct ModePlan {
  RecordCopy rec;
  uint32_t* row_ptr = nullptr;  // I_n + 1
  Chunk* chunks = nullptr;
  uint32_t n_chunks = 0;
  SplitRow* splits = nullptr;
  uint32_t n_splits = 0;
  uint32_t n_big_splits = 0;  // splits[0, n_big_splits) have > kSplitBig pieces
  uint32_t n_pieces = 0;
  uint64_t rows_nonempty = 0;
  uint64_t rows_empty = 0;
  ShardPlan shard;
  RowSubset subset;
};

struct Params {
  int order;
  uint32_t dims[kMaxOrder];
  uint32_t J[kMaxOrder];
  uint32_t R;
  uint32_t RP;
  float* A[kMaxOrder];
  float* B[kMaxOrder];
  float* Q[kMaxOrder];
};

// One blocked core phase (sgdt_core_blocked.cu): Psi, the rank's slice of
// it, the column-block width and the launch geometry of its steps.
struct CorePlan {
  bool valid = false;
  const uint32_t* batch = nullptr;
  int per_mode = 0;
  uint64_t m = 0, lo = 0, hi = 0;
  int world = 1, rank = 0;  // exchange group: the session's ranks (sharded) or itself
  double lr = 0.0, reg = 0.0;
  uint32_t T = 1, steps = 0, kstride = 0, js4 = 0, st = 0;
  int grid = 0;
  size_t smem = 0;
  uint32_t next = 0;  // next step to launch (sgdt_core_step checks the order)
};

struct Session {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;  // sampler run-ahead (Psi does not depend on the model)
  cudaEvent_t ev_start = nullptr, ev_core = nullptr, ev_samp = nullptr;
  cudaEvent_t ev_bar = nullptr;  // sgdt_stream_barrier
  int order = 0;
  int rank = 0, world = 1;  // sharded factor phase (multi-GPU)
  uint32_t dims[kMaxOrder] = {};
  uint32_t J[kMaxOrder] = {};
  uint32_t R = 0, RP = 0;
  uint32_t chunk_size = 2048;
  uint64_t nnz = 0, nnz_test = 0;

  RecordCopy train_rec, test_rec;
  ModePlan mode[kMaxOrder];
  std::vector<uint64_t> h_row_ptr[kMaxOrder];  // host copy of every mode's bucket offsets
  uint32_t piece_cap = 0;                       // rows of piece_partials

  Params P{};
  double* piece_partials = nullptr;  // max pieces x RP
  double* export_buf = nullptr;      // 2 x RP, boundary-row partials of the last mode run

  // peer publication (sgdt_set_peers): per-mode peer tables on the device,
  // the export-record slots (world x rec_stride fp64, slot = rank) and the
  // peers' record buffers
  PeerTable* d_peers = nullptr;  // kMaxOrder tables
  int npeers = 0;
  uint32_t rec_stride = 0;       // 3 + 2 RP: {n_export, row0, row1, g0[RP], g1[RP]}
  double* xrec = nullptr;
  double* peer_rec[kMaxPeers] = {};
  uint32_t* merge_rows = nullptr;  // 2
  double* merge_g = nullptr;       // 2 x RP

  // sampler state
  uint64_t* mt = nullptr;       // 312 words + position word
  uint64_t* mt_out = nullptr;   // raw engine outputs of the last draw run (mt_gen_kernel)
  uint64_t mt_out_cap = 0;
  uint64_t* mt_tent = nullptr;  // 313: the engine state after the run if nothing was rejected
  int* mt_flag = nullptr;       // set by draw_map_kernel when an output was rejected
  MtJump jump;                  // jump-ahead of long draw runs (sgdt_sampler.cu)
  uint32_t* pool = nullptr;     // nnz, persistent
  bool pool_valid = false;
  unsigned long long* head = nullptr;  // nnz stamped list heads
  uint32_t stamp = 0;
  uint32_t* draw_j = nullptr;   // m
  uint32_t* link = nullptr;     // m
  uint32_t* kprev = nullptr;    // m
  uint32_t* lprev = nullptr;    // m
  uint32_t* dval = nullptr;     // m
  // sgdt_set_pool_capture: the pool values each sampler run reads
  // (pre_j[i] = pool[j_i], pre_lo[i] = pool[i] before the run), 2 x cap
  bool capture_pre = false;
  uint32_t* pool_pre = nullptr;
  uint64_t pool_pre_cap = 0;
  uint32_t* d_delta = nullptr;  // 2 x delta_cap (device): draw targets, final values
  uint32_t* h_delta = nullptr;  // 4 x delta_cap (pinned): sgdt_pool_delta_view
  uint64_t delta_cap = 0;
  uint32_t* batch = nullptr;    // 2 x order x m: double-buffered Psi (one per mode when resampling)
  uint64_t batch_cap = 0;
  uint64_t last_batch_len = 0;
  uint64_t sampler_runs = 0;  // launch_sampler calls (sgdt_pool_delta: exactly one since delta_base)
  uint64_t delta_base = ~0ull;
  uint64_t delta_m = 0;       // m of the last sampler run
  uint32_t* last_batch = nullptr;  // points into batch
  // sgdt_sample_ahead: the next core phase's Psi, drawn on the side stream
  bool ahead_valid = false;
  uint64_t ahead_m = 0;
  int ahead_per_mode = 0;
  int ahead_slot = 0;      // batch slot holding it
  int core_slot = 0;       // batch slot read by the last enqueued core phase

  // core scratch (M samples)
  float* cs_a = nullptr;      // M x Jmax
  float* cs_c = nullptr;      // M x R
  float* cs_xhat = nullptr;   // M
  float* cs_x = nullptr;      // M
  ulonglong2* cs_part = nullptr;  // 2 x Jmax x grid stamped partials + per-CTA new-column words (sgdt_core.cu)
  uint32_t core_stamp = 0;        // last stamp used in cs_part
  uint64_t cs_cap = 0;
  int core_grid = 0, core_block = 0;

  // blocked / sharded core phase (sgdt_core_blocked.cu)
  int core_mode = 0;               // 0: cooperative column kernel, 1: blocked steps (single GPU)
  CorePlan cplan;
  double* core_x = nullptr;        // exchange buffer: 2 slots x world x core_x_stride fp64 (peer-visible)
  uint32_t core_x_stride = 0;
  double* core_peer_x[kMaxPeers + 1] = {};  // every rank's exchange buffer, by rank (sgdt_set_peers)
  double* core_part = nullptr;     // num_sms x core_x_stride: per-CTA vectors
  unsigned* core_ticket = nullptr;
  float *cb_a = nullptr, *cb_c = nullptr, *cb_xh = nullptr, *cb_x = nullptr;  // per-sample state (T < R)
  uint64_t cb_cap = 0;

  // eval
  double* ev_part = nullptr;
  double* ev_out = nullptr;
  double* h_ev_out = nullptr;  // pinned

  int* flag = nullptr;    // device numeric-error flag
  int* h_flag = nullptr;  // pinned mirror

  double* stage = nullptr;  // fp64 staging for model transfer
  uint64_t stage_cap = 0;
  double* xfer = nullptr;  // fp64 staging of the whole model (sgdt_run_epochs_host)
  uint64_t xfer_cap = 0;

  cudaEvent_t ev[4 + kMaxOrder] = {};
  cudaEvent_t ev_copy[kMaxOrder] = {};  // sgdt_factor_epoch_host: A^(n) landed in hx
  double* hx = nullptr;                 // pinned fp64 staging of A (sgdt_factor_epoch_host)
  uint64_t hx_cap = 0;
  std::vector<cudaEvent_t> tev;  // per-epoch phase events of sgdt_run_epochs (timing means)
  sgdt_timing timing{};
  bool timing_valid = false;
  uint64_t launches = 0;  // kernels launched by this session
};

// NVTX ranges around the enqueue of each phase and mode ("sgdt:core",
// "sgdt:factor:mode 2", ...): ncu --nvtx --nvtx-include "sgdt:factor:mode 2/"
// profiles one mode's launches.  Header-only NVTX v3: no-ops unless a tool
// injects itself.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
inline const char* nvtx_mode_name(int n) {
  static const char* names[kMaxOrder] = {"sgdt:factor:mode 0", "sgdt:factor:mode 1", "sgdt:factor:mode 2",
                                         "sgdt:factor:mode 3", "sgdt:factor:mode 4", "sgdt:factor:mode 5",
                                         "sgdt:factor:mode 6", "sgdt:factor:mode 7"};
  return names[n];
}

// error plumbing (sgdt_session.cu)
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

#define SGDT_CUDA(call)                                                              \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess) {                                                         \
      (void)cudaGetLastError(); /* clear a non-sticky error for the next call */     \
      return ::sgdt::fail(SGDT_ERR_INTERNAL, std::string(#call) + ": " +             \
                                                cudaGetErrorString(e_));             \
    }                                                                                \
  } while (0)

// kernels (launchers return cudaError_t)
int launch_sampler(Session& s, uint64_t m, uint32_t* out_batch, cudaStream_t st);
int launch_core(Session& s, const sgdt_core_hyper& h, const uint32_t* batches, uint64_t m,
                int per_mode_batches);
int launch_q_refresh(Session& s, int mode);
uint32_t core_block_width(const Session& s, uint64_t m_local, int grid, double step_us, uint32_t requested);
uint32_t core_block_kstride(const Session& s, uint32_t T);
uint32_t core_block_max_kstride(const Session& s);
int plan_core_geometry(Session& s, CorePlan& pl);
int launch_core_block_step(Session& s, uint32_t k);
int launch_factor_mode(Session& s, int n, const sgdt_factor_hyper& h, bool subset = false);
int launch_row_subsets(Session& s, int n, RowSubset& rs, cudaStream_t st);
int launch_factor_finish(Session& s, int n, const sgdt_factor_hyper& h, uint32_t k, const uint32_t* rows_dev,
                         const double* g_dev);
int launch_eval(Session& s, int which, double* rmse, double* mae);
int launch_cast_model(Session& s, int to_device, int n, double* stage);

}  // namespace sgdt
