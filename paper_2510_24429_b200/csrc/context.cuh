// The device-resident LP context (one per cclp_cu_ctx, one per shard):
// device memory, layouts, plans, the iteration's parameters and the setup /
// loop / view operations. Methods are defined in engine.cu (layouts, setup,
// iteration launches) and sharded.cu (shard construction).
#pragma once

#include "host_util.cuh"

namespace cclp_cu {

void gaussian_start(uint64_t seed, long long n, double* v);

struct Context {
  int device = 0;
  cudaStream_t stream = nullptr, side = nullptr;
  int m = 0, n = 0;
  long long nnz = 0;
  // unscaled matrix: CSC (reference layout) and CSR
  int *colptr = nullptr, *rowind = nullptr, *rowptr = nullptr, *colind = nullptr;
  double *val_csc = nullptr, *val_csr = nullptr;
  // scaled matrix values
  double *sval_csc = nullptr, *sval_csr = nullptr;
  double *c = nullptr, *l = nullptr, *u = nullptr, *b = nullptr;
  double *r = nullptr, *s = nullptr;
  bool equality = true;
  // partitions
  int Grow = 0, Gcol = 0, row_grid = 1, col_grid = 1;  // G = 0: pick from the mean row length
  int spmv_grid_r = 1, spmv_grid_c = 1, epi_grid = 1;
  int rpg_r = 1, rpg_c = 1;  // SpMV rows per lane group in flight (tuned)
  struct SidePlan {  // long-row segments of one SpMV side (SpmvPlan)
    int thr = 0x7fffffff, nseg = 0, nlong = 0;
    bool has_long = false;
    int4* seg = nullptr;
    int* lr_first = nullptr;
    double* part = nullptr;
    unsigned* cnt = nullptr;
    std::vector<long long> wrow, wseg;  // host weights while planning
  } plan_rows, plan_cols;
  void plan_side(bool rows_side, int G, SidePlan& sp);
  void plan_side_ptr(const int* dptr, int rows, int G, SidePlan& sp);
  int* plan_starts(bool rows_side, const SidePlan& sp, int grid);
  int* plan_starts_ptr(const int* dptr, int rows, const SidePlan& sp, int grid);
  // ---- column panels of the row SpMV: when the gathered x is larger than
  // the L2 can keep (C5: 400 MB), A is split by columns into panels of
  // kPanelBytes of x, stored panel-major (each panel a CSR over all rows with
  // its rows' entries in column order), and A x = sum over panels in panel
  // order, each panel's gathers L2-resident.
  static constexpr size_t kPanelBytes = size_t(48) << 20;
  struct Panel {
    int* ptr = nullptr;    // [m + 1]
    int* idx = nullptr;    // [nnz_k] global (gather-space) column indices
    int* perm = nullptr;   // [nnz_k] position in CSR(A) (values are gathered per solve)
    double* val = nullptr; // [nnz_k] scaled values
    long long nnz = 0;
    int G = 1;
    SidePlan sp;
    int* start = nullptr;
  };
  std::vector<Panel> panels;
  int panel_grid = 0;
  long long panel_gn = 0;          // shards: the full matrix's column count
  std::vector<int> panel_cb;       // shards: every shard's column bounds
  std::vector<int> panel_G_hint;   // shards: the full matrix's per-panel G
  void build_panels(long long gather_len);
  bool use_panels() const { return !panels.empty() && !exact; }
  PanelArgs panel_args(int k) const;
  SpmvPlan plan(bool rows_side) const;
  int* spmv_row_start = nullptr;  // [spmv_grid_r + 1]
  int* spmv_col_start = nullptr;  // [spmv_grid_c + 1]
  int *row_start = nullptr, *col_start = nullptr;
  bool exact = false;  // G = 1: reference-order (bit-identical) SpMV sums
  // state
  double* xc[3][2] = {};
  double *aty[2] = {}, *xsum[2] = {}, *atysum[2] = {};
  double *y[2] = {}, *ax[3] = {}, *ysum[2] = {}, *axsum[2] = {};
  double *rowp = nullptr, *colp = nullptr, *work_part = nullptr;
  unsigned* counter = nullptr;
  Ctrl* ctrl = nullptr;
  Ctrl* h_ctrl = nullptr;  // pinned, [4]
  LogEntry* log = nullptr;
  int log_cap = 4096;
  LogEntry* h_log = nullptr;
  double* thr = nullptr;
  int thr_cap = 0;
  unsigned long long* t0 = nullptr;
  double* scalars = nullptr;  // device scratch [16]
  double* h_scalars = nullptr;
  PowerCtrl* pctrl = nullptr;
  int* iflags = nullptr;    // [0] ruiz notdone, [1] amb row count, [2] amb col count
  int* amb_idx = nullptr;   // [2][256]
  double* wn = nullptr;     // n-vector scratch x2
  double* wn2 = nullptr;
  double* wm = nullptr;
  // outputs (device views) + pinned staging for snapshots
  double *vx = nullptr, *vy = nullptr, *vz = nullptr, *vrep = nullptr;
  double *h_sx = nullptr, *h_sy = nullptr, *h_sz = nullptr;
  // inline ladder snapshots: kSnapSlots device slots of x | z (n each) | y (m)
  double* snap_buf[kSnapSlots] = {};
  // host flags in pinned, device-mapped memory: [0] cancel request (mirrored
  // from the caller's flag by the host loop, read by the kernels every
  // iteration), [1] snapshots copied out by the host
  unsigned* h_flags = nullptr;
  const unsigned* d_flags = nullptr;
  unsigned* cancel_dev = nullptr;
  unsigned long long* stamps = nullptr;  // in-graph phase stamps (stamp_phase)
  unsigned long long* spec_sync = nullptr;  // speculative row products (IterParams::spec)
  std::atomic<int> abort_req{0};  // cclp_cu_request_cancel (any thread)
  void ensure_flags() {
    if (h_flags) return;
    h_flags = host_alloc<unsigned>(16);
    std::memset(h_flags, 0, 16 * sizeof(unsigned));
    void* dp = nullptr;
    CK(cudaHostGetDevicePointer(&dp, h_flags, 0));
    d_flags = static_cast<const unsigned*>(dp);
  }
  cudaEvent_t ev_snap = nullptr, ev_a = nullptr, ev_b = nullptr;
  // graph
  cudaGraphExec_t graph = nullptr;
  int graph_k = 0;
  IterParams params{};
  bool begun = false;
  long long launches = 0;
  double b_norm = 0, c_norm = 0;
  double norm_est = 0, omega = 0, tau = 0, sigma = 0;
  // host-side phase timings (seconds; stream synchronized at each border):
  // 0 upload, 1 csr build, 2 partition + spmv tuning, 3 norms, 4 ruiz,
  // 5 scale values, 6 power iteration, 7 state init + check(0),
  // 8 graph build, 9 loop, 10 result view + download
  static constexpr int kPhases = 11;
  double phase[kPhases] = {};
  std::chrono::steady_clock::time_point phase_t0;
  template <class T>
  T* alloc(size_t count) {
    void* p = nullptr;
    // +4 elements of slack: the bulk copies of the epilogues move whole
    // 16-byte units and may read one element past a vector's end (bulk_stream)
    ck(cudaMallocAsync(&p, (std::max<size_t>(count, 1) + 4) * sizeof(T), stream), "cudaMallocAsync");
    return static_cast<T*>(p);
  }
  void release(void* p) {
    if (p) cudaFreeAsync(p, stream);
  }
  // pinned host buffers with their sizes (returned to the process cache)
  std::vector<std::pair<void*, size_t>> pinned;
  template <class T>
  T* host_alloc(size_t count) {
    const size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
    void* p = pinned_alloc(bytes);
    pinned.emplace_back(p, bytes);
    return static_cast<T*>(p);
  }
  double* stage[2] = {nullptr, nullptr};
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
  void ensure_stage() {
    for (int b = 0; b < 2; ++b)
      if (!stage[b]) {
        stage[b] = host_alloc<double>(kStageChunk / sizeof(double));
        CK(cudaEventCreateWithFlags(&stage_ev[b], cudaEventDisableTiming));
      }
  }
  void h2d(void* dst, const void* src, size_t bytes) {
    if (bytes == 0) return;
    if (bytes < 2 * kStageChunk || is_pinned(src)) {
      CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, stream));
      return;
    }
    ensure_stage();
    size_t k = 0;
    for (size_t off = 0; off < bytes; off += kStageChunk, ++k) {
      const int b = static_cast<int>(k & 1);
      CK(cudaEventSynchronize(stage_ev[b]));  // the chunk's previous DMA (this or an earlier call)
      const size_t len = std::min(kStageChunk, bytes - off);
      par_memcpy(stage[b], static_cast<const char*>(src) + off, len);
      CK(cudaMemcpyAsync(static_cast<char*>(dst) + off, stage[b], len, cudaMemcpyHostToDevice, stream));
      CK(cudaEventRecord(stage_ev[b], stream));
    }
  }
  void d2h(void* dst, const void* src, size_t bytes) {  // synchronous on return
    if (bytes == 0) return;
    if (bytes < 2 * kStageChunk || is_pinned(dst)) {
      CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, stream));
      CK(cudaStreamSynchronize(stream));
      return;
    }
    ensure_stage();
    const size_t nch = (bytes + kStageChunk - 1) / kStageChunk;
    auto issue = [&](size_t k) {
      const size_t off = k * kStageChunk, len = std::min(kStageChunk, bytes - off);
      CK(cudaMemcpyAsync(stage[k & 1], static_cast<const char*>(src) + off, len, cudaMemcpyDeviceToHost,
                         stream));
      CK(cudaEventRecord(stage_ev[k & 1], stream));
    };
    issue(0);
    for (size_t k = 0; k < nch; ++k) {
      if (k + 1 < nch) issue(k + 1);
      CK(cudaEventSynchronize(stage_ev[k & 1]));
      const size_t off = k * kStageChunk, len = std::min(kStageChunk, bytes - off);
      par_memcpy(static_cast<char*>(dst) + off, stage[k & 1], len);
    }
  }
  void mark(int k) {
    CK(cudaStreamSynchronize(stream));
    const auto now = std::chrono::steady_clock::now();
    phase[k] = std::chrono::duration<double>(now - phase_t0).count();
    phase_t0 = now;
  }

  ~Context();
  void upload(const cclp_cu_lp* lp);
  void build_csr();
  void build_csr_from(const int* cptr, const int* ridx, const double* cval, int ncols, long long cnt);
  void init_aux(int dev);
  void partition();
  void tune_spmv();
  bool rows_equality = false;
  // SELL-32 copy of A' for the column product (k_spmv_cols_sell): structure
  // per long-row threshold, block ranges per column grid, values per solve.
  bool sell_on = false;
  static constexpr double kSellMaxPad = 1.25;
  int sell_thr = -1, sell_grid = 0, sell_nsl = 0, sell_bs = kSpmvBlock;
  long long* sell_off = nullptr;
  int* sell_start = nullptr;
  int* sell_idx = nullptr;
  double* sell_val = nullptr;
  std::vector<long long> sell_cum;  // host: slots before each slice
  void build_sell_cols();
  // SELL-G copy of A for the row product (k_spmv_rows_sellg): the same sums
  // as the CSR-G kernel, so it is chosen by timing (decided once).
  struct SellG {
    bool on = false, decided = false;
    int thr = -1, G = 0, grid = 0, bs = kSpmvBlock, nsl = 0;
    long long* off = nullptr;
    int* start = nullptr;
    int* idx = nullptr;
    double* val = nullptr;
  };
  SellG sgr, sgc;  // rows (k_spmv_rows_sellg), columns (k_spmv_cols_sellg)
  void build_sell_rows();
  void build_sellg(bool rows_side);
  void relative_report(const double* x, const double* y, const double* z, double* rep, double* abs_viol);
  void price(const double* y, const char* status, const unsigned char* skip, int phase1, double dtol, int bland,
             long long* entering, int* direction, double* violation);
  // SpMV geometry tuning folded into the first power iterations (results are
  // geometry-independent, so the candidates can do real work): both start
  // tables stay alive until the choice is made.
  bool tune_pending = false;
  int* tune_rows_st[3] = {nullptr, nullptr, nullptr};
  int* tune_cols_st[3] = {nullptr, nullptr, nullptr};
  int tune_sms = 148;
  int row_sms = 148;  // SMs the row product's grid is planned on (tune_spmv)
  cudaEvent_t tune_ev[96] = {};
  static constexpr int kSellTuneEvents = 64;
  cudaEvent_t sell_ev[kSellTuneEvents] = {};  // SELL-G geometry timing (build_sellg)
  void set_geometry(bool rows_side, int per_sm, int rpg);
  void choose_geometry(const std::vector<float> (&ms)[2][4]);
  void explicit_tune();
  void ensure_tuned() {
    if (tune_pending) explicit_tune();
  }
  int grow() const { return exact ? 1 : Grow; }
  int gcol() const { return exact ? 1 : Gcol; }
  void launch_spmv(bool transpose, const double* vec, double* out, bool scaled, const int* stop);
  double reduce(const double* a, const double* bvec, long long len, int mode);  // reproducible
  void launch_repro_max(int mode, const double* a, const double* bvec, long long len, bool pdl = false);
  void launch_repro_sum(int mode, const double* a, const double* bvec, long long len, const double* Mdev,
                        long long N, PowerCtrl* pc = nullptr, bool pdl = false);
  void repro_local_max(int mode, const double* a, const double* bvec, long long len, double* M);
  void repro_local_sums(int mode, const double* a, const double* bvec, long long len, const double* M,
                        long long N, double* S);
  void ruiz(int iterations);
  void ruiz_init();
  bool ruiz_maxima(const double* s_g, const double* r_g);
  void ruiz_update();
  void power_rows(const double* vg, double* w, bool scaled, bool pdl = false);
  void power_cols(const double* wg, double* u, bool scaled, bool pdl = false);
  // One k_spmv_range launch, programmatic when pdl (engine.cu).
  template <int G, bool LONG>
  void range_launch(bool pdl, int grid, const SpmvPlan& P, const int* ptr, const int* idx, const double* val,
                    const double* vec, double* out, int rpg, int accumulate);
  double power_norm(int iterations, uint64_t seed, bool scaled, bool pregenerated = false);
  double* h_v0 = nullptr;  // pinned start vector of the power iteration
  // h_v0 holds the start vector of seed v0_seed (a pure function of (seed, n)):
  // the default seed's is generated on a host thread during upload / CSR build
  std::thread v0_thread;
  unsigned long long v0_seed = ~0ull;
  // ---- sharded mode (sharded.cuh): this context is shard `shard_rank` of
  // `shard_count`, owning rows [r0, r0 + m) of A and columns [c0, c0 + n)
  bool own_stream = true;
  int shard_rank = 0, shard_count = 1, r0 = 0, c0 = 0, Sm = 0, Sn = 0;
  long long nnz_rows_slice = 0, nnz_cols_slice = 0;  // this shard's part of A (rows) / A' (rows)
  double* x_full = nullptr;  // [P * Sn] padded full x (gather source of the row SpMV)
  double* y_full = nullptr;  // [P * Sm] padded full y (gather source of the column SpMV)
  double* xpart = nullptr;   // [P][kRowParts + kColParts] exchanged report sums
  double* vparts = nullptr;  // [kRowParts + kColParts] report sums of the last view
  unsigned long long* push_flags = nullptr;  // [3][kMaxPushShards] peer epochs (push transport)
  unsigned* push_counter = nullptr;          // [2]
  bool ipc_buffers = false;                  // exchange buffers from cudaMalloc (CUDA IPC)
  std::vector<void*> ipc_owned;
  void setup(const cclp_cu_config& cfg);
  void init_state(const cclp_cu_config& cfg, const cclp_cu_tolerances& tol, const double* thresholds,
                  int nthr, bool launch_init);
  void shard_from_host(const cclp_cu_lp* lp, int rank, int P, const std::vector<int>& rb,
                       const std::vector<int>& cb, cudaStream_t shared, const std::vector<int>& panel_G);
  void begin(const cclp_cu_config& cfg, const cclp_cu_tolerances& tol, const double* thresholds,
             int nthr);
  void launch_iteration(bool init);
  void launch_rows_half(bool init);  // k_spmv_rows + k_dual
  void launch_cols_half(bool init);  // k_spmv_cols + k_primal
  void launch_dual(int ii);
  void launch_primal(int ii);
  static constexpr int kBulkMinRows = 256 * 1024;   // k_dual: bulk-copy ring from this many rows
  static constexpr int kBulkMinCols = 1024 * 1024;  // k_primal: from this many columns
  bool bulk_epilogue(bool rows_side) const;
  void build_graph(int k);
  void profile_kernels(long long iters, double* out);  // cclp_cu_profile_kernels
  void fetch_ctrl(Ctrl* dst);
  void extract_view(int view, const Ctrl& st);
};

}  // namespace cclp_cu
