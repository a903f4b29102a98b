// The engine's context (context.cuh): the device copy of the LP, CSR(A) built
// next to the reference's CSC, the SELL layouts and column panels, the SpMV
// plans and their tuning, the one-time setup on the device (Ruiz scaling,
// ||A|| power iteration, step sizes), the iteration's kernel launches and
// CUDA graphs, and the view extraction for results and snapshots. The C ABI
// over it is capi.cu (one device) and sharded.cu (row-block shards).
// Reference: run_pdhg, proj/src/pdhg.cpp:230-378.
#include "context.cuh"
#include "iter_kernels.cuh"
#include "setup_kernels.cuh"

namespace cclp_cu {

Context::~Context() {
  if (v0_thread.joinable()) v0_thread.join();
  cudaSetDevice(device);
  if (graph) cudaGraphExecDestroy(graph);
  if (stream) {
    for (void* q : ipc_owned) {  // cudaMalloc'ed (exported over IPC): not pool memory
      if (q == x_full) x_full = nullptr;
      if (q == y_full) y_full = nullptr;
      if (q == xpart) xpart = nullptr;
      if (q == push_flags) push_flags = nullptr;
    }
    void* ptrs[] = {colptr, rowind, rowptr, colind, val_csc, val_csr, sval_csc, sval_csr, c, l, u, b,
                    r, s, row_start, col_start, spmv_row_start, spmv_col_start, rowp, colp, work_part,
                    counter, ctrl, log, thr, t0, scalars, pctrl, iflags, amb_idx, wn, wn2, wm, vx, vy,
                    vz, vrep, plan_rows.seg, plan_rows.lr_first, plan_rows.part, plan_rows.cnt,
                    plan_cols.seg, plan_cols.lr_first, plan_cols.part, plan_cols.cnt, x_full, y_full,
                    xpart, vparts, push_flags, push_counter, sell_off, sell_start, sell_idx, sell_val,
                    sgr.off, sgr.start, sgr.idx, sgr.val, sgc.off, sgc.start, sgc.idx, sgc.val,
                    cancel_dev, stamps, spec_sync, ax[2], snap_buf[0], snap_buf[1]};
    static_assert(kSnapSlots == 2, "release list");
    for (void* p : ptrs) release(p);
    for (int k = 0; k < 3; ++k)
      for (int q = 0; q < 2; ++q) release(xc[k][q]);
    for (int q = 0; q < 2; ++q) {
      double* v[] = {aty[q], xsum[q], atysum[q], y[q], ax[q], ysum[q], axsum[q]};
      for (double* p : v) release(p);
    }
    for (auto& pn : panels) {
      void* pp[] = {pn.ptr, pn.idx, pn.perm, pn.val, pn.start, pn.sp.seg, pn.sp.lr_first, pn.sp.part, pn.sp.cnt};
      for (void* q : pp) release(q);
    }
    for (int k = 1; k < 3; ++k) {  // start tables not already owned as spmv_*_start
      if (tune_rows_st[k] != spmv_row_start) release(tune_rows_st[k]);
      if (tune_cols_st[k] != spmv_col_start) release(tune_cols_st[k]);
    }
    // pinned buffers may still be targets of queued copies
    cudaStreamSynchronize(stream);
    if (side) cudaStreamSynchronize(side);
  }
  for (void* q : ipc_owned) cudaFree(q);
  cudaGetLastError();
  for (auto& pb : pinned) pinned_release(pb.first, pb.second);
  for (auto& e : stage_ev)
    if (e) cudaEventDestroy(e);
  if (ev_snap) cudaEventDestroy(ev_snap);
  for (auto& e : tune_ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : sell_ev)
    if (e) cudaEventDestroy(e);
  if (ev_a) cudaEventDestroy(ev_a);
  if (ev_b) cudaEventDestroy(ev_b);
  if (stream && own_stream) cudaStreamDestroy(stream);
  if (side) cudaStreamDestroy(side);
}

// A context without a matrix: the device's pool, a stream and scratch
// allocation (the sharded coordinator's helper buffers).
void Context::init_aux(int dev) {
  device = dev;
  phase_t0 = std::chrono::steady_clock::now();
  ensure_pool(device);
  CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&ev_snap, cudaEventDisableTiming));
  CK(cudaEventCreate(&ev_a));
  CK(cudaEventCreate(&ev_b));
}

void Context::upload(const cclp_cu_lp* lp) {
  m = lp->m;
  n = lp->n;
  nnz = lp->colptr[n];
  phase_t0 = std::chrono::steady_clock::now();
  ensure_pool(device);
  CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&ev_snap, cudaEventDisableTiming));
  CK(cudaEventCreate(&ev_a));
  CK(cudaEventCreate(&ev_b));
  colptr = alloc<int>(n + 1);
  rowind = alloc<int>(nnz);
  val_csc = alloc<double>(nnz);
  c = alloc<double>(n);
  l = alloc<double>(n);
  u = alloc<double>(n);
  b = alloc<double>(m);
  r = alloc<double>(m);
  s = alloc<double>(n);
  h2d(colptr, lp->colptr, sizeof(int) * (n + 1));
  h2d(rowind, lp->rowind, sizeof(int) * nnz);
  h2d(val_csc, lp->val, sizeof(double) * nnz);
  h2d(c, lp->c, sizeof(double) * n);
  h2d(l, lp->col_lower, sizeof(double) * n);
  h2d(u, lp->col_upper, sizeof(double) * n);
  // equality form: b = row_lower (= row_upper); checked on the host view
  equality = true;
  for (int i = 0; i < m; ++i) {
    const double lo = lp->row_lower[i], hi = lp->row_upper[i];
    if (!(lo == hi && lo > -INFINITY && lo < INFINITY)) {
      equality = false;
      break;
    }
  }
  h2d(b, lp->row_lower, sizeof(double) * m);
  rows_equality = true;  // kkt entry points need the equality form (b = row bounds)
  for (int i = 0; i < m && rows_equality; ++i)
    rows_equality = lp->row_lower[i] == lp->row_upper[i] && std::isfinite(lp->row_lower[i]);
  if (m > 0 && n > 0 && nnz > 0) {  // the default seed's start vector, behind the ingest
    h_v0 = host_alloc<double>(n);
    v0_seed = 0;
    v0_thread = std::thread(gaussian_start, 0ull, static_cast<long long>(n), h_v0);
  }
  mark(0);
  build_csr();
  mark(1);
  partition();
  mark(2);
}

void Context::build_csr() { build_csr_from(colptr, rowind, val_csc, n, nnz); }

// CSR of the m x ncols matrix given by a device CSC (rows local, ascending
// within each column): a stable radix sort of the entries by row, so within
// a row the entries keep CSC order, i.e. ascending column.
void Context::build_csr_from(const int* cptr, const int* ridx, const double* cval, int ncols, long long cnt) {
  rowptr = alloc<int>(m + 1);
  colind = alloc<int>(cnt);
  val_csr = alloc<double>(cnt);
  if (cnt == 0) {
    CK(cudaMemsetAsync(rowptr, 0, sizeof(int) * (m + 1), stream));
    return;
  }
  int* col_of = alloc<int>(cnt);
  int* keys_out = alloc<int>(cnt);
  int* perm_in = alloc<int>(cnt);
  int* perm_out = alloc<int>(cnt);
  k_expand_major<<<blocks_for(ncols), kBlock, 0, stream>>>(cptr, ncols, col_of);
  k_iota<<<blocks_for(cnt), kBlock, 0, stream>>>(perm_in, cnt);
  CKL("expand");
  int bits = 1;
  while ((1LL << bits) < m) ++bits;
  size_t tmp_bytes = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, ridx, keys_out, perm_in, perm_out,
                                     static_cast<int>(cnt), 0, bits, stream));
  void* tmp = alloc<char>(tmp_bytes);
  CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, ridx, keys_out, perm_in, perm_out,
                                     static_cast<int>(cnt), 0, bits, stream));
  k_offsets_from_sorted<<<blocks_for(m + 1), kBlock, 0, stream>>>(keys_out, cnt, m, rowptr);
  k_gather_csr<<<blocks_for(cnt), kBlock, 0, stream>>>(perm_out, cnt, col_of, cval, colind, val_csr);
  CKL("csr");
  CK(cudaStreamSynchronize(stream));
  release(tmp);
  release(col_of);
  release(keys_out);
  release(perm_in);
  release(perm_out);
}

void Context::partition() {
  if (Grow == 0) Grow = pick_group(nnz, m);
  if (Gcol == 0) Gcol = pick_group(nnz, n);
  if (const char* e = dev_knob("CCLP_CU_G_ROWS")) Grow = std::atoi(e);  // A/B experiments only
  if (const char* e = dev_knob("CCLP_CU_G_COLS")) Gcol = std::atoi(e);
  // Setup kernels use nnz-balanced row ranges of `row_grid` / `col_grid`
  // blocks. The iteration's SpMV kernels run one full wave of resident
  // blocks (grid-stride over rows); the epilogues one wave of kTile-thread
  // blocks, so finalize reduces only that many partials.
  int sms = 148;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  epi_grid = sms;  // one epilogue block per SM (its shared-memory tile ring: bulk_stream)
  const long long cap = 148 * 4;
  row_grid = static_cast<int>(std::max<long long>(1, std::min<long long>(cap, (m + 31) / 32 + nnz / 1024)));
  col_grid = static_cast<int>(std::max<long long>(1, std::min<long long>(cap, (n + 31) / 32 + nnz / 1024)));
  row_start = alloc<int>(row_grid + 1);
  col_start = alloc<int>(col_grid + 1);
  k_partition<<<blocks_for(row_grid + 1), kBlock, 0, stream>>>(rowptr, m, row_grid, 8, row_start);
  k_partition<<<blocks_for(col_grid + 1), kBlock, 0, stream>>>(colptr, n, col_grid, 8, col_start);
  CKL("partition");
  rowp = alloc<double>(static_cast<size_t>(std::max(epi_grid, 148 * 8)) * kRowParts);
  colp = alloc<double>(static_cast<size_t>(std::max(epi_grid, 148 * 8)) * kColParts);
  // view kernels reuse rowp/colp with up to 148*4 blocks
  work_part = alloc<double>(148 * 8 * 6);  // up to 148*4 blocks x 6 level sums
  counter = alloc<unsigned>(4);
  CK(cudaMemsetAsync(counter, 0, sizeof(unsigned) * 4, stream));
  scalars = alloc<double>(16);
  h_scalars = host_alloc<double>(16);
  pctrl = alloc<PowerCtrl>(1);
  iflags = alloc<int>(4);
  amb_idx = alloc<int>(512);
  wn = alloc<double>(n);
  wn2 = alloc<double>(n);
  wm = alloc<double>(m);
  t0 = alloc<unsigned long long>(1);
  tune_spmv();
}

// Long-row segmentation of one SpMV side (see SpmvPlan): segments and their
// combine bookkeeping depend on the matrix only; the per-geometry part is the
// weight-balanced split of the row+segment sequence into `grid` blocks.
void Context::plan_side(bool rows_side, int G, SidePlan& sp) {
  plan_side_ptr(rows_side ? rowptr : colptr, rows_side ? m : n, G, sp);
}

void Context::plan_side_ptr(const int* dptr, int rows, int G, SidePlan& sp) {
  // rows past 32 G nonzeros (> 32 strided loads per lane) would leave their
  // lane group straggling behind the block: they go to whole warps instead
  sp.thr = 32 * G;
  int* d_count = alloc<int>(1);
  CK(cudaMemsetAsync(d_count, 0, sizeof(int), stream));
  k_count_long<<<blocks_for(rows), kBlock, 0, stream>>>(dptr, rows, sp.thr, d_count);
  CKL("count long");
  int nlong = 0;
  CK(cudaMemcpyAsync(&nlong, d_count, sizeof(int), cudaMemcpyDeviceToHost, stream));
  CK(cudaStreamSynchronize(stream));
  release(d_count);
  sp.has_long = nlong > 0;
  if (!sp.has_long) return;
  std::vector<int> ptr(static_cast<size_t>(rows) + 1);
  CK(cudaMemcpy(ptr.data(), dptr, sizeof(int) * (rows + 1), cudaMemcpyDeviceToHost));
  std::vector<int4> segs;
  std::vector<int> first;
  sp.wrow.assign(static_cast<size_t>(rows) + 1, 0);
  for (int i = 0; i < rows; ++i) {
    const int b = ptr[i], e = ptr[i + 1];
    long long w = 4;  // per-row overhead
    if (e - b > sp.thr) {
      const int lr = static_cast<int>(first.size());
      first.push_back(static_cast<int>(segs.size()));
      for (int q = b; q < e; q += kSegLen) segs.push_back(make_int4(i, q, std::min(q + kSegLen, e), lr));
    } else {
      w += e - b;
    }
    sp.wrow[i + 1] = sp.wrow[i] + w;
  }
  first.push_back(static_cast<int>(segs.size()));
  sp.wseg.assign(segs.size() + 1, 0);
  for (size_t k = 0; k < segs.size(); ++k) sp.wseg[k + 1] = sp.wseg[k] + (segs[k].z - segs[k].y) + 32;
  sp.nseg = static_cast<int>(segs.size());
  sp.nlong = nlong;
  sp.seg = alloc<int4>(segs.size());
  sp.lr_first = alloc<int>(first.size());
  sp.part = alloc<double>(segs.size());
  sp.cnt = alloc<unsigned>(nlong);
  CK(cudaMemcpyAsync(sp.seg, segs.data(), sizeof(int4) * segs.size(), cudaMemcpyHostToDevice, stream));
  CK(cudaMemcpyAsync(sp.lr_first, first.data(), sizeof(int) * first.size(), cudaMemcpyHostToDevice,
                     stream));
  CK(cudaMemsetAsync(sp.cnt, 0, sizeof(unsigned) * nlong, stream));
  CK(cudaStreamSynchronize(stream));
}

// Block starts [2 * (grid + 1)] for one geometry: rows then segments.
int* Context::plan_starts(bool rows_side, const SidePlan& sp, int grid) {
  return plan_starts_ptr(rows_side ? rowptr : colptr, rows_side ? m : n, sp, grid);
}

int* Context::plan_starts_ptr(const int* dptr, int rows, const SidePlan& sp, int grid) {
  int* st = alloc<int>(2 * (grid + 1));
  if (!sp.has_long) {  // device split by nonzeros + per-row overhead; no segments
    k_partition<<<blocks_for(grid + 1), kBlock, 0, stream>>>(dptr, rows, grid, 4, st);
    CK(cudaMemsetAsync(st + grid + 1, 0, sizeof(int) * (grid + 1), stream));
    CKL("plan partition");
    return st;
  }
  const long long Wr = sp.wrow.back(), W = Wr + sp.wseg.back();
  std::vector<int> h(2 * (grid + 1));
  for (int b = 0; b <= grid; ++b) {
    const long long t = W * b / grid;
    if (t <= Wr) {
      h[b] = static_cast<int>(std::lower_bound(sp.wrow.begin(), sp.wrow.end(), t) - sp.wrow.begin());
      h[grid + 1 + b] = 0;
    } else {
      h[b] = rows;
      h[grid + 1 + b] =
          static_cast<int>(std::lower_bound(sp.wseg.begin(), sp.wseg.end(), t - Wr) - sp.wseg.begin());
    }
    if (h[b] > rows) h[b] = rows;
    if (h[grid + 1 + b] > sp.nseg) h[grid + 1 + b] = sp.nseg;
  }
  h[grid] = rows;
  h[2 * grid + 1] = sp.nseg;
  CK(cudaMemcpy(st, h.data(), sizeof(int) * h.size(), cudaMemcpyHostToDevice));
  return st;
}

SpmvPlan Context::plan(bool rows_side) const {
  const SidePlan& sp = rows_side ? plan_rows : plan_cols;
  SpmvPlan P;
  P.start = rows_side ? spmv_row_start : spmv_col_start;
  P.grid = rows_side ? spmv_grid_r : spmv_grid_c;
  P.seg = sp.seg;
  P.lr_first = sp.lr_first;
  P.part = sp.part;
  P.cnt = sp.cnt;
  P.thr = (exact || !sp.has_long) ? 0x7fffffff : sp.thr;
  return P;
}

void Context::build_panels(long long gather_len) {
  long long pb = static_cast<long long>(kPanelBytes);
  if (const char* e = dev_knob("CCLP_CU_PANEL_BYTES")) pb = std::max(64LL, std::atoll(e));  // tests
  // Panels are defined on the ORIGINAL column space (a shard maps them into
  // its padded gather space), and a shard takes each panel's G from the full
  // matrix, so sharded sums equal the single-device sums bit for bit.
  const long long gn = panel_gn > 0 ? panel_gn : gather_len;
  const long long K = (gn * 8 + pb - 1) / pb;
  if (K < 3 || m == 0 || nnz == 0) return;  // x (nearly) fits the L2: one pass
  const long long W = (gn + K - 1) / K;
  auto to_gather = [&](long long c) -> long long {  // original column -> gather index
    if (panel_cb.empty()) return std::min(c, gather_len);
    const int P = static_cast<int>(panel_cb.size()) - 1;
    if (c >= gn) return static_cast<long long>(P) * Sn;
    int q = static_cast<int>(std::upper_bound(panel_cb.begin(), panel_cb.end(), static_cast<int>(c)) -
                             panel_cb.begin()) - 1;
    q = std::max(0, std::min(q, P - 1));
    return static_cast<long long>(q) * Sn + (c - panel_cb[q]);
  };
  int sms = 148;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  panel_grid = 2 * sms;
  int* cnt = alloc<int>(static_cast<size_t>(m) + 1);
  size_t tmp_bytes = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, cnt, m + 1, stream));
  void* tmp = alloc<char>(tmp_bytes);
  panels.resize(K);
  for (long long k = 0; k < K; ++k) {
    Panel& pn = panels[k];
    const int lo = static_cast<int>(to_gather(std::min(k * W, gn)));
    const int hi = static_cast<int>(to_gather(std::min((k + 1) * W, gn)));
    k_panel_count<<<blocks_for(m + 1), kBlock, 0, stream>>>(rowptr, colind, m, lo, hi, cnt);
    CKL("panel count");
    pn.ptr = alloc<int>(static_cast<size_t>(m) + 1);
    CK(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, pn.ptr, m + 1, stream));
    int total = 0;
    CK(cudaMemcpyAsync(&total, pn.ptr + m, sizeof(int), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    pn.nnz = total;
    pn.idx = alloc<int>(total);
    pn.perm = alloc<int>(total);
    pn.val = alloc<double>(total);
    k_panel_fill<<<blocks_for(m), kBlock, 0, stream>>>(rowptr, colind, m, lo, pn.ptr, pn.idx, pn.perm);
    CKL("panel fill");
    pn.G = k < static_cast<long long>(panel_G_hint.size()) ? panel_G_hint[k] : pick_group(pn.nnz, m);
    if (const char* e = dev_knob("CCLP_CU_PANEL_G")) pn.G = std::atoi(e);  // A/B experiments only
    plan_side_ptr(pn.ptr, m, pn.G, pn.sp);
    pn.start = plan_starts_ptr(pn.ptr, m, pn.sp, panel_grid);
    pn.sp.wrow.clear();
    pn.sp.wrow.shrink_to_fit();
    pn.sp.wseg.clear();
    pn.sp.wseg.shrink_to_fit();
  }
  release(tmp);
  release(cnt);
}

PanelArgs Context::panel_args(int k) const {
  const Panel& pn = panels[k];
  PanelArgs a;
  a.plan.start = pn.start;
  a.plan.grid = panel_grid;
  a.plan.seg = pn.sp.seg;
  a.plan.lr_first = pn.sp.lr_first;
  a.plan.part = pn.sp.part;
  a.plan.cnt = pn.sp.cnt;
  a.plan.thr = pn.sp.has_long ? pn.sp.thr : 0x7fffffff;
  a.ptr = pn.ptr;
  a.idx = pn.idx;
  a.val = pn.val;
  a.accumulate = k > 0 ? 1 : 0;
  return a;
}

// Picks the launch geometry of the two iteration SpMVs (blocks per SM, rows
// per lane group in flight) by timing candidates on this matrix. Each timed
// launch is preceded by the other half-step's SpMV so the L2 holds what it
// holds inside the iteration (C2's matrix alone fits the 126 MB L2; timing a
// kernel back to back would measure an L2-resident matrix). G (lanes per row)
// is fixed by the mean row length and long-row segments by the matrix, so
// every candidate produces bit-identical results.
void Context::tune_spmv() {
  int sms = 148;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  tune_sms = sms;
  CK(cudaMemsetAsync(wn, 0, sizeof(double) * std::max(n, 1), stream));
  CK(cudaMemsetAsync(wm, 0, sizeof(double) * std::max(m, 1), stream));
  plan_side(true, Grow, plan_rows);
  plan_side(false, Gcol, plan_cols);
  tune_rows_st[1] = plan_starts(true, plan_rows, sms);
  tune_rows_st[2] = plan_starts(true, plan_rows, 2 * sms);
  tune_cols_st[1] = plan_starts(false, plan_cols, sms);
  tune_cols_st[2] = plan_starts(false, plan_cols, 2 * sms);
  build_panels(x_full ? static_cast<long long>(shard_count) * Sn : n);
  // The single-device SELL-G row product starts while the last block of
  // k_primal still runs the decision tail on one SM (row_step): its grids
  // are multiples of the other SMs, so no block waits for that SM.
  row_sms = (x_full == nullptr && !use_panels() && sms > 1) ? sms - 1 : sms;
  if (const char* e = dev_knob("CCLP_CU_ROW_SMS")) row_sms = std::atoi(e);  // A/B experiments only
  plan_rows.wrow.clear();
  plan_rows.wrow.shrink_to_fit();
  plan_rows.wseg.clear();
  plan_rows.wseg.shrink_to_fit();
  plan_cols.wrow.clear();
  plan_cols.wrow.shrink_to_fit();
  plan_cols.wseg.clear();
  plan_cols.wseg.shrink_to_fit();
  set_geometry(true, 2, 1);
  set_geometry(false, 2, 1);
  tune_pending = true;
  // A device-wide context (not a shard) without column panels tunes inside
  // its first power iterations (power_norm); everything else now.
  const bool defer = x_full == nullptr && !use_panels() && dev_knob("CCLP_CU_TUNE_EAGER") == nullptr;
  if (!defer) explicit_tune();
}

void Context::set_geometry(bool rows_side, int per_sm, int rpg) {
  if (rows_side) {
    spmv_grid_r = tune_sms * per_sm;
    spmv_row_start = tune_rows_st[per_sm];
    rpg_r = rpg;
  } else {
    spmv_grid_c = tune_sms * per_sm;
    spmv_col_start = tune_cols_st[per_sm];
    rpg_c = rpg;
  }
}

// Candidates c = (blocks per SM, rows per group in flight) = (1 + c/2,
// 1 + c%2), judged in the order (2,1), (2,2), (1,1), (1,2): a later one
// replaces the best only when its median is 3% faster, so near-ties keep two
// blocks per SM and one row per group (the geometry that wins inside the
// iteration on random structure; C2 measured 71 vs 74 us/iteration).
// ms[side][cand] = samples.
void Context::choose_geometry(const std::vector<float> (&ms)[2][4]) {
  for (int side = 0; side < 2; ++side) {
    float best = 1e30f;
    int best_ps = 2, best_rpg = 1;
    for (int c : {2, 3, 0, 1}) {
      std::vector<float> t = ms[side][c];
      if (t.empty()) continue;
      std::sort(t.begin(), t.end());
      const float med = t[t.size() / 2];
      if (med < 0.97f * best) {
        best = med;
        best_ps = 1 + c / 2;
        best_rpg = 1 + c % 2;
      }
    }
    set_geometry(side == 0, best_ps, best_rpg);
  }
  release(tune_rows_st[3 - spmv_grid_r / tune_sms]);
  release(tune_cols_st[3 - spmv_grid_c / tune_sms]);
  tune_rows_st[3 - spmv_grid_r / tune_sms] = nullptr;
  tune_cols_st[3 - spmv_grid_c / tune_sms] = nullptr;
  tune_pending = false;
}

// Stand-alone tuning: each candidate timed between launches of the other
// side's SpMV (the cache state of the iteration), first sample discarded.
void Context::explicit_tune() {
  auto launch_side = [&](bool rows_side, int per_sm, int rpg) {
    set_geometry(rows_side, per_sm, rpg);
    const int grid = rows_side ? spmv_grid_r : spmv_grid_c;
    const SpmvPlan P = plan(rows_side);
    const bool lng = P.thr != 0x7fffffff;
    if (rows_side) {
      with_group_long(grow(), lng, [&](auto g, auto l) {
        k_spmv_range<decltype(g)::value, decltype(l)::value><<<grid, kSpmvBlock, 0, stream>>>(
            P, rowptr, colind, val_csr, GatherPlain{x_full ? x_full : wn}, wm, rpg);
      });
    } else {
      with_group_long(gcol(), lng, [&](auto g, auto l) {
        k_spmv_range<decltype(g)::value, decltype(l)::value><<<grid, kSpmvBlock, 0, stream>>>(
            P, colptr, rowind, val_csc, GatherPlain{y_full ? y_full : wm}, wn, rpg);
      });
    }
    CKL("tune spmv");
  };
  const char* force = dev_knob("CCLP_CU_RPG");
  std::vector<float> ms[2][4];
  const int reps = (nnz > 30'000'000) ? 4 : 6;
  for (int side = 0; side < 2; ++side) {
    const bool rows_side = side == 0;
    for (int c = 0; c < 4; ++c) {
      const int per_sm = 1 + c / 2, rpg = 1 + c % 2;
      if (force && std::atoi(force) != rpg) continue;
      for (int rep = 0; rep < reps; ++rep) {
        launch_side(!rows_side, 2, 1);
        CK(cudaEventRecord(ev_a, stream));
        launch_side(rows_side, per_sm, rpg);
        CK(cudaEventRecord(ev_b, stream));
        CK(cudaEventSynchronize(ev_b));
        float t = 0;
        CK(cudaEventElapsedTime(&t, ev_a, ev_b));
        if (rep > 0) ms[side][c].push_back(t);
      }
    }
  }
  choose_geometry(ms);
}

// SELL-32 layout of A' (SellPlan): per-slice widths ignore the columns the
// long-row segments sum; each block of the column grid gets a contiguous
// slice range of about equal slots + per-column overhead. CCLP_CU_SELL=0
// keeps the G-lane CSR column kernel (A/B).
void Context::build_sell_cols() {
  const char* e = dev_knob("CCLP_CU_SELL");
  sell_on = false;
  if ((e != nullptr && std::atoi(e) == 0) || n == 0 || nnz == 0 || !sval_csc) return;
  // Measured: SELL wins where the gathered y is large (round 1,
  // profiles/r1/history/r1_spmv_experiments.txt: C3 m = 0.4M -12 us, C4
  // m = 5M -40 us per column product) and, since its loop runs at 32
  // registers with two blocks per SM, also where y is cache-resident (round
  // 2, profiles/r2/history/r2_sell_cols_occupancy.txt: C2 m = 0.1M 25.4 ->
  // 22.8 us; round 1's pipelined loop lost 0.5 us there). The padding rule
  // below is the only condition (CCLP_CU_SELL=0 keeps the CSR-G kernel).
  const SpmvPlan P = plan(false);
  const int thr = P.thr;
  const int nsl = (n + 31) / 32;
  if (sell_thr == thr && sell_nsl < 0) return;  // padding too high (decided once)
  if (!sell_off || sell_thr != thr) {
    int* w = alloc<int>(nsl);
    k_sell_width<<<blocks_for(nsl), kBlock, 0, stream>>>(colptr, n, thr, nsl, w);
    CKL("sell width");
    std::vector<int> hw(nsl);
    CK(cudaMemcpyAsync(hw.data(), w, sizeof(int) * nsl, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    release(w);
    sell_cum.assign(static_cast<size_t>(nsl) + 1, 0);
    for (int q = 0; q < nsl; ++q) sell_cum[q + 1] = sell_cum[q] + 32LL * hw[q];
    // Slices pad every column to the slice's longest: worth it only when the
    // column lengths are near-uniform (C2, C3, C4: <= 1.25x the nonzeros;
    // Poisson-like lengths as in C5 pad ~2x and lose). A property of the
    // matrix alone, so the choice (and the summation order) is deterministic.
    if (static_cast<double>(sell_cum[nsl]) > kSellMaxPad * static_cast<double>(nnz)) {
      sell_thr = thr;
      sell_nsl = -1;  // remembered: no SELL for this threshold
      return;
    }
    release(sell_off);
    release(sell_idx);
    release(sell_val);
    sell_off = alloc<long long>(static_cast<size_t>(nsl) + 1);
    CK(cudaMemcpyAsync(sell_off, sell_cum.data(), sizeof(long long) * (nsl + 1), cudaMemcpyHostToDevice, stream));
    sell_idx = alloc<int>(static_cast<size_t>(std::max<long long>(sell_cum[nsl], 1)));
    sell_val = alloc<double>(static_cast<size_t>(std::max<long long>(sell_cum[nsl], 1)));
    sell_thr = thr;
    sell_nsl = nsl;
    sell_grid = 0;
  }
  k_sell_fill<<<blocks_for(static_cast<long long>(nsl) * 32), kBlock, 0, stream>>>(
      colptr, rowind, sval_csc, n, thr, nsl, sell_off, sell_idx, sell_val);
  CKL("sell fill");
  // block slice ranges for `grid` blocks: equal slots + per-column overhead
  auto starts = [&](int grid) {
    auto weight = [&](long long q) { return sell_cum[q] + 16LL * 32 * q; };
    const long long total = weight(nsl);
    std::vector<int> st(static_cast<size_t>(grid) + 1);
    for (int b = 0; b <= grid; ++b) {
      const long long target = total * b / grid;
      int lo = 0, hi = nsl;
      while (lo < hi) {
        const int mid = (lo + hi) / 2;
        if (weight(mid) >= target) hi = mid; else lo = mid + 1;
      }
      st[b] = b == grid ? nsl : lo;
    }
    int* d = alloc<int>(static_cast<size_t>(grid) + 1);
    CK(cudaMemcpyAsync(d, st.data(), sizeof(int) * (grid + 1), cudaMemcpyHostToDevice, stream));
    CK(cudaStreamSynchronize(stream));  // st is a host temporary
    return d;
  };
  if (sell_grid == 0 || (thr != 0x7fffffff && sell_grid != spmv_grid_c)) {
    release(sell_start);
    sell_bs = kSpmvBlock;
    sell_grid = spmv_grid_c;
    sell_start = starts(sell_grid);
    // Without long columns the block shape is free (every shape sums each
    // column in the same order): time 1024-thread blocks on the column grid
    // against 256-thread blocks on four times as many, keep the faster.
    if (thr == 0x7fffffff) {
      int* alt = starts(4 * spmv_grid_c);
      SellPlan S{sell_off, sell_start, colptr, sell_idx, sell_val, n, thr};
      const double* gy = y_full ? y_full : wm;  // shards gather from the padded full y
      auto time_it = [&](int bs) {
        std::vector<float> t;
        for (int rep = 0; rep < 4; ++rep) {
          CK(cudaEventRecord(ev_a, stream));
          if (bs == kSpmvBlock) {
            S.start = sell_start;
            k_sell_range<kSpmvBlock><<<spmv_grid_c, kSpmvBlock, 0, stream>>>(S, GatherPlain{gy}, wn);
          } else {
            S.start = alt;
            k_sell_range<256><<<4 * spmv_grid_c, 256, 0, stream>>>(S, GatherPlain{gy}, wn);
          }
          CK(cudaEventRecord(ev_b, stream));
          CK(cudaEventSynchronize(ev_b));
          float ms = 0;
          CK(cudaEventElapsedTime(&ms, ev_a, ev_b));
          if (rep > 0) t.push_back(ms);
        }
        std::sort(t.begin(), t.end());
        return t[t.size() / 2];
      };
      CKL("sell tune");
      const float t_big = time_it(kSpmvBlock), t_small = time_it(256);
      // and the grid-stride deal (no start table) on 1024-thread blocks
      int* keep_big = sell_start;
      S.start = nullptr;
      float t_gs;
      {
        std::vector<float> t;
        for (int rep = 0; rep < 4; ++rep) {
          CK(cudaEventRecord(ev_a, stream));
          k_sell_range<kSpmvBlock><<<spmv_grid_c, kSpmvBlock, 0, stream>>>(S, GatherPlain{gy}, wn);
          CK(cudaEventRecord(ev_b, stream));
          CK(cudaEventSynchronize(ev_b));
          float ms = 0;
          CK(cudaEventElapsedTime(&ms, ev_a, ev_b));
          if (rep > 0) t.push_back(ms);
        }
        std::sort(t.begin(), t.end());
        t_gs = t[t.size() / 2];
      }
      const char* fm = dev_knob("CCLP_CU_SELL_MODE");  // A/B: contig | small | gs
      int mode = 0;  // 0 contiguous 1024, 1 contiguous 256, 2 grid-stride 1024
      if (fm != nullptr) {
        mode = std::string(fm) == "small" ? 1 : (std::string(fm) == "gs" ? 2 : 0);
      } else {
        float best = t_big;
        if (t_small < 0.97f * best) { mode = 1; best = t_small; }
        if (t_gs < 0.97f * best) mode = 2;
      }
      if (mode == 1) {
        release(keep_big);
        sell_start = alt;
        sell_bs = 256;
        sell_grid = 4 * spmv_grid_c;
      } else if (mode == 2) {
        release(keep_big);
        release(alt);
        sell_start = nullptr;
        sell_bs = kSpmvBlock;
        sell_grid = spmv_grid_c;
      } else {
        release(alt);
      }
    }
  }
  sell_on = true;
}

// SELL-G layout of A (SellPlan with G lanes per row, the row kernel's own G):
// bit-identical to the CSR-G row product, kept only if a timing against it
// (in the tuned geometry) shows it 3% faster. Not with column panels.
// CCLP_CU_SELL_ROWS=0 disables it, =2 forces it (tests: bit-identity).
void Context::build_sell_rows() { build_sellg(true); }

void Context::build_sellg(bool rows_side) {
  SellG& S = rows_side ? sgr : sgc;
  const char* e = dev_knob(rows_side ? "CCLP_CU_SELL_ROWS" : "CCLP_CU_SELLG_COLS");
  const bool force = e != nullptr && std::atoi(e) == 2;
  const int cnt = rows_side ? m : n;
  const int* ptr = rows_side ? rowptr : colptr;
  const int* idx = rows_side ? colind : rowind;
  const double* sval = rows_side ? sval_csr : sval_csc;
  const double* uval = rows_side ? val_csr : val_csc;
  // the column side takes SELL-G only where the SELL-32 layout was not chosen
  // The column side measured slower inside the iteration than its stand-alone
  // timing suggested (C2: 31.4 vs 30.6 us), so it is opt-in there
  // (CCLP_CU_SELLG_COLS=1: timed, =2: forced).
  const bool opted = rows_side || (e != nullptr && std::atoi(e) >= 1);
  if ((e != nullptr && std::atoi(e) == 0) || !opted || cnt == 0 || nnz == 0 || !sval ||
      (rows_side && use_panels()) || (!rows_side && sell_on)) {
    S.on = false;
    return;
  }
  if (S.decided && !S.on) return;
  const SpmvPlan P = plan(rows_side);
  const int thr = P.thr, G = rows_side ? grow() : gcol(), R = 32 / G;
  const int nsl = (cnt + R - 1) / R;
  if (!S.off || S.thr != thr || S.G != G) {
    int* w = alloc<int>(nsl);
    k_sellg_width<<<blocks_for(nsl), kBlock, 0, stream>>>(ptr, cnt, thr, nsl, G, w);
    CKL("sellg width");
    std::vector<int> hw(nsl);
    CK(cudaMemcpyAsync(hw.data(), w, sizeof(int) * nsl, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    release(w);
    std::vector<long long> cum(static_cast<size_t>(nsl) + 1, 0);
    for (int q = 0; q < nsl; ++q) cum[q + 1] = cum[q] + 32LL * hw[q];
    // padded slots beyond 1.25x the nonzeros lose inside the iteration even
    // where a stand-alone timing says otherwise (C4 rows, G = 4: 1.40x,
    // +15 us); the rule depends on the matrix only
    if (!force && static_cast<double>(cum[nsl]) > kSellMaxPad * static_cast<double>(nnz)) {
      S.on = false;
      S.decided = true;
      return;
    }
    release(S.off);
    release(S.idx);
    release(S.val);
    release(S.start);
    S.off = alloc<long long>(static_cast<size_t>(nsl) + 1);
    CK(cudaMemcpyAsync(S.off, cum.data(), sizeof(long long) * (nsl + 1), cudaMemcpyHostToDevice, stream));
    S.idx = alloc<int>(static_cast<size_t>(std::max<long long>(cum[nsl], 1)));
    S.val = alloc<double>(static_cast<size_t>(std::max<long long>(cum[nsl], 1)));
    // block slice ranges for `grid` blocks: equal slots + per-row overhead
    auto starts = [&](int grid) {
      auto weight = [&](long long q) { return cum[q] + 16LL * R * q; };
      const long long total = weight(nsl);
      std::vector<int> st(static_cast<size_t>(grid) + 1);
      for (int b = 0; b <= grid; ++b) {
        const long long target = total * b / grid;
        int lo = 0, hi = nsl;
        while (lo < hi) {
          const int mid = (lo + hi) / 2;
          if (weight(mid) >= target) hi = mid; else lo = mid + 1;
        }
        st[b] = b == grid ? nsl : lo;
      }
      int* d = alloc<int>(static_cast<size_t>(grid) + 1);
      CK(cudaMemcpyAsync(d, st.data(), sizeof(int) * (grid + 1), cudaMemcpyHostToDevice, stream));
      CK(cudaStreamSynchronize(stream));
      return d;
    };
    S.thr = thr;
    S.G = G;
    S.nsl = nsl;
    k_sellg_fill<<<blocks_for(static_cast<long long>(nsl) * 32), kBlock, 0, stream>>>(
        ptr, idx, sval, cnt, thr, nsl, G, S.off, S.idx, S.val);
    CKL("sellg fill");
    // candidates: 1024-thread blocks on the side's grid (the only one with
    // long rows: the segments are planned for it), else also 2 x 1024 and
    // 8 x 256 per SM; against the CSR-G kernel in its tuned geometry, the
    // other side's product run between samples (the iteration's cache state)
    const bool lng = thr != 0x7fffffff;
    const int side_grid = rows_side ? spmv_grid_r : spmv_grid_c;
    const int side_rpg = rows_side ? rpg_r : rpg_c;
    const double* gv = rows_side ? (x_full ? x_full : wn) : (y_full ? y_full : wm);
    double* outv = rows_side ? wm : wn2;
    const SpmvPlan Po = plan(!rows_side);
    auto other_side = [&] {
      if (rows_side) {
        with_group_long(gcol(), Po.thr != 0x7fffffff, [&](auto g, auto l) {
          k_spmv_range<decltype(g)::value, decltype(l)::value><<<spmv_grid_c, kSpmvBlock, 0, stream>>>(
              Po, colptr, rowind, val_csc, GatherPlain{y_full ? y_full : wm}, wn2, rpg_c);
        });
      } else {
        with_group_long(grow(), Po.thr != 0x7fffffff, [&](auto g, auto l) {
          k_spmv_range<decltype(g)::value, decltype(l)::value><<<spmv_grid_r, kSpmvBlock, 0, stream>>>(
              Po, rowptr, colind, val_csr, GatherPlain{x_full ? x_full : wn}, wm, rpg_r);
        });
      }
    };
    struct Cand { int bs, grid; };
    const int side_sms = rows_side && !lng ? row_sms : tune_sms;
    std::vector<Cand> cands{{kSpmvBlock, side_grid / tune_sms * side_sms}};
    if (!lng) {
      if (cands[0].grid != 2 * side_sms) cands.push_back({kSpmvBlock, 2 * side_sms});
      cands.push_back({256, 8 * side_sms});
    }
    std::vector<int*> cand_start(cands.size());
    for (size_t ci = 0; ci < cands.size(); ++ci) cand_start[ci] = starts(cands[ci].grid);
    // variant 0: the CSR-G kernel in its tuned geometry; 1..: SELL-G candidates
    auto launch_variant = [&](size_t v) {
      with_group_long(G, lng, [&](auto g, auto l) {
        constexpr int GG = decltype(g)::value;
        constexpr bool LL = decltype(l)::value;
        if (v == 0) {
          k_spmv_range<GG, LL><<<side_grid, kSpmvBlock, 0, stream>>>(P, ptr, idx, uval, GatherPlain{gv}, outv,
                                                                   side_rpg);
          return;
        }
        const Cand& c = cands[v - 1];
        const SellPlan SP{S.off, cand_start[v - 1], ptr, S.idx, S.val, cnt, thr};
        if (c.bs == 256)
          k_sellg_range<GG, LL, 256><<<c.grid, 256, 0, stream>>>(SP, P, idx, uval, GatherPlain{gv}, outv);
        else
          k_sellg_range<GG, LL, kSpmvBlock><<<c.grid, kSpmvBlock, 0, stream>>>(SP, P, idx, uval, GatherPlain{gv},
                                                                               outv);
      });
    };
    // interleaved rounds (each variant once per round, the other side's
    // product before each sample, as in the iteration), so clock ramps and
    // drift weigh on every variant alike; round 0 is a warm-up; medians
    const size_t V = cands.size() + 1;
    constexpr int kRounds = 8;
    static_assert(2 * kRounds * 4 <= kSellTuneEvents, "event pool");
    for (size_t e = 0; e < 2 * kRounds * V; ++e)
      if (!sell_ev[e]) CK(cudaEventCreate(&sell_ev[e]));
    for (int round = 0; round < kRounds; ++round)
      for (size_t v = 0; v < V; ++v) {
        other_side();
        CK(cudaEventRecord(sell_ev[2 * (round * V + v)], stream));
        launch_variant(v);
        CK(cudaEventRecord(sell_ev[2 * (round * V + v) + 1], stream));
      }
    CK(cudaEventSynchronize(sell_ev[2 * (kRounds * V - 1) + 1]));  // one host wait
    std::vector<std::vector<float>> samples(V);
    for (int round = 1; round < kRounds; ++round)
      for (size_t v = 0; v < V; ++v) {
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, sell_ev[2 * (round * V + v)], sell_ev[2 * (round * V + v) + 1]));
        samples[v].push_back(ms);
      }
    auto median = [](std::vector<float> t) {
      std::sort(t.begin(), t.end());
      return t[t.size() / 2];
    };
    const float t_csr = median(samples[0]);
    // rows: SELL-G unless the timing finds it clearly (10%) slower — inside
    // the iteration it won on every matrix that passes the padding rule, and
    // a tighter margin let sample noise flip C2 back to CSR-G (+1 us)
    float best = force ? 1e30f : (rows_side ? 1.10f : 0.97f) * t_csr;
    int* best_start = nullptr;
    for (size_t ci = 0; ci < cands.size(); ++ci) {
      // 256-thread blocks must win by 5 %: launched after the epilogue with
      // PDL inside the iteration they run ~5 % slower than stand-alone
      // against 1024-thread blocks (C2: 28.0 vs 26.6 us in the graph at equal
      // stand-alone times), while where they win they win by far (C3: 86 vs
      // 106 us)
      const float t = median(samples[ci + 1]) * (cands[ci].bs == 256 ? 1.05f : 1.0f);
      if (t < best) {
        best = t;
        best_start = cand_start[ci];
        S.bs = cands[ci].bs;
        S.grid = cands[ci].grid;
      }
    }
    for (int* st : cand_start)
      if (st != best_start) release(st);
    CKL("sellg tune");
    S.decided = true;
    S.on = best_start != nullptr;
    S.start = best_start;
    if (!S.on) {
      release(S.off);
      release(S.idx);
      release(S.val);
      S.off = nullptr;
      S.idx = nullptr;
      S.val = nullptr;
    }
    return;
  }
  k_sellg_fill<<<blocks_for(static_cast<long long>(nsl) * 32), kBlock, 0, stream>>>(
      ptr, idx, sval, cnt, thr, nsl, G, S.off, S.idx, S.val);
  CKL("sellg fill");
}

// price() (simplex.cpp:266-296) on the device: see k_price.
void Context::price(const double* y_in, const char* status, const unsigned char* skip, int phase1, double dtol,
                    int bland, long long* entering, int* direction, double* violation) {
  if (!rows_equality) throw std::invalid_argument("price: LP must be in equality form");
  const long long total = static_cast<long long>(n) + m;
  const int grid = static_cast<int>(std::max<long long>(1, std::min<long long>(148 * 8, (total + kBlock - 1) / kBlock)));
  char* d_status = alloc<char>(static_cast<size_t>(std::max<long long>(total, 1)));
  unsigned char* d_skip = skip ? alloc<unsigned char>(static_cast<size_t>(std::max<long long>(total, 1))) : nullptr;
  PriceCand* part = alloc<PriceCand>(static_cast<size_t>(grid) + 1);
  h2d(wm, y_in, sizeof(double) * m);
  h2d(d_status, status, static_cast<size_t>(total));
  if (skip) h2d(d_skip, skip, static_cast<size_t>(total));
  k_price<<<grid, kBlock, 0, stream>>>(n, m, colptr, rowind, val_csc, c, wm, d_status, d_skip, phase1, dtol,
                                       bland, part);
  k_price_finish<<<1, 1, 0, stream>>>(part, grid, bland, part + grid);
  CKL("price");
  PriceCand out;
  CK(cudaMemcpyAsync(&out, part + grid, sizeof(out), cudaMemcpyDeviceToHost, stream));
  CK(cudaStreamSynchronize(stream));
  release(d_status);
  release(d_skip);
  release(part);
  *entering = out.j;
  *direction = out.dir;
  *violation = out.viol;
}

// relative_report + absolute_violation (kkt.cpp:106-149) of a host iterate
// on the unscaled equality-form LP; `rep` in cclp_cu_report order.
void Context::relative_report(const double* x, const double* y, const double* z, double* rep,
                              double* abs_viol) {
  if (!rows_equality) throw std::invalid_argument("relative_report: LP must be in equality form");
  if (!vx) {  // the view buffers (extract_view allocates the same set)
    vx = alloc<double>(n);
    vz = alloc<double>(n);
    vy = alloc<double>(m);
    vrep = alloc<double>(kRepN);
  }
  h2d(vx, x, sizeof(double) * n);
  h2d(vy, y, sizeof(double) * m);
  h2d(vz, z, sizeof(double) * n);
  launch_spmv(false, vx, wm, false, nullptr);  // ax = A x, reference order
  launch_spmv(true, vy, wn, false, nullptr);   // aty = A' y
  const int rb = static_cast<int>(std::max<long long>(1, std::min<long long>(148 * 4, (m + kBlock - 1) / kBlock)));
  const int cb = static_cast<int>(std::max<long long>(1, std::min<long long>(148 * 4, (n + kBlock - 1) / kBlock)));
  double* part = alloc<double>(static_cast<size_t>(rb) * kKktRowF + static_cast<size_t>(cb) * kKktColF + 16);
  double* rpart = part;
  double* cpart = part + static_cast<size_t>(rb) * kKktRowF;
  double* fin = cpart + static_cast<size_t>(cb) * kKktColF;
  k_kkt_rows<<<rb, kBlock, 0, stream>>>(m, wm, vy, b, rpart);
  k_kkt_cols<<<cb, kBlock, 0, stream>>>(n, vx, vz, wn, c, l, u, cpart);
  k_kkt_finish<<<1, 32, 0, stream>>>(rpart, m > 0 ? rb : 0, cpart, n > 0 ? cb : 0, fin);
  CKL("kkt");
  double f[kKktRowF + kKktColF];
  CK(cudaMemcpyAsync(f, fin, sizeof(f), cudaMemcpyDeviceToHost, stream));
  CK(cudaStreamSynchronize(stream));
  release(part);
  const double* rw = f;
  const double* cl = f + kKktRowF;
  rep[kRpNorm2] = std::sqrt(rw[0]);
  rep[kRdNorm2] = std::sqrt(cl[0]);
  rep[kRpInf] = std::max(rw[1], cl[2]);
  rep[kRdInf] = cl[1];
  rep[kPobj] = cl[4];
  rep[kDobj] = rw[2] + cl[5];
  rep[kGap] = std::abs(rep[kPobj] - rep[kDobj]);
  rep[kRelP] = rep[kRpNorm2] / (1.0 + std::sqrt(rw[3]));
  rep[kRelD] = rep[kRdNorm2] / (1.0 + std::sqrt(cl[6]));
  rep[kRelGap] = rep[kGap] / (1.0 + std::abs(rep[kPobj]) + std::abs(rep[kDobj]));
  rep[kMaxResid] = std::max({rep[kRelP], rep[kRelD], rep[kRelGap]});
  rep[kCompl] = cl[3];
  if (abs_viol) *abs_viol = std::max({rw[1], cl[2], cl[1], cl[3]});  // absolute_violation (:141-149)
}

void Context::launch_spmv(bool transpose, const double* vec, double* out, bool scaled,
                          const int* stop) {
  // kernel-level matvec (kernels.hpp:27-40): reference-order sums (G = 1)
  if (!transpose) {
    k_spmv<1><<<row_grid, kBlock, 0, stream>>>(rowptr, colind, scaled ? sval_csr : val_csr,
                                               GatherPlain{vec}, row_start, out, stop);
  } else {
    k_spmv<1><<<col_grid, kBlock, 0, stream>>>(colptr, rowind, scaled ? sval_csc : val_csc,
                                               GatherPlain{vec}, col_start, out, stop);
  }
  CKL("spmv");
}

// Reproducible reductions (repro_consts, setup_kernels.cuh): pass 1 the
// per-term maxima into scalars[0..K), pass 2 the exact level sums into
// scalars[2..2 + 3K), both on the stream. `N` is the GLOBAL term count (a
// shard passes the full length), `Mdev` the global maxima on the device.
void Context::launch_repro_max(int mode, const double* a, const double* bvec, long long len, bool pdl) {
  const int grid = blocks_for(std::max(len, 1LL), kBlock, 148 * 4);
  if (pdl && mode == 3) {  // the power iteration's
    launch_pdl(k_repro_max<3>, grid, kBlock, stream, a, bvec, len, work_part, counter + 1, scalars);
    return;
  }
  switch (mode) {
    case 0: k_repro_max<0><<<grid, kBlock, 0, stream>>>(a, bvec, len, work_part, counter + 1, scalars); break;
    case 1: k_repro_max<1><<<grid, kBlock, 0, stream>>>(a, bvec, len, work_part, counter + 1, scalars); break;
    case 2: k_repro_max<2><<<grid, kBlock, 0, stream>>>(a, bvec, len, work_part, counter + 1, scalars); break;
    default: k_repro_max<3><<<grid, kBlock, 0, stream>>>(a, bvec, len, work_part, counter + 1, scalars); break;
  }
  CKL("repro max");
}
void Context::launch_repro_sum(int mode, const double* a, const double* bvec, long long len, const double* Mdev,
                               long long N, PowerCtrl* pc, bool pdl) {
  const int grid = blocks_for(std::max(len, 1LL), kBlock, 148 * 4);
  double* out = scalars + 2;
  if (pdl && mode == 3) {
    launch_pdl(k_repro_sum<3>, grid, kBlock, stream, a, bvec, len, Mdev, N, work_part, counter + 1, out, pc);
    return;
  }
  switch (mode) {
    case 0: k_repro_sum<0><<<grid, kBlock, 0, stream>>>(a, bvec, len, Mdev, N, work_part, counter + 1, out); break;
    case 1: k_repro_sum<1><<<grid, kBlock, 0, stream>>>(a, bvec, len, Mdev, N, work_part, counter + 1, out); break;
    case 2: k_repro_sum<2><<<grid, kBlock, 0, stream>>>(a, bvec, len, Mdev, N, work_part, counter + 1, out); break;
    default:
      k_repro_sum<3><<<grid, kBlock, 0, stream>>>(a, bvec, len, Mdev, N, work_part, counter + 1, out, pc);
      break;
  }
  CKL("repro sum");
}
// Host-synced halves for the sharded setup: the local maxima, then (given
// the global maxima) the local exact level sums.
void Context::repro_local_max(int mode, const double* a, const double* bvec, long long len, double* M) {
  const int K = mode == 3 ? 2 : 1;
  launch_repro_max(mode, a, bvec, len);
  CK(cudaMemcpyAsync(h_scalars, scalars, sizeof(double) * K, cudaMemcpyDeviceToHost, stream));
  CK(cudaStreamSynchronize(stream));
  for (int k = 0; k < K; ++k) M[k] = h_scalars[k];
}
void Context::repro_local_sums(int mode, const double* a, const double* bvec, long long len, const double* M,
                               long long N, double* S) {
  const int K = mode == 3 ? 2 : 1;
  std::memcpy(h_scalars + 8, M, sizeof(double) * K);
  CK(cudaMemcpyAsync(scalars + 8, h_scalars + 8, sizeof(double) * K, cudaMemcpyHostToDevice, stream));
  launch_repro_sum(mode, a, bvec, len, scalars + 8, N);
  CK(cudaMemcpyAsync(h_scalars, scalars + 2, sizeof(double) * 3 * K, cudaMemcpyDeviceToHost, stream));
  CK(cudaStreamSynchronize(stream));
  for (int k = 0; k < 3 * K; ++k) S[k] = h_scalars[k];
}
double Context::reduce(const double* a, const double* bvec, long long len, int mode) {
  launch_repro_max(mode, a, bvec, len);
  launch_repro_sum(mode, a, bvec, len, scalars, len);
  CK(cudaMemcpyAsync(h_scalars, scalars + 2, sizeof(double) * 3, cudaMemcpyDeviceToHost, stream));
  CK(cudaStreamSynchronize(stream));
  return repro_final(h_scalars);
}

// Ruiz factors into r, s (scaling.cpp:46-90); ambiguous pow2_sqrt cases are
// evaluated with the host libm exactly as the reference does.
void Context::ruiz_init() {
  k_fill<<<blocks_for(m), kBlock, 0, stream>>>(r, m, 1.0);
  k_fill<<<blocks_for(n), kBlock, 0, stream>>>(s, n, 1.0);
  CKL("ruiz init");
}

// One pass's row / column maxima of |a_ij| r_i s_j (exact, order-free) into
// wm / wn; s_g and r_g are the gathered scales (this context's own r, s, or a
// shard's padded full copies). Returns whether any factor is outside [1/2, 2).
bool Context::ruiz_maxima(const double* s_g, const double* r_g) {
  double* rmax = wm;
  double* cmax = wn;
  auto absmax = [&](int G, int grid, const int* ptr, const int* idx, const double* val, const double* self,
                    const double* other, int is_row, const int* start, double* out) {
    with_group(G, [&](auto g) {
      k_scaled_absmax<decltype(g)::value><<<grid, kBlock, 0, stream>>>(ptr, idx, val, self, other, is_row,
                                                                        start, out);
    });
  };
  absmax(Grow, row_grid, rowptr, colind, val_csr, r, s_g, 1, row_start, rmax);
  absmax(Gcol, col_grid, colptr, rowind, val_csc, s, r_g, 0, col_start, cmax);
  CK(cudaMemsetAsync(iflags, 0, sizeof(int) * 4, stream));
  k_ruiz_notdone<<<blocks_for(m), kBlock, 0, stream>>>(rmax, m, iflags);
  k_ruiz_notdone<<<blocks_for(n), kBlock, 0, stream>>>(cmax, n, iflags);
  CKL("ruiz max");
  int hf[4];
  CK(cudaMemcpyAsync(hf, iflags, sizeof(hf), cudaMemcpyDeviceToHost, stream));
  CK(cudaStreamSynchronize(stream));
  return hf[0] != 0;
}

// r_i /= pow2_sqrt(rowmax_i), s_j /= pow2_sqrt(colmax_j) (scaling.cpp:23-25,
// :75-86); ambiguous pow2_sqrt cases are evaluated with the host libm
// exactly as the reference does.
void Context::ruiz_update() {
  double* rmax = wm;
  double* cmax = wn;
  k_ruiz_update<<<blocks_for(m), kBlock, 0, stream>>>(rmax, m, r, iflags + 1, amb_idx, 256);
  k_ruiz_update<<<blocks_for(n), kBlock, 0, stream>>>(cmax, n, s, iflags + 2, amb_idx + 256, 256);
  CKL("ruiz update");
  int hf[4];
  CK(cudaMemcpyAsync(hf, iflags, sizeof(hf), cudaMemcpyDeviceToHost, stream));
  CK(cudaStreamSynchronize(stream));
  for (int side_k = 0; side_k < 2; ++side_k) {
    const int cnt = hf[1 + side_k];
    if (cnt == 0) continue;
    if (cnt > 256) throw Error(CCLP_CU_ECUDA, "ruiz: too many ambiguous pow2_sqrt cases");
    std::vector<int> idx(cnt);
    CK(cudaMemcpy(idx.data(), amb_idx + 256 * side_k, sizeof(int) * cnt, cudaMemcpyDeviceToHost));
    double* mx = side_k == 0 ? rmax : cmax;
    double* sc = side_k == 0 ? r : s;
    for (int q = 0; q < cnt; ++q) {
      double v, cur;
      CK(cudaMemcpy(&v, mx + idx[q], sizeof(double), cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(&cur, sc + idx[q], sizeof(double), cudaMemcpyDeviceToHost));
      cur /= std::exp2(std::round(0.5 * std::log2(v)));  // pow2_sqrt, scaling.cpp:23-25
      CK(cudaMemcpy(sc + idx[q], &cur, sizeof(double), cudaMemcpyHostToDevice));
    }
  }
}

// Ruiz factors into r, s (scaling.cpp:46-90).
void Context::ruiz(int iterations) {
  ruiz_init();
  for (int t = 0; t < iterations; ++t) {
    if (!ruiz_maxima(s, r)) break;
    ruiz_update();
  }
}

// The power iteration's start vector, v_j = normal_distribution(mt19937_64(
// seed + 0x9e3779b97f4a7c15)) (pdhg.cpp:49-52), bit-identical to libstdc++ but
// parallel. libstdc++'s polar method draws attempts of exactly two engine
// outputs (generate_canonical<double, 53> on a 64-bit engine is u * 2^-64,
// clamped below 1), accepts those with 0 < r2 <= 1, and returns y*mult then
// x*mult per accepted attempt (mult = sqrt(-2 log(r2) / r2), then
// `* stddev + mean` = `* 1.0 + 0.0`). Attempt boundaries are therefore fixed
// in the raw engine stream: only the engine itself is serial. The calling
// thread generates raw chunks while a team of host threads decides the
// previous chunk's attempts, prefix-sums the accepted ones and writes their
// entries (checked against the oracle's sequential restatement in tests).
void gaussian_start(uint64_t seed, long long n, double* v) {
  if (n <= 0) return;
  std::mt19937_64 rng(seed + 0x9e3779b97f4a7c15ull);
  const long long pairs = (n + 1) / 2;  // the last one half-used when n is odd
  constexpr long long kAttempts = 1 << 19;  // per chunk
  // raw engine outputs, two chunks (uninitialized: filled before use)
  std::unique_ptr<uint64_t[]> buf[2];
  long long buf_cap[2] = {0, 0};
  const int T = static_cast<int>(std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
  auto canon = [](uint64_t u) {
    const double r = static_cast<double>(u) * 0x1p-64;
    return r >= 1.0 ? std::nextafter(1.0, 0.0) : r;
  };
  auto attempt = [&](const uint64_t* d, long long a, double& x, double& y, double& r2) {
    x = 2.0 * canon(d[2 * a]) - 1.0;
    y = 2.0 * canon(d[2 * a + 1]) - 1.0;
    r2 = x * x + y * y;
    return !(r2 > 1.0 || r2 == 0.0);
  };
  // decides chunk d's attempts and writes its accepted pairs from pair `base`
  auto process = [&](const uint64_t* d, long long na, long long base) -> long long {
    std::vector<long long> cnt(T + 1, 0);
    const long long per = (na + T - 1) / T;
    auto run = [&](auto&& body) {
      std::vector<std::thread> th;
      for (int t = 1; t < T; ++t) th.emplace_back(body, t);
      body(0);
      for (auto& x : th) x.join();
    };
    run([&](int t) {
      long long c = 0;
      double x, y, r2;
      for (long long a = t * per; a < std::min(na, (t + 1) * per); ++a) c += attempt(d, a, x, y, r2);
      cnt[t + 1] = c;
    });
    for (int t = 0; t < T; ++t) cnt[t + 1] += cnt[t];
    run([&](int t) {
      long long k = base + cnt[t];
      double x, y, r2;
      for (long long a = t * per; a < std::min(na, (t + 1) * per) && k < pairs; ++a) {
        if (!attempt(d, a, x, y, r2)) continue;
        const double mult = std::sqrt(-2 * std::log(r2) / r2);
        v[2 * k] = y * mult * 1.0 + 0.0;
        if (2 * k + 1 < n) v[2 * k + 1] = x * mult * 1.0 + 0.0;
        ++k;
      }
    });
    return cnt[T];
  };
  // Attempts to draw for `r` more pairs: the expected count (acceptance pi/4)
  // plus six standard deviations, capped at one chunk. Drawing more than
  // needed only discards engine outputs; drawing fewer costs another chunk.
  auto want = [&](long long r) {
    const double p = 0.78539816339744831;
    const double a = r / p + 6.0 * std::sqrt(r * (1.0 - p)) / p + 64.0;
    return std::min<long long>(kAttempts, static_cast<long long>(a));
  };
  auto fill = [&](int b, long long na) {
    if (buf_cap[b] < na) {
      buf[b].reset(new uint64_t[2 * na]);
      buf_cap[b] = na;
    }
    uint64_t* d = buf[b].get();
    for (long long i = 0; i < 2 * na; ++i) d[i] = rng();
  };
  long long done = 0;
  int cur = 0;
  long long na = want(pairs);
  fill(cur, na);
  while (true) {
    long long got = 0;
    std::thread worker([&, cur, na] { got = process(buf[cur].get(), na, done); });
    // the next chunk is drawn while this one is decided, only when this one
    // cannot be expected to finish the vector
    long long na_next = 0;
    if (na == kAttempts && done + static_cast<long long>(0.78 * na) < pairs) {
      na_next = want(pairs - done - static_cast<long long>(0.78 * na));
      fill(cur ^ 1, na_next);
    }
    worker.join();
    done += got;
    if (done >= pairs) break;
    cur ^= 1;
    if (na_next == 0) {  // short (rare): draw the remainder now
      na_next = want(pairs - done);
      fill(cur, na_next);
    }
    na = na_next;
  }
}

// estimate_matrix_norm (pdhg.cpp:46-65) on the scaled or unscaled matrix.
// Per iteration: w = A v and u = A' w with the iteration's tuned SpMV
// geometry (G lanes per row), nu = ||u|| and lambda = v.u in one reduction,
// then v = u / nu materialized (the reference's `v = u / norm`, :62).
double Context::power_norm(int iterations, uint64_t seed, bool scaled, bool pregenerated) {
  if (m == 0 || n == 0 || nnz == 0) {
    ensure_tuned();
    return 0.0;
  }
  // start vector: mt19937_64 + normal_distribution, as the reference (:49-52)
  if (!h_v0) h_v0 = host_alloc<double>(n);
  if (!pregenerated) {
    if (v0_thread.joinable()) v0_thread.join();
    if (v0_seed != seed) gaussian_start(seed, n, h_v0);
    v0_seed = seed;
  }
  const double* v0 = h_v0;
  double* v = wn;
  double* u = wn2;
  CK(cudaMemcpyAsync(v, v0, sizeof(double) * n, cudaMemcpyHostToDevice, stream));
  double nv = reduce(v, nullptr, n, 0);
  if (std::sqrt(nv) == 0.0) {
    k_fill<<<blocks_for(n), kBlock, 0, stream>>>(v, n, 1.0);
    nv = reduce(v, nullptr, n, 0);
  }
  PowerCtrl pc{std::sqrt(nv), 0.0, 0, 0};
  CK(cudaMemcpyAsync(pctrl, &pc, sizeof(pc), cudaMemcpyHostToDevice, stream));
  k_div_scalar<<<blocks_for(n), kBlock, 0, stream>>>(v, &pctrl->nu, v, n);  // v /= v.norm()
  // Deferred geometry tuning: the first K iterations cycle through the four
  // candidates (one warm-up round, then `reps` timed rounds) with events
  // around each product; one host sync after them picks the geometry.
  const bool rows_panels = scaled && use_panels();
  const int reps = (nnz > 30'000'000) ? 4 : 7;
  int K = 0;
  if (tune_pending && !rows_panels && iterations >= 4 * (reps + 1) && 4 * (reps + 1) * 3 <= 96) {
    K = 4 * (reps + 1);
    for (int e = 0; e < 3 * K; ++e)
      if (!tune_ev[e]) CK(cudaEventCreate(&tune_ev[e]));
  } else {
    ensure_tuned();
  }
  const char* force = dev_knob("CCLP_CU_RPG");
  for (int t = 0; t < iterations; ++t) {
    const int cand = t % 4;
    if (t < K) {
      set_geometry(true, 1 + cand / 2, 1 + cand % 2);
      set_geometry(false, 1 + cand / 2, 1 + cand % 2);
      CK(cudaEventRecord(tune_ev[3 * t], stream));
    } else if (t == K && K > 0) {
      CK(cudaEventSynchronize(tune_ev[3 * K - 1]));
      std::vector<float> ms[2][4];
      for (int q = 4; q < K; ++q) {  // round 0 is the warm-up
        const int c = q % 4;
        if (force && std::atoi(force) != 1 + c % 2) continue;
        float a = 0, b = 0;
        CK(cudaEventElapsedTime(&a, tune_ev[3 * q], tune_ev[3 * q + 1]));
        CK(cudaEventElapsedTime(&b, tune_ev[3 * q + 1], tune_ev[3 * q + 2]));
        ms[0][c].push_back(a);
        ms[1][c].push_back(b);
      }
      choose_geometry(ms);
    }
    // Past the timed tuning rounds the five launches are programmatic (PDL):
    // each kernel's launch overlaps its predecessor's tail and waits for it
    // (griddepcontrol.wait) before reading anything.
    const bool pdl = t >= K;
    power_rows(v, wm, scaled, pdl);  // w = A v (:57)
    if (t < K) CK(cudaEventRecord(tune_ev[3 * t + 1], stream));
    power_cols(wm, u, scaled, pdl);  // u = A' w (:58)
    if (t < K) CK(cudaEventRecord(tune_ev[3 * t + 2], stream));
    // nu = ||u||, lambda = v.u with the partition-free sums (sharded setups
    // reproduce them bit for bit)
    launch_repro_max(3, u, v, n, pdl);
    launch_repro_sum(3, u, v, n, scalars, n, pctrl, pdl);  // its last block finishes nu, lambda
    if (pdl)  // v = u / norm
      launch_pdl(k_div_scalar, blocks_for(n), kBlock, stream, static_cast<const double*>(u),
                 static_cast<const double*>(&pctrl->nu), v, static_cast<long long>(n));
    else
      k_div_scalar<<<blocks_for(n), kBlock, 0, stream>>>(u, &pctrl->nu, v, n);
    CKL("power");
  }
  if (tune_pending) ensure_tuned();  // fewer iterations than the tuning rounds
  CK(cudaMemcpyAsync(&pc, pctrl, sizeof(pc), cudaMemcpyDeviceToHost, stream));
  CK(cudaStreamSynchronize(stream));
  if (pc.zero) return 0.0;
  return std::sqrt(std::max(pc.lambda, 0.0));
}

// The power iteration's products on the tuned SpMV plans (sharded: the
// gathered vector is the padded full one).
template <int G, bool LONG>
void Context::range_launch(bool pdl, int grid, const SpmvPlan& P, const int* ptr, const int* idx, const double* val,
                           const double* vec, double* out, int rpg, int accumulate) {
  if (pdl)
    launch_pdl(k_spmv_range<G, LONG, GatherPlain>, grid, kSpmvBlock, stream, P, ptr, idx, val, GatherPlain{vec}, out,
               rpg, accumulate);
  else
    k_spmv_range<G, LONG><<<grid, kSpmvBlock, 0, stream>>>(P, ptr, idx, val, GatherPlain{vec}, out, rpg, accumulate);
}

void Context::power_rows(const double* vg, double* w, bool scaled, bool pdl) {
  const double* aval = scaled ? sval_csr : val_csr;
  if (scaled && use_panels()) {  // panel by panel
    for (int k = 0; k < static_cast<int>(panels.size()); ++k) {
      const PanelArgs a = panel_args(k);
      with_group_long(panels[k].G, a.plan.thr != 0x7fffffff, [&](auto g, auto l) {
        range_launch<decltype(g)::value, decltype(l)::value>(pdl, panel_grid, a.plan, a.ptr, a.idx, a.val, vg, w, 1,
                                                             a.accumulate);
      });
    }
  } else {
    const SpmvPlan Pr = plan(true);
    with_group_long(grow(), Pr.thr != 0x7fffffff, [&](auto g, auto l) {
      range_launch<decltype(g)::value, decltype(l)::value>(pdl, spmv_grid_r, Pr, rowptr, colind, aval, vg, w, rpg_r,
                                                           0);
    });
  }
}
void Context::power_cols(const double* wg, double* u, bool scaled, bool pdl) {
  const double* atval = scaled ? sval_csc : val_csc;
  const SpmvPlan Pc = plan(false);
  with_group_long(gcol(), Pc.thr != 0x7fffffff, [&](auto g, auto l) {
    range_launch<decltype(g)::value, decltype(l)::value>(pdl, spmv_grid_c, Pc, colptr, rowind, atval, wg, u, rpg_c, 0);
  });
}

void Context::launch_rows_half(bool init) {
  const IterParams& p = params;
  const int ii = init ? 1 : 0;
  if (use_panels()) {
    for (int k = 0; k < static_cast<int>(panels.size()); ++k) {
      const PanelArgs a = panel_args(k);
      with_group_long(panels[k].G, a.plan.thr != 0x7fffffff, [&](auto g, auto l) {
        launch_pdl(k_spmv_rows_panel<decltype(g)::value, decltype(l)::value>, panel_grid, kSpmvBlock, stream,
                   p, ii, a);
      });
    }
    launches += static_cast<long long>(panels.size()) - 1;
  } else if (p.use_sell_r) {
    with_group_long(grow(), p.plan_r.thr != 0x7fffffff, [&](auto g, auto l) {
      if (sgr.bs == 256)
        launch_pdl(k_spmv_rows_sellg<decltype(g)::value, decltype(l)::value, 256>, sgr.grid, 256, stream, p,
                   ii);
      else
        launch_pdl(k_spmv_rows_sellg<decltype(g)::value, decltype(l)::value, kSpmvBlock>, sgr.grid,
                   kSpmvBlock, stream, p, ii);
    });
  } else {
    with_group_long(grow(), p.plan_r.thr != 0x7fffffff, [&](auto g, auto l) {
      launch_pdl(k_spmv_rows<decltype(g)::value, decltype(l)::value>, spmv_grid_r, kSpmvBlock, stream, p,
                 ii);
    });
  }
  launch_dual(ii);
}

void Context::launch_cols_half(bool init) {
  const IterParams& p = params;
  const int ii = init ? 1 : 0;
  if (p.use_sell_cg) {
    with_group_long(gcol(), p.plan_c.thr != 0x7fffffff, [&](auto g, auto l) {
      if (sgc.bs == 256)
        launch_pdl(k_spmv_cols_sellg<decltype(g)::value, decltype(l)::value, 256>, sgc.grid, 256, stream, p, ii);
      else
        launch_pdl(k_spmv_cols_sellg<decltype(g)::value, decltype(l)::value, kSpmvBlock>, sgc.grid, kSpmvBlock,
                   stream, p, ii);
    });
  } else if (p.use_sell_c) {
    if (p.plan_c.thr != 0x7fffffff)
      launch_pdl(k_spmv_cols_sell<true, kSpmvBlock>, spmv_grid_c, kSpmvBlock, stream, p, ii);
    else if (sell_bs == 256)
      launch_pdl(k_spmv_cols_sell<false, 256>, sell_grid, 256, stream, p, ii);
    else
      launch_pdl(k_spmv_cols_sell<false, kSpmvBlock>, sell_grid, kSpmvBlock, stream, p, ii);
  } else {
    with_group_long(gcol(), p.plan_c.thr != 0x7fffffff, [&](auto g, auto l) {
      launch_pdl(k_spmv_cols<decltype(g)::value, decltype(l)::value>, spmv_grid_c, kSpmvBlock, stream, p, ii);
    });
  }
  launch_primal(ii);
}

// The streaming epilogues: one block per SM, the operand streams through the
// shared-memory ring of bulk copies (bulk_stream, iter_kernels.cuh) on long
// vectors, loaded by the threads on short ones (reg_stream: the same elements
// in the same order, so the results do not depend on the choice). Measured
// crossovers (profiles/r2/history/r2_epilogue_bulk_vs_reg.txt): k_dual's 7
// streams at 100k rows (C2) 3.8 vs 4.3 us, at 400k (C3) 8.9 vs 7.8 us;
// k_primal's 8 at 500k columns (C2) 14.8 vs 15.9 us, at 2.2M (C3) 45.9 vs
// 40.8 us.
bool Context::bulk_epilogue(bool rows_side) const {
  if (const char* e = dev_knob("CCLP_CU_EPI")) {  // tests: reg | bulk
    if (std::string(e) == "reg") return false;
    if (std::string(e) == "bulk") return true;
  }
  return rows_side ? m >= kBulkMinRows : n >= kBulkMinCols;
}
void Context::launch_dual(int ii) {
  if (bulk_epilogue(true)) {
    allow_smem(reinterpret_cast<const void*>(k_dual<true>), bulk_smem<kDualStreams>());
    launch_pdl_smem(k_dual<true>, epi_grid, kTile, bulk_smem<kDualStreams>(), stream, params, ii);
  } else {
    launch_pdl(k_dual<false>, epi_grid, kTile, stream, params, ii);
  }
}
void Context::launch_primal(int ii) {
  if (bulk_epilogue(false)) {
    allow_smem(reinterpret_cast<const void*>(k_primal<true>), bulk_smem<kPrimalStreams>());
    launch_pdl_smem(k_primal<true>, epi_grid, kTile, bulk_smem<kPrimalStreams>(), stream, params, ii);
  } else {
    launch_pdl(k_primal<false>, epi_grid, kTile, stream, params, ii);
  }
}

void Context::launch_iteration(bool init) {
  launch_rows_half(init);
  launch_cols_half(init);
  launches += kKernelsPerIteration;
}

void Context::build_graph(int k) {
  if (graph && graph_k == k) return;
  if (graph) {
    cudaGraphExecDestroy(graph);
    graph = nullptr;
  }
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
  const long long before = launches;
  for (int i = 0; i < k; ++i) launch_iteration(false);
  launches = before;
  CK(cudaStreamEndCapture(stream, &g));
  CK(cudaGraphInstantiate(&graph, g, 0));
  cudaGraphDestroy(g);
  graph_k = k;
}

void Context::begin(const cclp_cu_config& cfg, const cclp_cu_tolerances& tol,
                    const double* thresholds, int nthr) {
  exact = cfg.exact_spmv != 0;
  if (graph) {
    cudaGraphExecDestroy(graph);
    graph = nullptr;
  }
  k_stamp<<<1, 1, 0, stream>>>(t0);
  CKL("stamp");
  setup(cfg);
  init_state(cfg, tol, thresholds, nthr, true);
}

// Scaling, norms, ||A|| and the step sizes (pdhg.cpp:245-267).
void Context::setup(const cclp_cu_config& cfg) {
  phase_t0 = std::chrono::steady_clock::now();
  // the power iteration's start vector is host work: overlap it with the
  // device-side norms, Ruiz passes and value scaling
  // (the default seed's vector may still be in the making since upload: it
  // is joined only right before the power iteration)
  if (v0_thread.joinable() && v0_seed != cfg.seed) v0_thread.join();
  if (!h_v0) h_v0 = host_alloc<double>(n);
  std::thread rng_thread;
  if (m > 0 && n > 0 && nnz > 0 && v0_seed != cfg.seed) {
    v0_seed = cfg.seed;
    rng_thread = std::thread(gaussian_start, cfg.seed, static_cast<long long>(n), h_v0);
  }
  struct Joiner {
    std::thread& t;
    ~Joiner() { if (t.joinable()) t.join(); }
  } joiner{rng_thread};
  // norms on the unscaled model (pdhg.cpp:253-254)
  b_norm = std::sqrt(reduce(b, nullptr, m, 0));
  c_norm = std::sqrt(reduce(c, nullptr, n, 0));
  mark(3);
  ruiz(cfg.scaling_iterations);
  mark(4);
  if (!sval_csr) sval_csr = alloc<double>(nnz);
  if (!sval_csc) sval_csc = alloc<double>(nnz);
  k_scale_values<<<blocks_for(static_cast<long long>(m) * 32), kBlock, 0, stream>>>(
      rowptr, m, colind, val_csr, r, s, 1, sval_csr);
  k_scale_values<<<blocks_for(static_cast<long long>(n) * 32), kBlock, 0, stream>>>(
      colptr, n, rowind, val_csc, s, r, 0, sval_csc);
  CKL("scale");
  for (auto& pn : panels)  // panel-major copies of the scaled values
    if (pn.nnz > 0)
      k_gather_vals<<<blocks_for(pn.nnz), kBlock, 0, stream>>>(pn.perm, pn.nnz, sval_csr, pn.val);
  CKL("panel values");
  mark(5);
  if (rng_thread.joinable()) rng_thread.join();
  if (v0_thread.joinable()) v0_thread.join();
  norm_est = power_norm(cfg.norm_iterations, cfg.seed, true, true);
  mark(6);
  const double a_norm = norm_est > 0.0 ? norm_est : 1.0;
  omega = cfg.primal_weight;
  if (omega <= 0.0) {  // pdhg.cpp:260-265 on the scaled model
    const double cs = std::sqrt(reduce(c, s, n, 1));
    const double bs = std::sqrt(reduce(b, r, m, 1));
    omega = (cs > 0.0 && bs > 0.0) ? cs / bs : 1.0;
  }
  tau = cfg.step_scale * omega / a_norm;
  sigma = cfg.step_scale / (omega * a_norm);
}

// State buffers, control block, x_0 and (optionally) the initial products
// and check(0) (make_initial_state, pdhg.cpp:67-82; the first check block).
void Context::init_state(const cclp_cu_config& cfg, const cclp_cu_tolerances& tol,
                         const double* thresholds, int nthr, bool launch_init) {
  // state buffers
  auto alloc_n = [&](double*& p) { if (!p) p = alloc<double>(n); };
  auto alloc_m = [&](double*& p) { if (!p) p = alloc<double>(m); };
  for (int k = 0; k < 3; ++k)
    for (int q = 0; q < 2; ++q) alloc_n(xc[k][q]);
  for (int q = 0; q < 2; ++q) {
    alloc_n(aty[q]); alloc_n(xsum[q]); alloc_n(atysum[q]);
    alloc_m(y[q]); alloc_m(ax[q]); alloc_m(ysum[q]); alloc_m(axsum[q]);
  }
  alloc_m(ax[2]);
  for (int q = 0; q < 2; ++q) {
    CK(cudaMemsetAsync(y[q], 0, sizeof(double) * std::max(m, 1), stream));
    CK(cudaMemsetAsync(ysum[q], 0, sizeof(double) * std::max(m, 1), stream));
    CK(cudaMemsetAsync(axsum[q], 0, sizeof(double) * std::max(m, 1), stream));
    CK(cudaMemsetAsync(xsum[q], 0, sizeof(double) * std::max(n, 1), stream));
    CK(cudaMemsetAsync(atysum[q], 0, sizeof(double) * std::max(n, 1), stream));
  }
  if (!ctrl) {
    ctrl = alloc<Ctrl>(1);
    h_ctrl = host_alloc<Ctrl>(4);
    log = alloc<LogEntry>(log_cap);
    h_log = host_alloc<LogEntry>(log_cap);
  }
  Ctrl c0;
  std::memset(&c0, 0, sizeof c0);
  c0.stop = -1;
  c0.last_restart_resid = INFINITY;
  CK(cudaMemcpyAsync(ctrl, &c0, sizeof c0, cudaMemcpyHostToDevice, stream));
  if (nthr > thr_cap) {
    if (thr) release(thr);
    thr = alloc<double>(nthr);
    thr_cap = nthr;
  }
  if (nthr > 0)
    CK(cudaMemcpyAsync(thr, thresholds, sizeof(double) * nthr, cudaMemcpyHostToDevice, stream));
  k_init_x<<<blocks_for(n), kBlock, 0, stream>>>(l, u, s, n, xc[0][0]);
  CKL("init x");

  IterParams& p = params;
  p.m = m; p.n = n;
  p.rowptr = rowptr; p.colind = colind; p.aval = sval_csr;
  p.colptr = colptr; p.rowind = rowind; p.atval = sval_csc;
  p.row_start = row_start; p.col_start = col_start;
  p.row_grid = epi_grid; p.col_grid = epi_grid;  // partial counts for finalize
  p.plan_r = plan(true); p.plan_c = plan(false);
  p.rpg_rows = rpg_r; p.rpg_cols = rpg_c;
  build_sell_cols();
  build_sellg(true);
  build_sellg(false);
  p.use_sell_r = sgr.on ? 1 : 0;
  p.sell_r = SellPlan{sgr.off, sgr.start, rowptr, sgr.idx, sgr.val, m, sgr.thr};
  p.use_sell_cg = sgc.on ? 1 : 0;
  p.sell_cg = SellPlan{sgc.off, sgc.start, colptr, sgc.idx, sgc.val, n, sgc.thr};
  p.use_sell_c = sell_on ? 1 : 0;
  p.sell_c = SellPlan{sell_off, sell_start, colptr, sell_idx, sell_val, n, sell_thr};
  p.c = c; p.l = l; p.u = u; p.b = b; p.r = r; p.s = s;
  for (int k = 0; k < 3; ++k)
    for (int q = 0; q < 2; ++q) p.xc[k][q] = xc[k][q];
  for (int q = 0; q < 2; ++q) {
    p.aty[q] = aty[q]; p.xsum[q] = xsum[q]; p.atysum[q] = atysum[q];
    p.y[q] = y[q]; p.ax[q] = ax[q]; p.ysum[q] = ysum[q]; p.axsum[q] = axsum[q];
  }
  p.ax[2] = ax[2];
  p.rowp = rowp; p.colp = colp; p.counter = counter; p.ctrl = ctrl;
  p.log = log; p.log_cap = log_cap; p.log_interval = cfg.log_interval;
  p.tau = tau; p.sigma = sigma; p.eps_rel = tol.eps_rel; p.restart_factor = cfg.restart_factor;
  p.b_norm = b_norm; p.c_norm = c_norm; p.time_limit = cfg.time_limit;
  p.max_iter = cfg.max_iterations; p.check_interval = cfg.check_interval;
  p.nthr = nthr; p.thr = thr; p.t0_ns = t0;
  p.xg = nullptr; p.yg = nullptr; p.y_full_loc = nullptr; p.xpart_loc = nullptr;
  if (shard_count > 1 || x_full != nullptr) {  // sharded: gathers from the padded full vectors
    p.xg = x_full;
    p.yg = y_full;
    p.y_full_loc = y_full + static_cast<size_t>(shard_rank) * Sm;
    p.xpart_loc = xpart + shard_rank * (kRowParts + kColParts);
    p.time_limit = INFINITY;  // checked on the host so every shard stops together
    CK(cudaMemsetAsync(y_full, 0, sizeof(double) * std::max<size_t>(1, size_t(shard_count) * Sm), stream));
    CK(cudaMemcpyAsync(x_full + static_cast<size_t>(shard_rank) * Sn, xc[0][0], sizeof(double) * n,
                       cudaMemcpyDeviceToDevice, stream));
  }
  // inline snapshots and the per-iteration cancel (single device only: the
  // sharded solve halts for snapshots and agrees on stops on the host)
  const bool single = !(shard_count > 1 || x_full != nullptr);
  p.snap_inline = 0;
  p.stamps = nullptr;
  p.spec = nullptr;
  p.host_flags = nullptr;
  p.cancel_dev = nullptr;
  for (int k = 0; k < kSnapSlots; ++k) p.snap_x[k] = p.snap_y[k] = p.snap_z[k] = nullptr;
  if (single) {
    ensure_flags();
    if (!cancel_dev) cancel_dev = alloc<unsigned>(1);
    CK(cudaMemsetAsync(cancel_dev, 0, sizeof(unsigned), stream));
    p.host_flags = d_flags;
    p.cancel_dev = cancel_dev;
    if (!stamps) stamps = alloc<unsigned long long>(cclp_cu::kStampRing * 4);
    CK(cudaMemsetAsync(stamps, 0, sizeof(unsigned long long) * cclp_cu::kStampRing * 4, stream));
    p.stamps = stamps;
    // speculative row products (row_step) where one kernel computes the whole
    // row product of a step (not the column panels) and PDL is on
    const char* ek = dev_knob("CCLP_CU_SPEC");  // A/B experiments only
    if (p.use_sell_r && sgr.grid % row_sms == 0 && pdl_enabled() && (ek == nullptr || std::atoi(ek) != 0)) {
      if (!spec_sync) spec_sync = alloc<unsigned long long>(4);
      CK(cudaMemsetAsync(spec_sync, 0, sizeof(unsigned long long) * 4, stream));
      p.spec = spec_sync;
    }
    if (nthr > 0) {
      for (int k = 0; k < kSnapSlots; ++k) {
        if (!snap_buf[k]) snap_buf[k] = alloc<double>(2 * static_cast<size_t>(n) + m);
        p.snap_x[k] = snap_buf[k];
        p.snap_z[k] = snap_buf[k] + n;
        p.snap_y[k] = snap_buf[k] + 2 * static_cast<size_t>(n);
      }
      p.snap_inline = 1;
    }
  }
  // initial products and check(0)
  if (launch_init) launch_iteration(true);
  if (graph) {
    cudaGraphExecDestroy(graph);
    graph = nullptr;
  }
  mark(7);
  begun = true;
}

void Context::fetch_ctrl(Ctrl* dst) {
  CK(cudaMemcpyAsync(dst, ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, stream));
  CK(cudaStreamSynchronize(stream));
}

// Unscaled x, y, z (and a report) of a view of the current state into vx,
// vy, vz, vrep.
void Context::extract_view(int view, const Ctrl& st) {
  if (!vx) {
    vx = alloc<double>(n);
    vz = alloc<double>(n);
    vy = alloc<double>(m);
    vrep = alloc<double>(kRepN);
  }
  ViewParams v;
  v.it = params;
  int vv = view;
  if (vv == kViewCurEff) vv = st.R ? kViewAvg : kViewCur;
  v.view = vv;
  v.t = st.iteration;
  v.R_prev = st.R_prev;
  v.inv = st.window > 0 ? 1.0 / static_cast<double>(st.window) : 0.0;
  v.x_out = vx;
  v.y_out = vy;
  v.z_out = vz;
  v.rowp = rowp;
  v.colp = colp;
  v.counter = counter + 3;
  v.report = vrep;
  v.parts_out = vparts;
  const int gr = blocks_for(m, kBlock, 148 * 4);
  const int gc = blocks_for(n, kBlock, 148 * 4);
  k_view_rows<<<gr, kBlock, 0, stream>>>(v);
  k_view_cols<<<gc, kBlock, 0, stream>>>(v, gr);
  CKL("view");
}


// cclp_cu_profile_kernels: average device time per launch of the four
// iteration kernels, launched eagerly (no PDL, no graph) with events between
// them (the bench keeps it beside the in-graph split).
void Context::profile_kernels(long long iters, double* out) {
  if (!begun) throw std::invalid_argument("cclp_cu_profile_kernels: call cclp_cu_begin first");
  constexpr int K = kKernelsPerIteration;
  std::vector<cudaEvent_t> ev((K + 1) * iters);
  for (auto& e : ev) CK(cudaEventCreate(&e));
  const IterParams& p = params;
  for (long long i = 0; i < iters; ++i) {
    cudaEvent_t* e = &ev[(K + 1) * i];
    CK(cudaEventRecord(e[0], stream));
    if (use_panels()) {
      for (int k = 0; k < static_cast<int>(panels.size()); ++k) {
        const PanelArgs a = panel_args(k);
        with_group_long(panels[k].G, a.plan.thr != 0x7fffffff, [&](auto g, auto l) {
          k_spmv_rows_panel<decltype(g)::value, decltype(l)::value>
              <<<panel_grid, kSpmvBlock, 0, stream>>>(p, 0, a);
        });
      }
    } else if (p.use_sell_r) {
      with_group_long(grow(), p.plan_r.thr != 0x7fffffff, [&](auto g, auto l) {
        if (sgr.bs == 256)
          k_spmv_rows_sellg<decltype(g)::value, decltype(l)::value, 256>
              <<<sgr.grid, 256, 0, stream>>>(p, 0);
        else
          k_spmv_rows_sellg<decltype(g)::value, decltype(l)::value, kSpmvBlock>
              <<<sgr.grid, kSpmvBlock, 0, stream>>>(p, 0);
      });
    } else {
      with_group_long(grow(), p.plan_r.thr != 0x7fffffff, [&](auto g, auto l) {
        k_spmv_rows<decltype(g)::value, decltype(l)::value>
            <<<spmv_grid_r, kSpmvBlock, 0, stream>>>(p, 0);
      });
    }
    CK(cudaEventRecord(e[1], stream));
    launch_dual(0);
    CK(cudaEventRecord(e[2], stream));
    if (p.use_sell_cg) {
      with_group_long(gcol(), p.plan_c.thr != 0x7fffffff, [&](auto g, auto l) {
        if (sgc.bs == 256)
          k_spmv_cols_sellg<decltype(g)::value, decltype(l)::value, 256>
              <<<sgc.grid, 256, 0, stream>>>(p, 0);
        else
          k_spmv_cols_sellg<decltype(g)::value, decltype(l)::value, kSpmvBlock>
              <<<sgc.grid, kSpmvBlock, 0, stream>>>(p, 0);
      });
    } else if (p.use_sell_c) {
      if (p.plan_c.thr != 0x7fffffff)
        k_spmv_cols_sell<true, kSpmvBlock>
            <<<spmv_grid_c, kSpmvBlock, 0, stream>>>(p, 0);
      else if (sell_bs == 256)
        k_spmv_cols_sell<false, 256><<<sell_grid, 256, 0, stream>>>(p, 0);
      else
        k_spmv_cols_sell<false, kSpmvBlock>
            <<<sell_grid, kSpmvBlock, 0, stream>>>(p, 0);
    } else {
      with_group_long(gcol(), p.plan_c.thr != 0x7fffffff, [&](auto g, auto l) {
        k_spmv_cols<decltype(g)::value, decltype(l)::value>
            <<<spmv_grid_c, kSpmvBlock, 0, stream>>>(p, 0);
      });
    }
    CK(cudaEventRecord(e[3], stream));
    launch_primal(0);
    CK(cudaEventRecord(e[4], stream));
    launches += K;
  }
  CK(cudaStreamSynchronize(stream));
  double acc[K] = {0, 0, 0, 0};
  for (long long i = 0; i < iters; ++i)
    for (int k = 0; k < K; ++k) {
      float ms;
      CK(cudaEventElapsedTime(&ms, ev[(K + 1) * i + k], ev[(K + 1) * i + k + 1]));
      acc[k] += ms;
    }
  for (auto& e : ev) cudaEventDestroy(e);
  for (int k = 0; k < K; ++k) out[k] = iters ? acc[k] / iters : 0.0;
}

}  // namespace cclp_cu
