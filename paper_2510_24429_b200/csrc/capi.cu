// C ABI of the single-device engine (include/cclp_cu.h): create/solve/destroy,
// the kernel-level entry points and the measurement hooks. The solve's host
// protocol (cclp_cu_solve) keeps two CUDA-graph batches in flight on a
// launcher thread and runs the caller's sink and log on the calling thread.
// Reference: run_pdhg, proj/src/pdhg.cpp:230-378.
#include "capi_util.cuh"

extern "C" {

const char* cclp_cu_last_error(void) { return g_err.c_str(); }

void cclp_cu_gaussian_start(uint64_t seed, int64_t n, double* out) {
  cclp_cu::gaussian_start(seed, n, out);
}

const char* cclp_cu_stop_string(int32_t stop) {
  switch (stop) {  // pdhg.cpp:28-44
    case CCLP_CU_STOP_CONVERGED: return "converged";
    case CCLP_CU_STOP_ITERATION_LIMIT: return "iteration-limit";
    case CCLP_CU_STOP_TIME_LIMIT: return "time-limit";
    case CCLP_CU_STOP_CANCELLED: return "cancelled";
    case CCLP_CU_STOP_WON_BY_CROSSOVER: return "won-by-crossover";
    case CCLP_CU_STOP_NUMERICAL_ERROR: return "numerical-error";
  }
  return "unknown";
}

void cclp_cu_default_config(cclp_cu_config* cfg) {
  cfg->step_scale = 0.9;
  cfg->primal_weight = 0.0;
  cfg->restart_factor = 0.5;
  cfg->time_limit = INFINITY;
  cfg->norm_iterations = 100;
  cfg->scaling_iterations = 10;
  cfg->max_iterations = 2000000;
  cfg->check_interval = 1;
  cfg->seed = 0;
  cfg->log_interval = 0;
  cfg->deterministic = 1;
  cfg->poll_interval = 0;
  cfg->exact_spmv = 0;
}

void cclp_cu_default_tolerances(cclp_cu_tolerances* t) {
  t->eps_rel = 1e-6;
  t->eps_abs = 1e-6;
  t->eps_cross = 1e-2;
  t->decrement = 0.1;
}

int cclp_cu_create(const cclp_cu_lp* lp, int device, cclp_cu_ctx** out) {
  *out = nullptr;
  return guarded([&] {
    if (lp == nullptr || lp->m < 0 || lp->n < 0 || lp->colptr == nullptr)
      throw std::invalid_argument("cclp_cu_create: bad LP");
    cclp_cu::validate_csc(lp);  // before any device work
    cclp_cu::ck(cudaSetDevice(device), "cudaSetDevice");
    auto* ctx = new cclp_cu_ctx();
    ctx->c.device = device;
    try {
      ctx->c.upload(lp);
    } catch (...) {
      delete ctx;
      throw;
    }
    *out = ctx;
  });
}

int cclp_cu_create_from_file(const char* path, int device, cclp_cu_ctx** out, int32_t* m_out,
                             int32_t* n_out) {
  *out = nullptr;
  int fd = -1;
  void* map = MAP_FAILED;
  size_t len = 0;
  const int rc = guarded([&] {
    fd = open(path, O_RDONLY);
    if (fd < 0) throw std::invalid_argument(std::string("cclp_cu_create_from_file: cannot open ") + path);
    struct stat st;
    if (fstat(fd, &st) != 0 || st.st_size < 32) throw std::invalid_argument("cclp_cu_create_from_file: short file");
    len = static_cast<size_t>(st.st_size);
    map = mmap(nullptr, len, PROT_READ, MAP_SHARED, fd, 0);
    if (map == MAP_FAILED) throw std::invalid_argument("cclp_cu_create_from_file: mmap failed");
    const char* base = static_cast<const char*>(map);
    if (std::memcmp(base, "CCLPCSC1", 8) != 0) throw std::invalid_argument("cclp_cu_create_from_file: bad magic");
    int32_t mn[2];
    int64_t nnz;
    std::memcpy(mn, base + 8, sizeof mn);
    std::memcpy(&nnz, base + 16, sizeof nnz);
    const int32_t m = mn[0], n = mn[1];
    if (m < 0 || n < 0 || nnz < 0) throw std::invalid_argument("cclp_cu_create_from_file: bad header");
    size_t off = 32;
    auto take = [&](size_t bytes) {  // exact bound: the array ends inside the file
      const char* p = base + off;
      if (off + bytes > len) throw std::invalid_argument("cclp_cu_create_from_file: truncated file");
      off += bytes;
      off = (off + 7) / 8 * 8;
      return p;
    };
    cclp_cu_lp lp;
    lp.m = m;
    lp.n = n;
    lp.colptr = reinterpret_cast<const int32_t*>(take(sizeof(int32_t) * (static_cast<size_t>(n) + 1)));
    lp.rowind = reinterpret_cast<const int32_t*>(take(sizeof(int32_t) * static_cast<size_t>(nnz)));
    lp.val = reinterpret_cast<const double*>(take(sizeof(double) * static_cast<size_t>(nnz)));
    lp.c = reinterpret_cast<const double*>(take(sizeof(double) * n));
    lp.row_lower = reinterpret_cast<const double*>(take(sizeof(double) * m));
    lp.row_upper = reinterpret_cast<const double*>(take(sizeof(double) * m));
    lp.col_lower = reinterpret_cast<const double*>(take(sizeof(double) * n));
    lp.col_upper = reinterpret_cast<const double*>(take(sizeof(double) * n));
    if (lp.colptr[n] != nnz) throw std::invalid_argument("cclp_cu_create_from_file: colptr[n] != nnz");
    if (m_out) *m_out = m;
    if (n_out) *n_out = n;
    const int rc2 = cclp_cu_create(&lp, device, out);
    if (rc2 != CCLP_CU_OK) throw Error(rc2, g_err);
  });
  if (map != MAP_FAILED) munmap(map, len);
  if (fd >= 0) close(fd);
  return rc;
}

int cclp_cu_destroy(cclp_cu_ctx* ctx) {
  delete ctx;
  return CCLP_CU_OK;
}

int cclp_cu_begin(cclp_cu_ctx* ctx, const cclp_cu_config* cfg, const cclp_cu_tolerances* tol) {
  return guarded([&] {
    cclp_cu::ck(cudaSetDevice(ctx->c.device), "cudaSetDevice");
    validate_inputs(ctx, *cfg, *tol, nullptr, 0);
    cclp_cu_tolerances t = *tol;
    ctx->c.ensure_flags();
    ctx->c.h_flags[0] = ctx->c.h_flags[1] = 0u;
    ctx->c.begin(*cfg, t, nullptr, 0);
    // measurement mode: never converge, never hit the limit
    ctx->c.params.eps_rel = -1.0;
    ctx->c.params.max_iter = (1LL << 62);
    ctx->c.params.time_limit = INFINITY;
  });
}

int cclp_cu_advance(cclp_cu_ctx* ctx, int64_t iters, double* device_ms) {
  return guarded([&] {
    Context& C = ctx->c;
    if (!C.begun) throw std::invalid_argument("cclp_cu_advance: call cclp_cu_begin first");
    const int k = 32;
    C.build_graph(k);
    CK(cudaEventRecord(C.ev_a, C.stream));
    long long done = 0;
    while (done + k <= iters) {
      CK(cudaGraphLaunch(C.graph, C.stream));
      C.launches += cclp_cu::kKernelsPerIteration * k;
      done += k;
    }
    while (done < iters) {
      C.launch_iteration(false);
      ++done;
    }
    CK(cudaEventRecord(C.ev_b, C.stream));
    CK(cudaEventSynchronize(C.ev_b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, C.ev_a, C.ev_b));
    if (device_ms) *device_ms = ms;
  });
}

int cclp_cu_profile_kernels(cclp_cu_ctx* ctx, int64_t iters, double* out) {
  return guarded([&] { ctx->c.profile_kernels(iters, out); });
}

int cclp_cu_phase_profile(cclp_cu_ctx* ctx, double* out, int64_t* steps) {
  return guarded([&] {
    Context& C = ctx->c;
    if (!C.begun || C.stamps == nullptr)
      throw std::invalid_argument("cclp_cu_phase_profile: call cclp_cu_begin/advance first (single device)");
    constexpr int R = cclp_cu::kStampRing;
    std::vector<unsigned long long> st(R * 4);
    Ctrl ctl;
    CK(cudaStreamSynchronize(C.stream));
    CK(cudaMemcpy(st.data(), C.stamps, sizeof(unsigned long long) * R * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&ctl, C.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost));
    // steps t and t+1 both still in the ring: t in [it - R + 1, it - 2]
    std::vector<double> d[4];
    const long long it = ctl.iteration;
    for (long long t = std::max<long long>(1, it - R + 1); t + 1 < it; ++t) {
      const unsigned long long* a = &st[(t % R) * 4];
      const unsigned long long nxt = st[((t + 1) % R) * 4];
      const unsigned long long e[5] = {a[0], a[1], a[2], a[3], nxt};
      bool ok = true;
      for (int k = 0; k < 4; ++k) ok = ok && e[k] != 0 && e[k + 1] > e[k];
      if (!ok) continue;
      for (int k = 0; k < 4; ++k) d[k].push_back(1e-3 * static_cast<double>(e[k + 1] - e[k]));
    }
    for (int k = 0; k < 4; ++k) {
      if (d[k].empty()) { out[k] = 0.0; continue; }
      std::nth_element(d[k].begin(), d[k].begin() + d[k].size() / 2, d[k].end());
      out[k] = d[k][d[k].size() / 2];
    }
    if (steps) *steps = static_cast<int64_t>(d[0].size());
  });
}

void* cclp_cu_stream(cclp_cu_ctx* ctx) { return ctx ? static_cast<void*>(ctx->c.stream) : nullptr; }

int cclp_cu_describe(cclp_cu_ctx* ctx, int64_t* out, int32_t nout) {
  const Context& C = ctx->c;
  Ctrl st;
  std::memset(&st, 0, sizeof st);
  if (C.ctrl != nullptr && cudaMemcpy(&st, C.ctrl, sizeof st, cudaMemcpyDeviceToHost) != cudaSuccess)
    cudaGetLastError();
  const int64_t v[] = {C.m, C.n, C.nnz, C.grow(), C.gcol(), C.spmv_grid_r * 10 + C.rpg_r,
                       C.spmv_grid_c * 10 + C.rpg_c, C.launches,
                       static_cast<int64_t>(st.t_fin_start - st.t_cols_start),
                       static_cast<int64_t>(st.t_fin_end - st.t_fin_start),
                       // 10..20: phase timings in ns (Context::phase)
                       static_cast<int64_t>(1e9 * C.phase[0]), static_cast<int64_t>(1e9 * C.phase[1]),
                       static_cast<int64_t>(1e9 * C.phase[2]), static_cast<int64_t>(1e9 * C.phase[3]),
                       static_cast<int64_t>(1e9 * C.phase[4]), static_cast<int64_t>(1e9 * C.phase[5]),
                       static_cast<int64_t>(1e9 * C.phase[6]), static_cast<int64_t>(1e9 * C.phase[7]),
                       static_cast<int64_t>(1e9 * C.phase[8]), static_cast<int64_t>(1e9 * C.phase[9]),
                       static_cast<int64_t>(1e9 * C.phase[10]),
                       // 21, 22: block size of the SELL row / column product (0: CSR-G kernel)
                       C.sgr.on ? C.sgr.bs : 0, C.sell_on ? C.sell_bs : (C.sgc.on ? C.sgc.bs : 0),
                       // 23: the row product starts during the decision tail (row_step)
                       C.params.spec != nullptr ? 1 : 0};
  for (int i = 0; i < nout && i < static_cast<int>(sizeof(v) / sizeof(v[0])); ++i) out[i] = v[i];
  return CCLP_CU_OK;
}

int cclp_cu_matvec(cclp_cu_ctx* ctx, const double* x, double* out) {
  return guarded([&] {
    Context& C = ctx->c;
    CK(cudaSetDevice(C.device));
    CK(cudaMemcpyAsync(C.wn, x, sizeof(double) * C.n, cudaMemcpyHostToDevice, C.stream));
    C.launch_spmv(false, C.wn, C.wm, false, nullptr);
    CK(cudaMemcpyAsync(out, C.wm, sizeof(double) * C.m, cudaMemcpyDeviceToHost, C.stream));
    CK(cudaStreamSynchronize(C.stream));
  });
}

int cclp_cu_relative_report(cclp_cu_ctx* ctx, const double* x, const double* y, const double* z,
                            cclp_cu_report* out, double* abs_violation) {
  return guarded([&] {
    Context& C = ctx->c;
    CK(cudaSetDevice(C.device));
    double rep[cclp_cu::kRepN];
    C.relative_report(x, y, z, rep, abs_violation);
    copy_report(rep, out);
  });
}

int cclp_cu_price(cclp_cu_ctx* ctx, const double* y, const char* status, const uint8_t* skip, int32_t phase1,
                  double dtol, int32_t bland, int64_t* entering, int32_t* direction, double* violation) {
  return guarded([&] {
    Context& C = ctx->c;
    CK(cudaSetDevice(C.device));
    long long e = -1;
    int d = 0;
    C.price(y, status, skip, phase1, dtol, bland, &e, &d, violation);
    *entering = e;
    *direction = d;
  });
}

int cclp_cu_matvec_transpose(cclp_cu_ctx* ctx, const double* y, double* out) {
  return guarded([&] {
    Context& C = ctx->c;
    CK(cudaSetDevice(C.device));
    CK(cudaMemcpyAsync(C.wm, y, sizeof(double) * C.m, cudaMemcpyHostToDevice, C.stream));
    C.launch_spmv(true, C.wm, C.wn, false, nullptr);
    CK(cudaMemcpyAsync(out, C.wn, sizeof(double) * C.n, cudaMemcpyDeviceToHost, C.stream));
    CK(cudaStreamSynchronize(C.stream));
  });
}

int cclp_cu_ruiz(cclp_cu_ctx* ctx, int32_t iterations, double* row_scale, double* col_scale) {
  return guarded([&] {
    Context& C = ctx->c;
    CK(cudaSetDevice(C.device));
    C.ruiz(iterations);
    CK(cudaMemcpyAsync(row_scale, C.r, sizeof(double) * C.m, cudaMemcpyDeviceToHost, C.stream));
    CK(cudaMemcpyAsync(col_scale, C.s, sizeof(double) * C.n, cudaMemcpyDeviceToHost, C.stream));
    CK(cudaStreamSynchronize(C.stream));
  });
}

int cclp_cu_estimate_norm(cclp_cu_ctx* ctx, int32_t iterations, uint64_t seed, double* out) {
  return guarded([&] {
    Context& C = ctx->c;
    CK(cudaSetDevice(C.device));
    *out = C.power_norm(iterations, seed, false);
  });
}

int cclp_cu_solve(cclp_cu_ctx* ctx, const cclp_cu_config* cfg_in, const cclp_cu_tolerances* tol,
                  const double* thresholds, int32_t nthr, cclp_cu_sink_fn sink, void* sink_user,
                  const volatile uint8_t* cancel, cclp_cu_log_fn logfn, void* log_user,
                  double* x_out, double* y_out, double* z_out, cclp_cu_result* res) {
  return guarded([&] {
    Context& C = ctx->c;
    CK(cudaSetDevice(C.device));
    const cclp_cu_config cfg = *cfg_in;
    validate_inputs(ctx, cfg, *tol, thresholds, nthr);
    const auto wall0 = std::chrono::steady_clock::now();
    C.launches = 0;
    // First-touch the caller's result arrays on a host thread while the
    // device works, so the final device-to-host copies do not take page
    // faults (fresh pageable arrays cost ~4 ms on C2 otherwise).
    std::thread prefault([=, &C] {
      if (x_out) std::memset(x_out, 0, sizeof(double) * C.n);
      if (y_out) std::memset(y_out, 0, sizeof(double) * C.m);
      if (z_out) std::memset(z_out, 0, sizeof(double) * C.n);
    });
    struct JoinOnExit {
      std::thread& t;
      ~JoinOnExit() { if (t.joinable()) t.join(); }
    } prefault_join{prefault};
    const int k = cfg.poll_interval > 0 ? cfg.poll_interval : 64;
    // the log ring holds two batches in flight (at most one line per iteration)
    if (cfg.log_interval > 0 && C.log_cap < 4 * k) {
      C.release(C.log);
      C.log = nullptr;
      C.log_cap = 4 * k;
      C.h_log = C.host_alloc<cclp_cu::LogEntry>(C.log_cap);
      C.log = C.alloc<cclp_cu::LogEntry>(C.log_cap);
    }
    // cancel: the caller's flag (and cclp_cu_request_cancel) mirrored into
    // mapped memory that k_primal reads every iteration (pdhg.cpp:301)
    C.ensure_flags();
    C.abort_req.store(0);
    volatile unsigned* hf = C.h_flags;
    auto mirror_cancel = [&]() {
      if ((cancel != nullptr && *cancel) || C.abort_req.load(std::memory_order_relaxed)) hf[0] = 1u;
    };
    hf[0] = 0u;
    hf[1] = 0u;
    mirror_cancel();
    // three pinned staging sets of x | z (n) | y (m) for ladder snapshots:
    // cudaHostAlloc costs ~1 ms per MB, so it runs on a helper thread while
    // the setup works on the device, and is done before the loop's timer
    const size_t stage_bytes = sizeof(double) * 3 * (2 * static_cast<size_t>(C.n) + C.m);
    void* stage_p = nullptr;
    std::exception_ptr stage_err;
    std::thread stage_alloc;
    if (nthr > 0 && !C.h_sx)
      stage_alloc = std::thread([&] {
        try {
          stage_p = cclp_cu::pinned_alloc(stage_bytes);
        } catch (...) {
          stage_err = std::current_exception();
        }
      });
    struct JoinStage {
      std::thread& t;
      ~JoinStage() { if (t.joinable()) t.join(); }
    } stage_join{stage_alloc};
    C.begin(cfg, *tol, thresholds, nthr);
    if (stage_alloc.joinable()) {
      stage_alloc.join();
      if (stage_err) std::rethrow_exception(stage_err);
      C.pinned.emplace_back(stage_p, stage_bytes);
      C.h_sx = static_cast<double*>(stage_p);
    }
    const double setup_s =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
    C.build_graph(k);
    C.mark(8);
    CK(cudaEventRecord(C.ev_a, C.stream));

    // ---- host side of the loop ------------------------------------------
    // A launcher thread keeps two graph batches in flight (the device never
    // waits for the host between batches), mirrors the cancel flag, and
    // copies ladder snapshots out of their device slots on the side stream;
    // the calling thread receives log lines and snapshots through a queue, in
    // iteration order, and runs the caller's log and sink callbacks
    // (pdhg.cpp:332-358) while the device keeps iterating.
    struct Event {
      int kind;  // 0 log line, 1 snapshot (staging set `set`), 2 end of loop
      long long iteration;
      std::string line;
      int set = 0, thr_idx = 0, use_avg = 0;
      double maxresid = 0.0;
    };
    std::mutex mu;
    std::condition_variable cv;
    std::deque<Event> events;
    bool staging_busy[3] = {false, false, false};  // 0,1: slot snapshots; 2: host-extracted
    std::exception_ptr launcher_error;
    Ctrl st;
    auto push = [&](Event e) {
      std::lock_guard<std::mutex> g(mu);
      events.push_back(std::move(e));
      cv.notify_all();
    };
    auto set_ptr = [&](int set) { return C.h_sx + static_cast<size_t>(set) * (2 * static_cast<size_t>(C.n) + C.m); };
    auto acquire_set = [&](int set) {  // launcher: wait until the sink released it
      std::unique_lock<std::mutex> g(mu);
      cv.wait(g, [&] { return !staging_busy[set]; });
      staging_busy[set] = true;
    };

    std::thread launcher([&] {
      try {
        CK(cudaSetDevice(C.device));
        long long log_seen = 0;
        int snaps_copied = 0;
        auto emit_logs_upto = [&](const Ctrl& q, long long upto) {
          if (!logfn || cfg.log_interval <= 0) {
            log_seen = q.log_count;
            return;
          }
          for (long long i = std::max(log_seen, q.log_count - C.log_cap); i < q.log_count; ++i) {
            const auto& e = C.h_log[i % C.log_cap];
            if (e.iteration > upto) return;
            char line[160];
            std::snprintf(line, sizeof line, "%lld\t%.6e\t%.6e\t%.6e\t%.3f\n", e.iteration, e.rel_primal,
                          e.rel_dual, e.rel_gap, e.elapsed);
            push(Event{0, e.iteration, line});
            log_seen = i + 1;
          }
        };
        auto fetch_log = [&](const Ctrl& q) {
          if (!logfn || cfg.log_interval <= 0 || q.log_count == log_seen) return;
          CK(cudaMemcpyAsync(C.h_log, C.log, sizeof(cclp_cu::LogEntry) * C.log_cap, cudaMemcpyDeviceToHost,
                             C.side));
          CK(cudaStreamSynchronize(C.side));
        };
        // snapshot `idx`, extracted by the kernels into slot idx % kSnapSlots
        auto copy_inline = [&](const Ctrl& q, int idx) {
          const cclp_cu::SnapMeta& mt = q.snap_meta[idx % cclp_cu::kSnapSlots];
          const int set = idx % cclp_cu::kSnapSlots;
          acquire_set(set);
          CK(cudaMemcpyAsync(set_ptr(set), C.snap_buf[set], sizeof(double) * (2 * static_cast<size_t>(C.n) + C.m),
                             cudaMemcpyDeviceToHost, C.side));
          CK(cudaStreamSynchronize(C.side));
          hf[1] = static_cast<unsigned>(idx + 1);  // the device slot is free again
          emit_logs_upto(q, mt.iteration);
          push(Event{1, mt.iteration, {}, set, mt.thr_idx, mt.use_avg, mt.maxresid});
        };
        // a snapshot the loop halted for, or one requested at the final check
        auto copy_extracted = [&](const Ctrl& q) {
          acquire_set(2);
          C.extract_view(q.snap_use_avg ? cclp_cu::kViewAvg : cclp_cu::kViewCur, q);
          double* h = set_ptr(2);
          CK(cudaEventRecord(C.ev_snap, C.stream));
          CK(cudaStreamWaitEvent(C.side, C.ev_snap, 0));
          CK(cudaMemcpyAsync(h, C.vx, sizeof(double) * C.n, cudaMemcpyDeviceToHost, C.side));
          CK(cudaMemcpyAsync(h + C.n, C.vz, sizeof(double) * C.n, cudaMemcpyDeviceToHost, C.side));
          CK(cudaMemcpyAsync(h + 2 * static_cast<size_t>(C.n), C.vy, sizeof(double) * C.m, cudaMemcpyDeviceToHost,
                             C.side));
          CK(cudaStreamSynchronize(C.side));
          emit_logs_upto(q, q.snap_iteration);
          push(Event{1, q.snap_iteration, {}, 2, q.snap_thr_idx, q.snap_use_avg, q.snap_maxresid});
        };
        auto clear_halt = [&]() {
          const int zero[2] = {0, 0};
          CK(cudaMemcpyAsync(&C.ctrl->halt, &zero[0], sizeof(int), cudaMemcpyHostToDevice, C.stream));
          CK(cudaMemcpyAsync(&C.ctrl->snap_pending, &zero[1], sizeof(int), cudaMemcpyHostToDevice, C.stream));
          CK(cudaStreamSynchronize(C.stream));
        };
        auto process = [&](const Ctrl& q) {  // everything a finished batch reported
          fetch_log(q);
          while (snaps_copied < q.snaps_done) copy_inline(q, snaps_copied++);
          if (q.halt && q.snap_pending) {
            copy_extracted(q);
            clear_halt();
          }
          emit_logs_upto(q, LLONG_MAX);
        };
        cudaEvent_t evb[2];
        for (auto& e : evb) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        struct EvGuard {
          cudaEvent_t* e;
          ~EvGuard() { for (int i = 0; i < 2; ++i) cudaEventDestroy(e[i]); }
        } evguard{evb};
        auto launch_batch = [&](int slot) {
          CK(cudaGraphLaunch(C.graph, C.stream));
          C.launches += cclp_cu::kKernelsPerIteration * k;
          CK(cudaMemcpyAsync(&C.h_ctrl[slot], C.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, C.stream));
          CK(cudaEventRecord(evb[slot], C.stream));
        };
        auto wait_batch = [&](int slot) {  // polls, mirroring the cancel flag meanwhile
          while (true) {
            const cudaError_t e = cudaEventQuery(evb[slot]);
            if (e == cudaSuccess) return;
            if (e != cudaErrorNotReady) CK(e);
            mirror_cancel();
            std::this_thread::sleep_for(std::chrono::microseconds(20));
          }
        };
        Ctrl q;
        C.fetch_ctrl(&q);  // after the initial check
        process(q);
        if (q.stop < 0) {
          int cur = 0;
          launch_batch(cur);
          bool ahead = false;
          while (true) {
            if (!ahead) launch_batch(cur ^ 1);  // one batch ahead of the one waited for
            ahead = false;
            wait_batch(cur);
            q = C.h_ctrl[cur];
            const bool drained = q.stop >= 0 || q.halt;
            if (drained) wait_batch(cur ^ 1);  // exits at once: the device state is q
            process(q);
            if (q.stop >= 0) break;
            if (drained) {  // the halt was served: restart the pipeline
              launch_batch(cur);
              continue;
            }
            cur ^= 1;
          }
        }
        if (q.snap_pending && !q.halt) copy_extracted(q);  // the step that would extract it never ran
        emit_logs_upto(q, LLONG_MAX);
        st = q;
      } catch (...) {
        launcher_error = std::current_exception();
      }
      push(Event{2, 0, {}});
    });
    struct JoinLauncher {
      std::thread& t;
      ~JoinLauncher() { if (t.joinable()) t.join(); }
    } launcher_join{launcher};

    // calling thread: callbacks in order
    while (true) {
      Event e;
      {
        std::unique_lock<std::mutex> g(mu);
        cv.wait(g, [&] { return !events.empty(); });
        e = std::move(events.front());
        events.pop_front();
      }
      if (e.kind == 2) break;
      if (e.kind == 0) {
        logfn(e.line.c_str(), log_user);
        continue;
      }
      if (sink) {
        const double* h = set_ptr(e.set);
        cclp_cu_snapshot sp;
        sp.x = h;
        sp.z = h + C.n;
        sp.y = h + 2 * static_cast<size_t>(C.n);
        sp.m = C.m;
        sp.n = C.n;
        sp.threshold = thresholds[e.thr_idx];
        sp.maxresid = e.maxresid;
        sp.from_average = e.use_avg;
        sp.iteration = e.iteration;
        sink(&sp, sink_user);
      }
      std::lock_guard<std::mutex> g(mu);
      staging_busy[e.set] = false;
      cv.notify_all();
    }
    launcher.join();
    if (launcher_error) std::rethrow_exception(launcher_error);
    CK(cudaEventRecord(C.ev_b, C.stream));
    CK(cudaEventSynchronize(C.ev_b));
    float loop_ms = 0;
    CK(cudaEventElapsedTime(&loop_ms, C.ev_a, C.ev_b));
    C.mark(9);

    const int view = st.result_view;
    const int stop = st.stop;
    const bool rep_valid = st.result_report_valid != 0;
    C.extract_view(view, st);
    if (prefault.joinable()) prefault.join();
    C.d2h(x_out, C.vx, sizeof(double) * C.n);
    C.d2h(y_out, C.vy, sizeof(double) * C.m);
    C.d2h(z_out, C.vz, sizeof(double) * C.n);
    double rep[cclp_cu::kRepN];
    CK(cudaMemcpyAsync(rep, C.vrep, sizeof(rep), cudaMemcpyDeviceToHost, C.stream));
    CK(cudaStreamSynchronize(C.stream));
    C.mark(10);
    res->stop = stop;
    res->iterations = st.iteration;
    res->restarts = st.restarts;
    res->error_iteration = stop == CCLP_CU_STOP_NUMERICAL_ERROR ? st.error_iteration : -1;
    copy_report(rep_valid ? st.result_report : rep, &res->report);
    res->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
    res->norm_estimate = C.norm_est;
    res->omega = C.omega;
    res->tau = C.tau;
    res->sigma = C.sigma;
    res->setup_seconds = setup_s;
    res->loop_seconds = loop_ms * 1e-3;
    res->kernel_launches = C.launches;
    C.begun = false;
  });
}

int cclp_cu_request_cancel(cclp_cu_ctx* ctx) {
  if (ctx == nullptr) return CCLP_CU_EINVAL;
  ctx->c.abort_req.store(1);
  return CCLP_CU_OK;
}

int cclp_cu_run_pdhg(const cclp_cu_lp* lp, const cclp_cu_config* cfg, const cclp_cu_tolerances* tol,
                     const double* thresholds, int32_t nthr, cclp_cu_sink_fn sink, void* sink_user,
                     const volatile uint8_t* cancel, double* x_out, double* y_out, double* z_out,
                     cclp_cu_result* res, int device) {
  cclp_cu_ctx* ctx = nullptr;
  int rc = cclp_cu_create(lp, device, &ctx);
  if (rc != CCLP_CU_OK) return rc;
  rc = cclp_cu_solve(ctx, cfg, tol, thresholds, nthr, sink, sink_user, cancel, nullptr, nullptr,
                     x_out, y_out, z_out, res);
  cclp_cu_destroy(ctx);
  return rc;
}

}  // extern "C"
