// C ABI of the row-block sharded solve (cclp_cu_sharded_*, sharded.cuh) and
// its host helpers (partition, NCCL id).
#include "context.cuh"
#include "iter_kernels.cuh"
#include "setup_kernels.cuh"
#include "sharded.cuh"
#include "capi_util.cuh"

struct cclp_cu_sharded {
  cclp_cu::Sharded s;
};

extern "C" {

int cclp_cu_sharded_request_cancel(cclp_cu_sharded* ctx) {
  if (ctx == nullptr) return CCLP_CU_EINVAL;
  ctx->s.abort_req.store(1);
  return CCLP_CU_OK;
}

int cclp_cu_partition(const int32_t* ptr, int32_t rows, int32_t parts, int32_t* bounds) {
  return guarded([&] {
    if (ptr == nullptr || bounds == nullptr || rows < 0 || parts < 1)
      throw std::invalid_argument("cclp_cu_partition: bad arguments");
    cclp_cu::host_partition(ptr, rows, parts, 4, bounds);
  });
}

int cclp_cu_nccl_unique_id(uint8_t* out128) {
  return guarded([&] {
    auto& api = cclp_cu::nccl();
    if (!api.ok) throw Error(CCLP_CU_ENCCL, api.err);
    ncclUniqueId id;
    cclp_cu::nck(api.GetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out128, &id, sizeof(id));
  });
}

int cclp_cu_sharded_create(const cclp_cu_lp* lp, int device, int32_t nshards, int32_t rank,
                           int32_t nranks, const uint8_t* nccl_id, cclp_cu_sharded** out) {
  *out = nullptr;
  return guarded([&] {
    if (lp == nullptr || lp->m < 0 || lp->n < 0 || lp->colptr == nullptr)
      throw std::invalid_argument("cclp_cu_sharded_create: bad LP");
    if (nranks < 1 || rank < 0 || rank >= nranks || nshards < 1)
      throw std::invalid_argument("cclp_cu_sharded_create: bad rank / shard counts");
    if (nranks > 1 && nccl_id == nullptr)
      throw std::invalid_argument("cclp_cu_sharded_create: NCCL needs the unique id");
    cclp_cu::ck(cudaSetDevice(device), "cudaSetDevice");
    auto* ctx = new cclp_cu_sharded();
    try {
      ncclUniqueId id;
      if (nccl_id) std::memcpy(&id, nccl_id, sizeof(id));
      ctx->s.create(lp, device, nshards, rank, nranks, nccl_id ? &id : nullptr);
    } catch (...) {
      delete ctx;
      throw;
    }
    *out = ctx;
  });
}

int cclp_cu_sharded_create_hostcomm(const cclp_cu_lp* lp, int device, int32_t rank, int32_t nranks,
                                    const cclp_cu_host_comm* comm, cclp_cu_sharded** out) {
  *out = nullptr;
  return guarded([&] {
    if (lp == nullptr || lp->m < 0 || lp->n < 0 || lp->colptr == nullptr || comm == nullptr)
      throw std::invalid_argument("cclp_cu_sharded_create_hostcomm: bad arguments");
    if (nranks < 1 || rank < 0 || rank >= nranks)
      throw std::invalid_argument("cclp_cu_sharded_create_hostcomm: bad rank");
    cclp_cu::ck(cudaSetDevice(device), "cudaSetDevice");
    auto* ctx = new cclp_cu_sharded();
    try {
      ctx->s.create(lp, device, 1, rank, nranks, nullptr, comm);
    } catch (...) {
      delete ctx;
      throw;
    }
    *out = ctx;
  });
}

int cclp_cu_sharded_destroy(cclp_cu_sharded* ctx) {
  if (ctx) cudaSetDevice(ctx->s.device);
  delete ctx;
  return CCLP_CU_OK;
}

int cclp_cu_sharded_describe(cclp_cu_sharded* ctx, int64_t* out, int32_t nout) {
  const auto& S = ctx->s;
  std::vector<int64_t> v;
  v.push_back(S.P);
  for (int b : S.rb) v.push_back(b);
  for (int b : S.cb) v.push_back(b);
  v.push_back(S.launches);
  v.push_back(S.halo_x.on ? 1 : 0);
  v.push_back(S.halo_x.volume);
  v.push_back(S.halo_y.on ? 1 : 0);
  v.push_back(S.halo_y.volume);
  v.push_back(static_cast<int64_t>(S.shards.size()));  // this process's shards:
  for (const auto& sh : S.shards) {                   // rank, nnz of its A rows / A' rows
    v.push_back(sh->shard_rank);
    v.push_back(sh->nnz_rows_slice);
    v.push_back(sh->nnz_cols_slice);
  }
  for (int i = 0; i < nout && i < static_cast<int>(v.size()); ++i) out[i] = v[i];
  return CCLP_CU_OK;
}

int cclp_cu_sharded_begin(cclp_cu_sharded* ctx, const cclp_cu_config* cfg, const cclp_cu_tolerances* tol) {
  return guarded([&] {
    auto& S = ctx->s;
    cclp_cu::ck(cudaSetDevice(S.device), "cudaSetDevice");
    validate_inputs_eq(S.equality, *cfg, *tol, nullptr, 0);
    S.begin(*cfg, *tol, nullptr, 0);
    for (auto& sh : S.shards) {  // measurement mode: never converge, never hit the limit
      sh->params.eps_rel = -1.0;
      sh->params.max_iter = (1LL << 62);
    }
    if (S.graph) {
      cudaGraphExecDestroy(S.graph);
      S.graph = nullptr;
    }
  });
}

int cclp_cu_sharded_advance(cclp_cu_sharded* ctx, int64_t iters, double* device_ms) {
  return guarded([&] {
    auto& S = ctx->s;
    if (!S.begun) throw std::invalid_argument("cclp_cu_sharded_advance: call begin first");
    Context& C = S.s0();
    const int k = 16;
    CK(cudaEventRecord(C.ev_a, S.stream));
    long long done = 0;
    while (done + k <= iters) {
      S.run_batch(k);
      done += k;
    }
    while (done < iters) {
      S.launch_round(false);
      ++done;
    }
    CK(cudaEventRecord(C.ev_b, S.stream));
    CK(cudaEventSynchronize(C.ev_b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, C.ev_a, C.ev_b));
    if (device_ms) *device_ms = ms;
  });
}

int cclp_cu_sharded_solve(cclp_cu_sharded* ctx, const cclp_cu_config* cfg_in, const cclp_cu_tolerances* tol,
                          const double* thresholds, int32_t nthr, cclp_cu_sink_fn sink, void* sink_user,
                          const volatile uint8_t* cancel, double* x_out, double* y_out, double* z_out,
                          cclp_cu_result* res) {
  return guarded([&] {
    auto& S = ctx->s;
    cclp_cu::ck(cudaSetDevice(S.device), "cudaSetDevice");
    const cclp_cu_config cfg = *cfg_in;
    validate_inputs_eq(S.equality, cfg, *tol, thresholds, nthr);
    const auto wall0 = std::chrono::steady_clock::now();
    S.launches = 0;
    S.abort_req.store(0);
    S.begin(cfg, *tol, thresholds, nthr);
    const double setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
    const int k = cfg.poll_interval > 0 ? cfg.poll_interval : 32;
    S.build_graph(k);
    Context& C0 = S.s0();
    CK(cudaEventRecord(C0.ev_a, S.stream));
    Ctrl st;
    S.fetch_ctrl(&st);
    std::vector<double> hx(S.n), hy(S.m), hz(S.n);
    double sums[cclp_cu::kRowParts + cclp_cu::kColParts];
    bool cancelled = false, timed_out = false;
    while (true) {
      if (st.halt && st.snap_pending) {  // PdhgSnapshot of the better view (pdhg.cpp:346-358)
        S.assemble_view(st.snap_use_avg ? cclp_cu::kViewAvg : cclp_cu::kViewCur, st, hx.data(), hy.data(),
                        hz.data(), sums);
        if (sink) {
          cclp_cu_snapshot sp;
          sp.x = hx.data();
          sp.y = hy.data();
          sp.z = hz.data();
          sp.m = S.m;
          sp.n = S.n;
          sp.threshold = thresholds[st.snap_thr_idx];
          sp.maxresid = st.snap_maxresid;
          sp.from_average = st.snap_use_avg;
          sp.iteration = st.snap_iteration;
          sink(&sp, sink_user);
        }
        S.clear_halt();
        st.halt = 0;
      }
      if (st.stop >= 0) break;
      const bool want_cancel = (cancel != nullptr && *cancel) || S.abort_req.load(std::memory_order_relaxed);
      const bool want_time =
          std::isfinite(cfg.time_limit) &&
          std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count() > cfg.time_limit;
      using Req = cclp_cu::Sharded::StopReq;
      const Req req = S.agree(want_cancel ? Req::kStopCancel : want_time ? Req::kStopTime : Req::kStopNone);
      if (req != Req::kStopNone) {  // all ranks stop together, with the same reason
        cancelled = req == Req::kStopCancel;
        timed_out = req == Req::kStopTime;
        break;
      }
      S.run_batch(k);
      S.fetch_ctrl(&st);
    }
    CK(cudaEventRecord(C0.ev_b, S.stream));
    CK(cudaEventSynchronize(C0.ev_b));
    float loop_ms = 0;
    CK(cudaEventElapsedTime(&loop_ms, C0.ev_a, C0.ev_b));
    int view = st.result_view;
    int stop = st.stop;
    bool rep_valid = st.result_report_valid != 0;
    if (cancelled || timed_out) {
      stop = cancelled ? CCLP_CU_STOP_CANCELLED : CCLP_CU_STOP_TIME_LIMIT;
      view = cclp_cu::kViewCurEff;
      rep_valid = st.checked != 0;
      if (rep_valid) std::memcpy(st.result_report, st.R ? st.avg : st.cur, sizeof(st.result_report));
    }
    S.assemble_view(view, st, x_out, y_out, z_out, sums);
    double rep[cclp_cu::kRepN];
    cclp_cu::host_make_report(sums, sums + cclp_cu::kRowParts, C0.b_norm, C0.c_norm, rep);
    res->stop = stop;
    res->iterations = st.iteration;
    res->restarts = st.restarts;
    res->error_iteration = stop == CCLP_CU_STOP_NUMERICAL_ERROR ? st.error_iteration : -1;
    copy_report(rep_valid ? st.result_report : rep, &res->report);
    res->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
    res->norm_estimate = C0.norm_est;
    res->omega = C0.omega;
    res->tau = C0.tau;
    res->sigma = C0.sigma;
    res->setup_seconds = setup_s;
    res->loop_seconds = loop_ms * 1e-3;
    res->kernel_launches = S.launches;
    S.begun = false;
  });
}

}  // extern "C"
