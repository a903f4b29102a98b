// Shared device-side definitions for the cclp_cu PDHG engine (sm_100a).
//
// Layout in HBM (per context):
//   CSR(A)      rowptr i32[m+1], colind i32[nnz], val f64[nnz]   (row kernel)
//   CSR(A^T)    colptr i32[n+1], rowind i32[nnz], val f64[nnz]   (column kernel;
//               this is the reference's own CSC, types.hpp:31)
//   unscaled c,l,u f64[n], b f64[m] and the Ruiz factors s f64[n], r f64[m];
//   scaled copies of both value arrays. Scaled c/l/u/b are recomputed on the
//   fly with the reference's exact operations (apply_scaling,
//   scaling.cpp:29-44), so they cost no memory and match bit for bit.
//   State (ping-pong by iteration parity): y, ax, y_sum, ax_sum (m);
//   aty, x_sum, aty_sum (n); next-x candidates in 3 rotating slots x 2
//   (continue / restart) (n).
#pragma once

#include <cstdint>

namespace cclp_cu {

constexpr int kBlock = 256;       // setup / view kernels
constexpr int kSpmvBlock = 1024;  // lean SpMV kernels: fat blocks on contiguous row ranges
constexpr int kEpiBlock = 512;    // streaming epilogues (one wave, few partials)
constexpr int kKernelsPerIteration = 4;
constexpr int kRowParts = 8;   // per-block partials of the row kernel
constexpr int kColParts = 14;  // per-block partials of the column kernel

// Views a result or snapshot can be taken from.
enum View : int { kViewCur = 0, kViewAvg = 1, kViewCurEff = 2 };

// Report field order = ResidualReport (kkt.hpp:43-58).
enum Rep : int {
  kRpNorm2 = 0, kRdNorm2, kRpInf, kRdInf, kPobj, kDobj, kGap, kRelP, kRelD, kRelGap, kMaxResid,
  kCompl, kRepN
};

// Ladder snapshots are extracted by the iteration kernels themselves into one
// of kSnapSlots device slots (the step after the check that fired reads the
// checked state anyway) and copied out by the host on a side stream while
// the loop runs on; only when every slot still waits for the host does the
// loop fall back to halting.
constexpr int kSnapSlots = 2;
struct SnapMeta {
  long long iteration;
  double maxresid;
  int thr_idx, use_avg;
};

struct LogEntry {
  long long iteration;
  double rel_primal, rel_dual, rel_gap, elapsed;
};

// Device-resident control block: every decision of the reference loop body
// (pdhg.cpp:300-377) is taken here by the finalize tail of the column kernel.
struct Ctrl {
  long long iteration;   // t: number of steps taken (state index)
  long long window;      // iterates in the running sums of state t
  long long restarts;
  long long error_iteration;
  long long snap_iteration;
  long long log_count;
  int R;                 // restart decided at check(t), applied by step t
  int R_prev;            // restart applied by step t-1 (selects x_t)
  int stop;              // -1 while running, else PdhgStopReason
  int halt;              // a ladder snapshot is waiting for the host
  int next_threshold;
  int have_best;
  int snap_pending, snap_use_avg, snap_thr_idx;
  int result_view;       // View of the returned iterate
  int result_report_valid;
  int use_avg;
  int checked;           // cur/avg reports belong to the current iteration
  int snaps_done;        // snapshots extracted into slots (slot = index % kSnapSlots)
  int snap_rprev;        // x of the pending snapshot's state: xc[it % 3][snap_rprev]
  int pad2;
  double last_restart_resid;
  double snap_maxresid;
  double snap_inv;       // 1/window of the pending snapshot's state (average view)
  SnapMeta snap_meta[kSnapSlots];
  // timing probes (globaltimer ns) of the last step: column-kernel start
  // (block 0), finalize start and end
  unsigned long long t_cols_start, t_fin_start, t_fin_end;
  double cur[kRepN], avg[kRepN], best[kRepN], result_report[kRepN];
};

}  // namespace cclp_cu
