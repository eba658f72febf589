// paper_2307_08507_b200/csrc/solver.h -- per-call device workspace of the
// MDOT-PNCG solver (internal; see include/mdot.h for the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "../../include/mdot.h"
#include "internal.cuh"

namespace mdot {

void set_error(const char* fmt, ...);

struct Marg {           // marginals of one plan (rows then columns, [nrows + n])
  double* lm = nullptr; // log marginals
  double* m = nullptr;  // marginals
  double* s = nullptr;  // Sinkhorn direction
  double* g = nullptr;  // gradient
  double* bp = nullptr; // base potentials A, B this plan was evaluated at (K2s screen bounds)
};

struct Comm;

struct Workspace {
  cudaStream_t st = nullptr;
  Comm* comm = nullptr;
  int64_t row0 = 0;
  int64_t n = 0, nrows = 0;
  // 2-D (row x column) sharding (mdot_solve_sharded_2d): this rank owns the
  // block rows [row0, row0 + nrows) x columns [col0, col0 + n) of an n_glob x
  // n_glob problem; `comm` joins the ranks of this column block (other row
  // blocks: column sums), `comm_row` the ranks of this row block (other
  // column blocks: row sums).  Host control loop only.
  Comm* comm_row = nullptr;
  int64_t col0 = 0, n_glob = 0;
  bool two_d() const { return comm_row != nullptr; }
  // problem
  const void* Cdev = nullptr;
  const float* Xdev = nullptr;
  const float* Ydev = nullptr;
  void* owned_C = nullptr;
  float* owned_X = nullptr;
  float* owned_Y = nullptr;
  int otf = 0, c_f64 = 0, kind_fast = 0, d = 0;
  float scale = 0.f;
  bool host_io = false;
  bool exact_mode = false;
  int jacobi = 0;                   // MDOT_PROJ_PNCG_JACOBI: finalize writes grad / diag(Hessian) as s
  double gbar = 0.0;
  // device buffers (one allocation)
  void* base = nullptr;
  double *r = nullptr, *c = nullptr, *logr = nullptr, *logc = nullptr, *rho_r = nullptr, *sig_c = nullptr;
  double *U = nullptr, *V = nullptr, *u = nullptr, *v = nullptr, *tu = nullptr, *tv = nullptr;
  double *A = nullptr, *B = nullptr, *p = nullptr, *pprev = nullptr;
  Marg mg[2];
  Marg* cur = nullptr;
  Marg* trial = nullptr;
  double *rowpart = nullptr, *colpart = nullptr, *colm = nullptr, *cols = nullptr, *lr_ex = nullptr;
  double *blockpart = nullptr, *scal_dev = nullptr, *aux = nullptr;
  float4 *rowp = nullptr, *colp = nullptr;
  float* nrm = nullptr;              // [nrows + n] Z22b squared norms of X, Y rows (dot-form K2)
  bool use_nrm = false;             // set by load_problem for the dot recipe: prep writes them into .w
  unsigned int* ticket_flag = nullptr;
  unsigned int* ticket = nullptr;
  int* flag = nullptr;
  double* scal_host = nullptr;      // mapped pinned
  double* scal_host_dev = nullptr;  // its device alias
  int chunks = 1;
  EvalArgs eval{};
  struct { double* coltot = nullptr; } tot;
  alignas(64) unsigned char tmap[128];
  bool use_tma = false;
  int tma_grid = 0;
  int pers_grid = 0;                // persistent cooperative projection (0 = off)
  int persist_ncta = 0;             // persistent grid: 0 all co-resident CTAs, > 0 at most that many (batch
                                    // workers run side by side on slices of the grid), < 0 off
  unsigned int* pers_bar = nullptr;
  // K2s screen (screen.cu): graph-slot device control on the on-the-fly
  // cost, one rank, d in {2, 4, 8, 16}.  screen_cap: prep writes the bounds;
  // screen_now: the slots evaluate with K2s (dropped for the rest of a
  // projection once a graph kept more than screen_fmax of its entries)
  bool screen_cap = false, screen_now = false;
  bool screen_skip = false;   // the last probe kept > 8 screen_fmax: the next projection stays dense
  bool md_last = false;       // this projection is the solve's last MD step (set by the MD loop)
  float screen_T = 48.f;
  double screen_fmax = 0.004;
  float* sopA = nullptr;                  // [nrows padded to 128][32] K2s A operand rows (prep)
  float* sopB = nullptr;                  // [n padded to 256][32] K2s B operand rows (prep)
  double* sop_ymax = nullptr;             // max_j |y_j|
  unsigned long long* smin = nullptr;     // [2]
  unsigned long long* scount = nullptr;   // [2] kept, screened entries (zeroed per graph)
  int64_t screen_kept = 0, screen_total = 0, screen_slots = 0, screen_timed = 0;
  double screen_ms = 0.0;
  // stats
  int64_t evals = 0, fallbacks = 0, kernel_launches = 0, launches = 0;
  double kernel_ms = 0.0;
  double stage_ms[4] = {0, 0, 0, 0};
  int64_t stage_samples = 0;
  double last_mass = 1.0;
  int time_kernels = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;

  // device-resident control
  CtrlState* ctrl = nullptr;
  int* done_host = nullptr;
  int* ran_host = nullptr;
  cudaGraphExec_t gexec = nullptr;
  cudaStream_t cap_stream = nullptr;
  int gslots = 0;
  const void* gsig[9] = {};
  cudaEvent_t gev[2 * 65] = {};
  bool gev_made = false;

  // per-iteration trace (mdot_options.trace): host records in order; device
  // control paths write into trace_dev and are appended after each projection
  int64_t trace_cap = 0;            // 0 = off
  std::vector<mdot_trace_rec> trace_host;
  mdot_trace_rec* trace_dev = nullptr;
  long long* trace_len_dev = nullptr;
  void trace_add(const mdot_trace_rec& q) {
    if ((int64_t)trace_host.size() < trace_cap) trace_host.push_back(q);
  }
  void ctrl_trace_setup(CtrlState& h, int t);   // device controller: buffer + counter for this projection
  mdot_status ctrl_trace_collect();              // append the projection's device records

  ~Workspace() {   // error paths: release() and free_owned() are idempotent
    free_owned();
    release();
  }
  bool sharded() const;
  mdot_status alloc(cudaStream_t stream, int64_t n, int64_t nrows);
  mdot_status launch_slot_body(cudaStream_t s, int slot, bool timed, bool with_ctrl = false);
  mdot_status build_graph();
  mdot_status screen_counts(unsigned long long* hc);
  void release();
  mdot_status load_problem(const mdot_problem* pb, int64_t row0);
  void free_owned();
  mdot_status l2_reset();
  // MDOT_CHECKED builds: guard bands (in doubles from base) after each sub-buffer
  static constexpr size_t kGuardDbl = 64;
  std::vector<size_t> guards;
  mdot_status check_guards();
  mdot_status setup(const mdot_options& o);
  void set_gamma(double gb);
  mdot_status prep(int mode, double alpha, double beta, const double* s_dir, const double* Ain,
                   const double* Bin);
  // skip_k1: the fp32-entry partials of this point are already in
  // rowpart / colpart (an NC2 trial being completed)
  mdot_status evaluate(Marg* out, const double* gcur, const double* pcur, double* sc, bool skip_k1 = false);
  // NC2 scalar-only line-search trials (MDOT_NC2=1, sharded host
  // loop): K1 + this rank's contributions to phi'(alpha) and the mass, summed
  // over the ranks as 4 scalars instead of the column (and row) vectors
  bool nc2 = false;
  mdot_status nc2_trial(double* q);          // q[4]: sum p R 2^rho, sum R 2^rho, sum p C 2^sig, bad
  mdot_status nc2_prc(double* prc);          // <p, (r, c)> over the whole problem
  mdot_status launch_eval();                 // the fp32-entry K1 / K2 pass of evaluate
  mdot_status gauge_center(double* X, double* Y);
  mdot_status round_and_cost(float* P_out_dev, double* cost_F, double* cost_G);
};

mdot_status build_schedule(const mdot_schedule* s, std::vector<double>& g);
mdot_status project_pncg(Workspace& w, const mdot_options& o, int t, mdot_result* res);
mdot_status project_sinkhorn(Workspace& w, const mdot_options& o, int t, mdot_result* res);
mdot_status project_device(Workspace& w, const mdot_options& o, int t, mdot_result* res);
mdot_status project_persistent(Workspace& w, const mdot_options& o, int t, mdot_result* res);

}  // namespace mdot
