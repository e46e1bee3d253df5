// Shared declarations of libhsdla_b200 (sm_100a): context, error plumbing and the
// descriptor types of the multi-segment contraction kernel.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <map>
#include <string>
#include <mutex>
#include <set>
#include <utility>
#include <vector>

#include "../../include/hsdla_b200.h"

namespace hsdla {

// True the first time it is called for (key, current device): per-device one-time setup
// such as cudaFuncSetAttribute (function attributes are per device).
inline bool first_on_device(const void* key) {
  static std::mutex m;
  static std::set<std::pair<const void*, int>> seen;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(m);
  return seen.insert({key, dev}).second;
}

void set_error(const std::string& msg);

// Complex multiply of the DMMA contractions: 3 (default) = three real products per complex
// MAC (Re = P_re Q_re + P_im Q_im, Im = (P_re - P_im)(Q_re + Q_im) - P_re Q_re + P_im Q_im);
// 4 = the real embedding's four.  HSDLA_CMUL=4 selects the latter (A/B measurements).
inline int cmul_mode() {
  static int m = -1;
  if (m < 0) {
    const char* e = getenv("HSDLA_CMUL");
    m = (e && e[0] == '4' && e[1] == 0) ? 4 : 3;
  }
  return m;
}

// Sum planes of the three-product multiply for the pipeline's generated stacks (template path):
// HSDLA_PLANES=1 writes them in the expansion pass and runs the DADD-free contraction on them.
// Off by default: measured slower on B200 (C2 contraction 2.23-2.26 vs 2.18 ms; the extra
// plane loads and L2 footprint cost more than the DADDs they save, profiles/README.md).
inline bool planes_enabled() {
  static int m = -1;
  if (m < 0) {
    const char* e = getenv("HSDLA_PLANES");
    m = (e && e[0] == '1') ? 1 : 0;
  }
  return m == 1;
}

#define HS_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t _e = (call);                                                           \
    if (_e != cudaSuccess) {                                                           \
      ::hsdla::set_error(std::string(#call) + ": " + cudaGetErrorString(_e) + " (" +   \
                         __FILE__ + ":" + std::to_string(__LINE__) + ")");             \
      return HSDLA_ERR_CUDA;                                                           \
    }                                                                                  \
  } while (0)

#define HS_CHECK_LAUNCH() HS_CUDA(cudaGetLastError())

// One K-segment of a contraction: C += P^H Q over k rows.  P and Q are column-major
// complex128 with leading dims ldP / ldQ (elements); column c of P starts at P + c*ldP.
// `sel`/`P_alt`: device-side branch selection without a host round trip — when `sel` is
// non-null and *sel != 0 (the T set's Cholesky info: not HPD, or forced general path) the
// segment reads P_alt instead of P (builder.py:284-302 per-atom HPD dispatch).
struct Seg {
  const double2* P;
  const double2* Q;
  const double2* P_alt;
  const int* sel;
  long long ldP, ldQ;
  int k;
  int pad_;
  // Optional real "sum planes" of the three-product multiply, laid out like P / Q (element
  // row + col * ld, in doubles): Pd = Re P - Im P, Qs = Re Q + Im Q.  When every segment of a
  // launch has them the kernel stages them instead of forming the sums with DADDs.
  const double* Pd;
  const double* Qs;
};

enum ProbKind : int {
  PROB_GENERAL = 0,     // C = alpha*acc (+ beta*C if accumulate), all m x n entries
  PROB_TRI_LOWER = 1,   // lower(C) (+)= acc; strict upper untouched
  PROB_TRI_MIRROR = 2,  // lower(C) (+)= acc, then upper = conj(lower^T), diag imag = +0
};

struct Prob {
  double2* C;
  long long ldC;
  int m, n;  // output rows / cols (tri: m == n)
  int kind;
  int seg0, nseg;
  int accumulate;
  int tiles_m, tiles_n;  // tile grid (tri: tiles_m == tiles_n)
  int ntiles;            // tiles of this problem
  int nchunks;           // K chunks per tile (all tiles of a problem share the segments)
  long long it_base;     // first stream-K iteration (tile-chunk) of this problem
  int col_tile_lo, col_tile_hi;  // tri only: restrict to tile columns [lo, hi) (sharding)
  double2 alpha, beta;
  // TRI_MIRROR only, or nullptr: per group of panel_group lower tile columns, the count of its
  // finished tiles (the group of columns [p0, p1) is complete at the sum of tiles_m - tn); a
  // copy stream waits on each group's counter (one stream wait per copy) and copies the group's
  // finished tiles and mirrors to the host while the kernel runs.
  int* panel_done;
  int panel_group;  // tile columns per counter (panel_done[tn / panel_group]); 0 = 1
};

constexpr int kTile = 64;  // complex outputs per CTA tile edge

// Tile count of a problem (host side, also used for sharding).
int prob_tile_count(const Prob& p);

struct Arena;  // descriptor staging (defined in capi.cu)

}  // namespace hsdla

struct hsdla_ctx {
  // Key of the T preparation whose results sit in a build workspace (hsdla_build_args.reuse_t).
  struct TKey {
    const void* ws = nullptr;
    long long forms_off = -1, info_off = -1;  // workspace offsets (depend on n_basis, ld)
    const void *taa = nullptr, *tab = nullptr, *tbb = nullptr;
    long long t_ld = 0;
    int force = -1, joint = -1;
    std::vector<int> tdim, tdense;
    std::vector<double> u2;
  } tkey;
  // Joint-factor info per T set of the T preparation in tkey (0 = H takes the joint form).
  std::vector<int> joint_info;
  std::vector<int> joint_split;  // per T set: 1 = the joint factor uses the dense/diagonal split
  double joint_sigma = 0.0;      // common shift of the joint factors in tkey's workspace
  bool joint_pending = false;  // joint_info not read back yet (fresh T preparation in flight)
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;   // joint T factor, overlapping A/B generation
  cudaStream_t side2 = nullptr;  // T_AA forms + factor, beside the joint factor
  cudaStream_t copy = nullptr;  // D2H of finished H / S, overlapped with later compute
  cudaEvent_t copy_go = nullptr;
  cudaStream_t upload = nullptr;  // descriptor H2D, ahead of the compute stream
  cudaStream_t h2d = nullptr;     // host-sourced A / B uploads (hsdla_build_args.A_host)
  cudaEvent_t a_up = nullptr, b_up = nullptr;
  cudaEvent_t upload_done = nullptr;
  // Two in-flight builds (k-point pipelining): per-build events, flag and read-back area.
  struct BuildSlot {
    cudaEvent_t ev[8] = {};
    cudaEvent_t s_copied = nullptr, h_copied = nullptr, done = nullptr;
    int* flag_dev = nullptr;
    int* panel_cnt = nullptr;      // 2 x panel_cap counters (S, H) for streamed copies
    int panel_cap = 0;
    int* host_area = nullptr;      // mapped pinned (host view)
    int* host_area_dev = nullptr;  // device view of host_area
    int n_atoms = 0, n_tsets = 0;
    bool force = false, copies = false, pending = false;
    unsigned long long ticket = 0;
    std::vector<int> t_index;
    std::vector<int> joint;  // per T set: 1 = this build's H used the joint factor (2 = split)
    double sigma = 0.0;      // this build's joint shift (H -= sigma S after the contraction)
    int types = 0;           // template path: atom types (0 = per-atom path)
    int merged = 0;          // S and H in one contraction launch
    const void* h_dev = nullptr;  // this build's device H / S (copy hazards of the next build)
    const void* s_dev = nullptr;
    std::vector<cudaEvent_t> group_ev;  // debug (HSDLA_TIMELINE): end of each streamed group copy
  } slots[2];
  unsigned long long seq = 0;
  // Outcomes of builds completed before their ticket was finished (more than two in flight).
  struct Outcome {
    int rc = 0, nonfinite = 0;
    std::vector<int> info, hpd, joint;
    double sigma = 0.0;
    int types = 0, merged = 0;
    float ms[7] = {};
  };
  std::map<unsigned long long, Outcome> stash;
  cudaEvent_t fork = nullptr, join = nullptr, join2 = nullptr;
  cudaEvent_t epoch = nullptr;  // recorded at creation (debug timelines)
  int device = 0;
  int num_sms = 148;
  // stream-K fix-up workspace: per-CTA partial tiles and ready flags
  double* partials = nullptr;
  int* ready = nullptr;
  int partial_slots = 0;
  // Device descriptor arena and its pinned host staging twin.
  char* desc_dev = nullptr;
  char* stage_host = nullptr;
  size_t desc_cap = 0;
  size_t desc_off = 0;
  cudaEvent_t stage_done = nullptr;
  bool stage_pending = false;
  // Small device scratch: tile counters and flags; pinned mirrors for read-back.
  int* scratch_dev = nullptr;   // [64..95] operator flags, [96..97] build-slot flags
  int* scratch_host = nullptr;  // mapped pinned: [0..127] operator read-back, [128..327] build slots
  int* scratch_host_dev = nullptr;
};

namespace hsdla {
// Contraction launcher: uploads problems/segments through the ctx arena and launches
// the persistent DMMA kernel.  `counter_slot` picks the tile counter to use.
int launch_contract(hsdla_ctx* ctx, const std::vector<Prob>& probs,
                    const std::vector<Seg>& segs, int* flag_dev);
// TMA + mbarrier variant (contract_tma.cu); `probs` already tiled (it_base, nchunks set).
void plan_dp_waves(const std::vector<Prob>& probs, long long total, int grid, int* waves,
                   int* nch, long long* dp_it);
int launch_contract_tma(hsdla_ctx* ctx, const std::vector<Prob>& probs, long long total,
                        const std::vector<Seg>& segs, int* flag_dev);
// True when the TMA path has a better tile shape for these problems (96-row T applications).
bool tma_wants(const std::vector<Prob>& probs);
// Arena helpers.
int arena_begin(hsdla_ctx* ctx, size_t bytes);
void* arena_push(hsdla_ctx* ctx, const void* src, size_t bytes, void** host_ptr);
int arena_flush(hsdla_ctx* ctx);

// Small kernels (small.cu)
enum OperandPrep : int { PREP_COPY = 0, PREP_CONJ_TRANS = 1, PREP_HERM_FULL = 2,
                         PREP_TRIL = 3, PREP_TRIL_CONJ_TRANS = 4 };
int launch_prep(hsdla_ctx* ctx, int op, int rows, int cols, const double2* in, long long ldin,
                double2* out, long long ldout, double scale);
int launch_potrf_batched(hsdla_ctx* ctx, int n, int batch, const double2* T, long long ldt,
                         long long stride_t, double2* F, long long ldf, long long stride_f,
                         int* info_dev);
int launch_tprep(hsdla_ctx* ctx, cudaStream_t stream, int n_tsets, const int* tdim_dev, int mp,
                 const double2* taa, const double2* tab, const double2* tbb, long long t_ld,
                 double2* forms, int do_chol, int* info_dev);
// Joint factor L of [[T_AA, T_AB], [T_AB^H, T_BB]] per T set (ld 2*mp, in `joint`), with the
// dense-block / diagonal-tail split where tdense[t] < tdim[t] and T has that structure; info per
// set into info_dev and, if non-null, the mapped host views (info, split flag).
int launch_tjoint(cudaStream_t stream, int n_tsets, const int* tdim_dev, const int* tdense_dev,
                  int mp, const double2* taa, const double2* tab, const double2* tbb,
                  long long t_ld, double2* joint, int* info_dev, int* info_host_dev,
                  int* split_host_dev, const double* u2_dev, double sigma_fixed,
                  double* sigma_host_dev);
// C -= sigma S (full matrices): the shifted joint form's correction.
int launch_axpy_shift(hsdla_ctx* ctx, int n, double sigma, const double2* S, long long lds,
                      double2* C, long long ldc);
// Tail rows [d, m) of split joint T sets: atoms_dev[e] = (row offset, d, m, T set).
int launch_ttail(hsdla_ctx* ctx, const int4* atoms_dev, int n_atoms, int max_tail, int n_basis,
                 const double2* A, const double2* B, long long ld, double2* XY, double2* Z,
                 const double2* joint, long long lj);
int ab_generate(hsdla_ctx* ctx, const hsdla_ab_args* args);
// Per-type templates (abgen.cu): representative atoms reps[i] at the origin into rows toff[i]
// of At / Bt (ld ldt).
int ab_generate_templates(hsdla_ctx* ctx, const hsdla_ab_args* args, const std::vector<int>& reps,
                          const std::vector<long long>& toff, double2* At, double2* Bt,
                          long long ldt);
// Template expansion (expand.cu): for every atom block e (atoms_dev[e] = (atom, template row,
// height, -), first stacked row off_dev[e]) and column t, with phase z = e^{i K_t.x_atom}:
//   O0 = T0 z,  O1 = (scale1 ? ||udot||_row : 1) T1 z,  O2 = T1 z (if non-null),
// and the three-product sum planes Od = Re - Im, Os = Re + Im of O0 and O1 (if non-null).
struct ExpandOut {
  double2* O0;
  double* O0d;
  double* O0s;
  double2* O1;
  double* O1d;
  double* O1s;
  double2* O2;
  int scale1;
};
int launch_expand(hsdla_ctx* ctx, int n_basis, const double* kv, const double* pos,
                  const double* radial, int radial_stride, const int4* atoms_dev,
                  const long long* off_dev, int n_blocks, const double2* T0, const double2* T1,
                  long long ldt, const ExpandOut& o, long long ld);
int preload_expand();
// kind 0: o1/o2 = j_l(x), j'_l(x), (l_max+1) x n row-major; kind 1: o1 = Y_lm (complex,
// (l_max+1)^2 x n row-major) at unit directions in (n x 3).
int special_functions(hsdla_ctx* ctx, int kind, int l_max, int n, const double* in, double* o1,
                      double* o2);
int match_factors(hsdla_ctx* ctx, const hsdla_ab_args* s, const int64_t* f_row, double* fa,
                  double* fb, int64_t ldf);
int reduced_s_aa(hsdla_ctx* ctx, const hsdla_reduced_args* r);
int phase_matrix(hsdla_ctx* ctx, int n, int n_atoms, const double* kv, const double* pos,
                 double2* E, long long lde);
int hadamard_lower(hsdla_ctx* ctx, int n, const double2* W, long long ldw, const double2* G,
                   long long ldg, double2* C, long long ldc, int accumulate);
int launch_mirror(hsdla_ctx* ctx, int n, double2* C, long long ldc, int* flag_dev);
int launch_scale_rows(hsdla_ctx* ctx, int m, int n, const double* d, double2* B, long long ldb);
int launch_zero_rows(hsdla_ctx* ctx, double2* base, long long ld, int row0, int rows, int cols);
int launch_finite_check(hsdla_ctx* ctx, int m, int n, const double2* A, long long lda, int* flag);
// Load every kernel a build may launch and set its shared-memory limit, at context creation:
// with lazy module loading a first launch inside a build could load (and allocate for) the
// module while the copy stream waits on that build's own kernels (streamed copies).
int preload_contract();
int preload_contract_tma();
int preload_abgen();
int preload_small();
int preload_gaunt();
// Gaunt tensor over a quadrature grid (Y: n_y x npts rows of ld ldy) and the Gaunt-sum T block
// (gaunt.cu).
int gaunt_tensor(hsdla_ctx* ctx, int n_row, int n_pot, int npts, int ldy, const double2* Y,
                 const double* w, double2* G);
int gaunt_sum(hsdla_ctx* ctx, int n_full, int n_dense, int n_l, int n_pot, const double2* c,
              const double2* G, const double* diag, double unit, double2* out);
// Copy the non-finite flag and the Cholesky infos into mapped host memory (out[0] = flag,
// out[1..n] = info) with plain stores, keeping the D2H copy engine free for H / S.
int launch_publish(hsdla_ctx* ctx, const int* flag, const int* info, int n, int* out_mapped);
}  // namespace hsdla
