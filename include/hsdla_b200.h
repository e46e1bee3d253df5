/*
 * hsdla_b200.h — C ABI of the B200-native (sm_100a) muffin-tin H/S setup path.
 *
 * Drop-in boundary for the reference package `hsdla` (arXiv 1602.06589, HSDLA):
 * every entry point below replaces one reference interface, cited as
 * file:line under /root/reference/pkg/src/hsdla/.  All matrices are complex128
 * (`hsdla_c64`, layout-identical to numpy complex128 / C99 double _Complex),
 * column-major with an explicit leading dimension counted in elements, exactly
 * the `ComplexDense` convention (matrix.py:21-50).  Matrix pointers are DEVICE
 * pointers unless marked HOST.  Work is enqueued on the context's CUDA stream;
 * calls return after enqueueing unless documented otherwise.
 *
 * Status convention (mirrors LAPACK, kernels.py:266-272):
 *   0                      success
 *   < 0 and > -1000        -(1-based index of the invalid argument)
 *   HSDLA_ERR_*            library / CUDA failures (message: hsdla_last_error())
 * Cholesky returns its pivot through an explicit `info` output instead.
 */
#ifndef HSDLA_B200_H
#define HSDLA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  double re, im;
} hsdla_c64;

typedef struct hsdla_ctx hsdla_ctx;

#define HSDLA_OK 0
#define HSDLA_ERR_CUDA -1000        /* a CUDA call failed */
#define HSDLA_ERR_UNSUPPORTED -1001 /* e.g. l_sph above the compiled maximum */
#define HSDLA_ERR_NAN_INPUT -1002   /* NaN in the lower triangle of a Cholesky input (kernels.py:127-129) */
#define HSDLA_ERR_NONFINITE -1003   /* non-finite value in a mirrored output (matrix.py:224-225) */
#define HSDLA_ERR_ALLOC -1004

#define HSDLA_MAX_LSPH 14 /* compiled template range of the A/B generator */

/* ---- library / context ------------------------------------------------- */
int hsdla_version(void);
/* Real DMMA products per complex multiply-add in the contractions: 3 (default: Re = P_re Q_re +
 * P_im Q_im, Im = (P_re - P_im)(Q_re + Q_im) - P_re Q_re + P_im Q_im) or 4 (HSDLA_CMUL=4).
 * The ledger (builder.py:336-370) counts 8 flops per complex MAC either way. */
int hsdla_complex_mul_products(void);
const char* hsdla_last_error(void);
/* Context = stream + descriptor arena + pinned staging; `stream` is a cudaStream_t (NULL = legacy). */
int hsdla_ctx_create(hsdla_ctx** out, void* stream);
int hsdla_ctx_destroy(hsdla_ctx* ctx);
int hsdla_ctx_set_stream(hsdla_ctx* ctx, void* stream);
int hsdla_ctx_synchronize(hsdla_ctx* ctx);
/* Owner rank of 64-wide column panel `panel` when the H/S lower triangle is sharded over
 * n_shards GPUs: panels j and n_panels-1-j form one balanced pair. */
int hsdla_panel_owner(int n_panels, int n_shards, int panel);

/* ---- KernelBackend operator contract (kernels.py:46-151) ----------------- */

/* lower(C) += A^H A, A is k x n (ld lda), C is n x n; strict upper of C never read or written.
 * Replaces KernelBackend.hermitian_rank_k_update (kernels.py:56-63, zherk at :242-244). */
int hsdla_herk_lower(hsdla_ctx* ctx, int n, int k, const hsdla_c64* A, int64_t lda,
                     hsdla_c64* C, int64_t ldc);

/* lower(C) += X^H B + B^H X, X and B are k x n.
 * Replaces KernelBackend.hermitian_rank_2k_update (kernels.py:66-74, zher2k at :246-248). */
int hsdla_her2k_lower(hsdla_ctx* ctx, int n, int k, const hsdla_c64* X, int64_t ldx,
                      const hsdla_c64* B, int64_t ldb, hsdla_c64* C, int64_t ldc);

/* C = alpha * op(A) * B + beta * C, op(A) = A^H (conj_a != 0, A is k x m) or A (A is m x k).
 * C is m x n; with beta == 0 C is not read.  `workspace` must hold m*k elements when conj_a == 0.
 * Replaces KernelBackend.general_product (kernels.py:77-89, zgemm at :250-253). */
int hsdla_gemm(hsdla_ctx* ctx, int conj_a, int m, int n, int k, hsdla_c64 alpha,
               const hsdla_c64* A, int64_t lda, const hsdla_c64* B, int64_t ldb,
               hsdla_c64 beta, hsdla_c64* C, int64_t ldc, hsdla_c64* workspace);

/* X = alpha * T * A (+ X if accumulate), T is m x m Hermitian read from its lower
 * triangle with the diagonal's imaginary part ignored; A, X are m x n.
 * `workspace` holds m*m elements.  Replaces KernelBackend.hermitian_product
 * (kernels.py:92-104, zhemm at :255-258). */
int hsdla_hemm_lower(hsdla_ctx* ctx, int m, int n, hsdla_c64 alpha, const hsdla_c64* T,
                     int64_t ldt, const hsdla_c64* A, int64_t lda, int accumulate,
                     hsdla_c64* X, int64_t ldx, hsdla_c64* workspace);

/* Y = op(L) * A with L lower triangular m x m (strict upper ignored), op = ^H if conj_l.
 * `workspace` holds m*m elements.  Replaces KernelBackend.triangular_product
 * (kernels.py:107-116, ztrmm at :260-264). */
int hsdla_trmm_lower(hsdla_ctx* ctx, int conj_l, int m, int n, const hsdla_c64* L, int64_t ldl,
                     const hsdla_c64* A, int64_t lda, hsdla_c64* Y, int64_t ldy,
                     hsdla_c64* workspace);

/* Batched Cholesky of tril(T_b) into F_b (lower factor, zero strict upper), b < batch.
 * info_host[b] (HOST, filled before return; this call synchronises the stream):
 * 0 = HPD, j+1 = first non-positive/non-finite pivot j (zpotrf info), -1 = NaN in tril(T).
 * T_b is never modified.  Replaces KernelBackend.cholesky_factor (kernels.py:119-132). */
int hsdla_potrf_lower_batched(hsdla_ctx* ctx, int n, int batch, const hsdla_c64* T,
                              int64_t ldt, int64_t stride_t, hsdla_c64* F, int64_t ldf,
                              int64_t stride_f, int32_t* info_host);

/* ---- storage helpers (matrix.py) ----------------------------------------- */

/* Upper <- conj(lower^T), diag imag <- +0; *nonfinite_host (HOST) = 1 if any entry is not
 * finite (synchronises).  Replaces HermitianAccumulator.mirror_to_full (matrix.py:216-226). */
int hsdla_mirror_lower(hsdla_ctx* ctx, int n, hsdla_c64* C, int64_t ldc, int32_t* nonfinite_host);

/* *nonfinite_host = 1 if any element of the m x n window A (DEVICE, column-major, lda)
 * is NaN or Inf, else 0; synchronises the stream.  The guard of write_hsm1
 * (matrix.py:242-246), run in HBM before an HSM1 file is streamed out. */
int hsdla_check_finite(hsdla_ctx* ctx, int m, int n, const hsdla_c64* A, int64_t lda,
                       int32_t* nonfinite_host);

/* B[i, :] *= d[i] (d real, DEVICE).  Replaces scale_rows (matrix.py:229-239). */
int hsdla_scale_rows(hsdla_ctx* ctx, int m, int n, const double* d, hsdla_c64* B, int64_t ldb);

/* ---- matching coefficients (flapw.py:201-233 compute_AB) ----------------- */
typedef struct {
  int32_t n_atoms;
  int32_t n_basis;            /* N_G */
  const double* k_vectors;    /* DEVICE n_basis x 3, row-major (SystemSpec.k_vectors) */
  const double* positions;    /* DEVICE n_atoms x 3 */
  const double* rotations;    /* DEVICE n_atoms x 9, row-major 3x3 */
  const double* mt_radius;    /* DEVICE n_atoms */
  const double* radial;       /* DEVICE n_atoms x radial_stride x 5: per l {u, u', udot, udot', ||udot||} */
  int32_t radial_stride;      /* >= max l_sph + 1 */
  const int32_t* l_sph;       /* HOST n_atoms, each <= HSDLA_MAX_LSPH */
  const int64_t* row_offset;  /* HOST n_atoms: first row of atom a's (l_sph+1)^2 block */
  double omega;               /* cell volume */
  hsdla_c64* A;               /* DEVICE out, column-major, leading dim ld */
  hsdla_c64* B;               /* DEVICE out */
  hsdla_c64* B_scaled;        /* DEVICE out or NULL: ||udot|| * B (the build_S side effect, builder.py:207) */
  int64_t ld;
  double* udot_norms;         /* DEVICE out or NULL: per-row ||udot|| (flapw.py:232) */
} hsdla_ab_args;
int hsdla_ab_generate(hsdla_ctx* ctx, const hsdla_ab_args* args);

/* Spherical Bessel j_0..j_lmax and j'_0..j'_lmax at n arguments x >= 0 (DEVICE), row l of
 * j / jp = order l ((l_max+1) x n row-major): special.py:104-131 spherical_bessel_all on the
 * A/B generator's device code (same regimes and rounding).  l_max <= HSDLA_MAX_LSPH. */
int hsdla_spherical_bessel(hsdla_ctx* ctx, int l_max, int n, const double* x, double* j,
                           double* jp);
/* Y_lm, rows l^2+l+m, at n unit directions (DEVICE n x 3): special.py:139-179
 * spherical_harmonics_all on the generator's Legendre recurrence; Y is (l_max+1)^2 x n
 * row-major complex. */
int hsdla_spherical_harmonics(hsdla_ctx* ctx, int l_max, int n, const double* directions,
                              hsdla_c64* Y);

/* Radial match factors f_A, f_B (flapw.py:179-198 match_factors) on the device: row
 * f_row[a] + l (l <= l_sph[a]) of f_a / f_b (DEVICE, row-major, row stride ld_f >= n_basis)
 * receives the factors of atom a for every K-vector.  Uses n_atoms, n_basis, k_vectors,
 * mt_radius, radial, radial_stride and l_sph of `spec`; f_b may be NULL. */
int hsdla_match_factors(hsdla_ctx* ctx, const hsdla_ab_args* spec, const int64_t* f_row,
                        double* f_a, double* f_b, int64_t ld_f);

/* ---- Legendre-reduced A-side overlap (oracle.py:159-216 reduced_S_AA) ----- */
typedef struct {
  int32_t n_atoms;
  int32_t n_basis;
  const double* k_vectors;    /* DEVICE n_basis x 3 */
  const double* positions;    /* DEVICE n_atoms x 3 */
  const double* f;            /* DEVICE match factors, row f_row[a] + l, row stride ld_f */
  int64_t ld_f;
  const int64_t* f_row;       /* HOST n_atoms */
  const int32_t* l_top;       /* HOST n_atoms: rows l = 0..l_top[a] of atom a (<= HSDLA_MAX_LSPH) */
  const double* coef;         /* DEVICE per f row: (2l+1) / (4 pi) / W_l^2 */
  double scale;               /* (4 pi)^2 / Omega */
  hsdla_c64* S;               /* DEVICE out n_basis x n_basis, column-major, full (exactly Hermitian) */
  int64_t lds;
} hsdla_reduced_args;
int hsdla_reduced_s_aa(hsdla_ctx* ctx, const hsdla_reduced_args* args);

/* ---- per-type phase factorisation ---------------
 * When the atoms of a type share rotation, radial data, muffin-tin radius and T, every
 * coefficient block is its type's template times a column phase: A_a = A^_t diag(e_a), so
 * S and H are sums over types of (phase Gram) o (template Gram). */
/* E[a + t*lde] = exp(i K_t . x_a) (DEVICE k_vectors n_basis x 3, positions n_atoms x 3). */
int hsdla_phase_matrix(hsdla_ctx* ctx, int n_basis, int n_atoms, const double* k_vectors,
                       const double* positions, hsdla_c64* E, int64_t lde);
/* lower(C) (+)= W o G elementwise on i >= j (all DEVICE, column-major). */
int hsdla_hadamard_lower(hsdla_ctx* ctx, int n, const hsdla_c64* W, int64_t ldw,
                         const hsdla_c64* G, int64_t ldg, hsdla_c64* C, int64_t ldc, int accumulate);

/* ---- input side: Gaunt coefficients and T assembly ---- */
/* G[(i * n_row + j) * n_pot + k] = sum_p w[p] conj(Y[i][p]) Y[j][p] Y[k][p] (special.py:189-244):
 * Y DEVICE complex rows of ld ldy (row L = l^2 + l + m, e.g. hsdla_spherical_harmonics on the
 * quadrature directions), w DEVICE npts weights, G DEVICE out; n_row, n_pot <= rows of Y. */
int hsdla_gaunt_tensor(hsdla_ctx* ctx, int n_row, int n_pot, int npts, int64_t ldy,
                       const hsdla_c64* Y, const double* w, hsdla_c64* G);
/* One T block of assemble_T (flapw.py:306-363), DEVICE, column-major n_full x n_full:
 * out[p, q] = sum_k c[l(p), l(q), k] G[p, q, k] on the leading n_dense = n_l^2 block
 * (c: n_l x n_l x n_pot, G: n_dense x n_dense x n_pot, numpy C order), plus diag[l(p)] (may be
 * NULL) and `unit` on the diagonal. */
int hsdla_gaunt_sum(hsdla_ctx* ctx, int n_full, int n_l, int n_pot, const hsdla_c64* c,
                    const hsdla_c64* G, const double* diag, double unit, hsdla_c64* out);

/* ---- the composed build (builder.py:403-474 build_all) ------------------- */
typedef struct {
  int32_t n_atoms;
  int32_t n_basis;
  const int32_t* heights;     /* HOST n_atoms: coefficient block heights */
  const int64_t* row_offset;  /* HOST n_atoms: first row of each block in A/B */
  const int32_t* t_index;     /* HOST n_atoms: which T set each atom uses */
  int32_t n_tsets;
  const int32_t* t_dim;       /* HOST n_tsets: m of each T set (m <= height of its atoms) */
  const hsdla_c64* t_aa;      /* DEVICE n_tsets x (t_ld x t_ld), column-major, lower triangle read */
  const hsdla_c64* t_ab;      /* DEVICE, full */
  const hsdla_c64* t_bb;      /* DEVICE, lower triangle read */
  int64_t t_ld;
  const hsdla_c64* A;         /* DEVICE stacked coefficients, column-major R x n_basis, ld */
  const hsdla_c64* B;
  const hsdla_c64* B_scaled;  /* DEVICE or NULL: if NULL the build scales B by udot_norms itself */
  const double* udot_norms;   /* DEVICE R (used when B_scaled == NULL) */
  int64_t ld;
  int32_t force_general_path; /* BuildConfig.force_general_path (builder.py:284) */
  hsdla_c64* H;               /* DEVICE out n_basis x n_basis, full Hermitian after the call */
  hsdla_c64* S;
  int64_t ldh;
  void* workspace;            /* DEVICE scratch of hsdla_build_workspace_size() bytes */
  size_t workspace_bytes;
  /* column-panel sharding for multi-GPU tile partitioning; n_shards <= 1 = all.
   * With sharding only the lower tiles of owned 64-wide column panels are written, unmirrored. */
  int32_t shard_rank, n_shards;
  /* Optional HOST (pinned) destinations: when non-NULL the full H / S (ld ldh_host) are
   * copied back on a copy stream, overlapped with compute: S during the H phase; H during
   * the next k-point (pipelined builds) or, for the synchronous calls, panel by panel during
   * its own contraction (cuStreamWaitValue32 on per-panel tile counters; set
   * HSDLA_STREAM_COPIES=0 to copy H whole after its kernel).  Not with sharding. */
  hsdla_c64* H_host;
  hsdla_c64* S_host;
  int64_t ldh_host;
  /* With sharding: 1 = write the owned tiles together with their conjugate mirror, so H / S
   * must be full n_basis x n_basis matrices shared by all shards — e.g. the consumer rank's
   * buffers mapped into every rank through NVLink peer memory: the contraction epilogue then
   * is the gather (no separate collective, no mirror pass).  0 = lower tiles only. */
  int32_t shard_mirror;
  /* 1 = the T sets (t_aa/t_ab/t_bb contents) are unchanged since the previous build on this
   * context: the T forms and Cholesky factors still in `workspace` are reused and the T
   * preparation is skipped (T does not depend on the k-point).  Honoured only when the
   * workspace, T pointers, t_ld, t_dim and force_general_path also match that build. */
  int32_t reuse_t;
  /* H copy scheduling for host destinations: 0 = default (synchronous calls stream H panel
   * by panel during its contraction, pipelined calls copy it whole under the next k-point),
   * 1 = stream (e.g. the last k-point of a batch, which has no successor to hide under),
   * -1 = copy whole after the contraction. */
  int32_t stream_h_copy;
  /* H form.  0 = default: per T set, factor the 2m x 2m Hermitian
   * [[T_AA, T_AB], [T_AB^H, T_BB]] = L L^H once (with the T preparation, cached with it); where
   * it is positive definite the atom's whole H contribution is W^H W with W = L^H [A_a; B_a],
   * so H is one stacked rank-2R update (K = 2R) instead of the reference's ZHER2K + ZHERK
   * (K = 3R), equal to rounding.  Sets whose matrix is not HPD, force_general_path, and
   * 1 here (or HSDLA_JOINT=0) use the reference forms Z = T_AB^H A + 1/2 T_BB B and
   * Y = C^H A / X = T_AA A.  The first build after the T sets change waits (host) for the
   * T preparation to learn which form applies. */
  int32_t h_reference_form;
  /* Optional HOST (pinned) sources of A and B (column-major, ld ld_ab_host >= rows): the build
   * uploads them into the DEVICE buffers A / B itself (which it then writes), A first and B on
   * a copy stream while the A-part of S (A^H A) already runs; S is then accumulated in two
   * launches.  B_scaled must be NULL; not with sharding. */
  const hsdla_c64* A_host;
  const hsdla_c64* B_host;
  int64_t ld_ab_host;
  /* HOST n_tsets or NULL: dense-block size d <= t_dim of each T set ((l_nonsph+1)^2).  Where
   * d < t_dim and T is zero outside the leading d x d blocks except its diagonals (as the
   * reference's assemble_T builds it, flapw.py:306-363), the joint H form factors the 2d x 2d
   * dense part and one 2x2 block per tail row, and the T applications run with K = d plus an
   * elementwise tail; otherwise T is treated as dense. */
  const int32_t* t_dense;
  /* HOST n_tsets x (max t_dim) or NULL: ||udot||^2 of each row of the set's atoms (a row < 0 =
   * the set may not be shifted: its atoms differ in ||udot|| or have T smaller than their block).
   * With it the joint H form also covers T sets that are not HPD: every set is factored as
   * T + sigma diag(I, U^2) with one common sigma >= 0 and H = sum W^H W - sigma S, because
   * [A; B]^H sigma diag(I, U^2) [A; B] summed over the atoms is sigma S exactly.  Applied only
   * when every set can take that shift; otherwise non-HPD sets use the reference forms. */
  const double* t_udot2;
  /* HOST n_atoms or NULL (hsdla_setup_hs / hsdla_setup_hs_async only): atom type index in
   * [0, n_types).  The atoms of a type share rotation, muffin-tin radius, l_sph, radial data
   * and T set (exact equality; the caller groups them), so each coefficient block is a type
   * template times the column phase: A_a = A_type diag(e^{iK.x_a}) (flapw.py:216-232 with
   * the per-atom factors split off).  The build then evaluates the Bessel / Y_lm / match
   * factor recurrences once per (type, K), applies the joint T factor once per type
   * (W = L^H [A_type; B_type], builder.py:231-240 / :284-302 on the template) and writes A,
   * ||udot|| B, W1, W2 for every atom with its phase, together with the sum planes of the
   * three-product contraction, in one HBM-bound expansion pass.  Ignored (per-atom path) when
   * a type mixes T sets or heights, T is smaller than its block, or the sources are on the host. */
  const int32_t* atom_type;
  int32_t n_types;
} hsdla_build_args;

typedef struct {
  int32_t* hpd_mask;          /* HOST out n_atoms: 1 = Cholesky succeeded (HPD branch) */
  int32_t* chol_info;         /* HOST out n_tsets: potrf info per T set (-2 = not attempted) */
  int32_t nonfinite;          /* out: 1 if H or S holds a non-finite value */
  float ms_setup, ms_S, ms_H_ABBA_BB, ms_H_AA; /* out: CUDA-event phase times */
  float ms_contract_S, ms_contract_H;           /* out: the two triangular DMMA contraction launches */
  float ms_apply_Z, ms_apply_XY;                /* out: the batched T-application launches */
  float ms_total;                               /* out: first event to last kernel / copy */
  int32_t* joint_info;        /* HOST out n_tsets or NULL: 1 = H used the joint T factor for this set,
                                 2 = with the dense / diagonal-tail split */
  double joint_shift;         /* out: the common shift sigma of the joint form (0 = none) */
  int32_t template_types;     /* out: atom types of the template path (hsdla_build_args.atom_type),
                                 0 = per-atom generation / T applications */
  float ms_templates;         /* out: template path: the per-type generator's share of ms_setup
                                 (the rest of ms_setup is the HBM-bound expansion) */
  int32_t merged_sh;          /* out: 1 = S and H were one contraction launch (ms_contract_H is
                                 both, ms_contract_S ~ 0): a reused, all-joint T preparation */
} hsdla_build_result;

size_t hsdla_build_workspace_size(const hsdla_build_args* args);
/* 1 if `p` points into page-locked (pinned / registered) host memory, else 0. */
int hsdla_is_pinned(const void* p);
/* Enqueues the whole build (the T_AA HPD branch of the reference forms is selected on the
 * device from the Cholesky info; the H form per T set needs the joint factor's info on the
 * host, read once after a fresh T preparation while the S contraction is already queued) and
 * synchronises once at the end (info, flags, timings).  Returns HSDLA_ERR_NAN_INPUT on a NaN in
 * tril(T_AA) and HSDLA_ERR_NONFINITE on non-finite output (outputs still written). */
int hsdla_build_hs(hsdla_ctx* ctx, const hsdla_build_args* args, hsdla_build_result* result);

/* The whole per-k-point hot path, SystemSpec -> (H, S): `hsdla_ab_generate` into
 * args->A / B / B_scaled (ab->A etc. must alias them) with the T preparation overlapped on a
 * side stream, then the build.  Replaces compute_AB (flapw.py:201) + build_all (builder.py:403)
 * as called by the reference CLI's regenerate flow (cli.py:283-292, :310-325). */
int hsdla_setup_hs(hsdla_ctx* ctx, const hsdla_ab_args* ab, const hsdla_build_args* args,
                   hsdla_build_result* result);

/* Pipelined form for k-point batches: enqueue one k-point (ab may be NULL = A/B given) and
 * return at once with a ticket; `hsdla_build_finish` waits for that k-point's compute and
 * host copies and fills `result`.  Two builds may be in flight per context; the next
 * build's contractions wait for the previous build's copies when it writes the same device
 * H / S; alternating two device H / S pairs between consecutive k-points removes those waits,
 * so the copies of k-point i overlap the whole compute of k-point i+1.  Host destinations of
 * in-flight builds must differ. */
int hsdla_setup_hs_async(hsdla_ctx* ctx, const hsdla_ab_args* ab, const hsdla_build_args* args,
                         unsigned long long* ticket);
int hsdla_build_finish(hsdla_ctx* ctx, unsigned long long ticket, hsdla_build_result* result);

#ifdef __cplusplus
}
#endif
#endif /* HSDLA_B200_H */
