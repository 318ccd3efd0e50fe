/*
 * periscat_b200 -- C ABI of the B200 (sm_100a) hot path of the periscat
 * solver (arXiv 1412.7466): the per-iteration matrix-vector product of the
 * S-preconditioned Schur-complement GMRES solve for the inclusions'
 * outgoing cylindrical-harmonic coefficients beta.
 *
 * Every entry point replaces one operation of the reference's Python solver
 * API.  The reference package specifies these modules in SPEC.md but ships
 * only the empty-grating modules, so the cited interface is
 * the SPEC signature (SPEC.md line) or the present reference function
 * (/root/reference/pkg/src/periscat/<file>:<line>).
 *
 * Conventions
 *   - complex values are interleaved (re, im) doubles == numpy complex128;
 *   - coefficient vectors are row-major [rhs][inclusion][n + p], n = -p..p
 *     (the reference's order layout, geometry.py:382-385);
 *   - "host" pointers are read during the call only; "device" pointers are
 *     CUDA device memory owned by the caller (e.g. torch tensors);
 *   - stream may be NULL (legacy default stream) or a cudaStream_t;
 *   - calls on one context must be serialised; one context per GPU/process;
 *   - every function returns PS_OK or an error code; ps_last_error() gives
 *     the message.
 */
#ifndef PERISCAT_B200_H
#define PERISCAT_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define PS_OK 0
#define PS_ERR_ARG 1         /* bad argument (ValueError in the reference)        */
#define PS_ERR_DOMAIN 2      /* overlapping disks               */
#define PS_ERR_NUMERICAL 3   /* NaN/Inf in a Krylov vector           */
#define PS_ERR_CUDA 4        /* CUDA runtime failure                               */
#define PS_ERR_STATE 5       /* call order (e.g. "not factorized", eg:267-268)     */
#define PS_ERR_UNSUPPORTED 6 /* expansion order outside the compiled range         */

typedef struct ps_ctx ps_ctx;

/* ---- lifetime ---------------------------------------------------------- */
int ps_version(void);
/* Guard-band (canary) builds only (-DPS_CANARY, tools/canary_run.sh): bytes
 * found overwritten past the end of any context allocation so far (live ones
 * are checked now, freed ones were checked at free); -1 in normal builds. */
long long ps_canary_check(void);
/* Canary builds: a deliberate overrun of a fresh allocation; returns the
 * overwritten byte count the guard band saw (1), -1 in normal builds. */
long long ps_canary_selftest(void);
int ps_create(ps_ctx** out, int device);
void ps_destroy(ps_ctx* ctx);
const char* ps_last_error(const ps_ctx* ctx);
/* largest multipole order p the kernels are compiled for */
int ps_max_order(void);

/* ---- problem data (host inputs, uploaded once per solve) --------------- */

/* Inclusion centres, multipole order p, near-field copies P, period d,
 * middle-layer wavenumber k2.  Replaces the (centers, k, p) arguments of
 * multiscat.apply_T and ProblemConfig.multipole_order /
 * near_field_copies / period / k2 (geometry.py:323-333).
 * Returns PS_ERR_DOMAIN if two enclosing centres (or a centre and a phased
 * copy) coincide.  Resets the owned-target range to [0, M). */
int ps_set_geometry(ps_ctx* ctx, int M, int p, int copies, double period, double k2,
                    const double* centers_host /* [M][2] */);

/* Disk-overlap domain check with the reference's
 * ParticleSet.min_gap semantics (geometry.py:131-144): smallest centre
 * distance over all pairs and their +-d copies minus 2 radius (+inf for
 * fewer than two inclusions), computed on the device.  PS_ERR_DOMAIN when
 * negative (overlapping enclosing disks); *min_gap (may be NULL) gets it. */
int ps_check_overlap(ps_ctx* ctx, double radius, double* min_gap);
/* Owned target inclusions [t_begin, t_end) for target sharding across ranks
 * ("apply_T parallel over target particles"). */
int ps_set_target_range(ps_ctx* ctx, int t_begin, int t_end);

/* Bloch phases alpha = exp(i kappa d) per right-hand side (geometry.py:373-375). */
int ps_set_rhs_bloch(ps_ctx* ctx, int nrhs, const double* bloch_host /* complex [nrhs] */);

/* Scattering matrix (scatmat.ScatteringMatrix): diagonal s_n
 * (disks) or dense s_{ln} with per-inclusion rotation phases
 * (rotate_scattering_matrix; rot_host may be NULL). */
int ps_set_smatrix(ps_ctx* ctx, const double* S_host /* complex [L] or [L][L] */,
                   int diagonal, const double* rot_host /* [M] or NULL */);

/* Layer coupling geometry (curves of empty_grating.build_geometry,
 * empty_grating.py:113-119): Gamma1 / Gamma2 nodes as rows (x, y, nx, ny,
 * arc weight), the layer-2 left-wall nodes (x, y), the layer-2 expansion
 * centre x2 (geometry.py:398-406), J-expansion order Q and Rayleigh-Bloch
 * orders per direction nrb. */
int ps_set_layers(ps_ctx* ctx, int n1, const double* g1_host, int n2, const double* g2_host,
                  int nw, const double* w2_host, const double* x2_host, int Q, int nrb);

/* SVD factors of the column-scaled empty-grating matrix for right-hand side
 * irhs (empty_grating.factorize, empty_grating.py:259-261, numpy
 * u, s, vh = svd(A, full_matrices=False)), its column scaling, the
 * regularisation eps (geometry.py:338) and the incident right-hand side f
 * (empty_grating.py:241-245).  Only the rows the particle field touches and
 * the columns B reads (and c, d) are kept on the device; apply_pinv
 * (empty_grating.py:264-273) is then two restricted GEMVs. */
int ps_set_pinv(ps_ctx* ctx, int irhs, int nrow, int ncol, const double* U_host,
                const double* s_host, const double* Vh_host, const double* col_scale_host,
                double eps, const double* f_host, int col_c, int col_d);

/* Assemble the coupling blocks C (multiscat.multipole_to_targets_block,
 * SPEC.md:494-502) and B_phys (source_to_local_block) as
 * device matrices -- per RHS, Bloch weights folded in, C for the owned
 * source range and B for the owned targets -- if they fit in max_gb; every
 * later Schur matvec then streams them instead of regenerating the Graf
 * symbols.  Otherwise (or after any geometry / phase / range change) the
 * matrix-free kernels are used.  Call after ps_set_pinv. */
int ps_precompute_coupling(ps_ctx* ctx, double max_gb);
/* Single-RHS M2L kernel choice: 0 auto (symmetric K1s -- each Graf symbol
 * row serves the pair and its reverse -- when this context owns every
 * target, else tiled K1), 1 force tiled K1, 2 force K1s (full range only),
 * 3 force K1h: K1s's schedule with the Toeplitz applies on the FP64 tensor
 * cores (banded Hankel DMMA; measured slower than K1s, kept opt-in). */
int ps_set_k1_variant(ps_ctx* ctx, int variant);
/* Symbol store of the symmetric single-RHS M2L (K1s): the translation symbols
 * t_nu(x_m - x_j - l d) of every tile-pair batch depend only on the geometry,
 * so the first launch after ps_set_geometry writes them to device memory in
 * the kernel's shared-memory layout (2.5 GB at BASELINE cfg3) and every later
 * launch bulk-copies them instead of regenerating them (that store-fed kernel
 * also stages each sweep's coefficient rows in shared memory by TMA; the
 * environment variable PS_K1S_STAGE=0 keeps them as global loads).  max_gb bounds the
 * store (default 32; 0 regenerates the symbols in every launch); the store is
 * also skipped when it exceeds half the free device memory.  max_gb < 0 only
 * queries; *bytes (optional) = current store size. */
int ps_set_symbol_store(ps_ctx* ctx, double max_gb, size_t* bytes);
/* Multi-RHS M2L kernel choice: 0 auto (FP64 tensor cores, mma.sync f64, for
 * >= 12 RHS; below that one single-RHS launch per RHS), 1 force the DFMA
 * multi-RHS K1m, 2 force DMMA K1d. */
int ps_set_mrhs_variant(ps_ctx* ctx, int variant);
/* SM partitioning of ps_apply_schur for one RHS with the symmetric M2L and
 * pre-assembled coupling blocks: the M2L runs on (SM count - sms) CTAs in a
 * high-priority stream while the HBM-bound C -> A^+ -> B chain streams on the
 * other SMs (sms = 0: only the M2L tail is shared); sms < 0 runs them back
 * to back.  Default 4 (best at cfg3). */
int ps_set_overlap(ps_ctx* ctx, int sms);
/* Queue order of that SM partitioning: 0 (default) the coupling chain at the
 * step's fork, 1 behind K1s (K1s' CTAs dispatched first; slower at cfg3). */
int ps_set_overlap_order(ps_ctx* ctx, int k1_first);
/* Single-RHS M2L launches (ps_apply_T, ps_apply_T_blocks) use SM count - sms
 * CTAs, leaving SMs free for work the caller overlaps on other streams (the
 * multi-GPU driver runs the coupling chain and its NCCL all-reduce there).
 * Default 0. */
int ps_set_k1_reserve(ps_ctx* ctx, int sms);
/* 1 if the pre-assembled coupling blocks are in use, 0 if matrix-free. */
int ps_coupling_mode(const ps_ctx* ctx);

/* ---- hot path (device pointers) ---------------------------------------- */

/* a = T beta: all-pairs Graf M2L over the 2P+1 phased copies, self term
 * excluded (multiscat.apply_T).  beta [nrhs][M][L] for ALL
 * inclusions; out [nrhs][t_end-t_begin][L] for the owned targets. */
int ps_apply_T(ps_ctx* ctx, const void* beta_dev, void* out_dev, void* stream);
/* Multi-GPU symmetric split (one RHS): the symmetric M2L over part `part` of
 * `nparts` equal ranges of the unordered tile-pair list, for ALL M targets:
 * out [M][L] holds this part's contributions (each pair's forward and
 * reverse translations); summing the parts of all ranks (a reduce-scatter)
 * gives apply_T.  beta: the full coefficient vector [M][L]. */
/* Particle field at points (M2P; SPEC.md:619-627 eval_total_field_grid, the
 * "particle phased multipole sums" of the layer-2 representation, PAPER.md
 * Eq. repre3_mod): out[r][i] = sum_l bloch_r^l sum_j sum_n beta_r,j[n]
 * H_n(k2 rho) e^{i n phi}, (rho, phi) = polar(pts[i] - x_j - l d e_x).
 * beta [nrhs][M][L], pts [npts][2] f64, out [nrhs][npts]; device pointers.
 * Points inside a particle get its (invalid there) outgoing sum; callers
 * mask them. */
int ps_particle_field(ps_ctx* ctx, const void* beta, int npts, const double* pts, void* out,
                      void* stream);
/* ps_particle_field plus the derivative along the unit vector dirs[pt]
 * (dirs [npts][2] f64 device; out_dn [nrhs][npts]): the particle part of
 * the wall-discrepancy check (empty_grating.wall_discrepancy_residual's
 * extra_field, eg:396-433). */
int ps_particle_field_grad(ps_ctx* ctx, const void* beta, int npts, const double* pts,
                           const double* dirs, void* out, void* out_dn, void* stream);
int ps_apply_T_blocks(ps_ctx* ctx, int part, int nparts, const void* beta, void* out,
                      void* stream);
/* Epilogue of the split: y_own = v_own - S (a_own - B A^+ g) for the owned
 * targets (solver.apply_schur_operator), given the summed
 * M2L rows a_own and the all-reduced coupling rows g (NULL: uncoupled). */
int ps_schur_finish(ps_ctx* ctx, const void* v_own, const void* a_own, const void* g, void* y,
                    void* stream);

/* g = C beta restricted to sources [s_begin, s_end): particle field values
 * and normal derivatives on Gamma1 (negated), Gamma2 and the telescoped L2
 * wall discrepancy (multiscat.multipole_to_targets_block).
 * g [nrhs][nrow_c], overwritten. */
int ps_apply_C(ps_ctx* ctx, const void* beta_dev, void* g_dev, int s_begin, int s_end,
               void* stream);

/* y = v_own - S (T v - B_phys A^+ g), g = C v already reduced over ranks
 * (solver.apply_schur_operator).  v [nrhs][M][L] full,
 * y [nrhs][Mt][L]. */
int ps_apply_schur_g(ps_ctx* ctx, const void* v_dev, const void* g_dev, void* y_dev,
                     void* stream);

/* Single-rank convenience: g = C v over all sources, then ps_apply_schur_g. */
int ps_apply_schur(ps_ctx* ctx, const void* v_dev, void* y_dev, void* stream);

/* rhs = S B_phys A^+ f for the owned targets, [nrhs][Mt][L]. */
int ps_schur_rhs(ps_ctx* ctx, void* rhs_dev, void* stream);

/* x_empty restricted to (B columns, c, d) = A^+ (f - g), g = C beta reduced
 * over ranks (solve_full recovery).  x [nrhs][ncol_b + 2 nrb]. */
int ps_recover(ps_ctx* ctx, const void* g_dev, void* x_dev, void* stream);

/* ---- GMRES building blocks (device-resident Arnoldi) --- */

/* Arnoldi pieces for drivers that apply the operator themselves and, on
 * several ranks, all-reduce the partial results between the calls
 * (krylov.gmres_device for any device operator, parallel.gmres_dist; they
 * replace the reference-SPEC GMRES loop SPEC.md:549-557).  The per-RHS
 * Hessenberg / Givens / residual state stays in the context on the device;
 * the caller owns the Krylov basis V [maxit+1][nrhs][n] (Krylov-index major)
 * and the vectors.  Only ps_krylov_begin synchronises (NaN/Inf RHS check).
 *   begin : state from the (all-reduced) squared RHS norms, V_0 = b / ||b||
 *   dot   : h [nrhs][k] = <V_i^r, w^r>, i < k, this rank's n entries (frozen
 *           RHS give 0)
 *   axpy  : w^r -= sum_i h[r][i] V_i^r (active RHS)
 *   norm2 : nrm2 [nrhs] = sum |w^r|^2 over this rank's entries
 *   step  : column k = h1 + h2 (the two CGS2 passes, [nrhs][k+1] each) and
 *           ||w||^2 -> Givens update, V_{k+1} = w / ||w||; status [nrhs+1]
 *           (device) = relative residual per RHS, then a NaN/Inf flag
 *   freeze: active_host [nrhs] (0 = converged RHS, no further updates)
 *   solve : x = sum_i y_i V_i with R y = g, iters_host [nrhs] columns each */
int ps_krylov_begin(ps_ctx* ctx, int nrhs, long long n, int maxit, const void* b_dev,
                    const double* bnorm2_dev, void* V_dev, void* stream);
int ps_krylov_dot(ps_ctx* ctx, int k, const void* V_dev, const void* w_dev, void* h_dev,
                  void* stream);
int ps_krylov_axpy(ps_ctx* ctx, int k, const void* V_dev, const void* h_dev, void* w_dev,
                   void* stream);
int ps_krylov_norm2(ps_ctx* ctx, int nrhs, long long n, const void* w_dev, double* nrm2_dev,
                    void* stream);
int ps_krylov_step(ps_ctx* ctx, int k, const void* h1_dev, const void* h2_dev,
                   const double* wnorm2_dev, const void* w_dev, void* V_dev, double* status_dev,
                   void* stream);
int ps_krylov_freeze(ps_ctx* ctx, const int* active_host, void* stream);
int ps_krylov_solve(ps_ctx* ctx, const int* iters_host, const void* V_dev, void* x_dev,
                    void* stream);

/* Whole unrestarted GMRES on one device (single rank): zero initial guess,
 * CGS2 Arnoldi, Givens least squares on the device; stops per RHS at
 * relative residual <= tol or maxit.  rhs/x [nrhs][M][L];
 * iters_host [nrhs]; hist_host [nrhs][maxit+1] (may be NULL). */
int ps_gmres(ps_ctx* ctx, const void* rhs_dev, void* x_dev, double tol, int maxit,
             int* iters_host, double* hist_host, void* stream);

/* ---- empty-grating setup on the device --------- */

/* One discretised curve of empty_grating.build_geometry (empty_grating.py:
 * 113-119; geometry.py:188-254): host rows of 8 doubles per node
 *   x, y, nx, ny, speed, weight, t, arc_weight (= weight * speed). */
typedef struct ps_curve_desc {
  int n;
  const double* data;
} ps_curve_desc;

/* InterfaceSpec (geometry.py:67-96): y = mean + sum_j a_j sin(2 pi j x/d)
 * + b_j cos(2 pi j x/d), j = 1..; at most 8 coefficients of each kind. */
typedef struct ps_interface_desc {
  double mean;
  int nsin, ncos;
  const double* sin_coeffs;
  const double* cos_coeffs;
} ps_interface_desc;

/* Everything assemble_empty_system (empty_grating.py:139-256) reads from a
 * ProblemConfig (geometry.py:317-406) and its curves. */
typedef struct ps_empty_desc {
  double period, k1, k2, k3;
  double y0;                   /* artificial boundary (ProblemConfig.y0) */
  double eps;                  /* regularization (apply_pinv, eg:270) */
  int copies;                  /* near_field_copies P */
  int Q;                       /* j_expansion_order */
  int nrb;                     /* rb_modes_per_direction (odd) */
  double centers[6];           /* expansion_centers() 1, 2, 3 (geometry.py:398-406) */
  ps_curve_desc g1, g2;        /* top / bottom interface (sample_interface) */
  ps_curve_desc wall[3];       /* left walls L1, L2, L3; right walls are +d translates */
  ps_curve_desc lid_up, lid_down;   /* Gu at +y0, Gd at -y0 */
  ps_interface_desc top, bottom;    /* parametrisation for the off-grid Alpert nodes */
  int rule_n, rule_skip, rule_interp;   /* CorrectionRule (quadrature.py:41-56) */
  const double* rule_x;
  const double* rule_w;
} ps_empty_desc;

/* Assemble the column-scaled empty-grating matrix A and rhs f for every RHS
 * on the device (one launch; empty_grating.assemble_empty_system), take its
 * SVD with cuSOLVER (empty_grating.factorize, eg:259-261), and install the
 * restricted A^+ factors and the layer-coupling curves exactly as
 * ps_set_layers + ps_set_pinv would from host factors.  theta_host[nrhs]:
 * incidence angles (ProblemConfig.incident_angle, measured from +x); the
 * Bloch phases are the ones given to ps_set_rhs_bloch (call it first).
 * PS_ERR_NUMERICAL if an SVD does not converge. */
int ps_setup_empty(ps_ctx* ctx, const ps_empty_desc* desc, const double* theta_host);
/* Multi-GPU setup split ("each rank does 2 of the 16 RHS
 * SVDs, then broadcasts"): assemble every RHS but factorise only RHS
 * [rhs_begin, rhs_end); the other RHS get their restricted A^+ factors with
 * ps_import_pinv from a buffer the owning rank filled with ps_export_pinv and
 * broadcast (NCCL).  ps_pinv_bytes: size of that packed buffer (one RHS). */
int ps_setup_empty_range(ps_ctx* ctx, const ps_empty_desc* desc, const double* theta_host,
                         int rhs_begin, int rhs_end);
long long ps_pinv_bytes(const ps_ctx* ctx);
int ps_export_pinv(ps_ctx* ctx, int irhs, void* dst_dev, void* stream);
int ps_import_pinv(ps_ctx* ctx, int irhs, const void* src_dev, void* stream);
/* Rows/columns of the device-assembled A (856 x 781 at the BASELINE geometry). */
int ps_empty_shape(const ps_ctx* ctx, int* nrow, int* ncol);
/* Copy one RHS's device-assembled data back (any pointer may be NULL):
 * A complex [nrow][ncol] row-major (column-scaled, as EmptyGratingSystem.matrix),
 * f complex [nrow], col_scale [ncol], singular values s [ncol] (descending). */
int ps_get_empty(ps_ctx* ctx, int irhs, double* A_host, double* f_host, double* col_scale_host,
                 double* s_host);
/* Concurrent cuSOLVER streams used for the per-RHS SVDs (default 4). */
int ps_set_svd_workers(ps_ctx* ctx, int workers);
/* Device time of the last ps_setup_empty: assembly and SVD + factor restriction. */
int ps_setup_timings(const ps_ctx* ctx, double* assemble_ms, double* svd_ms);

/* ---- empty-grating fields at points --------------- */

/* Number of empty-grating unknowns (columns of A, 781 at the BASELINE
 * geometry) ps_recover_full returns; -1 if the factors carry no field rows. */
int ps_full_columns(const ps_ctx* ctx);
/* x = A^+ (f - g) over ALL columns, in the reference order mu1, sigma1, mu2,
 * sigma2, a2, a1, a3, c, d (empty_grating.py:154-156; the recovery of
 * solve_full), g = C beta reduced over ranks.  x [nrhs][ncol]. */
int ps_recover_full(ps_ctx* ctx, const void* g_dev, void* x_dev, void* stream);
/* Layer-field data for ps_layer_field when the factors came from ps_set_pinv
 * (ps_setup_empty sets them itself): k1, k3, expansion centres 1 and 3
 * (geometry.py:398-406) and the incident wave vector per RHS,
 * inc [nrhs][2] = k1 (cos theta, sin theta) (empty_grating.py:32-42). */
int ps_set_field_params(ps_ctx* ctx, double k1, double k3, const double* c1_host,
                        const double* c3_host, const double* inc_host);
/* Total empty-grating layer field at points (empty_grating.eval_empty_field,
 * eg:352-393, total=True: phased layer potentials of the bounding interfaces
 * + the layer's regular expansion + the incident wave in layer 1) from x of
 * ps_recover_full.  pts [npts][2] f64 and layer [npts] int (1, 2, 3; other
 * values give 0) on the device; out [nrhs][npts] complex.  Plain smooth
 * quadrature: keep points ~5 node spacings off the interfaces (lp:244-246). */
int ps_layer_field(ps_ctx* ctx, const void* x_dev, int npts, const double* pts_dev,
                   const int* layer_dev, void* out_dev, void* stream);
/* Values and derivatives along dirs[pt] of the layer field (incident wave in
 * layer 1 only if incident != 0: eval_empty_field total=True/False) -- the
 * empty-grating part of wall_discrepancy_residual (eg:396-433), with the
 * derivative kernels N / T of layerpot._kernel_values_diff (lp:67-91) and
 * the regular-wave gradients (sf:86-125). */
int ps_layer_field_grad(ps_ctx* ctx, const void* x_dev, int npts, const double* pts_dev,
                        const int* layer_dev, const double* dirs_dev, int incident,
                        void* out_dev, void* out_dn_dev, void* stream);
/* The empty-grating matrix of one RHS when the factors came from host SVDs
 * (ps_setup_empty keeps its own): A_host the COLUMN-SCALED matrix
 * (EmptyGratingSystem.matrix, row-major complex [m][ncol]), f_host [m],
 * col_scale_host [ncol] (empty_grating.py:246-255). */
int ps_set_empty_system(ps_ctx* ctx, int irhs, int m, int ncol, const double* A_host,
                        const double* f_host, const double* col_scale_host);
/* Empty-grating rows of the coupled residual (solve_empty's
 * residual, eg:289-290): per RHS out_dev[2r] = ||A (x / cs) + C beta - f||^2
 * and out_dev[2r+1] = ||f||^2, x [nrhs][ncol] all unknowns (ps_recover_full),
 * g_dev [nrhs][nrow_c] = C beta (NULL: zero). */
int ps_empty_residual(ps_ctx* ctx, const void* x_dev, const void* g_dev, double* out_dev,
                      void* stream);

/* ---- particle scattering matrix ------------------- */

/* Star-shaped particle r(t) = a1 + a2 cos(a3 t) (ParticleShape,
 * geometry.py:99-113) sampled by geometry.sample_particle (geometry.py:
 * 224-256) at centre 0, rotation 0: host rows of 8 doubles per node
 * (x, y, nx, ny, speed, weight, t, arc_weight), n >= 64 nodes. */
typedef struct ps_particle_desc {
  double k2, kp;                      /* exterior (layer 2) and particle wavenumbers */
  double base_radius, bump_amplitude; /* a1, a2 */
  int lobes;                          /* a3 */
  int n;
  const double* curve;
  int rule_n, rule_skip, rule_interp; /* Alpert correction rule (quadrature.py:41-56) */
  const double* rule_x;
  const double* rule_w;
} ps_particle_desc;

/* Scattering matrix s_ln, |l|, |n| <= p, of one particle from the Mueller
 * BIE (scatmat.scattering_matrix): the
 * 2n x 2n Nystrom system of Eqs. intg1-intg2 assembled on the device, solved
 * for the 2p+1 incident regular waves (in-house Gauss-Jordan with partial
 * pivoting on the device, scatmat.cu gj_*), projected onto outgoing
 * coefficients.  S_host: complex [2p+1][2p+1] row-major (row l, column n);
 * residual (may be NULL): ||A X - B|| / ||B|| of the discrete solve.
 * PS_ERR_NUMERICAL for a singular system or non-finite entries. */
int ps_scattering_matrix(ps_ctx* ctx, const ps_particle_desc* desc, int p, double* S_host,
                         double* residual);

/* ---- instrumentation ---------------------------------------------------- */
/* Record CUDA events around every K1 (M2L) launch of this context. */
int ps_profile(ps_ctx* ctx, int enable);
/* Kernel launches issued so far, and total/launch count of timed K1 runs
 * (synchronises on the recorded events). */
int ps_stats(ps_ctx* ctx, long long* launches, double* k1_ms, long long* k1_count);
int ps_stats_reset(ps_ctx* ctx);
/* Mean timeline of the SM-partitioned single-RHS Schur steps run with
 * profiling on (ms from the step's fork): out3 = {K1s end, coupling-chain
 * end, step end}; *count = steps folded. */
int ps_timeline(ps_ctx* ctx, double* out3, long long* count);

/* ---- roofline denominator ---------------------------------------------- */
/* DFMA-chain FP64 throughput of the device (TFLOP/s, 2 flops per FMA). */
int ps_dfma_peak(int device, double* tflops, double* ms);
/* Same kernel launched back to back for ~seconds (sustained clock under the
 * power cap): the denominator for kernels timed inside a long step. */
int ps_dfma_sustained(int device, double seconds, double* tflops);
/* FP64 tensor-core (mma.sync m8n8k4 f64) throughput of the device, TFLOP/s. */
int ps_dmma_peak(int device, double* tflops);

#ifdef __cplusplus
}
#endif
#endif /* PERISCAT_B200_H */
