/* prismdg_b200.h -- C ABI of the B200-native prism-DG hot path.
 *
 * The reference (`prismdg`, pure Python + numpy) has no FFI: its "operator API"
 * is the module-level functions of external2d.py / internal3d.py / columns.py /
 * mesh.py.  Each entry below replaces one of them (cited per entry) and is
 * bound by ctypes in paper_2605_16082_b200/_lib.py; INTEGRATION.md shows the
 * binding a maintainer adds to the reference side.
 *
 * Conventions
 *  - Every field pointer is a DEVICE pointer (caller-owned, e.g. a torch CUDA
 *    tensor), FP64, in the device layouts of csrc/common.cuh:
 *      C3  [3][nt]            2D nodal field           (reference: (nt,3))
 *      P6  [6][L][nt]         prism nodal field        (reference: (P,6), p = c*L+l)
 *      P6N [N][6][L][nt]      N-component prism field  (reference: (P,6,N))
 *      FAC [3][2][2][L][nt]   lateral flux factor      (reference: (nt,L,3,2,2))
 *      MASS [36][L][nt]       prism mass               (reference: (P,6,6))
 *      BAND d [36][L][nc], u [18][L][nc], w [18][L][nc]  (reference: BandedColumnMatrix)
 *  - `els` (optional, device int32, n_els entries) selects columns exactly like
 *    the reference's `els=` argument; NULL means all columns.
 *  - `stream` is a cudaStream_t; every call is asynchronous and stream ordered.
 *  - Return value: 0 on success, PDG_ERR_CUDA on a launch/API error.  Numerical
 *    failures (dry columns, zero pivots, CFL) are written by the kernels to the
 *    context error word and read with pdg_last_error(); codes map 1:1 onto the
 *    reference exceptions (errors.py:16-52).
 *  - The library never allocates on the hot path; workspaces are sized once.
 */
#ifndef PRISMDG_B200_H
#define PRISMDG_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PDG_OK 0
#define PDG_ERR_DRY 1           /* DryColumn(column, depth)       */
#define PDG_ERR_ZERO_PIVOT 2    /* ZeroPivot(layer, node)         */
#define PDG_ERR_SINGULAR_MASS 3 /* SingularMass                   */
#define PDG_ERR_CFL 4           /* CflViolation(ratio)            */
#define PDG_ERR_DEGENERATE 5    /* DegenerateLayer                */
#define PDG_ERR_SHAPE 6         /* ShapeMismatch                  */
#define PDG_ERR_NONPOS_LENGTH 7 /* NonPositiveLength              */
#define PDG_ERR_CUDA 100

typedef struct pdg_err {
  int code;
  int pad;
  long long i0, i1;
  double val;
} pdg_err;

typedef struct pdg_ctx pdg_ctx;

/* Mesh2D geometry + connectivity, HOST arrays in the reference (nt,3) layout
 * (mesh.py:35-54).  Copied, transposed and owned by the context. */
typedef struct pdg_mesh_desc {
  int nt;
  const double* j2d;   /* (nt)   */
  const double* dphx;  /* (nt,3) */
  const double* dphy;
  const double* elen;
  const double* enx;
  const double* eny;
  const double* b;     /* (nt,3) bed at the corners */
  const int64_t* nbr;  /* (nt,3) */
  const int64_t* nbrk;
  const int64_t* btag;
  double min_edge;
} pdg_mesh_desc;

/* ---- Mesh2D setup on device (mesh.py:79-127, 187-228) ---------------------------------------
 * pdg_mesh_build: nodal coordinates, J2D, grad phi, edge lengths/normals and the edge pairing
 * (nbr, nbrk, btag; bit-exact with the reference's dict pass via a stable radix sort).  All DEVICE
 * pointers in the reference (nt,3) layout; tri int64 (nt,3).  err: code 8 = NonPositiveArea.
 * pdg_hilbert_perm: hilbert_reorder's permutation (stable sort of the order-`order` curve distance). */
int pdg_mesh_build(int nt, long long nv, const double* vx, const double* vy, const double* vb, const long long* tri,
                   double* x, double* y, double* b, double* j2d, double* dphx, double* dphy, double* elen,
                   double* enx, double* eny, long long* nbr, long long* nbrk, long long* btag, pdg_err* err,
                   void* stream);
int pdg_hilbert_perm(int nt, int order, const double* x, const double* y, long long* perm, void* stream);

/* ---- context ------------------------------------------------------------------------- */
int pdg_ctx_create(const pdg_mesh_desc* mesh, int device, pdg_ctx** out);
int pdg_ctx_destroy(pdg_ctx* ctx);
/* sigma fractions (L+1 host doubles, mesh.py:389) -- np.linspace(0, 1, L+1) */
int pdg_ctx_set_layers(pdg_ctx* ctx, int L, const double* fracs);
/* partitioned runs: columns 0..nown-1 are owned (computed), nown..nt-1 are ghost columns whose
 * values arrive by halo exchange.  Default nown = nt. */
int pdg_ctx_set_owned(pdg_ctx* ctx, int nown);
/* synchronises `stream`, returns and clears the first recorded device error */
int pdg_last_error(pdg_ctx* ctx, void* stream, int* code, long long* i0, long long* i1, double* val);
const char* pdg_cuda_error_string(void);
/* occupancy variant of a kernel family (0 F3D->2D, 1 vertical implicit, 2 vertical explicit, 3 r, 4 w~, 5 stage RHS):
 * value = min resident 128-thread blocks per SM (1, 3, 4) or 8/9/10 = shared-memory variant of the
 * F3D->2D / stage-RHS kernels (64-thread blocks); < 0 queries.  Returns the previous value. */
int pdg_tune(int key, int value);
/* number of kernel launches issued by this context since creation */
long long pdg_launch_count(pdg_ctx* ctx);

/* ---- 2D external mode (external2d.py) -------------------------------------------------- */
/* mode 0: external_tendencies (external2d.py:259-268) -> d_eta, d_qx, d_qy
 * mode 1: rhs_free_surface / rhs_depth_momentum residuals (external2d.py:128-256)
 * outputs are [3][n_rows] with n_rows = n_els (or nt). f3d2d is [2][3][nt]. */
int pdg_ext2d_eval(pdg_ctx* ctx, const double* eta, const double* qx, const double* qy, const double* f3d2d,
                   const double* source, const double* patm, int has_bc, double eta_bc, double g, double rho0,
                   const int* els, int n_els, int mode, double* out_eta, double* out_qx, double* out_qy,
                   void* stream);
/* subcycle_external (external2d.py:296-353): `state` [3 field][3][nt] advanced in place
 * by m SSP-RK3 substeps; qbar, f2d are [2][3][nt]; bc_vals (host, 3*m values: eta_bc at
 * each RK stage time) or NULL for no prescribed open-boundary level.  check_cfl != 0
 * runs check_cfl (external2d.py:271-283) on device first. */
int pdg_ext2d_subcycle(pdg_ctx* ctx, double* state, int m, double dt, double g, double rho0, const double* f3d2d,
                       const double* source, const double* patm, const double* bc_vals, double* qbar, double* f2d,
                       int check_cfl, void* stream);
/* the same sub-cycle one RK stage at a time, so a partitioned run can exchange the stage state
 * (halo) between stages: begin (CFL check, Q0 copy, Qbar = 0), rk_stage(0|1|2), end (Qbar /= m, F2D) */
int pdg_ext2d_subcycle_begin(pdg_ctx* ctx, const double* state, double g, double dt, int check_cfl, double* qbar,
                             void* stream);
/* stage 0: Y = S0 + dt d(X); 1: Y = 3/4 S0 + 1/4 (X + dt d(X)); 2: Y = S0/3 + 2/3 (X + dt d(X)), qbar += Y.Q */
int pdg_ext2d_rk_stage(pdg_ctx* ctx, int stage, const double* X, const double* S0, double* Y, double dt, double g,
                       double rho0, const double* f3d2d, const double* source, const double* patm, int has_bc,
                       double eta_bc, double* qbar, void* stream);
/* one RK stage over the columns els[0..n_els) only (partitioned runs: the columns next to ghost
 * columns first, then the interior while the halo exchange of the boundary values is in flight) */
int pdg_ext2d_rk_stage_cols(pdg_ctx* ctx, int stage, const double* X, const double* S0, double* Y, double dt,
                            double g, double rho0, const double* f3d2d, double* qbar, const int* els, int n_els,
                            void* stream);
int pdg_ext2d_subcycle_end(pdg_ctx* ctx, const double* state, const double* f3d2d, int m, double dt, double* qbar,
                           double* f2d, void* stream);
/* check_cfl on device; writes the ratio to ratio_dev[0] (device) and the error word */
int pdg_ext2d_cfl(pdg_ctx* ctx, const double* eta, double g, double dt, double* ratio_dev, void* stream);
/* apply_mh / apply_mh_inv (columns.py:45-69) on n triangles: v [nc][3][n], j2d [n] */
int pdg_apply_mh(const double* v, const double* j2d, int n, int nc, int inverse, double* out, pdg_err* err,
                 void* stream);

int pdg_eos(const double* T, const double* S, long long n, double alpha, double beta, double tref, double sref,
            double* out, void* stream);                                    /* eos_density external2d.py:81-87 */

/* ---- 3D internal mode (internal3d.py); eta_g = the grid's free surface (C3), geometry is
 *      rebuilt on device from (eta_g, mesh b, sigma fractions) -------------------------------- */
int pdg_prism_mass(pdg_ctx* ctx, const double* eta_g, const int* els, int n_els, double* mass,
                   void* stream);                                          /* prism_mass :114-123 */
/* mass_apply / mass_solve (:126-151): mass [36][L][nt], f/out [nc][6][L][nt]; solve != 0 -> LU */
int pdg_mass_op(int L, int nt, int nc, int solve, const double* mass, const double* f, double* out, pdg_err* err,
                void* stream);
/* project_transport (:164-181); mass NULL -> exact Kronecker form; qsum [2][3][nt] (column
 * sum of q) and htot [3][nt] (2 sum Jz) optional */
int pdg_project_transport(pdg_ctx* ctx, const double* eta_g, const double* ux, const double* uy, const double* mass,
                          const int* els, int n_els, double* q, double* qsum, double* htot, void* stream);
int pdg_column_sum(int nt, int L, int ncomp, const double* f, double* out, void* stream);   /* :184-187 */
int pdg_total_thickness(pdg_ctx* ctx, const double* eta_g, double* htot, void* stream); /* mesh.py:422 */
/* (Qbar - sum_col q) / H  and  consistent_transport (:190-208) */
int pdg_mismatch(pdg_ctx* ctx, const double* qbar, const double* qsum, const double* htot, double* mis,
                 void* stream);
int pdg_consistent_transport(pdg_ctx* ctx, const double* eta_g, const double* q, const double* mis, const int* els,
                             int n_els, double* out, void* stream);
int pdg_lateral_flux_factor(pdg_ctx* ctx, const double* eta_g, const double* q, double g, const int* els, int n_els,
                            double* fac, void* stream);                      /* :275-314 */
/* compute_r (:327-405) incl. the top-down sweep; from_T != 0 applies the linear EOS inline */
int pdg_compute_r(pdg_ctx* ctx, const double* eta_g, const double* rho_or_T, int from_T, double alpha, double tref,
                  double g, const int* els, int n_els, double* r, void* stream);
int pdg_compute_w(pdg_ctx* ctx, const double* eta_g, const double* q, const double* ux, const double* uy,
                  const double* fac, const int* els, int n_els, double* w, void* stream);   /* :434-502 */
/* compute_wtilde (:505-541); mis != NULL -> qbar = qb + Jz mis and its factor on the fly */
int pdg_compute_wtilde(pdg_ctx* ctx, const double* eta_g, const double* qb, const double* fac, const double* mis,
                       double g, const int* els, int n_els, double* w, void* stream);
/* horizontal_rhs (ncomp 2, :695-751) / tracer_horizontal_rhs (ncomp 1, :754-792) without the
 * explicit diffusion term (pdg_horizontal_diffusion adds it) */
int pdg_horizontal_rhs(pdg_ctx* ctx, const double* eta_g, const double* u, int ncomp, const double* q_adv,
                       const double* fac, const double* r, const double* mass, double f, double rho0, int mass_terms,
                       const int* els, int n_els, double* out, void* stream);
/* _horizontal_diffusion (:549-692; the reference raises at :665/:676, so this is the patched
 * oracle of tests/golden/hdiff.npz): out += scale * D(f).  ncomp 2 + wall_mirror 1: momentum
 * (kappa_h, walls mirrored); ncomp 1 + wall_mirror 0: tracer (nu_h, walls insulated).
 * mode 0: out is the prism residual [ncomp][6][L][nt] (rows of els, else the owned columns);
 * mode 1: out is its column sum [ncomp][3][nt] (:184-187, the F3D->2D forcing).  kh == 0: no-op. */
int pdg_horizontal_diffusion(pdg_ctx* ctx, const double* eta_g, const double* f, int ncomp, double kh,
                             int wall_mirror, double scale, int mode, const int* els, int n_els, double* out,
                             void* stream);
int pdg_mass_terms(int L, int nt, const double* mass, const double* u, const double* r, double f, double rho0,
                   double* out, void* stream);                             /* :745-750 over all rows */
int pdg_stress_rhs(pdg_ctx* ctx, const double* ux, const double* uy, double tsx, double tsy, double cd, const int* els,
                   int n_els, double* out, void* stream);                  /* :919-934 */

/* ---- column solvers (columns.py) ------------------------------------------------------------ */
/* solve_r_column (kind 0, :95-122) / solve_w_column (kind 1, :125-151): rhs/out [nc][6][L][ncol] */
int pdg_solve_sweep(int kind, int ncol, int L, int nc, const double* rhs, const double* j2d, const int* layers,
                    double* out, pdg_err* err, void* stream);
/* solve_banded_column (:292-348); gu/gw receive the propagation tiles (may alias u/w) */
int pdg_solve_banded(int ncol, int L, int nc, const double* d, const double* u, const double* w, double* gu,
                     double* gw, const double* rhs, double* x, pdg_err* err, void* stream);
int pdg_apply_banded(int ncol, int L, int nc, const double* d, const double* u, const double* w, const double* x,
                     double* y, void* stream);                               /* :356-366 */
int pdg_build_implicit(long long P, const double* mass, const double* d, const double* u, const double* w, double dt,
                       double* od, double* ou, double* ow, void* stream);    /* internal3d.py:902-906 */
/* solve_tridiagonal (:507-531): arrays [n][nb] (batch contiguous), work [n][nb] */
int pdg_solve_tridiagonal(int nb, int n, const double* lower, const double* diag, const double* upper,
                          const double* rhs, double* x, double* work, pdg_err* err, void* stream);
/* assemble_vertical_operator (internal3d.py:800-899): outputs compact over the selected columns */
int pdg_assemble_vertical(pdg_ctx* ctx, const double* eta_g, const double* wt, const double* wm, double kh, double kv,
                          double n0, int order, const int* els, int n_els, double* d, double* u, double* w,
                          void* stream);

/* ---- domain decomposition on the device (partition.py decompose(device=...)) ---- */
/* split_ranges: raw split points k = 1..P-1 (first prefix whose prism weight reaches k W / P) of the
 * DEVICE int64 weights [n]; raw: HOST [P-1] (the host applies the non-empty / capacity clamps) */
int pdg_split_search(const long long* w, int n, int P, long long* raw, void* stream);
/* ghost rings (1..depth, breadth first over edge neighbours) of the owned range [lo, hi): DEVICE
 * ghosts (ascending global ids) and rings, capacity nt - (hi - lo); n_ghosts: HOST */
int pdg_partition_rings(pdg_ctx* ctx, int lo, int hi, int depth, int* ghosts, int* rings, int* n_ghosts,
                        void* stream);

/* ---- halo exchange (partitioned runs): field = nplanes planes of nt doubles; buf = [nplanes][n] */
int pdg_halo_pack(const double* field, long long nplanes, int nt, const int* idx, int n, double* buf, void* stream);
int pdg_halo_unpack(const double* buf, long long nplanes, int nt, const int* idx, int n, double* field, void* stream);

/* ---- NCCL halo exchange of a partitioned run (csrc/comm.cu).
 * The library binds the process's NCCL at run time (pdg_comm_load(path of libnccl.so.2)); rank 0
 * creates the 128-byte unique id, the caller broadcasts it (torch.distributed bootstrap).  A plan
 * lists per peer the owned columns to send and the ghost slots to fill (host int32 lists, copied).
 * start: pack + grouped ncclSend/ncclRecv on the plan's communication stream (after the pack);
 * finish: `stream` waits for the transfers, then unpacks.  Work launched on `stream` between the
 * two overlaps the exchange; every call is stream ordered and CUDA-graph capturable. */
typedef struct pdg_comm pdg_comm;
typedef struct pdg_halo_plan pdg_halo_plan;
int pdg_comm_load(const char* libnccl_path);
const char* pdg_comm_error_string(void);
int pdg_comm_unique_id(void* id128);
int pdg_comm_init(const void* id128, int rank, int nranks, int device, pdg_comm** out);
int pdg_comm_destroy(pdg_comm* comm);
int pdg_halo_plan_create(pdg_comm* comm, int nt, int npeers, const int* peers, const int* nsend,
                         const int* const* send_idx, const int* nrecv, const int* const* recv_idx, int max_planes,
                         pdg_halo_plan** out);
int pdg_halo_plan_destroy(pdg_halo_plan* plan);
int pdg_halo_start(pdg_halo_plan* plan, int nfields, double* const* fields, const long long* nplanes, void* stream);
int pdg_halo_finish(pdg_halo_plan* plan, int nfields, double* const* fields, const long long* nplanes, void* stream);
/* blocking exchanges under the SURVEY section 8b names: the 2D sub-cycle state (9 C3 planes, the
 * all-rings plan) and ring-1 3D fields (start + finish) */
int pdg_halo_2d(pdg_halo_plan* plan, double* state9, void* stream);
int pdg_halo_3d(pdg_halo_plan* plan, int nfields, double* const* fields, const long long* nplanes, void* stream);

/* ---- device-initiated halo exchange over NVLink peer memory (csrc/p2p.cu; SURVEY.md section 8e
 * "LSA peer stores (2D)").  No NCCL: every rank owns an inbox (per peer: an epoch flag and a
 * double-buffered receive window) that its peers map -- pdg_p2p_local exports the CUDA IPC handle
 * (64 bytes) or raw pointer and the per-peer offsets, pdg_p2p_connect maps a peer's inbox.
 * start: per peer one kernel stores the packed boundary values into the peer's window and
 * publishes the epoch (release, system scope); finish: per peer one kernel waits for the epoch
 * (acquire) and unpacks.  Epochs are device-resident: stream ordered, CUDA-graph capturable. */
typedef struct pdg_p2p pdg_p2p;
int pdg_p2p_create(int nt, int npeers, const int* peers, const int* nsend, const int* const* send_idx,
                   const int* nrecv, const int* const* recv_idx, int max_planes, int device, pdg_p2p** out);
int pdg_p2p_destroy(pdg_p2p* plan);
int pdg_p2p_local(pdg_p2p* plan, void* ipc_handle64, void** raw, long long* win_off, long long* flag_off);
int pdg_p2p_connect(pdg_p2p* plan, int slot, const void* ipc_handle64, void* raw, long long win_off,
                    long long flag_off);
int pdg_p2p_start(pdg_p2p* plan, int nfields, double* const* fields, const long long* nplanes, void* stream);
int pdg_p2p_finish(pdg_p2p* plan, int nfields, double* const* fields, const long long* nplanes, void* stream);

/* device-to-device copy of `bytes` on `stream` (csrc/hostio.cu) */
int pdg_copy_d2d(void* dst, const void* src, long long bytes, void* stream);

/* ---- host I/O layout conversion (set_state / get_state of the drop-in; csrc/hostio.cu):
 * rows [ncols][L][nk] = columns [c0, c0 + ncols) of a reference-layout field ((P, nk) with
 * p = c L + l, or (nt, nk) with L = 1) in a device staging buffer  <->  planes [nk][L][nt] */
int pdg_rows_to_planes(const double* rows, int ncols, int L, int nk, double* planes, int nt, int c0, void* stream);
int pdg_planes_to_rows(const double* planes, int nt, int c0, int ncols, int L, int nk, double* rows, void* stream);

/* ---- fused IMEX stage entries (the stepper) ---------------- */
/* F3D->2D = column sum of horizontal_rhs(u, q, fac(q)) + stress_rhs  -> [2][3][nt] */
int pdg_step_f3d2d(pdg_ctx* ctx, const double* eta_u, const double* u, const double* q, const double* r, double g,
                   double f, double rho0, double tsx, double tsy, double cd, double* f3d2d, void* stream);
/* the same with rsum (optional) = the per-column layer sum of jm (r_top + r_bot) from pdg_step_r:
 * the tile-staged kernel then loads no r (the F3D->2D mass term is linear in r) */
int pdg_step_f3d2d_rsum(pdg_ctx* ctx, const double* eta_u, const double* u, const double* q, const double* r,
                        const double* rsum, double g, double f, double rho0, double tsx, double tsy, double cd,
                        double* f3d2d, void* stream);
/* the stepper's baroclinic head from T (EOS inline) -> r [2][6][L][nt]; with the tile-staged
 * kernel also rsum [2][3][nt] (*rsum_written = 1) */
int pdg_step_r(pdg_ctx* ctx, const double* eta_g, const double* T, double alpha, double tref, double g, double* r,
               double* rsum, int* rsum_written, void* stream);
/* stage right-hand sides: ncomp 2: M0 u0 + dt (F_h(u, q + Jz mis) + stress + M1 F2D/H1);
 * ncomp 1: M0 T0 + dt F_T(T, q + Jz mis) */
int pdg_step_rhs(pdg_ctx* ctx, int ncomp, const double* eta_u, const double* eta0, const double* eta1,
                 const double* u, const double* u0, const double* q, const double* mis, const double* r,
                 const double* f2d, double g, double f, double rho0, double tsx, double tsy, double cd, double dt,
                 double* out, void* stream);
/* both stage right-hand sides in one pass (shared q~ / flux factor / masses) */
int pdg_step_rhs_ut(pdg_ctx* ctx, const double* eta_u, const double* eta0, const double* eta1, const double* u,
                    const double* T, const double* u0, const double* T0, const double* q, const double* mis,
                    const double* r, const double* f2d, double g, double f, double rho0, double tsx, double tsy,
                    double cd, double dt, double* out_u, double* out_T, void* stream);
/* pdg_step_rhs_ut and w~ of the stage into w [6][L][nt] (pdg_compute_wtilde with q~ = q + Jz mis):
 * formed in the same bottom-up layer loop, which already forms q~ and its lateral flux factor */
int pdg_step_rhs_ut_w(pdg_ctx* ctx, const double* eta_u, const double* eta0, const double* eta1, const double* u,
                      const double* T, const double* u0, const double* T0, const double* q, const double* mis,
                      const double* r, const double* f2d, double g, double f, double rho0, double tsx, double tsy,
                      double cd, double dt, double* out_u, double* out_T, double* w, void* stream);
/* vertical stage: implicit (M1 - dt A) x = rhs by block Thomas, or explicit x = M1^-1 (rhs + dt A xin),
 * A = assemble_vertical_operator(eta_u, wt, w_m = (z(eta1) - z(eta0)) / dt_mesh, kh, kv) in registers */
int pdg_step_vertical(pdg_ctx* ctx, int ncomp, int implicit, const double* eta_u, const double* eta0,
                      const double* eta1, double dt_mesh, const double* wt, double kh, double kv, double n0, int order,
                      double dt, const double* rhs, const double* xin, double* x, void* stream);
/* the same over a list of owned columns (partitioned runs: boundary columns first, then the interior
 * while the ring-1 exchange of the boundary result is in flight) */
int pdg_step_vertical_cols(pdg_ctx* ctx, int ncomp, int implicit, const double* eta_u, const double* eta0,
                           const double* eta1, double dt_mesh, const double* wt, double kh, double kv, double n0,
                           int order, double dt, const double* rhs, const double* xin, double* x, const int* cols,
                           int ncols, void* stream);

/* explicit vertical stage of momentum (ncomp 2) and tracer in one pass */
/* diagnostics_2d (external2d.py:366-380) and budget_3d (internal3d.py:942-951) of the resident state
 * in one fused pass: S [3][3][nt] (eta, qx, qy), u [2][6][L][nt], T [6][L][nt]; out (device, 10
 * doubles): 2D volume, 2D energy, eta min, eta max, 3D volume, momentum x, momentum y, tracer
 * mass, T min, T max.  work: device scratch of pdg_diagnostics_work_doubles(ctx) doubles.
 * Deterministic (fixed reduction order). */
int pdg_step_diagnostics(pdg_ctx* ctx, const double* S, const double* u, const double* T, double g, double* work,
                         double* out, void* stream);
int pdg_diagnostics_work_doubles(pdg_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif
