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

/* ---- context ------------------------------------------------------------------------- */
int pdg_ctx_create(const pdg_mesh_desc* mesh, int device, pdg_ctx** out);
int pdg_ctx_destroy(pdg_ctx* ctx);
/* sigma fractions (L+1 host doubles, mesh.py:389) -- np.linspace(0, 1, L+1) */
int pdg_ctx_set_layers(pdg_ctx* ctx, int L, const double* fracs);
/* synchronises `stream`, returns and clears the first recorded device error */
int pdg_last_error(pdg_ctx* ctx, void* stream, int* code, long long* i0, long long* i1, double* val);
const char* pdg_cuda_error_string(void);
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
/* check_cfl on device; writes the ratio to ratio_dev[0] (device) and the error word */
int pdg_ext2d_cfl(pdg_ctx* ctx, const double* eta, double g, double dt, double* ratio_dev, void* stream);
/* apply_mh / apply_mh_inv (columns.py:45-69) on n triangles: v [nc][3][n], j2d [n] */
int pdg_apply_mh(const double* v, const double* j2d, int n, int nc, int inverse, double* out, pdg_err* err,
                 void* stream);

#ifdef __cplusplus
}
#endif
#endif
