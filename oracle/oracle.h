/* oracle.h -- fp64 CPU oracle for AbstractSplat (arXiv 2503.00308).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code with
 * the CUDA path (paper_2503_00308_b200/) and neither side includes the other.
 *
 * Everything is double precision.  Citations: P:L = /root/reference/PAPER.md line L.
 * The readings of silent / ambiguous points are listed in DESIGN.md ("Readings") and
 * referred to here by their ids (G1..G19, H1..H5, O1..).
 *
 * Affine-form layout used at this ABI (D7): a form over n variables
 * xi in [-1,1]^n is 2(n+1) doubles  [lA_0..lA_{n-1}, lb, uA_0..uA_{n-1}, ub]
 * meaning  lA.xi + lb <= y(xi) <= uA.xi + ub.
 */
#ifndef ABSPLAT_ORACLE_H
#define ABSPLAT_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define OR_NVMAX 9

typedef struct {
  double fx, fy, cx, cy;   /* intrinsics K = [[fx,0,cx],[0,fy,cy]] */
  int32_t W, H;            /* image size */
  double euler[3];         /* XYZ Euler of camera->world: R_c2w = Rz(e2) Ry(e1) Rx(e0) (G9) */
  double t[3];             /* camera centre in world */
} or_camera;

typedef struct {
  double eps_t[3];   /* translation half-widths (m); 0 = not perturbed */
  double eps_R[3];   /* Euler half-widths (rad) */
  double t_off[3];   /* centre offset of the translation box */
  double R_off[3];   /* centre offset of the Euler box */
  int32_t t_frame;   /* 0 = world axes, 1 = nominal camera axes */
  int32_t parts[6];  /* uniform partition count per pose axis (tx,ty,tz,e0,e1,e2) (G18) */
  /* Optional explicit partition (NEXT-3 refinement, P:470 (2)): n_explicit > 0 replaces the
   * uniform grid by n_explicit sub-boxes, bounds [n][9][2] = (lo, hi) per box axis in the
   * box's own units (t offsets, Euler offsets, group shifts 0..2), each inside the box. */
  int32_t n_explicit;
  const double* explicit_bounds;
  /* Adaptive Taylor order (NEXT-3, P:470 (3): "increase k until Eps falls below the given
   * tolerance"): k_tol > 0 picks, per Gaussian, the smallest k >= 8 with Eps <= k_tol, at most
   * k_max; k_tol <= 0 keeps k = 8 (G14). */
  double k_tol;
  int32_t k_max;
  /* NEXT-4: 1 = conic bounds by back-substitution through MatrixInv (CROWN-style, P:141,
   * P:486) instead of the forward forms; 0 = forward (reading G3). */
  int32_t inv_backward;
} or_pose_box;

typedef struct {
  int32_t n_groups;           /* 0..3 shared mean-shift groups */
  const int32_t* group_of;    /* [N], -1 = none; may be NULL when n_groups == 0 */
  const double* dir;          /* [n_groups][3] shift direction */
  const double* shift_lo;     /* [n_groups] */
  const double* shift_hi;     /* [n_groups] */
  int32_t parts[3];           /* partition count per group variable */
  const float* col_lo;        /* [N][3] or NULL (colour interval) */
  const float* col_hi;
  const float* op_lo;         /* [N] or NULL (opacity interval) */
  const float* op_hi;
  /* [N][3] or NULL: per-Gaussian private mean offsets (world axes, metres), independent of
   * every other Gaussian.  They enter each Gaussian's forms as three
   * private variables after the shared ones; depth comparisons treat them as independent. */
  const float* priv_lo;
  const float* priv_hi;
} or_scene_box;

typedef struct {
  int64_t pairs;            /* sum over (sub-box, tile) of |L_T| */
  int64_t active_pairs;     /* sum over (sub-box, pixel) of Gaussians not culled at the pixel */
  int64_t uncertain_pairs;  /* unordered pairs with Ind = '?' (step 13) */
  int64_t fails;            /* MatrixInv FAIL Gaussians (summed over sub-boxes) */
  int64_t straddles;        /* depth straddles d_min (G8) */
  int64_t dropped;          /* Gaussians with d_hi <= d_min */
  int64_t order_violations; /* pairs breaking the (kappa,index) order structure (must be 0) */
  int32_t kmax;             /* max |L_T| */
  int32_t n_sub;            /* number of sub-boxes P */
  int32_t n_vars;           /* n */
  int32_t pad;
} or_stats;

/* Abstract render.  lo/hi: [H][W][3] doubles.
 * mode 0 = windowed blend (prefix products + exception windows, step 13 order structure),
 * mode 1 = direct blend (Ind recomputed for every pair at every pixel, Alg. 3 literal),
 * mode 2 = mode 0 intersected, on tiles whose pairs are all certain, with BlendInd evaluated
 *          with linear relations along the sorted fold.
 * nthreads <= 0: OpenMP default.  Returns 0 on success, <0 on argument error. */
int or_render_bounds(int64_t N, const float* mean, const float* chol, const float* opacity,
                     const float* color, const or_camera* cam, const or_pose_box* box,
                     const or_scene_box* sbox, int32_t tile, int32_t mode, int32_t nthreads,
                     double* lo, double* hi, or_stats* stats);

/* Union (step 22) over the sub-boxes [sub_begin, sub_end) only, windowed blend, all
 * tiles.  An empty range gives the identities of the union's min / max (lo = 1, hi = 0), so
 * ranges combine by elementwise min / max into the full render (sub-box sharding, §8(e)). */
int or_render_subboxes(int64_t N, const float* mean, const float* chol, const float* opacity,
                       const float* color, const or_camera* cam, const or_pose_box* box,
                       const or_scene_box* sbox, int32_t tile, int32_t sub_begin, int32_t sub_end,
                       int32_t nthreads, double* lo, double* hi, or_stats* stats);

/* Same semantics at selected pixels only, computed without tiles: every non-dropped
 * Gaussian culled per pixel, direct blend.  `tile` is accepted for symmetry and unused
 * (results do not depend on the tile size, reading O1).  lo/hi: [npix][3]. */
int or_pixel_bounds(int64_t N, const float* mean, const float* chol, const float* opacity,
                    const float* color, const or_camera* cam, const or_pose_box* box,
                    const or_scene_box* sbox, int32_t tile, int64_t npix, const int32_t* px,
                    const int32_t* py, int32_t nthreads, double* lo, double* hi);

/* Restricted render: only the tiles listed (tile ids ty*ntx+tx) are computed; other
 * pixels of lo/hi are left untouched.  Used for bounded CPU baselines. */
int or_render_tiles(int64_t N, const float* mean, const float* chol, const float* opacity,
                    const float* color, const or_camera* cam, const or_pose_box* box,
                    const or_scene_box* sbox, int32_t tile, int64_t ntiles, const int32_t* tiles,
                    int32_t nthreads, double* lo, double* hi, or_stats* stats);

/* Concrete GaussianSplat (Alg. 1 l.2-11) at one pose.  shifts: [n_groups]
 * group shift values (may be NULL if n_groups == 0).  blend 0 = BlendSort (Alg. 2,
 * stable ascending-index ties), 1 = BlendInd (Alg. 3, index tie-break G6),
 * 2 = BlendInd with the paper's strict Ind (no tie-break).
 * px/py NULL => whole image, img [H][W][3]; else img [npix][3]. */
int or_render_concrete(int64_t N, const float* mean, const float* chol, const float* opacity,
                       const float* color, const or_camera* cam, int32_t n_groups,
                       const int32_t* group_of, const double* dir, const double* shifts,
                       int32_t blend, int64_t npix, const int32_t* px, const int32_t* py,
                       int32_t nthreads, double* img);

/* Concrete blends on explicit inputs (Alg. 2 / Alg. 3).  a[N], c[N][3], d[N] -> pc[3]. */
void or_blend_sort(int64_t N, const double* a, const double* c, const double* d, double* pc);
void or_blend_ind(int64_t N, const double* a, const double* c, const double* d, int32_t tiebreak,
                  double* pc);

/* Relaxation primitives on forms (layout above).  n <= OR_NVMAX. */
void or_form_conc(int32_t n, const double* f, double* lo, double* hi);
void or_form_mul(int32_t n, const double* f, const double* g, double* out);  /* R1 */
void or_form_sq(int32_t n, const double* f, double* out);                    /* R2 */
/* Table 2 Exp relaxation of a scalar interval [xl,xh] -> (slope,intercept) lower & upper */
void or_exp_relax(double xl, double xh, double* lo_slope, double* lo_icpt, double* hi_slope,
                  double* hi_icpt);
/* Table 2 Ind relaxation: returns 1 (certainly >0), 0 (certainly <=0), -1 ('?'). */
int32_t or_ind_relax(double xl, double xh);

/* MatrixInv (Alg. 4) on a 2x2 matrix of forms X[4] (row-major, each 2(n+1)).
 * X0 = inverse of the centre of conc X (P:470 (1)).  Outputs Conic[4] forms with the
 * Eps widening applied (lXinv lower / uXinv upper, union P:573), eps, rho_bar.
 * Returns 0 ok, 1 FAIL(det<=0), 2 FAIL(rho>=1). */
int32_t or_matrix_inv(int32_t n, const double* X, int32_t k, double* conic, double* eps,
                      double* rho);
/* Same input / output as or_matrix_inv, with the conic bounds by back-substitution (NEXT-4). */
int32_t or_matrix_inv_bwd(int32_t n, const double* X, int32_t k, double* conic, double* eps,
                          double* rho);

/* Pose forms of sub-box `sub` (step 1): R (world->camera) [9 forms] and t [3 forms],
 * plus the number of variables.  Returns number of sub-boxes, or <0 on error. */
int32_t or_pose_forms(const or_camera* cam, const or_pose_box* box, const or_scene_box* sbox,
                      int32_t sub, double* R, double* t, int32_t* nvars);

/* Per-Gaussian forms for sub-box `sub` (steps 2-11).  Output per Gaussian, see
 * OR_GREC_* offsets in oracle.cpp documentation; fields (each a form of 2(n+1)):
 * uc[3], d, up[2], Mp[2][3], X[3] (00,01,11), conic[4], W[2][3], D2, DU[2]
 * followed by scalars: flags, eps, rho, kappa, mu_lo[2], mu_hi[2], r2.  */
int32_t or_gaussian_forms(int64_t N, const float* mean, const float* chol, const float* opacity,
                          const float* color, const or_camera* cam, const or_pose_box* box,
                          const or_scene_box* sbox, int32_t sub, double* out, int32_t* nvars);
int32_t or_gaussian_forms_stride(int32_t n);

#ifdef __cplusplus
}
#endif
#endif
