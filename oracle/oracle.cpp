// oracle.cpp -- fp64 CPU oracle of the AbstractSplat hot path (arXiv 2503.00308).
//
// TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs.  It shares no code, header, table or constant
// generator with the CUDA path in paper_2503_00308_b200/; neither includes the other.
//
// Plain, slow, scalar fp64.  It follows SURVEY.md §8(c) steps 0-22, i.e. the paper's
// Alg. 1 lifted to affine forms (§3.3) with MatrixInv (Alg. 4,
// P:417-449) at line 8 and BlendInd (Alg. 3) at line 11, in the paper's order
// and notation.  P:L = PAPER.md line L.  The readings of points the paper leaves silent
// (G1..G19, H1..H5) are listed in DESIGN.md; each is cited where it is used.
//
// Pins (tests/test_oracle_*.py): Example 1, the 1x1 closed form of Alg. 4,
// Lemma 1 containment, Lemma 2, the d^4 identity of l.9-10, zero-width box ==
// concrete render, Theorem 1 containment under pose sampling, brute-force pose grid on
// C1, relaxation sandwich tests (Prop. 1 / Table 2), colour-box closed form.
#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

constexpr int NV = OR_NVMAX;
constexpr double TAU = 1e-12;     // cull threshold on a (G12)
constexpr double D_MIN = 0.01;    // near plane (G8)
constexpr int K_TAYLOR = 8;       // Taylor order k (P:550 footnote, G14)
constexpr double W_CAP = 1e12;    // |W| sanity cap: larger => FAIL (reading O3)

// ---------------------------------------------------------------- affine forms (D7)
struct Aff {  // A . xi + b
  double A[NV];
  double b;
};
struct Form {  // lo(xi) <= y(xi) <= hi(xi) for all xi in [-1,1]^n
  Aff lo, hi;
};



inline Aff aff_zero() {
  Aff a;
  for (int k = 0; k < NV; ++k) a.A[k] = 0.0;
  a.b = 0.0;
  return a;
}
inline Aff aff_scale(const Aff& a, double c) {
  Aff r;
  for (int k = 0; k < NV; ++k) r.A[k] = c * a.A[k];
  r.b = c * a.b;
  return r;
}
inline Aff aff_add(const Aff& a, const Aff& b) {
  Aff r;
  for (int k = 0; k < NV; ++k) r.A[k] = a.A[k] + b.A[k];
  r.b = a.b + b.b;
  return r;
}
inline double aff_min(const Aff& a, int n) {  // min over the box
  double v = a.b;
  for (int k = 0; k < n; ++k) v -= std::fabs(a.A[k]);
  return v;
}
inline double aff_max(const Aff& a, int n) {
  double v = a.b;
  for (int k = 0; k < n; ++k) v += std::fabs(a.A[k]);
  return v;
}
inline double aff_eval(const Aff& a, const double* xi, int n) {
  double v = a.b;
  for (int k = 0; k < n; ++k) v += a.A[k] * xi[k];
  return v;
}

Form constant(double v) {  // "constant relation"
  Form f;
  f.lo = aff_zero();
  f.hi = aff_zero();
  f.lo.b = v;
  f.hi.b = v;
  return f;
}
// concretisation: conc(f) = [lb - |lA|_1, ub + |uA|_1]
void conc(const Form& f, int n, double& lo, double& hi) {
  lo = aff_min(f.lo, n);
  hi = aff_max(f.hi, n);
}
// R0: Add (Table 1) -- exact
Form add(const Form& f, const Form& g) {
  Form r;
  r.lo = aff_add(f.lo, g.lo);
  r.hi = aff_add(f.hi, g.hi);
  return r;
}
// R0: multiplication by a constant c (Mul / Mmul with a constant operand) -- exact
Form scale(const Form& f, double c) {
  Form r;
  if (c >= 0) {
    r.lo = aff_scale(f.lo, c);
    r.hi = aff_scale(f.hi, c);
  } else {
    r.lo = aff_scale(f.hi, c);
    r.hi = aff_scale(f.lo, c);
  }
  return r;
}
Form add_const(const Form& f, double c) {
  Form r = f;
  r.lo.b += c;
  r.hi.b += c;
  return r;
}
// LS(f,c) / US(f,c): lower / upper affine function of c*f
Aff LS(const Form& f, double c) { return c >= 0 ? aff_scale(f.lo, c) : aff_scale(f.hi, c); }
Aff US(const Form& f, double c) { return c >= 0 ? aff_scale(f.hi, c) : aff_scale(f.lo, c); }

// R1: Mul of two forms (Table 1 Mul/Mmul; rule G1, fixed McCormick planes):
//   lower = LS(f, y_lo) + LS(g, x_lo) - x_lo*y_lo     ((x-x_lo)(y-y_lo) >= 0)
//   upper = US(f, y_hi) + US(g, x_lo) - x_lo*y_hi     ((x-x_lo)(y-y_hi) <= 0)
Form mul(const Form& f, const Form& g, int n) {
  double xl, xh, yl, yh;
  conc(f, n, xl, xh);
  conc(g, n, yl, yh);
  Form r;
  r.lo = aff_add(LS(f, yl), LS(g, xl));
  r.lo.b -= xl * yl;
  r.hi = aff_add(US(f, yh), US(g, xl));
  r.hi.b -= xl * yh;
  return r;
}
// R2: square of one form (rule G2): lower = tangent at p = clamp(0, x_lo, x_hi),
// upper = chord through (x_lo, x_lo^2), (x_hi, x_hi^2).
Form sq(const Form& f, int n) {
  double xl, xh;
  conc(f, n, xl, xh);
  double p = std::min(std::max(0.0, xl), xh);
  Form r;
  r.lo = LS(f, 2.0 * p);
  r.lo.b -= p * p;
  r.hi = US(f, xl + xh);
  r.hi.b -= xl * xh;
  return r;
}

// ---------------------------------------------------------------- rotation (G9)
// R_c2w = Rz(e2) Ry(e1) Rx(e0)  ("XYZ Euler angles")
void mat3_mul(const double* A, const double* B, double* C) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0;
      for (int k = 0; k < 3; ++k) s += A[3 * i + k] * B[3 * k + j];
      C[3 * i + j] = s;
    }
}
void rot_x(double a, double* M, bool deriv) {
  double c = std::cos(a), s = std::sin(a);
  if (!deriv) {
    double m[9] = {1, 0, 0, 0, c, -s, 0, s, c};
    std::memcpy(M, m, sizeof m);
  } else {
    double m[9] = {0, 0, 0, 0, -s, -c, 0, c, -s};
    std::memcpy(M, m, sizeof m);
  }
}
void rot_y(double a, double* M, bool deriv) {
  double c = std::cos(a), s = std::sin(a);
  if (!deriv) {
    double m[9] = {c, 0, s, 0, 1, 0, -s, 0, c};
    std::memcpy(M, m, sizeof m);
  } else {
    double m[9] = {-s, 0, c, 0, 0, 0, -c, 0, -s};
    std::memcpy(M, m, sizeof m);
  }
}
void rot_z(double a, double* M, bool deriv) {
  double c = std::cos(a), s = std::sin(a);
  if (!deriv) {
    double m[9] = {c, -s, 0, s, c, 0, 0, 0, 1};
    std::memcpy(M, m, sizeof m);
  } else {
    double m[9] = {-s, -c, 0, c, -s, 0, 0, 0, 0};
    std::memcpy(M, m, sizeof m);
  }
}
// R_c2w(e) and, if which >= 0, its partial derivative w.r.t. e[which]
void rot_c2w(const double* e, int which, double* R) {
  double X[9], Y[9], Z[9], T[9];
  rot_x(e[0], X, which == 0);
  rot_y(e[1], Y, which == 1);
  rot_z(e[2], Z, which == 2);
  mat3_mul(Z, Y, T);
  mat3_mul(T, X, R);
}

// ---------------------------------------------------------------- box / sub-boxes (a0)
struct Axis {
  double lo, hi;  // full range of the parameter offset
  int parts;
};
struct VarDef {
  int axis;       // 0..2 translation, 3..5 Euler, 6..8 group shift
  double c, r;    // parameter = c + r * xi
};
struct SubBox {
  int n;   // form variables: the shared ones (v[0..ns)) then the private mean offsets
  int ns;  // shared variables (pose axes and group shifts)
  VarDef v[NV];
  double fixed[9];  // parameter value on every axis when xi = 0 (centre or fixed value)
};

struct Problem {
  int64_t N;
  const float *mean, *chol, *opacity, *color;
  or_camera cam;
  or_pose_box box;
  int n_groups;
  const int32_t* group_of;
  double dir[3][3];
  const float *col_lo, *col_hi, *op_lo, *op_hi;
  const float *priv_lo, *priv_hi;  // per-Gaussian private mean offsets (NEXT-2)
  int n_priv;                      // 3 when present, else 0
  Axis axes[9];
  int n_sub;
};

int setup_problem(Problem& P, int64_t N, const float* mean, const float* chol, const float* opacity,
                  const float* color, const or_camera* cam, const or_pose_box* box,
                  const or_scene_box* sbox) {
  if (N < 0 || !cam || !box) return -1;
  if (N > 0 && (!mean || !chol || !opacity || !color)) return -1;
  P.N = N;
  P.mean = mean;
  P.chol = chol;
  P.opacity = opacity;
  P.color = color;
  P.cam = *cam;
  P.box = *box;
  P.n_groups = sbox ? sbox->n_groups : 0;
  if (P.n_groups < 0 || P.n_groups > 3) return -1;
  P.group_of = sbox ? sbox->group_of : nullptr;
  if (P.n_groups > 0 && !P.group_of) return -1;
  P.col_lo = sbox ? sbox->col_lo : nullptr;
  P.col_hi = sbox ? sbox->col_hi : nullptr;
  P.op_lo = sbox ? sbox->op_lo : nullptr;
  P.op_hi = sbox ? sbox->op_hi : nullptr;
  P.priv_lo = sbox ? sbox->priv_lo : nullptr;
  P.priv_hi = sbox ? sbox->priv_hi : nullptr;
  if ((P.priv_lo == nullptr) != (P.priv_hi == nullptr)) return -1;
  P.n_priv = P.priv_lo ? 3 : 0;
  for (int64_t i = 0; P.priv_lo && i < 3 * N; ++i)
    if (!(P.priv_lo[i] <= P.priv_hi[i]) || !std::isfinite(P.priv_lo[i]) ||
        !std::isfinite(P.priv_hi[i]))
      return -1;
  if ((P.col_lo == nullptr) != (P.col_hi == nullptr)) return -1;
  if ((P.op_lo == nullptr) != (P.op_hi == nullptr)) return -1;
  for (int a = 0; a < 3; ++a) {
    if (!(box->eps_t[a] >= 0) || !(box->eps_R[a] >= 0)) return -1;
    P.axes[a] = {box->t_off[a] - box->eps_t[a], box->t_off[a] + box->eps_t[a], box->parts[a]};
    P.axes[3 + a] = {box->R_off[a] - box->eps_R[a], box->R_off[a] + box->eps_R[a],
                     box->parts[3 + a]};
  }
  for (int g = 0; g < 3; ++g) {
    if (g < P.n_groups) {
      for (int b = 0; b < 3; ++b) P.dir[g][b] = sbox->dir[3 * g + b];
      if (!(sbox->shift_hi[g] >= sbox->shift_lo[g])) return -1;
      P.axes[6 + g] = {sbox->shift_lo[g], sbox->shift_hi[g], sbox->parts[g]};
    } else {
      for (int b = 0; b < 3; ++b) P.dir[g][b] = 0;
      P.axes[6 + g] = {0, 0, 1};
    }
  }
  P.n_sub = 1;
  int nvar = 0;
  for (int a = 0; a < 9; ++a) {
    if (P.axes[a].parts < 1) return -1;
    bool var = P.axes[a].hi > P.axes[a].lo;
    if (!var && P.axes[a].parts != 1) return -1;  // partitions only on perturbed axes
    if (var) ++nvar;
    P.n_sub *= P.axes[a].parts;
  }
  if (box->n_explicit < 0) return -1;
  if (box->k_tol > 0 && (box->k_max < K_TAYLOR || box->k_max > 64)) return -1;
  if (box->n_explicit > 0) {  // explicit partition: each sub-box inside the box
    if (!box->explicit_bounds) return -1;
    for (int s = 0; s < box->n_explicit; ++s)
      for (int a = 0; a < 9; ++a) {
        const double lo = box->explicit_bounds[(s * 9 + a) * 2];
        const double hi = box->explicit_bounds[(s * 9 + a) * 2 + 1];
        if (!(lo <= hi) || lo < P.axes[a].lo || hi > P.axes[a].hi) return -1;
      }
    P.n_sub = box->n_explicit;
  }
  if (nvar + P.n_priv > NV) return -1;
  if (cam->W <= 0 || cam->H <= 0) return -1;
  return 0;
}

// sub-box s: multi-index over axes (axis 0 fastest), uniform split (G18)
SubBox make_subbox_shared(const Problem& P, int s);
SubBox make_subbox(const Problem& P, int s) {
  SubBox B = make_subbox_shared(P, s);
  B.ns = B.n;
  B.n += P.n_priv;
  return B;
}
SubBox make_subbox_shared(const Problem& P, int s) {
  SubBox B;
  B.n = 0;
  if (P.box.n_explicit > 0) {  // explicit partition: centre / half-width of each axis
    for (int a = 0; a < 9; ++a) {
      const double lo = P.box.explicit_bounds[(s * 9 + a) * 2];
      const double hi = P.box.explicit_bounds[(s * 9 + a) * 2 + 1];
      const double c = 0.5 * (lo + hi);
      if (P.axes[a].hi > P.axes[a].lo) {  // a variable of the full box (possibly zero width here)
        B.v[B.n++] = {a, c, 0.5 * (hi - lo)};
      }
      B.fixed[a] = c;
    }
    return B;
  }
  int rem = s;
  for (int a = 0; a < 9; ++a) {
    const Axis& ax = P.axes[a];
    int m = rem % ax.parts;
    rem /= ax.parts;
    if (ax.hi > ax.lo) {
      double w = ax.hi - ax.lo;
      double c = ax.lo + w * (2.0 * m + 1.0) / (2.0 * ax.parts);
      double r = w / (2.0 * ax.parts);
      B.v[B.n++] = {a, c, r};
      B.fixed[a] = c;
    } else {
      B.fixed[a] = ax.lo;
    }
  }
  return B;
}

// ---------------------------------------------------------------- step 1: pose forms
struct Pose {
  Form R[9];  // world->camera rotation R = R_c2w^T (l.2)
  Form t[3];  // camera centre
  Form g[3];  // group shift parameters
};

Pose pose_forms(const Problem& P, const SubBox& B) {
  Pose pose;
  const int n = B.ns;  // the pose depends on the shared variables only
  // Euler centre of this sub-box
  double ec[3];
  for (int k = 0; k < 3; ++k) ec[k] = P.cam.euler[k] + B.fixed[3 + k];
  double Rc[9];
  rot_c2w(ec, -1, Rc);
  double dR[3][9];
  for (int k = 0; k < 3; ++k) rot_c2w(ec, k, dR[k]);
  // Lagrange remainder of the first-order Taylor expansion: each entry of R_c2w is a sum of
  // m_ab products of sines/cosines whose second partials are bounded by 1, so
  // |R(ec+delta) - R(ec) - dR.delta| <= 1/2 m_ab (sum_k |delta_k|)^2  (step 1, G9).
  static const double m[9] = {1, 2, 2, 1, 2, 2, 1, 1, 1};
  double rsum = 0;
  for (int i = 0; i < n; ++i)
    if (B.v[i].axis >= 3 && B.v[i].axis < 6) rsum += B.v[i].r;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      // R_ab = R_c2w[b][a]
      int src = 3 * b + a;
      Form f = constant(Rc[src]);
      for (int i = 0; i < n; ++i) {
        int ax = B.v[i].axis;
        if (ax >= 3 && ax < 6) {
          double s = dR[ax - 3][src] * B.v[i].r;
          f.lo.A[i] = s;
          f.hi.A[i] = s;
        }
      }
      double w = 0.5 * m[src] * rsum * rsum;
      f.lo.b -= w;
      f.hi.b += w;
      pose.R[3 * a + b] = f;
    }
  // translation: t = t0 + Mf (offset), Mf = I (world) or R_c2w(nominal euler) (camera axes)
  double Mf[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  if (P.box.t_frame == 1) rot_c2w(P.cam.euler, -1, Mf);
  for (int a = 0; a < 3; ++a) {
    Form f = constant(P.cam.t[a]);
    for (int b = 0; b < 3; ++b) {
      f.lo.b += Mf[3 * a + b] * B.fixed[b];
      f.hi.b += Mf[3 * a + b] * B.fixed[b];
    }
    for (int i = 0; i < n; ++i) {
      int ax = B.v[i].axis;
      if (ax < 3) {
        double s = Mf[3 * a + ax] * B.v[i].r;
        f.lo.A[i] = s;
        f.hi.A[i] = s;
      }
    }
    pose.t[a] = f;
  }
  for (int g = 0; g < 3; ++g) {
    Form f = constant(B.fixed[6 + g]);
    for (int i = 0; i < n; ++i)
      if (B.v[i].axis == 6 + g) {
        f.lo.A[i] = B.v[i].r;
        f.hi.A[i] = B.v[i].r;
      }
    pose.g[g] = f;
  }
  return pose;
}

// ---------------------------------------------------------------- steps 2-11 per Gaussian
enum { GF_DROP = 1, GF_STRADDLE = 2, GF_FAIL = 4 };

struct GRec {
  int flags;
  Form uc[3], d, up[2], Mp[2][3], X[3], conic[4], W[2][3], D2, DU[2];
  double eps, rho;
  int k;                // Taylor order used by MatrixInv
  double kappa;         // sort key: mid of d's forms at xi = 0 (step 12)
  double mu_lo[2], mu_hi[2], r2;  // footprint (step 11, G12)
  double o_lo, o_hi, c_lo[3], c_hi[3];
};

// Adaptive order (P:470 (3)): the smallest k >= k0 with Eps(k) = |X0|_F rho^(k+1) / (1 - rho)
// <= tol, at most kmax (tol <= 0: k0).  rho^(k+1) by repeated multiplication (reproducible).
int adaptive_k(double nx0, double rho, int k0, double tol, int kmax) {
  if (!(tol > 0)) return k0;
  double r = 1.0;
  for (int i = 0; i < k0 + 1; ++i) r *= rho;
  int k = k0;
  while (k < kmax && nx0 * r / (1.0 - rho) > tol) {
    r *= rho;
    ++k;
  }
  return k;
}

// MatrixInv (Alg. 4) on forms X[4] (row-major).  Returns 0 / 1 (det<=0) / 2 (rho>=1)
// k < 0 selects the order adaptively: k = adaptive_k(|X0|_F, rho, 8, k_tol, k_max).
int matrix_inv(const Form* X, int n, int k, Form* conic, double& eps, double& rho,
               double k_tol = 0.0, int k_max = 8, int* k_used = nullptr, bool backward = false) {
  // (1) X0 = inverse of the centre matrix of the input set (P:470, P:550 footnote)
  double Xc[4];
  for (int e = 0; e < 4; ++e) {
    double lo, hi;
    conc(X[e], n, lo, hi);
    Xc[e] = 0.5 * (lo + hi);
  }
  double det = Xc[0] * Xc[3] - Xc[1] * Xc[2];
  eps = 0;
  rho = 0;
  if (!(det > 0)) return 1;  // G11 / reading O2: non-positive centre determinant => FAIL
  double X0[4] = {Xc[3] / det, -Xc[1] / det, -Xc[2] / det, Xc[0] / det};
  // l.1  IXX0 = I - Mmul(X, X0)   (exact: X0 constant)
  Form E[4];
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) {
      Form s = scale(X[2 * a + 0], -X0[0 * 2 + b]);
      s = add(s, scale(X[2 * a + 1], -X0[1 * 2 + b]));
      E[2 * a + b] = add_const(s, a == b ? 1.0 : 0.0);
    }
  // l.2  Assert Norm(IXX0) < 1, with the interval Frobenius upper bound (R5, G13)
  double ss = 0;
  for (int e = 0; e < 4; ++e) {
    double lo, hi;
    conc(E[e], n, lo, hi);
    double mx = std::max(std::fabs(lo), std::fabs(hi));
    ss += mx * mx;
  }
  rho = std::sqrt(ss);
  if (!(rho < 1.0)) return 2;
  if (k < 0) {
    const double nx = std::sqrt(X0[0] * X0[0] + X0[1] * X0[1] + X0[2] * X0[2] + X0[3] * X0[3]);
    k = adaptive_k(nx, rho, 8, k_tol, k_max);
  }
  if (k_used) *k_used = k;
  // l.3  Xa = Mmul(X0, Pow(IXX0, i)), i = 0..k ; Pow as a left fold P^i = P^{i-1} . E
  //      (Mmul of two form matrices uses R1, or R2 when both operands are the same form)
  std::vector<Form> Pw(4), Pn(4);
  Form Xp[4];
  for (int e = 0; e < 4; ++e) Xp[e] = constant(0.0);
  std::vector<double> Bl((k + 1) * 4), Bh((k + 1) * 4);  // bounds of P^i entries (backward)
  for (int i = 0; i <= k; ++i) {
    if (i == 0) {
      Pw[0] = constant(1.0);
      Pw[1] = constant(0.0);
      Pw[2] = constant(0.0);
      Pw[3] = constant(1.0);
    } else if (i == 1) {
      for (int e = 0; e < 4; ++e) Pw[e] = E[e];
    } else {
      for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) {
          Form acc = constant(0.0);
          for (int l = 0; l < 2; ++l) {
            const Form& f = Pw[2 * a + l];
            const Form& g = E[2 * l + b];
            // at i = 2 the operand P^1_al is literally E_al: same form iff (a,l) == (l,b)
            bool same = (i == 2) && (a == l) && (l == b);
            acc = add(acc, same ? sq(f, n) : mul(f, g, n));
          }
          Pn[2 * a + b] = acc;
        }
      Pw = Pn;
    }
    for (int e = 0; e < 4; ++e) conc(Pw[e], n, Bl[i * 4 + e], Bh[i * 4 + e]);
    // Xa = X0 . P^i (exact), l.4 Xp = Sum(Xa)
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) {
        Form xa = add(scale(Pw[0 * 2 + b], X0[2 * a + 0]), scale(Pw[1 * 2 + b], X0[2 * a + 1]));
        Xp[2 * a + b] = add(Xp[2 * a + b], xa);
      }
  }
  // l.5  Eps = Norm(X0) * Norm(IXX0)^(k+1) / (1 - Norm(IXX0))
  double nx0 = std::sqrt(X0[0] * X0[0] + X0[1] * X0[1] + X0[2] * X0[2] + X0[3] * X0[3]);
  eps = nx0 * std::pow(rho, k + 1) / (1.0 - rho);
  // l.6-7  lXinv = Xp - Eps, uXinv = Xp + Eps; union of the two sets
  for (int e = 0; e < 4; ++e) {
    conic[e] = Xp[e];
    conic[e].lo.b -= eps;
    conic[e].hi.b += eps;
  }
  if (!backward) return 0;
  // NEXT-4 (CROWN-style back-substitution): the lower / upper affine bound of
  // each conic entry by propagating its coefficients backwards through
  // Xp = X0 + X0 sum_i P^i, P^i = P^{i-1} E with the same R1 planes (R2 at i = 2 on the
  // diagonal) down to E = I - X X0, affine in the box variables, so the product relaxations
  // are not compounded.  The planes use the forward pass's bounds of P^{i-1} and E.
  double El[4], Eh[4];
  for (int e = 0; e < 4; ++e) conc(E[e], n, El[e], Eh[e]);
  // lower affine bound of  cst + sum_{i=1..top} sum_e lam[i][e] P^i_e   (P^1 = E)
  auto backsub = [&](std::vector<double> lam, int top, double cst) -> Aff {
    double mu[4] = {0, 0, 0, 0};
    for (int i = top; i >= 2; --i)
      for (int c = 0; c < 2; ++c)
        for (int d = 0; d < 2; ++d) {
          const double lm = lam[i * 4 + 2 * c + d];
          if (lm == 0.0) continue;
          for (int l = 0; l < 2; ++l) {
            const double xl = Bl[(i - 1) * 4 + 2 * c + l];
            const double yl = El[2 * l + d], yh = Eh[2 * l + d];
            // R1: lower plane yl f + xl g - xl yl, upper plane yh f + xl g - xl yh (squares
            // E_cc E_cc included: their lower plane is the tangent at the lower end, reading O17)
            const double yy = lm >= 0 ? yl : yh;
            lam[(i - 1) * 4 + 2 * c + l] += lm * yy;
            mu[2 * l + d] += lm * xl;
            cst -= lm * xl * yy;
          }
        }
    Aff r = aff_zero();
    r.b = cst;
    for (int e = 0; e < 4; ++e) {
      const double ce = mu[e] + lam[4 + e];
      r = aff_add(r, ce >= 0 ? aff_scale(E[e].lo, ce) : aff_scale(E[e].hi, ce));
    }
    return r;
  };
  // intermediate bounds by back-substitution too (CROWN): level by level, each
  // entry of P^i is bounded by propagating it back to E with the (already refined) bounds
  // of the levels below, intersected with its forward bound (both are sound)
  for (int i = 2; i <= k; ++i)
    for (int e = 0; e < 4; ++e)
      for (int side = 0; side < 2; ++side) {
        const double sg = side == 0 ? 1.0 : -1.0;
        std::vector<double> lam((k + 1) * 4, 0.0);
        lam[i * 4 + e] = sg;
        const Aff b = backsub(lam, i, 0.0);
        double lo = b.b;
        for (int v = 0; v < n; ++v) lo -= std::fabs(b.A[v]);
        if (side == 0)
          Bl[i * 4 + e] = std::max(Bl[i * 4 + e], lo);
        else
          Bh[i * 4 + e] = std::min(Bh[i * 4 + e], -lo);
      }
  for (int out = 0; out < 4; ++out) {
    const int oa = out / 2, ob = out % 2;
    for (int side = 0; side < 2; ++side) {
      const double sg = side == 0 ? 1.0 : -1.0;  // lower bound of sg * Conic_ab
      std::vector<double> lam((k + 1) * 4, 0.0);
      for (int i = 1; i <= k; ++i)
        for (int m = 0; m < 2; ++m) lam[i * 4 + 2 * m + ob] = sg * X0[2 * oa + m];
      const Aff bnd = backsub(lam, k, sg * X0[out]);  // i = 0 term: X0 . I
      // keep, per entry and side, the tighter (by concretisation) of the forward form and
      // the back-substituted bound: both are sound
      auto lower_of = [&](const Aff& a) {
        double v = a.b;
        for (int t = 0; t < n; ++t) v -= std::fabs(a.A[t]);
        return v;
      };
      if (side == 0) {
        Aff cand = bnd;
        cand.b -= eps;
        if (lower_of(cand) > lower_of(conic[out].lo)) conic[out].lo = cand;
      } else {
        Aff cand = aff_scale(bnd, -1.0);
        cand.b += eps;
        if (-lower_of(aff_scale(cand, -1.0)) < -lower_of(aff_scale(conic[out].hi, -1.0)))
          conic[out].hi = cand;
      }
    }
  }
  return 0;
}

GRec gaussian_setup(const Problem& P, const SubBox& B, const Pose& pose, int64_t i) {
  const int n = B.n;
  GRec G;
  G.flags = 0;
  const or_camera& C = P.cam;
  // scene parameters of Gaussian i (D1)
  double uw[3], Mw[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int b = 0; b < 3; ++b) uw[b] = (double)P.mean[3 * i + b];
  const float* ch = P.chol + 6 * i;  // lower triangle row-major: m00 m10 m11 m20 m21 m22
  Mw[0] = ch[0];
  Mw[3] = ch[1];
  Mw[4] = ch[2];
  Mw[6] = ch[3];
  Mw[7] = ch[4];
  Mw[8] = ch[5];
  int grp = (P.n_groups > 0) ? P.group_of[i] : -1;
  // l.2  uc = Mmul(R, Add(uw, -t))  (the group shift adds s*dir to uw)
  Form v[3];
  for (int b = 0; b < 3; ++b) {
    Form w = constant(uw[b]);
    if (grp >= 0 && grp < P.n_groups) w = add(w, scale(pose.g[grp], P.dir[grp][b]));
    if (P.n_priv) {  // private offset: centre + radius * eta_b, eta_b = variable ns + b
      const double lo = P.priv_lo[3 * i + b], hi = P.priv_hi[3 * i + b];
      w = add_const(w, 0.5 * (lo + hi));
      w.lo.A[B.ns + b] += 0.5 * (hi - lo);
      w.hi.A[B.ns + b] += 0.5 * (hi - lo);
    }
    v[b] = add(w, scale(pose.t[b], -1.0));
  }
  for (int a = 0; a < 3; ++a) {
    Form acc = constant(0.0);
    for (int b = 0; b < 3; ++b) acc = add(acc, mul(pose.R[3 * a + b], v[b], n));
    G.uc[a] = acc;
  }
  // l.3  Mc = Mmul(R, Mw)  (Mw constant: exact)
  Form Mc[9];
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < 3; ++c) {
      Form acc = constant(0.0);
      for (int b = 0; b < 3; ++b) acc = add(acc, scale(pose.R[3 * a + b], Mw[3 * b + c]));
      Mc[3 * a + c] = acc;
    }
  // l.7  d = uc[2]
  G.d = G.uc[2];
  // l.4  J = [[fx*uc2, 0, -fx*uc0], [0, fy*uc2, -fy*uc1]]
  Form J00 = scale(G.uc[2], C.fx), J02 = scale(G.uc[0], -C.fx);
  Form J11 = scale(G.uc[2], C.fy), J12 = scale(G.uc[1], -C.fy);
  // l.5  up = Mmul(K, uc)
  G.up[0] = add(scale(G.uc[0], C.fx), scale(G.uc[2], C.cx));
  G.up[1] = add(scale(G.uc[1], C.fy), scale(G.uc[2], C.cy));
  // l.6  Mp = Mmul(J, Mc)  (zero entries of J contribute exactly 0)
  for (int c = 0; c < 3; ++c) {
    G.Mp[0][c] = add(mul(J00, Mc[0 * 3 + c], n), mul(J02, Mc[2 * 3 + c], n));
    G.Mp[1][c] = add(mul(J11, Mc[1 * 3 + c], n), mul(J12, Mc[2 * 3 + c], n));
  }
  // l.8  X = Mmul(Mp, Mp^T): diagonal with R2, off-diagonal computed once and mirrored (G5)
  Form X00 = constant(0.0), X11 = constant(0.0), X01 = constant(0.0);
  for (int c = 0; c < 3; ++c) {
    X00 = add(X00, sq(G.Mp[0][c], n));
    X11 = add(X11, sq(G.Mp[1][c], n));
    X01 = add(X01, mul(G.Mp[0][c], G.Mp[1][c], n));
  }
  G.X[0] = X00;
  G.X[1] = X01;
  G.X[2] = X11;
  Form Xm[4] = {X00, X01, X01, X11};
  G.k = K_TAYLOR;
  const bool bwd = P.box.inv_backward != 0;
  int st = (P.box.k_tol > 0)
               ? matrix_inv(Xm, n, -1, G.conic, G.eps, G.rho, P.box.k_tol, P.box.k_max, &G.k, bwd)
               : matrix_inv(Xm, n, K_TAYLOR, G.conic, G.eps, G.rho, 0.0, 8, nullptr, bwd);
  if (st != 0) G.flags |= GF_FAIL;
  // l.9 pieces: W = Mmul(Conic, Mp) (association G4), D2 = Mul(d,d), DU = Mul(d, up)
  if (!(G.flags & GF_FAIL)) {
    for (int a = 0; a < 2; ++a)
      for (int c = 0; c < 3; ++c) {
        Form acc = constant(0.0);
        for (int b = 0; b < 2; ++b) acc = add(acc, mul(G.conic[2 * a + b], G.Mp[b][c], n));
        G.W[a][c] = acc;
      }
    // numeric sanity cap (reading O3): a W this large carries no information
    for (int a = 0; a < 2; ++a)
      for (int c = 0; c < 3; ++c) {
        double lo, hi;
        conc(G.W[a][c], n, lo, hi);
        if (!(std::fabs(lo) <= W_CAP && std::fabs(hi) <= W_CAP)) G.flags |= GF_FAIL;
      }
  }
  if (G.flags & GF_FAIL)
    for (int a = 0; a < 2; ++a)
      for (int c = 0; c < 3; ++c) G.W[a][c] = constant(0.0);
  G.D2 = sq(G.d, n);
  G.DU[0] = mul(G.d, G.up[0], n);
  G.DU[1] = mul(G.d, G.up[1], n);
  // opacity / colour intervals (scene box)
  G.o_lo = P.op_lo ? (double)P.op_lo[i] : (double)P.opacity[i];
  G.o_hi = P.op_hi ? (double)P.op_hi[i] : (double)P.opacity[i];
  for (int ch3 = 0; ch3 < 3; ++ch3) {
    G.c_lo[ch3] = P.col_lo ? (double)P.col_lo[3 * i + ch3] : (double)P.color[3 * i + ch3];
    G.c_hi[ch3] = P.col_hi ? (double)P.col_hi[3 * i + ch3] : (double)P.color[3 * i + ch3];
  }
  // step 10: near plane (G8)
  double dl, dh;
  conc(G.d, n, dl, dh);
  if (!(dh > D_MIN) || !(G.o_hi > TAU)) {
    G.flags |= GF_DROP;
  } else if (dl <= D_MIN) {
    G.flags |= GF_STRADDLE;
  }
  // step 12 key
  G.kappa = 0.5 * (G.d.lo.b + G.d.hi.b);
  // step 11 footprint (G12): mu = up/d over [max(d_lo, d_min), d_hi]
  G.r2 = 0;
  G.mu_lo[0] = G.mu_lo[1] = G.mu_hi[0] = G.mu_hi[1] = 0;
  if (!(G.flags & GF_DROP)) {
    double de = std::max(dl, D_MIN);
    for (int a = 0; a < 2; ++a) {
      double ul, uh;
      conc(G.up[a], n, ul, uh);
      double q[4] = {ul / de, ul / dh, uh / de, uh / dh};
      G.mu_lo[a] = std::min(std::min(q[0], q[1]), std::min(q[2], q[3]));
      G.mu_hi[a] = std::max(std::max(q[0], q[1]), std::max(q[2], q[3]));
    }
    double x00l, x00h, x11l, x11h;
    conc(X00, n, x00l, x00h);
    conc(X11, n, x11l, x11h);
    double de2 = de * de;
    double lam = (x00h + x11h) / (de2 * de2);  // >= lambda_max(Sigma_2D), X = d^4 Sigma_2D
    double scut = 2.0 * std::log(G.o_hi / TAU);
    G.r2 = scut * lam;
  }
  return G;
}

// culling test of Gaussian G against a rectangle of pixel centres (G12, reading O1).
// The method's cull is per pixel (x0 == x1, y0 == y1): a Gaussian is dropped at pixel u
// iff dist^2(u, mu-rect) > s_cut * lambda_bar, which implies a <= tau there.  A tile's
// list L_T (tile rectangle) is a superset of every per-pixel list inside it, so TS is a
// pure performance knob: rounding is monotone, so dist^2(rect) <= dist^2(u) in fp too.
bool culled(const GRec& G, double x0, double x1, double y0, double y1) {
  double dx = std::max(0.0, std::max(G.mu_lo[0] - x1, x0 - G.mu_hi[0]));
  double dy = std::max(0.0, std::max(G.mu_lo[1] - y1, y0 - G.mu_hi[1]));
  return dx * dx + dy * dy > G.r2;
}

// step 13: three-valued Ind(d_i - d_j) with the index tie-break (G6).
// returns 1 (j certainly in front of i), 0 (certainly not), -1 ('?')
// Variables k >= ns are private to each Gaussian (NEXT-2): independent in d_i and d_j, so
// their slopes add in absolute value instead of cancelling.
int ind_class(const GRec& Gi, int64_t i, const GRec& Gj, int64_t j, int n, int ns) {
  double dl = Gi.d.lo.b - Gj.d.hi.b, du = Gi.d.hi.b - Gj.d.lo.b;
  double s1 = 0, s2 = 0;
  for (int k = 0; k < ns; ++k) {
    s1 += std::fabs(Gi.d.lo.A[k] - Gj.d.hi.A[k]);
    s2 += std::fabs(Gi.d.hi.A[k] - Gj.d.lo.A[k]);
  }
  for (int k = ns; k < n; ++k) {
    s1 += std::fabs(Gi.d.lo.A[k]) + std::fabs(Gj.d.hi.A[k]);
    s2 += std::fabs(Gi.d.hi.A[k]) + std::fabs(Gj.d.lo.A[k]);
  }
  dl -= s1;  // lower bound of d_i - d_j over the box
  du += s2;  // upper bound
  if (i > j) {
    if (dl >= 0) return 1;
    if (du < 0) return 0;
  } else {
    if (dl > 0) return 1;
    if (du <= 0) return 0;
  }
  return -1;
}

// steps 14-17: effective-opacity interval of Gaussian G at pixel centre u (G7).
// Returns false (and a = [0,0]) when G is culled at u (reading O1).
bool opacity_bounds(const GRec& G, const double u[2], int n, double& alo, double& ahi) {
  if (culled(G, u[0], u[0], u[1], u[1])) {
    alo = 0.0;
    ahi = 0.0;
    return false;
  }
  if (G.flags & GF_FAIL) {
    alo = 0.0;
    ahi = G.o_hi;
    return true;
  }
  // 14: x_a = Add(Mul(d, d, u_a), -Mul(d, up_a)) ; u_a > 0
  Form x[2];
  for (int a = 0; a < 2; ++a) x[a] = add(scale(G.D2, u[a]), scale(G.DU[a], -1.0));
  // 15: q = Mmul(x, W)
  Form s = constant(0.0);
  for (int c = 0; c < 3; ++c) {
    Form q = add(mul(x[0], G.W[0][c], n), mul(x[1], G.W[1][c], n));
    // 16: s = Mmul(q, q^T) = sum_c q_c^2 (R2)
    s = add(s, sq(q, n));
  }
  double sl, sh;
  conc(s, n, sl, sh);
  sl = std::max(sl, 0.0);
  // 17: a = o * Exp(-1/2 s): Table 2 Exp relaxation followed by concretisation gives
  //     [exp(z_lo), exp(z_hi)] with z = -s/2 (R3)
  alo = G.o_lo * std::exp(-0.5 * sh);
  ahi = G.o_hi * std::exp(-0.5 * sl);
  if (G.flags & GF_STRADDLE) alo = 0.0;
  return true;
}

// ---------------------------------------------------------------- per sub-box data
struct SubData {
  SubBox B;
  std::vector<GRec> G;
};

void build_subdata(const Problem& P, int s, SubData& S) {
  S.B = make_subbox(P, s);
  Pose pose = pose_forms(P, S.B);
  S.G.resize(P.N);
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t i = 0; i < P.N; ++i) S.G[i] = gaussian_setup(P, S.B, pose, i);
}

struct TileList {
  std::vector<int64_t> L;                 // Gaussian ids in (kappa, index) order
  std::vector<std::vector<int>> EF, EG;   // exception positions (ascending)
  int64_t uncertain = 0, violations = 0;
};

void tile_rect(const or_camera& C, int ts, int tile, double& x0, double& x1, double& y0,
               double& y1) {
  int ntx = (C.W + ts - 1) / ts;
  int tx = tile % ntx, ty = tile / ntx;
  x0 = tx * ts + 0.5;
  x1 = std::min((tx + 1) * ts, (int)C.W) - 0.5;
  y0 = ty * ts + 0.5;
  y1 = std::min((ty + 1) * ts, (int)C.H) - 0.5;
}

// steps 12-13: L_T, its order, and the '?' pairs
void build_tile_list(const Problem& P, const SubData& S, int ts, int tile, bool classify,
                     TileList& T) {
  double x0, x1, y0, y1;
  tile_rect(P.cam, ts, tile, x0, x1, y0, y1);
  T.L.clear();
  for (int64_t i = 0; i < P.N; ++i) {
    const GRec& G = S.G[i];
    if (G.flags & GF_DROP) continue;
    if (culled(G, x0, x1, y0, y1)) continue;
    T.L.push_back(i);
  }
  std::stable_sort(T.L.begin(), T.L.end(), [&](int64_t a, int64_t b) {
    return S.G[a].kappa < S.G[b].kappa;  // stable: ties keep ascending index
  });
  if (!classify) return;
  const int K = (int)T.L.size();
  const int n = S.B.n;
  T.EF.assign(K, {});
  T.EG.assign(K, {});
  for (int p = 0; p < K; ++p)
    for (int q = 0; q < K; ++q) {
      if (q == p) continue;
      int c = ind_class(S.G[T.L[p]], T.L[p], S.G[T.L[q]], T.L[q], n, S.B.ns);
      if (c == -1) {
        if (q < p)
          T.EF[p].push_back(q);
        else
          T.EG[p].push_back(q);
        if (q > p) ++T.uncertain;
      } else if ((q < p && c == 0) || (q > p && c == 1)) {
        ++T.violations;  // order structure of step 13 broken (must not happen)
      }
    }
}

// steps 18-19, windowed form: prefix products + exception windows (uses step 13 structure).
// unc_only: sum the contributions of the uncertain positions only (E_F or E_G non-empty;
// reading O20's interval part)
void blend_windowed(const SubData& S, const TileList& T, const double* alo, const double* ahi,
                    double pc_lo[3], double pc_hi[3], bool unc_only = false) {
  const int K = (int)T.L.size();
  std::vector<double> Pb(K + 1), Pl(K + 1);
  Pb[0] = 1.0;
  Pl[0] = 1.0;
  for (int p = 0; p < K; ++p) {
    Pb[p + 1] = Pb[p] * (1.0 - alo[p]);
    Pl[p + 1] = Pl[p] * (1.0 - ahi[p]);
  }
  for (int c = 0; c < 3; ++c) pc_lo[c] = pc_hi[c] = 0.0;
  for (int p = 0; p < K; ++p) {
    double Tb, Tl;
    const std::vector<int>& ef = T.EF[p];
    if (ef.empty()) {
      Tb = Pb[p];
    } else {
      int h = ef[0];
      Tb = Pb[h];
      size_t e = 0;
      for (int q = h; q < p; ++q) {
        if (e < ef.size() && ef[e] == q) {
          ++e;
          continue;
        }
        Tb *= 1.0 - alo[q];
      }
    }
    Tl = Pl[p];
    for (int q : T.EG[p]) Tl *= 1.0 - ahi[q];
    if (unc_only && ef.empty() && T.EG[p].empty()) continue;
    const GRec& G = S.G[T.L[p]];
    for (int c = 0; c < 3; ++c) {
      pc_hi[c] += Tb * ahi[p] * G.c_hi[c];
      pc_lo[c] += Tl * alo[p] * G.c_lo[c];
    }
  }
}

// steps 18-19, direct form: Alg. 3 with interval operands, Ind recomputed per pair
void blend_direct(const SubData& S, const std::vector<int64_t>& L, const double* alo,
                  const double* ahi, double pc_lo[3], double pc_hi[3]) {
  const int K = (int)L.size();
  const int n = S.B.n;
  for (int c = 0; c < 3; ++c) pc_lo[c] = pc_hi[c] = 0.0;
  for (int p = 0; p < K; ++p) {
    double Tb = 1.0, Tl = 1.0;  // T_hi over F(i), T_lo over G(i)
    for (int q = 0; q < K; ++q) {
      if (q == p) continue;  // Ind(d_i - d_i) = 0
      int c = ind_class(S.G[L[p]], L[p], S.G[L[q]], L[q], n, S.B.ns);
      if (c == 1) {
        Tb *= 1.0 - alo[q];
        Tl *= 1.0 - ahi[q];
      } else if (c == -1) {
        Tl *= 1.0 - ahi[q];
      }
    }
    const GRec& G = S.G[L[p]];
    for (int c = 0; c < 3; ++c) {
      pc_hi[c] += Tb * ahi[p] * G.c_hi[c];
      pc_lo[c] += Tl * alo[p] * G.c_lo[c];
    }
  }
}

// ---------------------------------------------------------------- NEXT-1: linear blend
// Effective opacity as an affine form (Alg. 1 l.10 with the linear relations kept):
// z = -s/2 from the s forms of steps 14-16; Table 2's Exp relaxation (R3) kept linear:
// lower = tangent at z_lo, e^{z_lo} (1 + z - z_lo), applied to z's lower form; upper = chord
// over [z_lo, z_hi] (slope m = (e^{z_hi} - e^{z_lo}) / (z_hi - z_lo) >= 0; e^{z_hi} at zero
// width), applied to z's upper form; times [o_lo, o_hi] >= 0.  FAIL: [0, o_hi]; straddle:
// lower 0.  Returns false when culled at u (a = 0).
bool opacity_form(const GRec& G, const double u[2], int n, Form& a) {
  if (culled(G, u[0], u[0], u[1], u[1])) return false;
  if (G.flags & GF_FAIL) {
    a = constant(0.0);
    a.hi.b = G.o_hi;
    return true;
  }
  Form x[2];
  for (int c = 0; c < 2; ++c) x[c] = add(scale(G.D2, u[c]), scale(G.DU[c], -1.0));
  Form sf = constant(0.0);
  for (int c = 0; c < 3; ++c) {
    Form q = add(mul(x[0], G.W[0][c], n), mul(x[1], G.W[1][c], n));
    sf = add(sf, sq(q, n));
  }
  double sl, sh;
  conc(sf, n, sl, sh);
  sl = std::max(sl, 0.0);
  const Form z = scale(sf, -0.5);  // z.lo = -s.hi / 2, z.hi = -s.lo / 2
  const double zl = -0.5 * sh, zh = -0.5 * sl;
  const double el = std::exp(zl), eh = std::exp(zh);
  const double m = (zh > zl) ? (eh - el) / (zh - zl) : eh;
  const Form lower = add_const(scale(z, G.o_lo * el), G.o_lo * el * (1.0 - zl));
  const Form upper = add_const(scale(z, G.o_hi * m), G.o_hi * (el - m * zl));
  a.lo = lower.lo;
  a.hi = upper.hi;
  if (G.flags & GF_STRADDLE) a.lo = aff_zero();
  return true;
}

// BlendInd (Alg. 3) with linear relations along the sorted fold (reading O20):
// T_0 = 1, T_{i+1} = Mul(T_i, 1 - a_i) (R1) over every position.  A certain position i (no
// uncertain partner: F(i) = before(i), every later Gaussian certainly behind) contributes
// Mul(T_i, a_i) c_i (R1; c in [c_lo, c_hi] >= 0 scales the lower / upper form); an uncertain
// one contributes its interval term [T_lo a_lo c_lo, T_hi a_hi c_hi] of the interval blend,
// passed in as unc_lo / unc_hi (zero on exception-free lists, where this is the plain fold).
// Culled Gaussians (a = 0) are skipped.
void blend_linear(const SubData& S, const TileList& TL, const std::vector<char>& act,
                  const std::vector<Form>& a, const double unc_lo[3], const double unc_hi[3],
                  double pc_lo[3], double pc_hi[3]) {
  const int n = S.B.n;
  const std::vector<int64_t>& L = TL.L;
  Form T = constant(1.0);
  Form pc[3] = {constant(0.0), constant(0.0), constant(0.0)};
  for (size_t p = 0; p < L.size(); ++p) {
    if (!act[p]) continue;
    const GRec& G = S.G[L[p]];
    if (TL.EF[p].empty() && TL.EG[p].empty()) {
      const Form ta = mul(T, a[p], n);
      for (int c = 0; c < 3; ++c) {
        Form t;
        t.lo = aff_scale(ta.lo, G.c_lo[c]);
        t.hi = aff_scale(ta.hi, G.c_hi[c]);
        pc[c] = add(pc[c], t);
      }
    }
    Form om;  // 1 - a
    om.lo = aff_scale(a[p].hi, -1.0);
    om.lo.b += 1.0;
    om.hi = aff_scale(a[p].lo, -1.0);
    om.hi.b += 1.0;
    T = mul(T, om, n);
  }
  for (int c = 0; c < 3; ++c) {
    pc_lo[c] = aff_min(pc[c].lo, n) + unc_lo[c];
    pc_hi[c] = aff_max(pc[c].hi, n) + unc_hi[c];
  }
}

// steps 20-21 finalise (union step 22 by the caller)
inline void finalise(double N, double pc_lo[3], double pc_hi[3]) {
  for (int c = 0; c < 3; ++c) {
    double l = pc_lo[c] - N * TAU, h = pc_hi[c] + N * TAU;
    pc_lo[c] = std::min(std::max(l, 0.0), 1.0);
    pc_hi[c] = std::min(std::max(h, 0.0), 1.0);
  }
}

void set_threads(int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
}

int render_tiles_impl(const Problem& P, int ts, const std::vector<int>& tiles, int mode,
                      double* lo, double* hi, or_stats* st, int sb0 = 0, int sb1 = -1) {
  const or_camera& C = P.cam;
  int64_t pairs = 0, active = 0, unc = 0, viol = 0, fails = 0, strad = 0, drop = 0;
  int kmax = 0;
  int nvars = 0;
  if (sb1 < 0) sb1 = P.n_sub;
  if (sb0 >= sb1) {  // empty union: the identities of step 22's min / max
    const int ntx = (C.W + ts - 1) / ts;
    for (int tile : tiles) {
      const int tx = tile % ntx, ty = tile / ntx;
      for (int py = ty * ts; py < std::min((ty + 1) * ts, (int)C.H); ++py)
        for (int px = tx * ts; px < std::min((tx + 1) * ts, (int)C.W); ++px)
          for (int c = 0; c < 3; ++c) {
            lo[3 * ((size_t)py * C.W + px) + c] = 1.0;
            hi[3 * ((size_t)py * C.W + px) + c] = 0.0;
          }
    }
  }
  for (int s = sb0; s < sb1; ++s) {
    SubData S;
    build_subdata(P, s, S);
    nvars = S.B.n;
    for (int64_t i = 0; i < P.N; ++i) {
      if (S.G[i].flags & GF_DROP) {
        ++drop;
        continue;
      }
      if (S.G[i].flags & GF_FAIL) ++fails;
      if (S.G[i].flags & GF_STRADDLE) ++strad;
    }
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : pairs, active, unc, viol) reduction(max : kmax)
    for (size_t ti = 0; ti < tiles.size(); ++ti) {
      int tile = tiles[ti];
      TileList T;
      build_tile_list(P, S, ts, tile, mode != 1, T);
      const int K = (int)T.L.size();
      pairs += K;
      unc += T.uncertain;
      viol += T.violations;
      kmax = std::max(kmax, K);
      std::vector<double> alo(K), ahi(K);
      int ntx = (C.W + ts - 1) / ts;
      int tx = tile % ntx, ty = tile / ntx;
      for (int py = ty * ts; py < std::min((ty + 1) * ts, (int)C.H); ++py)
        for (int px = tx * ts; px < std::min((tx + 1) * ts, (int)C.W); ++px) {
          double u[2] = {px + 0.5, py + 0.5};
          for (int p = 0; p < K; ++p) active += opacity_bounds(S.G[T.L[p]], u, S.B.n, alo[p], ahi[p]);
          double pl[3], ph[3];
          if (mode == 1)
            blend_direct(S, T.L, alo.data(), ahi.data(), pl, ph);
          else
            blend_windowed(S, T, alo.data(), ahi.data(), pl, ph);
          finalise((double)P.N, pl, ph);
          if (mode == 2) {
            // NEXT-1: linear-relation blend (certain positions as forms, uncertain ones as
            // interval terms, O20), intersected with the interval blend (both sound)
            std::vector<char> act(K);
            std::vector<Form> af(K);
            for (int p = 0; p < K; ++p) act[p] = opacity_form(S.G[T.L[p]], u, S.B.n, af[p]);
            double ul[3] = {0, 0, 0}, uh[3] = {0, 0, 0};
            if (T.uncertain > 0) blend_windowed(S, T, alo.data(), ahi.data(), ul, uh, true);
            double ql[3], qh[3];
            blend_linear(S, T, act, af, ul, uh, ql, qh);
            finalise((double)P.N, ql, qh);
            for (int c = 0; c < 3; ++c) {
              pl[c] = std::max(pl[c], ql[c]);
              ph[c] = std::min(ph[c], qh[c]);
            }
          }
          size_t o = 3 * ((size_t)py * C.W + px);
          for (int c = 0; c < 3; ++c) {
            if (s == sb0) {
              lo[o + c] = pl[c];
              hi[o + c] = ph[c];
            } else {  // step 22: union over sub-boxes
              lo[o + c] = std::min(lo[o + c], pl[c]);
              hi[o + c] = std::max(hi[o + c], ph[c]);
            }
          }
        }
    }
  }
  if (st) {
    st->pairs = pairs;
    st->active_pairs = active;
    st->uncertain_pairs = unc;
    st->order_violations = viol;
    st->fails = fails;
    st->straddles = strad;
    st->dropped = drop;
    st->kmax = kmax;
    st->n_sub = sb1 > sb0 ? sb1 - sb0 : 0;
    st->n_vars = nvars;
    st->pad = 0;
  }
  return 0;
}

// ---------------------------------------------------------------- form <-> flat arrays
void form_from(const double* p, int n, Form& f) {
  f.lo = aff_zero();
  f.hi = aff_zero();
  for (int k = 0; k < n; ++k) f.lo.A[k] = p[k];
  f.lo.b = p[n];
  for (int k = 0; k < n; ++k) f.hi.A[k] = p[n + 1 + k];
  f.hi.b = p[2 * n + 1];
}
void form_to(const Form& f, int n, double* p) {
  for (int k = 0; k < n; ++k) p[k] = f.lo.A[k];
  p[n] = f.lo.b;
  for (int k = 0; k < n; ++k) p[n + 1 + k] = f.hi.A[k];
  p[2 * n + 1] = f.hi.b;
}

// concrete rendering quantities of one Gaussian at one pose (Alg. 1 l.2-10 literal)
struct Concrete {
  bool keep;
  double d, up[2], Conic[4], Mp[6];
};
Concrete concrete_gaussian(const float* mean, const float* chol, int64_t i, const double* R,
                           const double* t, const double* shift3, const or_camera& C) {
  Concrete r;
  double uw[3], Mw[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int b = 0; b < 3; ++b) uw[b] = (double)mean[3 * i + b] + shift3[b];
  const float* ch = chol + 6 * i;
  Mw[0] = ch[0];
  Mw[3] = ch[1];
  Mw[4] = ch[2];
  Mw[6] = ch[3];
  Mw[7] = ch[4];
  Mw[8] = ch[5];
  double uc[3], Mc[9];
  for (int a = 0; a < 3; ++a) {  // l.2
    double s = 0;
    for (int b = 0; b < 3; ++b) s += R[3 * a + b] * (uw[b] - t[b]);
    uc[a] = s;
  }
  mat3_mul(R, Mw, Mc);  // l.3
  double J[6] = {C.fx * uc[2], 0, -C.fx * uc[0], 0, C.fy * uc[2], -C.fy * uc[1]};  // l.4
  r.up[0] = C.fx * uc[0] + C.cx * uc[2];  // l.5
  r.up[1] = C.fy * uc[1] + C.cy * uc[2];
  for (int a = 0; a < 2; ++a)  // l.6
    for (int c = 0; c < 3; ++c) {
      double s = 0;
      for (int b = 0; b < 3; ++b) s += J[3 * a + b] * Mc[3 * b + c];
      r.Mp[3 * a + c] = s;
    }
  r.d = uc[2];  // l.7
  double X[4];
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) {
      double s = 0;
      for (int c = 0; c < 3; ++c) s += r.Mp[3 * a + c] * r.Mp[3 * b + c];
      X[2 * a + b] = s;
    }
  double det = X[0] * X[3] - X[1] * X[2];  // l.8 Inv (closed-form 2x2)
  r.Conic[0] = X[3] / det;
  r.Conic[1] = -X[1] / det;
  r.Conic[2] = -X[2] / det;
  r.Conic[3] = X[0] / det;
  r.keep = r.d > D_MIN && det > 0;
  return r;
}
double concrete_alpha(const Concrete& g, double o, const double u[2]) {
  // l.9  q = Mmul(Add(Mul(d,d,u), -Mul(d,up)), Conic, Mp)
  double x[2] = {g.d * g.d * u[0] - g.d * g.up[0], g.d * g.d * u[1] - g.d * g.up[1]};
  double xc[2] = {x[0] * g.Conic[0] + x[1] * g.Conic[2], x[0] * g.Conic[1] + x[1] * g.Conic[3]};
  double qq = 0;
  for (int c = 0; c < 3; ++c) {
    double q = xc[0] * g.Mp[c] + xc[1] * g.Mp[3 + c];
    qq += q * q;
  }
  return o * std::exp(-0.5 * qq);  // l.10
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

void or_form_conc(int32_t n, const double* f, double* lo, double* hi) {
  Form F;
  form_from(f, n, F);
  conc(F, n, *lo, *hi);
}
void or_form_mul(int32_t n, const double* f, const double* g, double* out) {
  Form F, Gf;
  form_from(f, n, F);
  form_from(g, n, Gf);
  form_to(mul(F, Gf, n), n, out);
}
void or_form_sq(int32_t n, const double* f, double* out) {
  Form F;
  form_from(f, n, F);
  form_to(sq(F, n), n, out);
}
void or_exp_relax(double xl, double xh, double* lo_slope, double* lo_icpt, double* hi_slope,
                  double* hi_icpt) {
  // Table 2: lower exp(xl)(x - xl) + exp(xl); upper chord
  double el = std::exp(xl), eh = std::exp(xh);
  *lo_slope = el;
  *lo_icpt = el - el * xl;
  double sl = (xh > xl) ? (eh - el) / (xh - xl) : el;
  *hi_slope = sl;
  *hi_icpt = el - sl * xl;
}
int32_t or_ind_relax(double xl, double xh) {
  // Table 2 with Ind(x) = (x > 0)
  if (xl > 0) return 1;
  if (xh <= 0) return 0;
  return -1;
}

int32_t or_matrix_inv_bwd(int32_t n, const double* X, int32_t k, double* conic, double* eps,
                          double* rho) {
  if (n < 0 || n > NV || k < 1) return -1;
  Form Xf[4], Cf[4];
  for (int e = 0; e < 4; ++e) form_from(X + e * 2 * (n + 1), n, Xf[e]);
  int st = matrix_inv(Xf, n, k, Cf, *eps, *rho, 0.0, 8, nullptr, true);
  if (st == 0)
    for (int e = 0; e < 4; ++e) form_to(Cf[e], n, conic + e * 2 * (n + 1));
  return st;
}

int32_t or_matrix_inv(int32_t n, const double* X, int32_t k, double* conic, double* eps,
                      double* rho) {
  if (n < 0 || n > NV || k < 0) return -1;
  Form Xf[4], Cf[4];
  for (int e = 0; e < 4; ++e) form_from(X + e * 2 * (n + 1), n, Xf[e]);
  int st = matrix_inv(Xf, n, k, Cf, *eps, *rho);
  if (st == 0)
    for (int e = 0; e < 4; ++e) form_to(Cf[e], n, conic + e * 2 * (n + 1));
  return st;
}

int32_t or_pose_forms(const or_camera* cam, const or_pose_box* box, const or_scene_box* sbox,
                      int32_t sub, double* R, double* t, int32_t* nvars) {
  Problem P;
  if (setup_problem(P, 0, nullptr, nullptr, nullptr, nullptr, cam, box, sbox) != 0) return -1;
  if (sub < 0 || sub >= P.n_sub) return -1;
  SubBox B = make_subbox(P, sub);
  Pose pose = pose_forms(P, B);
  const int n = B.ns;
  for (int e = 0; e < 9; ++e) form_to(pose.R[e], n, R + e * 2 * (n + 1));
  for (int e = 0; e < 3; ++e) form_to(pose.t[e], n, t + e * 2 * (n + 1));
  *nvars = n;
  return P.n_sub;
}

int32_t or_gaussian_forms_stride(int32_t n) { return 28 * 2 * (n + 1) + 10; }

int32_t or_gaussian_forms(int64_t N, const float* mean, const float* chol, const float* opacity,
                          const float* color, const or_camera* cam, const or_pose_box* box,
                          const or_scene_box* sbox, int32_t sub, double* out, int32_t* nvars) {
  Problem P;
  if (setup_problem(P, N, mean, chol, opacity, color, cam, box, sbox) != 0) return -1;
  if (sub < 0 || sub >= P.n_sub) return -1;
  SubData S;
  build_subdata(P, sub, S);
  const int n = S.B.n;
  const int fs = 2 * (n + 1);
  const int stride = or_gaussian_forms_stride(n);
  for (int64_t i = 0; i < N; ++i) {
    const GRec& G = S.G[i];
    double* o = out + (size_t)i * stride;
    int f = 0;
    for (int a = 0; a < 3; ++a) form_to(G.uc[a], n, o + fs * f++);
    form_to(G.d, n, o + fs * f++);
    for (int a = 0; a < 2; ++a) form_to(G.up[a], n, o + fs * f++);
    for (int a = 0; a < 2; ++a)
      for (int c = 0; c < 3; ++c) form_to(G.Mp[a][c], n, o + fs * f++);
    for (int a = 0; a < 3; ++a) form_to(G.X[a], n, o + fs * f++);
    for (int a = 0; a < 4; ++a) form_to(G.conic[a], n, o + fs * f++);
    for (int a = 0; a < 2; ++a)
      for (int c = 0; c < 3; ++c) form_to(G.W[a][c], n, o + fs * f++);
    form_to(G.D2, n, o + fs * f++);
    for (int a = 0; a < 2; ++a) form_to(G.DU[a], n, o + fs * f++);
    double* sc = o + fs * f;  // f == 28
    sc[0] = G.flags;
    sc[1] = G.eps;
    sc[2] = G.rho;
    sc[3] = G.kappa;
    sc[4] = G.mu_lo[0];
    sc[5] = G.mu_lo[1];
    sc[6] = G.mu_hi[0];
    sc[7] = G.mu_hi[1];
    sc[8] = G.r2;
    sc[9] = G.k;
  }
  *nvars = n;
  return P.n_sub;
}

int or_render_bounds(int64_t N, const float* mean, const float* chol, const float* opacity,
                     const float* color, const or_camera* cam, const or_pose_box* box,
                     const or_scene_box* sbox, int32_t tile, int32_t mode, int32_t nthreads,
                     double* lo, double* hi, or_stats* stats) {
  Problem P;
  if (setup_problem(P, N, mean, chol, opacity, color, cam, box, sbox) != 0) return -1;
  if (tile < 1 || mode < 0 || mode > 2 || !lo || !hi) return -1;
  set_threads(nthreads);
  int ntx = (cam->W + tile - 1) / tile, nty = (cam->H + tile - 1) / tile;
  std::vector<int> tiles(ntx * nty);
  for (int k = 0; k < ntx * nty; ++k) tiles[k] = k;
  return render_tiles_impl(P, tile, tiles, mode, lo, hi, stats);
}

int or_render_subboxes(int64_t N, const float* mean, const float* chol, const float* opacity,
                       const float* color, const or_camera* cam, const or_pose_box* box,
                       const or_scene_box* sbox, int32_t tile, int32_t sub_begin, int32_t sub_end,
                       int32_t nthreads, double* lo, double* hi, or_stats* stats) {
  Problem P;
  if (setup_problem(P, N, mean, chol, opacity, color, cam, box, sbox) != 0) return -1;
  if (tile < 1 || !lo || !hi || sub_begin < 0 || sub_end > P.n_sub || sub_begin > sub_end) return -1;
  set_threads(nthreads);
  int ntx = (cam->W + tile - 1) / tile, nty = (cam->H + tile - 1) / tile;
  std::vector<int> tiles(ntx * nty);
  for (int k = 0; k < ntx * nty; ++k) tiles[k] = k;
  return render_tiles_impl(P, tile, tiles, 0, lo, hi, stats, sub_begin, sub_end);
}

int or_render_tiles(int64_t N, const float* mean, const float* chol, const float* opacity,
                    const float* color, const or_camera* cam, const or_pose_box* box,
                    const or_scene_box* sbox, int32_t tile, int64_t ntiles, const int32_t* tiles,
                    int32_t nthreads, double* lo, double* hi, or_stats* stats) {
  Problem P;
  if (setup_problem(P, N, mean, chol, opacity, color, cam, box, sbox) != 0) return -1;
  if (tile < 1 || !lo || !hi || ntiles < 0) return -1;
  int ntx = (cam->W + tile - 1) / tile, nty = (cam->H + tile - 1) / tile;
  std::vector<int> tl(ntiles);
  for (int64_t k = 0; k < ntiles; ++k) {
    if (tiles[k] < 0 || tiles[k] >= ntx * nty) return -1;
    tl[k] = tiles[k];
  }
  set_threads(nthreads);
  return render_tiles_impl(P, tile, tl, 0, lo, hi, stats);
}

int or_pixel_bounds(int64_t N, const float* mean, const float* chol, const float* opacity,
                    const float* color, const or_camera* cam, const or_pose_box* box,
                    const or_scene_box* sbox, int32_t tile, int64_t npix, const int32_t* px,
                    const int32_t* py, int32_t nthreads, double* lo, double* hi) {
  Problem P;
  if (setup_problem(P, N, mean, chol, opacity, color, cam, box, sbox) != 0) return -1;
  if (tile < 1 || npix < 0) return -1;
  set_threads(nthreads);
  for (int64_t k = 0; k < npix; ++k)
    if (px[k] < 0 || px[k] >= cam->W || py[k] < 0 || py[k] >= cam->H) return -1;
  for (int s = 0; s < P.n_sub; ++s) {
    SubData S;
    build_subdata(P, s, S);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t k = 0; k < npix; ++k) {
      // tile-free definition: every non-dropped Gaussian, culled per pixel (O1)
      std::vector<int64_t> L;
      double u[2] = {px[k] + 0.5, py[k] + 0.5};
      for (int64_t i = 0; i < P.N; ++i) {
        if (S.G[i].flags & GF_DROP) continue;
        if (culled(S.G[i], u[0], u[0], u[1], u[1])) continue;
        L.push_back(i);
      }
      const int K = (int)L.size();
      std::vector<double> alo(K), ahi(K);
      for (int p = 0; p < K; ++p) opacity_bounds(S.G[L[p]], u, S.B.n, alo[p], ahi[p]);
      double pl[3], ph[3];
      blend_direct(S, L, alo.data(), ahi.data(), pl, ph);
      finalise((double)P.N, pl, ph);
      for (int c = 0; c < 3; ++c) {
        if (s == 0) {
          lo[3 * k + c] = pl[c];
          hi[3 * k + c] = ph[c];
        } else {
          lo[3 * k + c] = std::min(lo[3 * k + c], pl[c]);
          hi[3 * k + c] = std::max(hi[3 * k + c], ph[c]);
        }
      }
    }
  }
  return 0;
}

void or_blend_sort(int64_t N, const double* a, const double* c, const double* d, double* pc) {
  // Alg. 2: as, cs = Sort(a, d), Sort(c, d) (stable: ties by ascending index)
  std::vector<int64_t> idx(N);
  for (int64_t i = 0; i < N; ++i) idx[i] = i;
  std::stable_sort(idx.begin(), idx.end(), [&](int64_t x, int64_t y) { return d[x] < d[y]; });
  double Ts = 1.0;  // Ts[i] = Prod(vs, i-1)
  pc[0] = pc[1] = pc[2] = 0.0;
  for (int64_t r = 0; r < N; ++r) {
    int64_t i = idx[r];
    for (int ch = 0; ch < 3; ++ch) pc[ch] += Ts * a[i] * c[3 * i + ch];
    Ts *= 1.0 - a[i];  // vs[i] = 1 - as[i]
  }
}

void or_blend_ind(int64_t N, const double* a, const double* c, const double* d, int32_t tiebreak,
                  double* pc) {
  // Alg. 3: V[i,j] = 1 - a[j] Ind(d[i] - d[j]); T[i] = Prod_j V[i,j]
  pc[0] = pc[1] = pc[2] = 0.0;
  for (int64_t i = 0; i < N; ++i) {
    double T = 1.0;
    for (int64_t j = 0; j < N; ++j) {
      if (j == i) continue;
      bool ind = d[i] - d[j] > 0;
      if (tiebreak && d[i] == d[j] && j < i) ind = true;  // G6
      if (ind) T *= 1.0 - a[j];
    }
    for (int ch = 0; ch < 3; ++ch) pc[ch] += T * a[i] * c[3 * i + ch];
  }
}

int or_render_concrete(int64_t N, const float* mean, const float* chol, const float* opacity,
                       const float* color, const or_camera* cam, int32_t n_groups,
                       const int32_t* group_of, const double* dir, const double* shifts,
                       int32_t blend, int64_t npix, const int32_t* px, const int32_t* py,
                       int32_t nthreads, double* img) {
  if (!cam || N < 0 || n_groups < 0 || n_groups > 3) return -1;
  if (n_groups > 0 && (!group_of || !dir || !shifts)) return -1;
  set_threads(nthreads);
  double Rc2w[9], R[9];
  rot_c2w(cam->euler, -1, Rc2w);
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) R[3 * a + b] = Rc2w[3 * b + a];
  std::vector<Concrete> G(N);
  for (int64_t i = 0; i < N; ++i) {
    double sh[3] = {0, 0, 0};
    int g = n_groups > 0 ? group_of[i] : -1;
    if (g >= 0 && g < n_groups)
      for (int b = 0; b < 3; ++b) sh[b] = shifts[g] * dir[3 * g + b];
    G[i] = concrete_gaussian(mean, chol, i, R, cam->t, sh, *cam);
  }
  // keep only d > d_min (G8); the blend follows with depths d
  std::vector<int64_t> keep;
  for (int64_t i = 0; i < N; ++i)
    if (G[i].keep) keep.push_back(i);
  const int64_t M = keep.size();
  std::vector<double> dk(M), ck(3 * M);
  for (int64_t r = 0; r < M; ++r) {
    dk[r] = G[keep[r]].d;
    for (int ch = 0; ch < 3; ++ch) ck[3 * r + ch] = color[3 * keep[r] + ch];
  }
  const int64_t total = px ? npix : (int64_t)cam->W * cam->H;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t k = 0; k < total; ++k) {
    int x = px ? px[k] : (int)(k % cam->W);
    int y = px ? py[k] : (int)(k / cam->W);
    double u[2] = {x + 0.5, y + 0.5};
    std::vector<double> a(M);
    for (int64_t r = 0; r < M; ++r) a[r] = concrete_alpha(G[keep[r]], opacity[keep[r]], u);
    double pc[3];
    if (blend == 0)
      or_blend_sort(M, a.data(), ck.data(), dk.data(), pc);
    else
      or_blend_ind(M, a.data(), ck.data(), dk.data(), blend == 1, pc);
    for (int ch = 0; ch < 3; ++ch) img[3 * k + ch] = pc[ch];
  }
  return 0;
}

}  // extern "C"
