// k_setup.cu -- rows a0-a5 of the hot path: sub-box pose forms (k_pose) and the per-Gaussian
// fp64 setup (k_setup): Alg. 1 lines 2-8 lifted to affine forms, MatrixInv (Alg. 4) at line 8,
// the line-9 pieces W = Conic Mp, D2 = d^2, DU = d up, the depth key and the footprint.
//
// PAPER.md references: Alg. 1; MatrixInv P:417-449 with X0 = inverse of the centre
// (P:470); relaxations G1/G2; Euler convention P:624 (G9).
#include <cmath>

#include "internal.cuh"

namespace absplat {

// ----------------------------------------------------------------------------- k_pose
// R_c2w = Rz(e2) Ry(e1) Rx(e0) and its partial derivatives.
__device__ void rc2w(const double e[3], int which, double R[9]) {
  double c0, s0, c1, s1, c2, s2;
  sincos(e[0], &s0, &c0);
  sincos(e[1], &s1, &c1);
  sincos(e[2], &s2, &c2);
  double X[9] = {1, 0, 0, 0, c0, -s0, 0, s0, c0};
  double Y[9] = {c1, 0, s1, 0, 1, 0, -s1, 0, c1};
  double Z[9] = {c2, -s2, 0, s2, c2, 0, 0, 0, 1};
  if (which == 0) {
    double d[9] = {0, 0, 0, 0, -s0, -c0, 0, c0, -s0};
    for (int k = 0; k < 9; ++k) X[k] = d[k];
  } else if (which == 1) {
    double d[9] = {-s1, 0, c1, 0, 0, 0, -c1, 0, -s1};
    for (int k = 0; k < 9; ++k) Y[k] = d[k];
  } else if (which == 2) {
    double d[9] = {-s2, -c2, 0, c2, -s2, 0, 0, 0, 0};
    for (int k = 0; k < 9; ++k) Z[k] = d[k];
  }
  double T[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) T[3 * i + j] = Z[3 * i] * Y[j] + Z[3 * i + 1] * Y[3 + j] + Z[3 * i + 2] * Y[6 + j];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) R[3 * i + j] = T[3 * i] * X[j] + T[3 * i + 1] * X[3 + j] + T[3 * i + 2] * X[6 + j];
}

// One thread per sub-box: a0 (uniform partition or explicit list) + a1 (pose forms).
__global__ void k_pose(BoxParams bp, PoseDev* out) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= bp.n_sub) return;
  PoseDev P;
  int n = 0;
  int axis[NVMAX];
  double rr[NVMAX];
  double fixed[9];
  int rem = s;
  for (int a = 0; a < 9; ++a) {
    if (bp.sub) {  // explicit partition (NEXT-3 refinement): centre / half-width per axis
      const double lo = bp.sub[(s * 9 + a) * 2], hi = bp.sub[(s * 9 + a) * 2 + 1];
      fixed[a] = 0.5 * (lo + hi);
      if (bp.hi[a] > bp.lo[a]) {  // a variable of the full box (possibly zero width here)
        axis[n] = a;
        rr[n] = 0.5 * (hi - lo);
        ++n;
      }
      continue;
    }
    const int p = bp.parts[a];
    const int m = rem % p;
    rem /= p;
    if (bp.hi[a] > bp.lo[a]) {
      const double w = bp.hi[a] - bp.lo[a];
      fixed[a] = bp.lo[a] + w * (2.0 * m + 1.0) / (2.0 * p);
      axis[n] = a;
      rr[n] = w / (2.0 * p);
      ++n;
    } else {
      fixed[a] = bp.lo[a];
    }
  }
  P.n = n;
  for (int e = 0; e < 9; ++e)
    for (int k = 0; k <= NVMAX; ++k) P.Rl[e][k] = P.Ru[e][k] = 0.0;
  for (int e = 0; e < 3; ++e)
    for (int k = 0; k <= NVMAX; ++k) P.t[e][k] = P.g[e][k] = 0.0;
  for (int k = 0; k < NVMAX; ++k) P.gslope[k] = 0.0;

  double ec[3] = {bp.euler0[0] + fixed[3], bp.euler0[1] + fixed[4], bp.euler0[2] + fixed[5]};
  double Rc[9], dR[3][9];
  rc2w(ec, -1, Rc);
  for (int k = 0; k < 3; ++k) rc2w(ec, k, dR[k]);
  double rsum = 0.0;
  for (int i = 0; i < n; ++i)
    if (axis[i] >= 3 && axis[i] < 6) rsum += rr[i];
  // number of sin/cos product terms per entry of R_c2w (each with |2nd partials| <= 1)
  const double mcount[9] = {1, 2, 2, 1, 2, 2, 1, 1, 1};
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      const int src = 3 * b + a;  // R (world->camera) = R_c2w^T
      const double w = 0.5 * mcount[src] * rsum * rsum;
      P.Rl[3 * a + b][NVMAX] = Rc[src] - w;
      P.Ru[3 * a + b][NVMAX] = Rc[src] + w;
      for (int i = 0; i < n; ++i)
        if (axis[i] >= 3 && axis[i] < 6) {
          const double sl = dR[axis[i] - 3][src] * rr[i];
          P.Rl[3 * a + b][i] = sl;
          P.Ru[3 * a + b][i] = sl;
        }
    }
  for (int e = 0; e < 9; ++e) {
    double v = P.Rl[e][NVMAX];
    for (int i = 0; i < n; ++i) v -= fabs(P.Rl[e][i]);
    P.Rcl[e] = v;
  }
  // translation: t0 + Mf * offset, Mf = I or R_c2w(nominal Euler) (reading O10)
  double Mf[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  if (bp.t_frame == 1) rc2w(bp.euler0, -1, Mf);
  for (int a = 0; a < 3; ++a) {
    double c = bp.t0[a];
    for (int b = 0; b < 3; ++b) c += Mf[3 * a + b] * fixed[b];
    P.t[a][NVMAX] = c;
    for (int i = 0; i < n; ++i)
      if (axis[i] < 3) P.t[a][i] = Mf[3 * a + axis[i]] * rr[i];
  }
  for (int gi = 0; gi < 3; ++gi) {
    P.g[gi][NVMAX] = fixed[6 + gi];
    for (int i = 0; i < n; ++i)
      if (axis[i] == 6 + gi) P.g[gi][i] = rr[i];
  }
  // common depth slope: derivative of d = R_2.(uw - t) w.r.t. the translation variables
  for (int i = 0; i < n; ++i)
    if (axis[i] < 3) {
      double v = 0.0;
      for (int c = 0; c < 3; ++c) v -= Rc[3 * c + 2] * Mf[3 * c + axis[i]] * rr[i];
      P.gslope[i] = v;
    }
  out[s] = P;
}

void launch_pose(const BoxParams& bp, PoseDev* out, cudaStream_t st) {
  k_pose<<<(bp.n_sub + 63) / 64, 64, 0, st>>>(bp, out);
}

// ----------------------------------------------------------------------------- k_setup
// Layout: 4 lanes (n <= 3), 8 lanes (n <= 7) or 16 lanes per Gaussian, lane k holding
// coefficient k of the lower and the upper affine function of every form (k < NV: slope of
// xi_k, k == NV: constant, k > NV: zero padding).  Concretisation is a shuffle reduction over
// the group.  This keeps the
// ~40 live forms of Alg. 1 + MatrixInv in registers (2 doubles per form per lane) instead
// of spilling ~10 KB per thread.  All control flow is uniform across the Gaussians of a
// warp (selects, no data-dependent branches) so the shuffles stay converged.
namespace {
constexpr unsigned FULL = 0xffffffffu;

struct HL {  // this lane's coefficient of a form: lower, upper
  double l, u;
};

// lanes per Gaussian: 4 when the n + 1 coefficients fit (n <= 3), 8 (n <= 7), else 16
template <int NV>
constexpr int lanes_for() {
  return (NV + 1 <= 4) ? 4 : ((NV + 1 <= 8) ? 8 : 16);
}

template <int W>
__device__ __forceinline__ double hsum(double v) {
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o, W);
  return v;
}

template <int NV>
struct Lane {
  static constexpr int W = lanes_for<NV>();
  int k;
  __device__ __forceinline__ bool slope() const { return k < NV; }
  __device__ __forceinline__ bool cst() const { return k == NV; }
  // conc(f) = [lb - |lA|_1, ub + |uA|_1]
  __device__ __forceinline__ void conc(const HL& f, double& mn, double& mx) const {
    const double a = slope() ? -fabs(f.l) : (cst() ? f.l : 0.0);
    const double b = slope() ? fabs(f.u) : (cst() ? f.u : 0.0);
    mn = hsum<W>(a);
    mx = hsum<W>(b);
  }
  __device__ __forceinline__ HL constant(double v) const {
    const double c = cst() ? v : 0.0;
    return HL{c, c};
  }
  // c * f (exact; sides swap for c < 0)
  __device__ __forceinline__ HL scale(const HL& f, double c) const {
    return (c >= 0) ? HL{c * f.l, c * f.u} : HL{c * f.u, c * f.l};
  }
  __device__ __forceinline__ void axpy(HL& acc, const HL& f, double c) const {
    acc.l += c * ((c >= 0) ? f.l : f.u);
    acc.u += c * ((c >= 0) ? f.u : f.l);
  }
  __device__ __forceinline__ void add_const(HL& f, double lo, double hi) const {
    if (cst()) {
      f.l += lo;
      f.u += hi;
    }
  }
  // acc += x*y, fixed McCormick planes (G1)
  __device__ __forceinline__ void mul_acc(HL& acc, const HL& x, const HL& y) const {
    double xl, xh, yl, yh;
    conc(x, xl, xh);
    conc(y, yl, yh);
    acc.l += yl * ((yl >= 0) ? x.l : x.u) + xl * ((xl >= 0) ? y.l : y.u);
    acc.u += yh * ((yh >= 0) ? x.u : x.l) + xl * ((xl >= 0) ? y.u : y.l);
    add_const(acc, -(xl * yl), -(xl * yh));
  }
  // the same with the operands' concretised bounds given (each form is concretised once and
  // reused by every product it enters: the shuffle reductions dominate this kernel)
  __device__ __forceinline__ void mul_acc_b(HL& acc, const HL& x, double xl, const HL& y, double yl,
                                            double yh) const {
    acc.l += yl * ((yl >= 0) ? x.l : x.u) + xl * ((xl >= 0) ? y.l : y.u);
    acc.u += yh * ((yh >= 0) ? x.u : x.l) + xl * ((xl >= 0) ? y.u : y.l);
    add_const(acc, -(xl * yl), -(xl * yh));
  }
  __device__ __forceinline__ void sq_acc_b(HL& acc, const HL& x, double xl, double xh) const {
    const double p = fmin(fmax(0.0, xl), xh);
    const double tp = 2.0 * p, sh = xl + xh;
    acc.l += tp * ((tp >= 0) ? x.l : x.u);
    acc.u += sh * ((sh >= 0) ? x.u : x.l);
    add_const(acc, -(p * p), -(xl * xh));
  }
  // acc += x*x: tangent at p = clamp(0, x_lo, x_hi), chord (G2)
  __device__ __forceinline__ void sq_acc(HL& acc, const HL& x) const {
    double xl, xh;
    conc(x, xl, xh);
    const double p = fmin(fmax(0.0, xl), xh);
    const double tp = 2.0 * p, sh = xl + xh;
    acc.l += tp * ((tp >= 0) ? x.l : x.u);
    acc.u += sh * ((sh >= 0) ? x.u : x.l);
    add_const(acc, -(p * p), -(xl * xh));
  }
};
}  // namespace

template <int NV>
__global__ void __launch_bounds__(128, 4) k_setup(SetupArgs A) {
  __shared__ PoseDev sp;
  __shared__ unsigned long long s_wsmax;
  if (threadIdx.x == 0) s_wsmax = 0ull;
  {
    const double* src = reinterpret_cast<const double*>(A.pose);
    double* dst = reinterpret_cast<double*>(&sp);
    for (int k = threadIdx.x; k < (int)(sizeof(PoseDev) / sizeof(double)); k += blockDim.x)
      dst[k] = src[k];
  }
  __syncthreads();
  constexpr int W = lanes_for<NV>();
  const Lane<NV> L{(int)(threadIdx.x & (W - 1))};
  const int k = L.k;
  const int64_t gi = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / W;
  const bool live = gi < A.N;
  const int64_t i = live ? gi : (A.N - 1);  // dead lane groups mirror the last Gaussian
  const int kc = (k < NV) ? k : NVMAX;      // coefficient slot in the pose tables
  const bool real = k <= NV;
  auto pose_R = [&](int e) -> HL {
    return real ? HL{sp.Rl[e][kc], sp.Ru[e][kc]} : HL{0.0, 0.0};
  };
  const double fx = A.fx, fy = A.fy, cx = A.cx, cy = A.cy;
  // ---- l.2 uc = Mmul(R, Add(uw, -t)); group shift adds s*dir to uw
  const int grp = A.group_of ? A.group_of[i] : -1;
  HL v[3];
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    double c = real ? -sp.t[b][kc] : 0.0;
    if (grp >= 0 && real) c += A.dir[grp][b] * sp.g[grp][kc];
    if (L.cst()) c += (double)A.mean[3 * i + b];
    if (A.priv_lo) {  // private offset (NEXT-2): centre + radius * eta_b, eta_b = slot ns + b
      const double lo = A.priv_lo[3 * i + b], hi = A.priv_hi[3 * i + b];
      if (L.cst()) c += 0.5 * (lo + hi);
      if (k == A.ns + b) c += 0.5 * (hi - lo);
    }
    v[b] = HL{c, c};
  }
  double vl[3], vh[3];
#pragma unroll
  for (int b = 0; b < 3; ++b) L.conc(v[b], vl[b], vh[b]);
  const double* Rlo = sp.Rcl;  // the R forms' lower bounds, from k_pose
  HL uc[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    HL acc{0.0, 0.0};
#pragma unroll
    for (int b = 0; b < 3; ++b)
      L.mul_acc_b(acc, pose_R(3 * a + b), Rlo[3 * a + b], v[b], vl[b], vh[b]);
    uc[a] = acc;
  }
  // ---- l.4 J, l.5 up = K uc, l.7 d = uc_2
  const HL d = uc[2];
  HL up0 = L.scale(uc[0], fx);
  L.axpy(up0, uc[2], cx);
  HL up1 = L.scale(uc[1], fy);
  L.axpy(up1, uc[2], cy);
  const HL J00 = L.scale(d, fx), J02 = L.scale(uc[0], -fx);
  const HL J11 = L.scale(d, fy), J12 = L.scale(uc[1], -fy);
  // ---- l.3 Mc = Mmul(R, Mw) (exact, Mw constant), l.6 Mp = Mmul(J, Mc)
  const float* ch = A.chol + 6 * i;
  const double Mw[9] = {ch[0], 0.0, 0.0, ch[1], ch[2], 0.0, ch[3], ch[4], ch[5]};
  double j00l, j02l, j11l, j12l, tmp;
  L.conc(J00, j00l, tmp);
  L.conc(J02, j02l, tmp);
  L.conc(J11, j11l, tmp);
  L.conc(J12, j12l, tmp);
  HL Mp[2][3];
  double Mpl[2][3], Mph[2][3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    HL Mc[3];
    double mcl[3], mch[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      HL acc{0.0, 0.0};
#pragma unroll
      for (int b = 0; b < 3; ++b) L.axpy(acc, pose_R(3 * a + b), Mw[3 * b + c]);
      Mc[a] = acc;
      L.conc(acc, mcl[a], mch[a]);
    }
    HL m0{0.0, 0.0}, m1{0.0, 0.0};
    L.mul_acc_b(m0, J00, j00l, Mc[0], mcl[0], mch[0]);
    L.mul_acc_b(m0, J02, j02l, Mc[2], mcl[2], mch[2]);
    L.mul_acc_b(m1, J11, j11l, Mc[1], mcl[1], mch[1]);
    L.mul_acc_b(m1, J12, j12l, Mc[2], mcl[2], mch[2]);
    Mp[0][c] = m0;
    Mp[1][c] = m1;
    L.conc(m0, Mpl[0][c], Mph[0][c]);
    L.conc(m1, Mpl[1][c], Mph[1][c]);
  }
  // ---- l.8 X = Mmul(Mp, Mp^T) (X01 once, mirrored: G5)
  HL X00{0.0, 0.0}, X01{0.0, 0.0}, X11{0.0, 0.0};
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    L.sq_acc_b(X00, Mp[0][c], Mpl[0][c], Mph[0][c]);
    L.sq_acc_b(X11, Mp[1][c], Mpl[1][c], Mph[1][c]);
    L.mul_acc_b(X01, Mp[0][c], Mpl[0][c], Mp[1][c], Mpl[1][c], Mph[1][c]);
  }
  // ---- l.8 Conic = MatrixInv(X; X0, k) (Alg. 4)
  bool ok = true;
  double x00l, x00h, x01l, x01h, x11l, x11h;
  L.conc(X00, x00l, x00h);
  L.conc(X01, x01l, x01h);
  L.conc(X11, x11l, x11h);
  const double c00 = 0.5 * (x00l + x00h), c01 = 0.5 * (x01l + x01h), c11 = 0.5 * (x11l + x11h);
  const double det = c00 * c11 - c01 * c01;
  if (!(det > 0.0)) ok = false;  // reading O2
  const double dsafe = ok ? det : 1.0;
  const double X0[4] = {c11 / dsafe, -c01 / dsafe, -c01 / dsafe, c00 / dsafe};
  HL E[4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const HL& xa0 = (a == 0) ? X00 : X01;
      const HL& xa1 = (a == 0) ? X01 : X11;
      HL e = L.scale(xa0, -X0[b]);
      L.axpy(e, xa1, -X0[2 + b]);
      if (a == b) L.add_const(e, 1.0, 1.0);
      E[2 * a + b] = e;
    }
  double ss = 0.0, Elo[4], Ehi[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    L.conc(E[e], Elo[e], Ehi[e]);
    const double m = fmax(fabs(Elo[e]), fabs(Ehi[e]));
    ss += m * m;
  }
  const double rho = sqrt(ss);
  if (!(rho < 1.0)) ok = false;  // Alg. 4 line 2
  // Taylor order: k = 8 (G14), or adaptively the smallest k >= 8 with
  // Eps(k) = |X0|_F rho^(k+1) / (1 - rho) <= k_tol, at most k_max (P:470 (3)); the decision
  // uses the oracle's operation order without FMA contraction
  int k_own = KTAYLOR;
  if (A.k_tol > 0.0 && ok) {
    const double nx = __dsqrt_rn(__dadd_rn(
        __dadd_rn(__dadd_rn(__dmul_rn(X0[0], X0[0]), __dmul_rn(X0[1], X0[1])), __dmul_rn(X0[2], X0[2])),
        __dmul_rn(X0[3], X0[3])));
    double r = 1.0;
    for (int t = 0; t < KTAYLOR + 1; ++t) r = __dmul_rn(r, rho);
    const double den = __dsub_rn(1.0, rho);
    while (k_own < A.k_max && __ddiv_rn(__dmul_rn(nx, r), den) > A.k_tol) {
      r = __dmul_rn(r, rho);
      ++k_own;
    }
  }
  const int k_warp = __reduce_max_sync(FULL, k_own);  // uniform trip count for the shuffles
  HL P[4], S[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    P[e] = E[e];
    S[e] = E[e];
  }
  // NEXT-4 back-substitution needs the forward bounds of every P^i entry (level 1 = E)
  constexpr int KB = 33;
  double Bl[KB][4], Bh[KB][4];
  const bool bwd = A.inv_backward != 0;
  if (bwd) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      Bl[1][e] = Elo[e];
      Bh[1][e] = Ehi[e];
    }
  }
  double Plo[4], Phi[4];  // concretised P^{it-1} (level 1: E)
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    Plo[e] = Elo[e];
    Phi[e] = Ehi[e];
  }
#pragma unroll 1
  for (int it = 2; it <= k_warp; ++it) {
    const bool acc = it <= k_own;  // beyond this Gaussian's order: computed, not summed
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      HL q0{0.0, 0.0}, q1{0.0, 0.0};  // row a of P^it = P^{it-1} E (O5)
      if (it == 2 && a == 0) {
        L.sq_acc_b(q0, P[0], Plo[0], Phi[0]);
      } else {
        L.mul_acc_b(q0, P[2 * a + 0], Plo[2 * a + 0], E[0], Elo[0], Ehi[0]);
      }
      L.mul_acc_b(q0, P[2 * a + 1], Plo[2 * a + 1], E[2], Elo[2], Ehi[2]);
      L.mul_acc_b(q1, P[2 * a + 0], Plo[2 * a + 0], E[1], Elo[1], Ehi[1]);
      if (it == 2 && a == 1) {
        L.sq_acc_b(q1, P[3], Plo[3], Phi[3]);
      } else {
        L.mul_acc_b(q1, P[2 * a + 1], Plo[2 * a + 1], E[3], Elo[3], Ehi[3]);
      }
      P[2 * a + 0] = q0;
      P[2 * a + 1] = q1;
      if (acc) {
        S[2 * a + 0].l += q0.l;
        S[2 * a + 0].u += q0.u;
        S[2 * a + 1].l += q1.l;
        S[2 * a + 1].u += q1.u;
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      L.conc(P[e], Plo[e], Phi[e]);
      if (bwd && it < KB) {
        Bl[it][e] = Plo[e];
        Bh[it][e] = Phi[e];
      }
    }
  }
  const double nx0 = sqrt(X0[0] * X0[0] + X0[1] * X0[1] + X0[2] * X0[2] + X0[3] * X0[3]);
  const double rs = ok ? rho : 0.0;
  const double eps = nx0 * pow(rs, (double)(k_own + 1)) / (1.0 - rs);
  HL conic[4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      HL xp = L.constant(X0[2 * a + b]);  // Xp = X0 + X0 S
      L.axpy(xp, S[b], X0[2 * a]);
      L.axpy(xp, S[2 + b], X0[2 * a + 1]);
      L.add_const(xp, -eps, eps);      // l.6-7, union
      conic[2 * a + b] = xp;
    }
  if (bwd) {  // uniform over the warp (the refinement shuffles); FAIL Gaussians' results unused
    // NEXT-4 (reading O17): lower affine bound of  cst + sum_{i=1..top} (init + [i == top] lam0) . P^i
    // by propagating the coefficients backwards through P^i = P^{i-1} E with the fixed R1
    // planes (squares included) and the operand bounds Bl / Bh, down to E (affine in xi).
    // The recursion is on scalars (uniform over the lanes); the result is this lane's
    // coefficient of the bound.
    auto backsub = [&](int top, const double (&lam0)[4], const double (&init)[4], double cst) {
      double lam[4], mu[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int e = 0; e < 4; ++e) lam[e] = lam0[e];
#pragma unroll 1
      for (int it = top; it >= 2; --it) {
        double nxt[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) nxt[e] = init[e];
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int dd = 0; dd < 2; ++dd) {
            const double lm = lam[2 * c + dd];
            if (lm == 0.0) continue;
#pragma unroll
            for (int l = 0; l < 2; ++l) {
              const double xl = Bl[it - 1][2 * c + l];
              const double yl = Bl[1][2 * l + dd], yh = Bh[1][2 * l + dd];
              const double yy = lm >= 0 ? yl : yh;
              nxt[2 * c + l] += lm * yy;
              mu[2 * l + dd] += lm * xl;
              cst -= lm * xl * yy;
            }
          }
#pragma unroll
        for (int e = 0; e < 4; ++e) lam[e] = nxt[e];
      }
      double rl = L.cst() ? cst : 0.0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const double ce = mu[e] + lam[e];  // P^1 = E
        rl += ce * (ce >= 0 ? E[e].l : E[e].u);
      }
      return rl;
    };
    // intermediate bounds by back-substitution as well (CROWN), level by level,
    // intersected with the forward ones; levels past this Gaussian's order run for the
    // uniform shuffle trip count and are unused
    const double zero4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 1
    for (int it = 2; it <= k_warp && it < KB; ++it)
#pragma unroll 1
      for (int e = 0; e < 4; ++e)
#pragma unroll 1
        for (int side = 0; side < 2; ++side) {
          const double sg = side == 0 ? 1.0 : -1.0;
          double unit[4] = {0.0, 0.0, 0.0, 0.0};
          unit[e] = sg;
          const double rl = backsub(it, unit, zero4, 0.0);
          double lo, hi;
          L.conc(HL{rl, rl}, lo, hi);
          if (side == 0)
            Bl[it][e] = fmax(Bl[it][e], lo);
          else
            Bh[it][e] = fmin(Bh[it][e], -lo);
        }
#pragma unroll 1
    for (int out = 0; out < 4; ++out) {
      const int oa = out >> 1, ob = out & 1;
#pragma unroll 1
      for (int side = 0; side < 2; ++side) {
        const double sg = side == 0 ? 1.0 : -1.0;  // lower bound of sg * Conic_ab
        double init[4] = {0.0, 0.0, 0.0, 0.0};
        init[0 + ob] = sg * X0[2 * oa];      // coefficient on P^i_{0 ob}, every level
        init[2 + ob] = sg * X0[2 * oa + 1];  // on P^i_{1 ob}
        const double rl = backsub(k_own, init, init, sg * X0[out]);  // i = 0: X0 . I
        // per entry and side the tighter (by concretisation) of the forward form and the
        // back-substituted bound (both sound)
        double a0, a1, b0, b1;
        if (side == 0) {
          const double cand = rl - (L.cst() ? eps : 0.0);
          L.conc(HL{cand, cand}, a0, a1);
          L.conc(HL{conic[out].l, conic[out].l}, b0, b1);
          if (ok && a0 > b0) conic[out].l = cand;
        } else {
          const double cand = -rl + (L.cst() ? eps : 0.0);
          L.conc(HL{cand, cand}, a0, a1);
          L.conc(HL{conic[out].u, conic[out].u}, b0, b1);
          if (ok && a1 < b1) conic[out].u = cand;
        }
      }
    }
  }
  // ---- l.9 pieces: W = Mmul(Conic, Mp) (G4), D2 = Mul(d,d), DU = Mul(d, up)
  HotRec<NV>* H = reinterpret_cast<HotRec<NV>*>(A.hot) + i;
  float wv[6][2];
  float wcv[6][2];
  double cnl[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    double h;
    L.conc(conic[e], cnl[e], h);
  }
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      HL acc{0.0, 0.0};
      L.mul_acc_b(acc, conic[2 * a + 0], cnl[2 * a + 0], Mp[0][c], Mpl[0][c], Mph[0][c]);
      L.mul_acc_b(acc, conic[2 * a + 1], cnl[2 * a + 1], Mp[1][c], Mpl[1][c], Mph[1][c]);
      double lo, hi;
      L.conc(acc, lo, hi);
      if (!(fabs(lo) <= WCAP && fabs(hi) <= WCAP)) ok = false;  // reading O3
      wv[3 * a + c][0] = (float)acc.l;
      wv[3 * a + c][1] = (float)acc.u;
      wcv[3 * a + c][0] = (float)lo;
      wcv[3 * a + c][1] = (float)hi;
    }
  double dl, dh, u0l, u0h, u1l, u1h;
  L.conc(d, dl, dh);
  L.conc(up0, u0l, u0h);
  L.conc(up1, u1l, u1h);
  HL D2{0.0, 0.0}, DU0{0.0, 0.0}, DU1{0.0, 0.0};
  L.sq_acc_b(D2, d, dl, dh);
  L.mul_acc_b(DU0, d, dl, up0, u0l, u0h);
  L.mul_acc_b(DU1, d, dl, up1, u1l, u1h);
  // ---- depth decisions, key, footprint (steps 10-12; G8, G12, O4)
  const double dcl = __shfl_sync(FULL, d.l, NV, W), dcu = __shfl_sync(FULL, d.u, NV, W);
  double s1 = L.slope() ? fabs(d.l - sp.gslope[k]) : 0.0;
  double s2 = L.slope() ? fabs(d.u - sp.gslope[k]) : 0.0;
  s1 = hsum<W>(s1);
  s2 = hsum<W>(s2);
  if (live && real) {
    H->d2[0][k] = D2.l;
    H->d2[1][k] = D2.u;
    H->du[0][0][k] = DU0.l;
    H->du[0][1][k] = DU0.u;
    H->du[1][0][k] = DU1.l;
    H->du[1][1][k] = DU1.u;
#pragma unroll
    for (int e = 0; e < 6; ++e) {
      H->w[e][0][k] = ok ? wv[e][0] : 0.f;
      H->w[e][1][k] = ok ? wv[e][1] : 0.f;
    }
    PairRec<NV>* PR = reinterpret_cast<PairRec<NV>*>(A.pair) + i;
    PR->dl[k] = d.l;
    PR->du[k] = d.u;
  }
  int fl = ok ? 0 : F_FAIL;
  const float olo = A.op_lo ? A.op_lo[i] : A.opacity[i];
  const float ohi = A.op_hi ? A.op_hi[i] : A.opacity[i];
  if (!(dh > DMIN) || !((double)ohi > TAU))
    fl |= F_DROP;
  else if (dl <= DMIN)
    fl |= F_STRADDLE;
  if (live && k == 0) {
    const double kappa = 0.5 * (dcl + dcu);
    double mu[4] = {0, 0, 0, 0}, r2 = 0.0;
    if (!(fl & F_DROP)) {
      const double de = fmax(dl, DMIN);
      const double ul[2] = {u0l, u1l}, uh[2] = {u0h, u1h};
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        const double q0 = ul[a] / de, q1 = ul[a] / dh, q2 = uh[a] / de, q3 = uh[a] / dh;
        mu[a] = fmin(fmin(q0, q1), fmin(q2, q3));
        mu[2 + a] = fmax(fmax(q0, q1), fmax(q2, q3));
      }
      const double de2 = de * de;
      const double lam = (x00h + x11h) / (de2 * de2);  // >= lambda_max(Sigma_2D)
      r2 = 2.0 * log((double)ohi / TAU) * lam;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) H->mu[e] = mu[e];
    H->r2 = r2;
    H->pad0 = 0.0;
#pragma unroll
    for (int e = 0; e < 6; ++e) {
      H->wc[e][0] = ok ? wcv[e][0] : 0.f;
      H->wc[e][1] = ok ? wcv[e][1] : 0.f;
    }
    H->o[0] = olo;
    H->o[1] = ohi;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      H->clo[c] = A.col_lo ? A.col_lo[3 * i + c] : A.color[3 * i + c];
      H->chi[c] = A.col_hi ? A.col_hi[3 * i + c] : A.color[3 * i + c];
    }
    H->flags = fl;
    PairRec<NV>* PR = reinterpret_cast<PairRec<NV>*>(A.pair) + i;
    const double ws = fmax(0.5 * (dcu - dcl) + fmax(s1, s2), 0.0);  // bit-pattern max below
    PR->kappa = kappa;
    PR->ws = ws;
    A.kkey[i] = (fl & F_DROP) ? ~0ull : key_of_double(kappa);
    A.kval[i] = (int32_t)i;
    if (!(fl & F_DROP)) atomicMax(&s_wsmax, (unsigned long long)__double_as_longlong(ws));
  }
  // block-aggregated counters (one vote per Gaussian: lane 0 of each lane group)
  const bool head = live && k == 0;
  const int nf = __syncthreads_count(head && (fl & F_FAIL) && !(fl & F_DROP));
  const int ns = __syncthreads_count(head && (fl & F_STRADDLE));
  const int nd = __syncthreads_count(head && (fl & F_DROP));
  if (threadIdx.x == 0) {
    if (s_wsmax) atomicMax(A.wsmax, s_wsmax);  // block max (ws >= 0: bits order like values)
    if (nf) atomicAdd(&A.counters[0], (unsigned long long)nf);
    if (ns) atomicAdd(&A.counters[1], (unsigned long long)ns);
    if (nd) atomicAdd(&A.counters[2], (unsigned long long)nd);
  }
}

void launch_setup(int nv, const SetupArgs& a, cudaStream_t st) {
  const int threads = 128;  // 32 (n <= 3), 16 (n <= 7) or 8 Gaussians per block
  const int64_t total = a.N * (nv + 1 <= 4 ? 4 : (nv + 1 <= 8 ? 8 : 16));
  const unsigned blocks = (unsigned)((total + threads - 1) / threads);
  if (a.N <= 0) return;
  switch (nv) {
#define CASE(K) \
  case K:       \
    k_setup<K><<<blocks, threads, 0, st>>>(a); \
    break;
    CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9)
#undef CASE
    default:
      break;
  }
}

}  // namespace absplat
