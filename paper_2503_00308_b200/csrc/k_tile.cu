// k_tile.cu -- rows a8-a10, the hot loop: per (pixel, Gaussian) opacity bounds (Alg. 1 lines
// 9-10 lifted: x = d^2 u - d up, q = x W, s = q q^T, a = o exp(-s/2)) and the
// transmittance scan + bounded blend (Alg. 3, interval reading O7), with the
// finalise/union epilogue.
//
// A work item is one 16x8 pixel block of a tile (128 threads, one pixel each; 8x8 / 64
// threads for 8-pixel tiles) over one chunk of the tile's Gaussian list (sorted by
// (kappa, index)).  The list is streamed through shared
// memory in batches of BS: the staging step turns each Gaussian's fp64 record into
// block-centred fp32 forms (B = u_c D2 - DU at the block centre u_c, so the per-pixel
// x = B + (u - u_c) D2 avoids the d^2 u - d up cancellation; H2) and fp64 per-row /
// per-column squared distances for the exact per-pixel cull (reading O1); Gaussians whose
// footprint misses the whole block are skipped.  Every thread then walks the batch for its
// pixel in order: FP32 on CUDA cores.
//
// Work is a list of (tile, chunk) items, longest first, pulled by persistent CTAs from an
// atomic counter (load balance).  A chunk is scanned with lookback / lookahead
// margins covering its positions' exception windows, so chunks of one tile compose front to
// back in k_merge with multiplications only.
//
// Uncertain depth pairs (rotation / scene boxes; step 13) are handled in the walk itself
// with a per-CTA ring in global memory (L2-resident): position q writes (T_hi before q,
// 1 - a_lo, 1 - a_hi, deferred T_lo a_lo) for its pixel; T_hi of a position with earlier
// uncertain partners is re-multiplied over its window [h, q) skipping E_F (no division,
// H3); the lower contribution of a position with later uncertain partners is deferred and
// finalised at g = max E_G, when all of E_G's (1 - a_hi) are known.
#include <algorithm>
#include <cfloat>
#include <cstdio>

#include "internal.cuh"

#ifndef KT2_MINB  // k_tile2 CTAs per SM (launch bounds; the batch size is clamped to match)
#define KT2_MINB 4
#endif

namespace absplat {

namespace {
constexpr unsigned FULLM = 0xffffffffu;
constexpr float LOG2E_HALF = 0.72134752044448170368f;  // log2(e) / 2

// A work item is one BX x 8 pixel block (BX = 16, or 8 for 8-pixel tiles), one thread per
// pixel; every warp covers an 8 x 4 quadrant so the warp-level cull stays compact.
constexpr int SBY = 8;           // block height
constexpr int NPART = 4;         // staging threads per Gaussian
__host__ __device__ __forceinline__ int block_w(int ts) { return ts >= 16 ? 16 : 8; }
__host__ __device__ __forceinline__ int pix_x(int t, int bx) {
  return bx == 16 ? ((t >> 5) & 1) * 8 + (t & 7) : (t & 7);
}
__host__ __device__ __forceinline__ int pix_y(int t, int bx) {
  return bx == 16 ? (t >> 6) * 4 + ((t >> 3) & 3) : (t >> 3);
}
__host__ __device__ __forceinline__ int pix_of(int x, int y, int bx) {
  return bx == 16 ? ((y >> 2) * 2 + (x >> 3)) * 32 + (y & 3) * 8 + (x & 7) : y * 8 + x;
}
constexpr int FB = 48;           // finalisation records staged in shared memory per batch
constexpr int EG8 = 60;          // E_G operands precomputed per staged finalisation record
constexpr int TL8 = 32;          // T_hi window operands precomputed per position

template <int NV>
struct alignas(16) SRec {
  static constexpr int C = NV + 1;
  static constexpr int CP = (C + 3) & ~3;  // padded for 16-byte vector loads
  // x_a lower forms (for the concretised x_lo_a only): B_a + du_a * D2_lo
  float2 XB[CP];            // (B_lo,0, B_lo,1) per coefficient
  float d2lo[CP];
  // q_c = mul(x0, W_0c) + mul(x1, W_1c) with the x-side McCormick terms folded into affine
  // functions of the pixel offset du, and the W-side terms in mid / radius form:
  //   q_lo,k = plo + du0 q0lo + du1 q1lo + x0 wm0 - |x0| wr0 + x1 wm1 - |x1| wr1
  //   q_hi,k = phi + du0 q0hi + du1 q1hi + x0 wm0 + |x0| wr0 + x1 wm1 + |x1| wr1
  // stored as mid / radius:  q_lo,k = m - r,  q_hi,k = m + r  with
  //   m = pm + du0 q0m + du1 q1m + x0 wm0 + x1 wm1,  r = pr + du0 q0r + du1 q1r + |x0| wr0 + |x1| wr1
  // kept as (mid, radius) pairs so both evaluate with one packed FFMA2 per term:
  //   P = (pm, pr), Q0 = (q0m, q0r), Q1 = (q1m, q1r), W0 = (wm0, wr0), W1 = (wm1, wr1)
  float2 P[3][CP], Q0[3][CP], Q1[3][CP], W0[3][CP], W1[3][CP];
  float2 WC[6];             // concretised W, [a*3+c]: ((lo + hi) / 2, (lo - hi) / 2)
  float o[2];
  float ctr[2];  // the form centre (block-local pixels, integer valued): see stage_forms
  float clo[3], chi[3];
  int flags;                // F_* of the Gaussian
  int pmf, ph, pg, pnF, pnG;  // position metadata (PM_*, h, g, |E_F|, |E_G|)
  int pfb, pfe;             // finalisation records [pfb, pfe) (absolute: F0 is subtracted in
                            // the walk, so phase A does not wait for the batch's F0 load)
  long long peoff;          // offset of E_F(p) then E_G(p) in exc[]
  unsigned long long mf0, mf1;  // E_F(p) bits over [h, h+128)
  // precomputed ring operands of the T_hi window: positions h + tlo[t]
  int tmode;                // 0 none, 1 dense (tlo = kept), 2 sparse (tlo = E_F), 3 slow
  int nT;
  unsigned char tlo[TL8];
  double r2;
};
// finalisation record of q' (finalised at g = max E_G(q')) staged in shared memory:
// T_lo(q') a_lo(q') = w(q') (1 - a_hi,g) prod_{r in E_G(q') \ {g}} (1 - a_hi,r), with the
// ring positions r = q' + off precomputed (culled positions, factor exactly 1, left out)
struct alignas(16) FinS {
  int qq;                   // q' (tile-local); -1: nothing to do in this block / chunk
  short n;                  // operand count, -1 = slow path (bits or exception lists)
  short pad;
  float clo[3];
  unsigned char off[EG8];
};

// Staging of one Gaussian for a block centred at (ucx, ucy) with half-extents (hx, hy): fp64
// arithmetic, one rounding.  The forms are centred on the block pixel corner nearest the
// Gaussian's mean (the middle of its mean rectangle, clamped to the block; S.ctr), so the fp32
// per-pixel offsets du are exact and small where the opacity is large (any centre gives the
// same forms up to fp32 rounding; the block centre cancels more bits).
// x_a lower form: u_a D2_lo - DU_a,hi = B_lo,a + du_a D2_lo with B_lo,a = uc_a D2_lo - DU_a,hi
// (u_a > 0 selects D2's lower side, step 14); upper: B_hi,a + du_a D2_hi.
// LS(x_a, w) = w >= 0 ? w x_lo,a : w x_hi,a  and  US(x_a, w) = w >= 0 ? w x_hi,a : w x_lo,a
// (R1 with the constant w = conc W), both affine in du_a.
template <int NV>
__device__ __forceinline__ void stage_forms(SRec<NV>& S, const HotRec<NV>* H, double ucx,
                                            double ucy, double hx, double hy, int part) {
  // NPART threads per Gaussian; thread `part` stages coefficients k = part, part + NPART,
  // ... of every channel, so all of its record loads are independent and issue together
  constexpr int C = NV + 1;
  constexpr int KP = (C + NPART - 1) / NPART;
  const double hh[2] = {hx, hy};
  double uc[2];
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const double o = (a ? ucy : ucx) - hh[a];
    const double rc = fmin(fmax(rint(0.5 * (H->mu[a] + H->mu[2 + a]) - o), 0.0), 2.0 * hh[a]);
    uc[a] = o + rc;
    if (part == 0) S.ctr[a] = (float)rc;
  }
  double wl[6], wh[6];  // concretised W, [a*3+c]
#pragma unroll
  for (int e = 0; e < 6; ++e) {
    wl[e] = H->wc[e][0];
    wh[e] = H->wc[e][1];
  }
  if (part == NPART - 1) {
#pragma unroll
    for (int e = 0; e < 6; ++e) {
      S.WC[e] = make_float2((float)(0.5 * (wl[e] + wh[e])), (float)(0.5 * (wl[e] - wh[e])));
    }
  }
#pragma unroll 1
  for (int i = 0; i < KP; ++i) {
    const int k = part + NPART * i;
    if (k >= C) break;
    const double d2l = H->d2[0][k], d2h = H->d2[1][k];
    double blo[2], bhi[2];
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      blo[a] = uc[a] * d2l - H->du[a][1][k];
      bhi[a] = uc[a] * d2h - H->du[a][0][k];
    }
    float wa[6], wb[6];
#pragma unroll
    for (int e = 0; e < 6; ++e) {
      wa[e] = H->w[e][0][k];
      wb[e] = H->w[e][1][k];
    }
    // x lower forms
    S.XB[k] = make_float2((float)blo[0], (float)blo[1]);
    S.d2lo[k] = (float)d2l;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double w0l = wl[c], w0h = wh[c], w1l = wl[3 + c], w1h = wh[3 + c];
      const double plo = w0l * (w0l >= 0 ? blo[0] : bhi[0]) + w1l * (w1l >= 0 ? blo[1] : bhi[1]);
      const double phi = w0h * (w0h >= 0 ? bhi[0] : blo[0]) + w1h * (w1h >= 0 ? bhi[1] : blo[1]);
      const double q0lo = w0l * (w0l >= 0 ? d2l : d2h), q1lo = w1l * (w1l >= 0 ? d2l : d2h);
      const double q0hi = w0h * (w0h >= 0 ? d2h : d2l), q1hi = w1h * (w1h >= 0 ? d2h : d2l);
      S.P[c][k] = make_float2((float)(0.5 * (plo + phi)), (float)(0.5 * (phi - plo)));
      S.Q0[c][k] = make_float2((float)(0.5 * (q0lo + q0hi)), (float)(0.5 * (q0hi - q0lo)));
      S.Q1[c][k] = make_float2((float)(0.5 * (q1lo + q1hi)), (float)(0.5 * (q1hi - q1lo)));
      const double a0 = wa[c], b0 = wb[c], a1 = wa[3 + c], b1 = wb[3 + c];
      S.W0[c][k] = make_float2((float)(0.5 * (a0 + b0)), (float)(0.5 * (b0 - a0)));
      S.W1[c][k] = make_float2((float)(0.5 * (a1 + b1)), (float)(0.5 * (b1 - a1)));
    }
  }
}

// steps 14-16 for one pixel at offset (du0, du1) from the record's form centre: the lower / upper
// forms of s as pairs S[k] = (s_lo,k, s_hi,k).  Each (m, r) term is one packed FFMA2 (same
// order as the scalar formulas); R2's plane selection LS(q, 2p) / US(q, qmin + qmax) is
// written select-free as tp m - |tp| r and sm m + |sm| r (two FFMA2 per coefficient).
template <int NV>
__device__ __forceinline__ void s_forms(const SRec<NV>& R, float du0, float du1,
                                        float2 (&S)[NV + 1]) {
  constexpr int C = NV + 1;
  // 14: concretised lower bound of x_a = Add(Mul(d,d,u_a), -Mul(d, up_a))
  const float2 DU = make_float2(du0, du1);
  const float2 xc = __ffma2_rn(DU, make_float2(R.d2lo[NV], R.d2lo[NV]), R.XB[NV]);
  float x0 = xc.x, x1 = xc.y;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const float2 v = __ffma2_rn(DU, make_float2(R.d2lo[k], R.d2lo[k]), R.XB[k]);
    x0 -= fabsf(v.x);
    x1 -= fabsf(v.y);
  }
  const float2 D0 = make_float2(du0, du0), D1 = make_float2(du1, du1);
  const float2 X0 = make_float2(x0, fabsf(x0)), X1 = make_float2(x1, fabsf(x1));
  const float2 Y0 = make_float2(-x0, x0), Y1 = make_float2(-x1, x1);
  // 15-16: q_c = mul(x0, W_0c) + mul(x1, W_1c) (R1); s = sum_c sq(q_c) (R2)
#pragma unroll
  for (int k = 0; k < C; ++k) S[k] = make_float2(0.f, 0.f);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    float ql[C], qh[C];
    float2 MR[C];
#pragma unroll
    for (int k = 0; k < C; ++k) {
      // m = pm + du0 q0m + du1 q1m + x0 wm0 + x1 wm1,  r = pr + du0 q0r + du1 q1r + |x0| wr0 + |x1| wr1
      float2 mr = __ffma2_rn(D0, R.Q0[c][k], R.P[c][k]);
      mr = __ffma2_rn(D1, R.Q1[c][k], mr);
      mr = __ffma2_rn(X0, R.W0[c][k], mr);
      mr = __ffma2_rn(X1, R.W1[c][k], mr);
      if (k == NV) {  // constant: q_lo -= x0 W_lo,0c + x1 W_lo,1c, q_hi -= x0 W_hi,0c + x1 W_hi,1c
        mr = __ffma2_rn(Y0, R.WC[c], mr);
        mr = __ffma2_rn(Y1, R.WC[3 + c], mr);
      }
      MR[k] = mr;
      ql[k] = mr.x - mr.y;
      qh[k] = mr.x + mr.y;
    }
    float qmin = ql[NV], qmax = qh[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      qmin -= fabsf(ql[k]);
      qmax += fabsf(qh[k]);
    }
    const float p = fminf(fmaxf(0.f, qmin), qmax);
    const float tp = 2.f * p, sm = qmin + qmax;
    // tp sel(ql, qh) = tp m - |tp| r and sm sel(qh, ql) = sm m + |sm| r
    const float2 T = make_float2(tp, sm), TA = make_float2(-fabsf(tp), fabsf(sm));
#pragma unroll
    for (int k = 0; k < C; ++k) {
      S[k] = __ffma2_rn(T, make_float2(MR[k].x, MR[k].x), S[k]);
      S[k] = __ffma2_rn(TA, make_float2(MR[k].y, MR[k].y), S[k]);
    }
    S[NV] = __ffma2_rn(make_float2(-p, -qmin), make_float2(p, qmax), S[NV]);
  }
}

// steps 14-17 for one pixel at offset (du0, du1) from the record's form centre: (a_lo, a_hi)
template <int NV>
__device__ __forceinline__ void opacity(const SRec<NV>& R, float du0, float du1, float& alo,
                                        float& ahi) {
  float2 S[NV + 1];
  s_forms<NV>(R, du0, du1, S);
  float smin = S[NV].x, smax = S[NV].y;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    smin -= fabsf(S[k].x);
    smax += fabsf(S[k].y);
  }
  smin = fmaxf(smin, 0.f);
  // 17: a = o * Exp(-s/2) concretised (O11)
  alo = R.o[0] * exp2f(-LOG2E_HALF * smax);
  ahi = R.o[1] * exp2f(-LOG2E_HALF * smin);
}

// steps 14-16 for one pixel, keeping s's lower / upper forms (NEXT-1 linear blend)
template <int NV>
__device__ __forceinline__ void opacity_sforms(const SRec<NV>& R, float du0, float du1,
                                               float (&sl)[NV + 1], float (&sh)[NV + 1]) {
  float2 S[NV + 1];
  s_forms<NV>(R, du0, du1, S);
#pragma unroll
  for (int k = 0; k <= NV; ++k) {
    sl[k] = S[k].x;
    sh[k] = S[k].y;
  }
}

// R1 McCormick product of two forms given as (lo[C], hi[C]) coefficient arrays (slopes then
// constant), fp32: out = mul(f, g) with the fixed planes of reading G1
template <int NV>
__device__ __forceinline__ void form_mul(const float (&fl)[NV + 1], const float (&fh)[NV + 1],
                                         const float (&gl)[NV + 1], const float (&gh)[NV + 1],
                                         float (&ol)[NV + 1], float (&oh)[NV + 1]) {
  float xl = fl[NV], xh = fh[NV], yl = gl[NV], yh = gh[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    xl -= fabsf(fl[k]);
    xh += fabsf(fh[k]);
    yl -= fabsf(gl[k]);
    yh += fabsf(gh[k]);
  }
  // lower = LS(f, y_lo) + LS(g, x_lo) - x_lo y_lo ; upper = US(f, y_hi) + US(g, x_lo) - x_lo y_hi
#pragma unroll
  for (int k = 0; k <= NV; ++k) {
    const float lf = yl >= 0.f ? fl[k] : fh[k], lg = xl >= 0.f ? gl[k] : gh[k];
    const float uf = yh >= 0.f ? fh[k] : fl[k], ug = xl >= 0.f ? gh[k] : gl[k];
    ol[k] = fmaf(yl, lf, xl * lg);
    oh[k] = fmaf(yh, uf, xl * ug);
  }
  ol[NV] -= xl * yl;
  oh[NV] -= xl * yh;
}
}  // namespace


// Ring layout (per CTA): [slot][component][pixel] floats, so a warp's load of one component
// is one contiguous 128-byte line.  Components: 0 T_hi before q, 1 (1 - a_lo,q),
// 2 (1 - a_hi,q), 3 deferred T_lo a_lo,q.  RS = float offset of (slot, comp) without pixel.
template <int SBP>
__device__ __forceinline__ int RS(int pos, int comp, int rmask) {
  return ((pos & rmask) * 4 + comp) * SBP;
}

// Skip ring: bit (p & 255) of s_skip[8] says position p's Gaussian misses the whole block
// (a = 0 for every pixel, so its factors (1 - a) are exactly 1 and its own contributions
// exactly 0).  skip_win returns the bits of positions [base, base + 128).
__device__ __forceinline__ void skip_win(const unsigned* sk, int base, unsigned long long& m0,
                                         unsigned long long& m1) {
  unsigned w[4];
  const int sh = base & 31, wi = base >> 5;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    w[k] = __funnelshift_r(sk[(wi + k) & 7], sk[(wi + k + 1) & 7], sh);
  m0 = ((unsigned long long)w[1] << 32) | w[0];
  m1 = ((unsigned long long)w[3] << 32) | w[2];
}

// product of ring component `comp` over the positions base + i for the set bits i of the
// 128-bit mask (m0, m1); loads are issued in groups of 8 so they overlap.  rf = ring + pix.
// product of ring component `comp` over the positions list[0 .. n) (an exception list in
// global memory), in order; list entries and ring values are loaded 8 at a time
template <int SBP>
__device__ __noinline__ float exc_prod(const float* rf, const int32_t* list, int n, int comp,
                                       int rmask) {
  float prod = 1.f;
  for (int e0 = 0; e0 < n; e0 += 8) {
    int idx[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) idx[u] = e0 + u < n ? list[e0 + u] : -1;
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = idx[u] >= 0 ? rf[RS<SBP>(idx[u], comp, rmask)] : 1.f;
#pragma unroll
    for (int u = 0; u < 8; ++u) prod *= v[u];
  }
  return prod;
}

// product of ring component 1 over the window [h, q) minus the sorted list ef[0 .. nf)
// (T_hi of a long window, dense case), ring values loaded 8 at a time
template <int SBP>
__device__ __noinline__ float window_prod(const float* rf, int h, int q, const int32_t* ef, int nf,
                                          int rmask) {
  float prod = 1.f;
  int e = 0;
  int nextF = nf > 0 ? ef[0] : 0x7fffffff;
  for (int r0 = h; r0 < q; r0 += 8) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = r0 + u < q ? rf[RS<SBP>(r0 + u, 1, rmask)] : 1.f;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int r = r0 + u;
      if (r >= q) break;
      if (r == nextF) {
        ++e;
        nextF = e < nf ? ef[e] : 0x7fffffff;
      } else {
        prod *= v[u];
      }
    }
  }
  return prod;
}

template <int SBP>
__device__ __forceinline__ float ring_prod(const float* rf, unsigned long long m0,
                                           unsigned long long m1, int base, int comp, int rmask) {
  float prod = 1.f;
  while (m0 | m1) {
    float v[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      int idx = -1;
      if (m0) {
        idx = base + __ffsll((long long)m0) - 1;
        m0 &= m0 - 1;
      } else if (m1) {
        idx = base + 64 + __ffsll((long long)m1) - 1;
        m1 &= m1 - 1;
      }
      v[t] = idx >= 0 ? rf[RS<SBP>(idx, comp, rmask)] : 1.f;
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) prod *= v[t];
  }
  return prod;
}

#ifndef KT1_MINB8
#define KT1_MINB8 8  // 8x8 blocks: 8 CTAs per SM bound (C5 1.80 -> ~1.72 ms; 9 spilled)
#endif
template <int NV, int BX>
__global__ void __launch_bounds__(BX * SBY, BX == 16 ? 5 : KT1_MINB8) k_tile(TileArgs A) {
  if (A.ovf && *A.ovf) return;  // sizes outgrown: the render is repeated
  constexpr int SBX = BX;         // block width
  constexpr int SBP = SBX * SBY;  // threads per CTA = pixels per work item
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_work;
  __shared__ unsigned s_skip[8];
  __shared__ int s_F[2];
  const int ts = A.ts;
  const int nsbx = ts / SBX;        // blocks per tile row
  const int nsub = nsbx * (ts / SBY);
  const int BS = A.bs;
  SRec<NV>* srec = reinterpret_cast<SRec<NV>*>(smem_raw);
  double* cx2 = reinterpret_cast<double*>(srec + BS);  // [BS][SBX]
  double* cy2 = cx2 + (size_t)BS * SBX;                // [BS][SBY]
  FinS* fins = reinterpret_cast<FinS*>(cy2 + (size_t)BS * SBY);  // [FB]
  const bool has_exc = A.pm != nullptr;
  const int pix = threadIdx.x;
  float* rf = has_exc ? reinterpret_cast<float*>(A.ring) + (size_t)blockIdx.x * A.R * SBP * 4 + pix
                      : nullptr;
  const int lx = pix_x(pix, SBX), ly = pix_y(pix, SBX);
  const float lxh = (float)lx + 0.5f, lyh = (float)ly + 0.5f;  // minus the record's form centre
  unsigned active = 0;
  const int nwork = A.n_items * nsub;

  for (;;) {
    if (threadIdx.x == 0) s_work = atomicAdd(A.counter, 1);
    __syncthreads();
    const int w = s_work;
    __syncthreads();
    if (w >= nwork) break;
    const int islot = A.order[w / nsub];
    const int sub = w % nsub;
    const int4 it = A.items[islot];
    if (it.x < 0) continue;  // padding
    const int tile = it.x, pbeg = it.y, pend = it.z, iflags = it.w;
    const int4 it2 = A.items2[islot];
    const int scan0 = it2.x, scan1 = it2.y, anext = it2.z;  // scan [A, L), record at A_next
    const int rmask = (1 << ((iflags >> 8) & 0xff)) - 1;     // per-item ring length - 1
    DCHECK(islot >= 0 && islot < A.n_items && tile >= 0 && tile < A.ntiles);
    DCHECK(0 <= scan0 && scan0 <= pbeg && pbeg <= pend && pend <= scan1 && rmask < A.R);
    DCHECK(A.tbegin[tile] + scan1 <= A.tend[tile]);
    const int tx = tile % A.ntx, ty = tile / A.ntx;
    const int ox = tx * ts + (sub % nsbx) * SBX, oy = ty * ts + (sub / nsbx) * SBY;  // origin
    const int64_t tb = A.tbegin[tile];
    const double ucx = ox + 0.5 * SBX, ucy = oy + 0.5 * SBY;  // block centre
    const bool iexc = has_exc && (iflags & IT_EXC);
    const bool in_img = (ox + lx < A.W) && (oy + ly < A.H);
    const double bx0 = ox + 0.5, bx1 = fmin((double)(ox + SBX), (double)A.W) - 0.5;
    const double by0 = oy + 0.5, by1 = fmin((double)(oy + SBY), (double)A.H) - 0.5;
    const bool block_live = ox < A.W && oy < A.H;
    float Tb = 1.f, Tl = 1.f, ahc[3] = {0.f, 0.f, 0.f}, alc[3] = {0.f, 0.f, 0.f};
    float recb = 1.f, recl = 1.f;  // running products at A_next (chunk composition)
    bool rec = false;

    for (int b0 = scan0; b0 < scan1; b0 += BS) {
      const int nb = min(BS, scan1 - b0);
      // finalisation records of the batch: fin_rec[F0, F1) (sorted by finalising position);
      // thread 0 loads the bounds now and publishes them through shared memory after its
      // phase A work, so no thread waits on (or spills) them
      int f0l = 0, f1l = 0;
      if (threadIdx.x == 0 && iexc) {
        f0l = A.finstart[tb + b0];
        f1l = A.finstart[tb + b0 + nb];
      }
      __syncthreads();
      // ---- phase A: fp64 record -> block-centred fp32 forms, whole-block cull (same exact
      //      test as the per-pixel one, on the block rectangle) into the skip ring, cull
      //      tables and position metadata.  Metadata and cull tables: one thread per
      //      Gaussian, taken from the highest thread ids (idle in the staging loop when
      //      NPART * nb < SBP); staging: four threads per Gaussian (stage_forms splits the
      //      coefficients).  Every thread evaluates the cull itself.
      for (int j = SBP - 1 - (int)threadIdx.x; j < nb; j += SBP) {
        const int64_t gp = tb + b0 + j;
        const int32_t g = A.vals[gp];
        const HotRec<NV>* H = reinterpret_cast<const HotRec<NV>*>(A.hot) + g;
        SRec<NV>& S = srec[j];
        const double mxl = H->mu[0], myl = H->mu[1], mxh = H->mu[2], myh = H->mu[3];
        const double r2 = H->r2;
        bool skip;
        {
          const double dx = fmax(0.0, fmax(__dsub_rn(mxl, bx1), __dsub_rn(bx0, mxh)));
          const double dy = fmax(0.0, fmax(__dsub_rn(myl, by1), __dsub_rn(by0, myh)));
          skip = !block_live || __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)) > r2;
        }
        const int bit = (b0 + j) & 255;
        if (skip)
          atomicOr(&s_skip[bit >> 5], 1u << (bit & 31));
        else
          atomicAnd(&s_skip[bit >> 5], ~(1u << (bit & 31)));
        int pmf = 0;
        if (iexc) {
          const int4 m = A.pm[gp];
          pmf = m.x;
          S.ph = m.y;
          S.pg = m.z;
          S.pnF = m.w;
          S.pnG = A.nG[gp];
          S.peoff = A.eoff[gp];
          S.pfb = A.finstart[gp];
          S.pfe = A.finstart[gp + 1];
          const ulonglong2 mf = A.mF[gp];
          S.mf0 = mf.x;
          S.mf1 = mf.y;
        } else {
          S.pfb = S.pfe = 0;
        }
        S.tmode = 0;
        S.nT = 0;
        S.pmf = pmf;
        S.flags = H->flags | (skip ? F_SKIP : 0);
        S.r2 = r2;
        // colours / opacity are read by the blend even for skipped (a = 0) entries
        S.o[0] = H->o[0];
        S.o[1] = H->o[1];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          S.clo[c] = H->clo[c];
          S.chi[c] = H->chi[c];
        }
        if (!skip) {
#pragma unroll
          for (int l = 0; l < SBX; ++l) {
            const double x = ox + l + 0.5;
            const double dx = fmax(0.0, fmax(__dsub_rn(mxl, x), __dsub_rn(x, mxh)));
            cx2[j * SBX + l] = __dmul_rn(dx, dx);
          }
#pragma unroll
          for (int l = 0; l < SBY; ++l) {
            const double y = oy + l + 0.5;
            const double dy = fmax(0.0, fmax(__dsub_rn(myl, y), __dsub_rn(y, myh)));
            cy2[j * SBY + l] = __dmul_rn(dy, dy);
          }
        }
      }
      for (int jj = threadIdx.x; jj < NPART * nb; jj += SBP) {
        const int j = jj / NPART, part = jj % NPART;
        const HotRec<NV>* H = reinterpret_cast<const HotRec<NV>*>(A.hot) + A.vals[tb + b0 + j];
        bool skip;
        {
          const double dx = fmax(0.0, fmax(__dsub_rn(H->mu[0], bx1), __dsub_rn(bx0, H->mu[2])));
          const double dy = fmax(0.0, fmax(__dsub_rn(H->mu[1], by1), __dsub_rn(by0, H->mu[3])));
          skip = !block_live || __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)) > H->r2;
        }
        if (!skip) stage_forms<NV>(srec[j], H, ucx, ucy, 0.5 * SBX, 0.5 * SBY, part);
      }
      if (threadIdx.x == 0) {
        s_F[0] = f0l;
        s_F[1] = f1l;
      }
      __syncthreads();
      // ---- phase B (needs the batch's skip bits): T_hi window operands per position and
      //      the batch's finalisation records, both skip-filtered
      if (iexc) {
        // (warp 0 builds the window lists while the other warps stage the finalisation
        //  records below)
        for (int j = threadIdx.x < 32 ? (int)threadIdx.x : nb; j < nb; j += 32) {
          SRec<NV>& S = srec[j];
          const int pmf = S.pmf, qpos = b0 + j;
          // (a skipped q contributes nothing: no T_hi needed)
          if (!(pmf & PM_EF) || (S.flags & F_SKIP) || qpos < pbeg || qpos >= pend || (pmf & PM_OVF))
            continue;
          const int h = S.ph, wlen = qpos - h;
          const unsigned long long v0 = wlen >= 64 ? ~0ull : ((1ull << wlen) - 1ull);
          const unsigned long long v1 =
              wlen <= 64 ? 0ull : (wlen >= 128 ? ~0ull : ((1ull << (wlen - 64)) - 1ull));
          // factors of skipped positions are exactly 1: leave them out of both lists
          unsigned long long k0, k1;
          skip_win(s_skip, h, k0, k1);
          const unsigned long long e0 = S.mf0 & ~k0, e1 = S.mf1 & ~k1;
          const unsigned long long f0 = ~S.mf0 & ~k0 & v0, f1 = ~S.mf1 & ~k1 & v1;
          const int nef = __popcll(e0) + __popcll(e1), nkept = __popcll(f0) + __popcll(f1);
          const bool dense = !(nkept > nef + 2);
          unsigned long long m0 = dense ? f0 : e0;
          unsigned long long m1 = dense ? f1 : e1;
          const int cnt = dense ? nkept : nef;
          int nT = 0;
          if (cnt <= TL8) {
            S.tmode = dense ? 1 : 2;
            for (; m0; m0 &= m0 - 1) S.tlo[nT++] = (unsigned char)(__ffsll((long long)m0) - 1);
            for (; m1; m1 &= m1 - 1) S.tlo[nT++] = (unsigned char)(64 + __ffsll((long long)m1) - 1);
          } else {
            S.tmode = 3;
            if (A.dbg) atomicAdd(A.dbg + DBG_TMODE3, 1ull);
          }
          S.nT = nT;
        }
      }
      // finalisation records of the batch with their ring operands (skip-filtered)
      const int F0 = s_F[0];
      for (int t = (int)threadIdx.x - 32; t < min(s_F[1] - F0, FB); t += SBP - 32) {
        if (t < 0) break;
        const FinRec fr = A.fin_rec[F0 + t];
        FinS& F = fins[t];
        const int qq = fr.qq;
        F.clo[0] = fr.clo[0];
        F.clo[1] = fr.clo[1];
        F.clo[2] = fr.clo[2];
        F.qq = -1;
        F.n = 0;
        if (qq < pbeg || qq >= pend) continue;  // another chunk's position
        if (fr.flags & PM_OVF) {
          F.qq = qq;
          F.n = -1;
          continue;
        }
        // q' within 128 positions of g: its skip bit is still in the ring.  A culled q' has
        // a_lo = 0 (nothing to finalise); culled positions in E_G(q') have factor 1.
        const int qb = qq & 255;
        if ((s_skip[qb >> 5] >> (qb & 31)) & 1u) continue;
        F.qq = qq;
        unsigned long long k0, k1;
        skip_win(s_skip, qq + 1, k0, k1);
        // g = max E_G(q') is the highest bit; its factor comes from the walk's register
        unsigned long long g0 = fr.mg.x & ~k0, g1 = fr.mg.y;
        if (g1) {
          g1 &= ~(1ull << (63 - __clzll((long long)g1)));
          g1 &= ~k1;
        } else {
          g0 &= ~(1ull << (63 - __clzll((long long)fr.mg.x)));
        }
        if (__popcll(g0) + __popcll(g1) > EG8) {
          F.n = -1;
          continue;
        }
        int n = 0;
        for (; g0; g0 &= g0 - 1) F.off[n++] = (unsigned char)__ffsll((long long)g0);
        for (; g1; g1 &= g1 - 1) F.off[n++] = (unsigned char)(64 + __ffsll((long long)g1));
        F.n = (short)n;
      }
      __syncthreads();
      // ---- walk the batch in (kappa, index) order
      for (int j = 0; j < nb; ++j) {
        const SRec<NV>& R = srec[j];
        const int flags = R.flags, pmf = R.pmf;
        const int qpos = b0 + j;  // tile-local position
        if (qpos == anext) {
          recb = Tb;
          recl = Tl;
          rec = true;
        }
        if ((flags & F_SKIP) && pmf == 0) continue;  // a = 0 on the whole block: no effect
        const bool main = qpos >= pbeg && qpos < pend;  // else lookback / lookahead margin
        float alo = 0.f, ahi = 0.f;
        bool keep = false;
        if (!(flags & F_SKIP)) {
          keep = in_img && !(__dadd_rn(cx2[j * SBX + lx], cy2[j * SBY + ly]) > R.r2);
          if (__any_sync(FULLM, keep)) {
            if (flags & F_FAIL) {
              ahi = keep ? R.o[1] : 0.f;
            } else {
              float l, h;
              opacity<NV>(R, lxh - R.ctr[0], lyh - R.ctr[1], l, h);
              alo = keep ? ((flags & F_STRADDLE) ? 0.f : l) : 0.f;
              ahi = keep ? h : 0.f;
            }
          }
        }
        active += (keep && main) ? 1u : 0u;
        if (pmf & PM_STORE) {
          // (1 - a_hi) is read only through E_G of earlier partners (q has PM_EF), the
          // deferred lower term only at q's own finalisation (PM_EG)
          const int rs = RS<SBP>(qpos, 0, rmask);
          if (pmf & PM_HSTART) rf[rs] = Tb;  // read only as some window's base
          rf[rs + SBP] = 1.f - alo;
          if (pmf & PM_EF) rf[rs + 2 * SBP] = 1.f - ahi;
          if (pmf & PM_EG) rf[rs + 3 * SBP] = Tl * alo;
        }
        // upper: T_hi over before(q) \ E_F(q).  Dense windows (mostly E_F): multiply the
        // window [h, q) skipping E_F.  Sparse windows: divide the running product by the
        // E_F factors when that is numerically safe (both products far from underflow),
        // else fall back to the window product (H3).
        float tbv = Tb;
        // (a_hi = 0 on this pixel: its upper contribution is exactly 0, no T_hi needed)
        if (main && (pmf & PM_EF) && !(flags & F_SKIP) && ahi > 0.f) {
          const int wlen = qpos - R.ph;
          DCHECK(wlen > 0 && wlen <= rmask && R.ph >= scan0);
          DCHECK(!(pmf & PM_OVF) || (R.peoff >= 0 && R.peoff + R.pnF <= A.nexc));
          if (!(pmf & PM_OVF)) {
            bool done = false;
            if (R.tmode == 1) {  // dense: T_hi before h times the kept factors
              float pr = rf[RS<SBP>(R.ph, 0, rmask)];
#pragma unroll 4
              for (int t = 0; t < R.nT; ++t) pr *= rf[RS<SBP>(R.ph + R.tlo[t], 1, rmask)];
              tbv = pr;
              done = true;
            } else if (R.tmode == 2) {  // sparse: divide the running product (guarded, H3)
              float dfac = 1.f;
#pragma unroll 4
              for (int t = 0; t < R.nT; ++t) dfac *= rf[RS<SBP>(R.ph + R.tlo[t], 1, rmask)];
              if (dfac >= 1e-20f && Tb >= 1e-25f) {
                tbv = Tb / dfac;
                done = true;
              } else if (A.dbg) {
                atomicAdd(A.dbg + DBG_THI_DIV_UNSAFE, 1ull);
              }
            }
            if (!done) {  // many operands or unsafe division: window product from the bits
              if (A.dbg) atomicAdd(A.dbg + DBG_THI_BITS, 1ull);
              const unsigned long long v0 = wlen >= 64 ? ~0ull : ((1ull << wlen) - 1ull);
              const unsigned long long v1 =
                  wlen <= 64 ? 0ull : (wlen >= 128 ? ~0ull : ((1ull << (wlen - 64)) - 1ull));
              tbv = rf[RS<SBP>(R.ph, 0, rmask)] * ring_prod<SBP>(rf, ~R.mf0 & v0, ~R.mf1 & v1, R.ph, 1, rmask);
            }
          } else {  // long window: exception lists from global memory
            if (A.dbg) atomicAdd(A.dbg + DBG_THI_OVF, 1ull);
            bool done = false;
            if (wlen > 2 * R.pnF + 8) {
              const float dfac = exc_prod<SBP>(rf, A.exc + R.peoff, R.pnF, 1, rmask);
              if (dfac >= 1e-20f && Tb >= 1e-25f) {
                tbv = Tb / dfac;
                done = true;
              }
            }
            if (!done && A.dbg) atomicAdd(A.dbg + DBG_THI_OVF_WINDOW, 1ull);
            if (!done)
              tbv = rf[RS<SBP>(R.ph, 0, rmask)] *
                    window_prod<SBP>(rf, R.ph, qpos, A.exc + R.peoff, R.pnF, rmask);
          }
        }
        // (unc_only: the interval terms of uncertain positions only, O20)
        const float wb = (main && (!A.unc_only || (pmf & (PM_EF | PM_EG)))) ? tbv * ahi : 0.f;
#pragma unroll
        for (int c = 0; c < 3; ++c) ahc[c] = fmaf(wb, R.chi[c], ahc[c]);
        // lower: T_lo over before(q) (E_G(q) empty) or deferred to max E_G(q)
        if (main && !(pmf & PM_EG) && (!A.unc_only || (pmf & PM_EF))) {
          const float wl = Tl * alo;
#pragma unroll
          for (int c = 0; c < 3; ++c) alc[c] = fmaf(wl, R.clo[c], alc[c]);
        }
        Tb = fmaf(-Tb, alo, Tb);
        Tl = fmaf(-Tl, ahi, Tl);
        // finalise deferred lower contributions of earlier partners whose last later
        // partner is q:  T_lo(q') = T_lo,before(q') prod_{r in E_G(q')} (1 - a_hi,r)
        for (int f = R.pfb - F0; f < R.pfe - F0; ++f) {
          float tl;
          const float* clo;
          if (f < FB) {
            const FinS& F = fins[f];
            if (F.qq < 0) continue;  // another chunk's position, or culled in this block
            DCHECK(qpos - F.qq > 0 && qpos - F.qq <= rmask && F.qq >= scan0);
            clo = F.clo;
            tl = rf[RS<SBP>(F.qq, 3, rmask)];
            if (tl == 0.f) continue;  // q' missed this pixel (a_lo = 0): the term is exactly 0
            if (F.n >= 0) {
              tl *= 1.f - ahi;  // g itself
#pragma unroll 4
              for (int e = 0; e < F.n; ++e) tl *= rf[RS<SBP>(F.qq + F.off[e], 2, rmask)];
            } else {
              if (A.dbg) atomicAdd(A.dbg + DBG_FIN_SLOW, 1ull);
              const FinRec& fr = A.fin_rec[F0 + f];
              if (!(fr.flags & PM_OVF)) {
                tl *= ring_prod<SBP>(rf, fr.mg.x, fr.mg.y, fr.qq + 1, 2, rmask);
              } else {
                if (A.dbg) atomicAdd(A.dbg + DBG_FIN_OVF, 1ull);
                tl *= exc_prod<SBP>(rf, A.exc + fr.eoff + fr.nF, fr.nG, 2, rmask);
              }
            }
          } else {
            const FinRec& fr = A.fin_rec[F0 + f];
            if (fr.qq < pbeg || fr.qq >= pend) continue;  // another chunk's position
            if (A.dbg) atomicAdd(A.dbg + DBG_FIN_UNSTAGED, 1ull);
            clo = fr.clo;
            tl = rf[RS<SBP>(fr.qq, 3, rmask)];
            if (tl == 0.f) continue;
            if (!(fr.flags & PM_OVF)) {
              tl *= ring_prod<SBP>(rf, fr.mg.x, fr.mg.y, fr.qq + 1, 2, rmask);
            } else {
              if (A.dbg) atomicAdd(A.dbg + DBG_FIN_OVF, 1ull);
              tl *= exc_prod<SBP>(rf, A.exc + fr.eoff + fr.nF, fr.nG, 2, rmask);
            }
          }
#pragma unroll
          for (int c = 0; c < 3; ++c) alc[c] = fmaf(tl, clo[c], alc[c]);
        }
      }
    }
    // ---- epilogue
    if (iflags & IT_SINGLE) {
      // +- N tau, clamp to [0,1], union over sub-boxes (steps 20-22)
      const int px = ox + lx, py = oy + ly;
      int64_t o = -1;
      if (A.tile_slot) {
        o = ((int64_t)A.tile_slot[tile] * ts * ts + (int64_t)(py - ty * ts) * ts + (px - tx * ts)) * 3;
      } else if (in_img) {
        o = ((int64_t)py * A.W + px) * 3;
      }
      if (o >= 0) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          float l = fminf(fmaxf(alc[c] - A.ntau, 0.f), 1.f);
          float h = fminf(fmaxf(ahc[c] + A.ntau, 0.f), 1.f);
          if (A.unc_only) {
            l = alc[c];
            h = ahc[c];
          }
          if (!in_img) l = h = 0.f;
          if (A.first) {
            A.lo[o + c] = l;
            A.hi[o + c] = h;
          } else {
            A.lo[o + c] = fminf(A.lo[o + c], l);
            A.hi[o + c] = fmaxf(A.hi[o + c], h);
          }
        }
      }
    } else {
      // chunk partial: sums relative to the chunk start and the chunk's transmittance
      if (!rec) {
        recb = Tb;
        recl = Tl;
      }
      float4* dst = reinterpret_cast<float4*>(A.partial + (((size_t)islot * nsub + sub) * SBP + pix) * 8);
      dst[0] = make_float4(ahc[0], ahc[1], ahc[2], recb);
      dst[1] = make_float4(alc[0], alc[1], alc[2], recl);
    }
  }
  // active (pixel, Gaussian) pairs
  unsigned v = active;
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(FULLM, v, s);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(A.active, (unsigned long long)v);
}

// ---- bulk-async (TMA engine) staging helpers: 1-D cp.async.bulk global -> shared with an
// mbarrier completing on the transferred bytes (SASS: UBLKCP / SYNCS)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// order this thread's earlier generic-proxy accesses to shared memory before async-proxy
// (bulk copy) writes to it
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ======================================================================== v2 tile kernel
// Work item = one 16x16 pixel block of a tile (TS >= 16) over one chunk of its list, 128
// threads, TWO pixels per thread: lane (x, y) of warp quadrant (qx, qy) owns the pixels
// (8 qx + x, 8 qy + y) and (8 qx + x, 8 qy + y + 4) -- same column, so the x_0 form and the
// du_0 / x_0 part of every q coefficient are shared, and the per-Gaussian coefficients loaded
// from shared memory serve both pixels.  The per-pixel arithmetic runs pixel-packed: every
// FFMA2 / FADD2 lane is one of the two pixels (the coefficient is the broadcast operand), the
// blend state and the exception ring hold float2 pairs.  Same steps and same per-pixel
// operations as k_tile (which keeps TS = 8).
constexpr int B2 = 16;   // block edge (pixels)
constexpr int T2 = 128;  // threads per block
constexpr int P2 = 256;  // pixels per block
__host__ __device__ __forceinline__ int v2_x(int t) { return ((t >> 5) & 1) * 8 + (t & 7); }
__host__ __device__ __forceinline__ int v2_y(int t) { return (t >> 6) * 8 + ((t >> 3) & 3); }

// Form centres: the per-pixel forms are evaluated in fp32 as x = x_b + du D2 and
// m = p_m + du q_m around a centre.  Around the 16x16 block centre (|du| up to 8) these sums
// cancel many bits for a small Gaussian far from it (the random sweeps' cases above 1e-4, up to
// 2.4e-4).  Each record is therefore centred on the block pixel corner nearest its mean (exact
// per-record offsets, ~0.5% of the kernel): the offsets are small where the opacity is large
// (sweep median error 3.7e-6 -> 6e-7, no case above 1e-4).  Measured and dropped: centring on
// each warp's 8x8 quadrant (every centre-dependent term, or only the q-form constants), 7-8% of
// the kernel for half the offsets.
template <int NV>
struct alignas(16) SRec2 {
  static constexpr int C = NV + 1;
  static constexpr int CP = (C + 3) & ~3;
  // lower x forms at the record's form centre ctr: x_lo,a,k(u) = xb_a[k] + du_a d2[k]
  float xb0[CP], xb1[CP], d2[CP];
  // q_c's (mid, radius) coefficients as affine functions of (du0, du1, x0, |x0|, x1, |x1|):
  //   m = pm + du0 q0m + du1 q1m + x0 wm0 + x1 wm1,  r = pr + du0 q0r + du1 q1r + |x0| wr0 + |x1| wr1
  float4 A[3][C];    // (pm, pr, q0m, q0r)
  float4 B[3][C];    // (wm0, wr0, q1m, q1r)
  float2 W1[3][CP];  // (wm1, wr1)
  float4 WC[3];      // concretised W_0c, W_1c as (mid0, half0, mid1, half1)
  float o[2];
  float ctr[2];      // the form centre (block-local pixels, integer valued)
  float clo[3], chi[3];
  int flags;
  int pmf, ph, pg, pnF, pnG;
  int pfb, pfe;
  long long peoff;
  unsigned long long mf0, mf1;
  int tmode;
  int nT;
  unsigned char tlo[TL8];
  double r2;
};

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 bc(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }

template <int NV>
__device__ __forceinline__ void stage_forms2(SRec2<NV>& S, const HotRec<NV>* H, double ucx,
                                             double ucy, int part) {
  constexpr int C = NV + 1;
  constexpr int KP = (C + NPART - 1) / NPART;
  const double uc[2] = {ucx, ucy};
  // the forms are centred on the block pixel corner nearest the Gaussian's mean (the middle
  // of its mean rectangle, clamped to the block), so the offsets are small where the opacity
  // is large; any centre gives the same forms up to fp32 rounding
  double ctr[2];
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const double o = uc[a] - 0.5 * B2;
    const double rc = fmin(fmax(rint(0.5 * (H->mu[a] + H->mu[2 + a]) - o), 0.0), (double)B2);
    ctr[a] = o + rc;
    if (part == 0) S.ctr[a] = (float)rc;
  }
  double wl[6], wh[6];
#pragma unroll
  for (int e = 0; e < 6; ++e) {
    wl[e] = H->wc[e][0];
    wh[e] = H->wc[e][1];
  }
  if (part == NPART - 1) {
#pragma unroll
    for (int c = 0; c < 3; ++c)
      S.WC[c] = make_float4((float)(0.5 * (wl[c] + wh[c])), (float)(0.5 * (wh[c] - wl[c])),
                            (float)(0.5 * (wl[3 + c] + wh[3 + c])),
                            (float)(0.5 * (wh[3 + c] - wl[3 + c])));
  }
#pragma unroll 1
  for (int i = 0; i < KP; ++i) {
    const int k = part + NPART * i;
    if (k >= C) break;
    const double d2l = H->d2[0][k], d2h = H->d2[1][k];
    float wa[6], wb[6];
#pragma unroll
    for (int e = 0; e < 6; ++e) {
      wa[e] = H->w[e][0][k];
      wb[e] = H->w[e][1][k];
    }
    S.d2[k] = (float)d2l;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double w1l = wl[3 + c], w1h = wh[3 + c];
      const double a0 = wa[c], b0 = wb[c], a1 = wa[3 + c], b1 = wb[3 + c];
      const double q1lo = w1l * (w1l >= 0 ? d2l : d2h), q1hi = w1h * (w1h >= 0 ? d2h : d2l);
      S.B[c][k] = make_float4((float)(0.5 * (a0 + b0)), (float)(0.5 * (b0 - a0)),
                              (float)(0.5 * (q1lo + q1hi)), (float)(0.5 * (q1hi - q1lo)));
      S.W1[c][k] = make_float2((float)(0.5 * (a1 + b1)), (float)(0.5 * (b1 - a1)));
    }
    // the centre-dependent terms
    double blo[2], bhi[2];
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      blo[a] = ctr[a] * d2l - H->du[a][1][k];
      bhi[a] = ctr[a] * d2h - H->du[a][0][k];
    }
    S.xb0[k] = (float)blo[0];
    S.xb1[k] = (float)blo[1];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double w0l = wl[c], w0h = wh[c], w1l = wl[3 + c], w1h = wh[3 + c];
      const double plo = w0l * (w0l >= 0 ? blo[0] : bhi[0]) + w1l * (w1l >= 0 ? blo[1] : bhi[1]);
      const double phi = w0h * (w0h >= 0 ? bhi[0] : blo[0]) + w1h * (w1h >= 0 ? bhi[1] : blo[1]);
      const double q0lo = w0l * (w0l >= 0 ? d2l : d2h), q0hi = w0h * (w0h >= 0 ? d2h : d2l);
      S.A[c][k] = make_float4((float)(0.5 * (plo + phi)), (float)(0.5 * (phi - plo)),
                              (float)(0.5 * (q0lo + q0hi)), (float)(0.5 * (q0hi - q0lo)));
    }
  }
}

// steps 14-17 for the thread's two pixels at offsets (du0, DU1) from the record's form centre
// (du0 shared; DU1 = (du1 of pixel 0, of pixel 1)): returns (a_lo, a_hi) pairs.  Same
// per-pixel operations as s_forms / opacity.
template <int NV>
__device__ __forceinline__ void opacity2(const SRec2<NV>& R, float du0, float2 DU1, float2& alo,
                                         float2& ahi) {
  constexpr int C = NV + 1;
  // 14: concretised lower bounds of x_0 (shared by the column) and x_1 (per pixel)
  float x0 = fmaf(du0, R.d2[NV], R.xb0[NV]);
#pragma unroll
  for (int k = 0; k < NV; ++k) x0 -= fabsf(fmaf(du0, R.d2[k], R.xb0[k]));
  float2 X1 = __ffma2_rn(DU1, bc(R.d2[NV]), bc(R.xb1[NV]));
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const float2 v = __ffma2_rn(DU1, bc(R.d2[k]), bc(R.xb1[k]));
    X1 = __fadd2_rn(X1, f2(-fabsf(v.x), -fabsf(v.y)));
  }
  const float2 AX1 = f2(fabsf(X1.x), fabsf(X1.y));
  const float2 D0 = bc(du0), X0 = f2(x0, fabsf(x0));
  float2 SL[C], SH[C];
#pragma unroll
  for (int k = 0; k < C; ++k) SL[k] = SH[k] = f2(0.f, 0.f);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    // 15: q_c = mul(x0, W_0c) + mul(x1, W_1c) as (mid, radius) forms, per pixel
    float2 M[C], RR[C];
    const float4 wc = R.WC[c];
#pragma unroll
    for (int k = 0; k < C; ++k) {
      const float4 a = R.A[c][k];
      const float4 b = R.B[c][k];
      const float2 w1 = R.W1[c][k];
      float2 mr = __ffma2_rn(D0, f2(a.z, a.w), f2(a.x, a.y));
      mr = __ffma2_rn(X0, f2(b.x, b.y), mr);
      if (k == NV) mr = __ffma2_rn(bc(-x0), f2(wc.x, wc.y), mr);  // - x0 conc W_0c
      float2 m = __ffma2_rn(DU1, bc(b.z), bc(mr.x));
      m = __ffma2_rn(X1, bc(w1.x), m);
      float2 r = __ffma2_rn(DU1, bc(b.w), bc(mr.y));
      r = __ffma2_rn(AX1, bc(w1.y), r);
      if (k == NV) {  // - x1 conc W_1c
        m = __ffma2_rn(X1, bc(-wc.z), m);
        r = __ffma2_rn(X1, bc(-wc.w), r);
      }
      M[k] = m;
      RR[k] = r;
    }
    // concretised q: q_lo = m - r, q_hi = m + r
    float2 qmin = __fadd2_rn(M[NV], f2(-RR[NV].x, -RR[NV].y));
    float2 qmax = __fadd2_rn(M[NV], RR[NV]);
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const float2 ql = __fadd2_rn(M[k], f2(-RR[k].x, -RR[k].y));
      const float2 qh = __fadd2_rn(M[k], RR[k]);
      qmin = __fadd2_rn(qmin, f2(-fabsf(ql.x), -fabsf(ql.y)));
      qmax = __fadd2_rn(qmax, f2(fabsf(qh.x), fabsf(qh.y)));
    }
    // 16: s += sq(q_c): lower tangent at p = clamp(0, qmin, qmax), upper chord (R2), with the
    // side selection written as tp m - |tp| r and sm m + |sm| r
    const float2 P = f2(fminf(fmaxf(0.f, qmin.x), qmax.x), fminf(fmaxf(0.f, qmin.y), qmax.y));
    const float2 TP = __fadd2_rn(P, P), SM = __fadd2_rn(qmin, qmax);
    const float2 NTP = f2(-fabsf(TP.x), -fabsf(TP.y)), ASM = f2(fabsf(SM.x), fabsf(SM.y));
#pragma unroll
    for (int k = 0; k < C; ++k) {
      SL[k] = __ffma2_rn(TP, M[k], SL[k]);
      SL[k] = __ffma2_rn(NTP, RR[k], SL[k]);
      SH[k] = __ffma2_rn(SM, M[k], SH[k]);
      SH[k] = __ffma2_rn(ASM, RR[k], SH[k]);
    }
    SL[NV] = __ffma2_rn(f2(-P.x, -P.y), P, SL[NV]);
    SH[NV] = __ffma2_rn(f2(-qmin.x, -qmin.y), qmax, SH[NV]);
  }
  float2 smin = SL[NV], smax = SH[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    smin = __fadd2_rn(smin, f2(-fabsf(SL[k].x), -fabsf(SL[k].y)));
    smax = __fadd2_rn(smax, f2(fabsf(SH[k].x), fabsf(SH[k].y)));
  }
  // 17: a = o Exp(-s/2) concretised (O11)
  alo = f2(R.o[0] * exp2f(-LOG2E_HALF * smax.x), R.o[0] * exp2f(-LOG2E_HALF * smax.y));
  ahi = f2(R.o[1] * exp2f(-LOG2E_HALF * fmaxf(smin.x, 0.f)),
           R.o[1] * exp2f(-LOG2E_HALF * fmaxf(smin.y, 0.f)));
}

// ring of the v2 kernel: [slot][component][thread] float2 (the thread's two pixels)
__device__ __forceinline__ int RS2(int pos, int comp, int rmask) {
  return ((pos & rmask) * 4 + comp) * T2;
}
__device__ __noinline__ float2 exc_prod2(const float2* rf, const int32_t* list, int n, int comp,
                                         int rmask) {
  float2 prod = f2(1.f, 1.f);
  for (int e0 = 0; e0 < n; e0 += 8) {
    int idx[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) idx[u] = e0 + u < n ? list[e0 + u] : -1;
    float2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = idx[u] >= 0 ? rf[RS2(idx[u], comp, rmask)] : f2(1.f, 1.f);
#pragma unroll
    for (int u = 0; u < 8; ++u) prod = mul2(prod, v[u]);
  }
  return prod;
}
__device__ __noinline__ float2 window_prod2(const float2* rf, int h, int q, const int32_t* ef,
                                            int nf, int rmask) {
  float2 prod = f2(1.f, 1.f);
  int e = 0;
  int nextF = nf > 0 ? ef[0] : 0x7fffffff;
  for (int r0 = h; r0 < q; r0 += 8) {
    float2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = r0 + u < q ? rf[RS2(r0 + u, 1, rmask)] : f2(1.f, 1.f);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int r = r0 + u;
      if (r >= q) break;
      if (r == nextF) {
        ++e;
        nextF = e < nf ? ef[e] : 0x7fffffff;
      } else {
        prod = mul2(prod, v[u]);
      }
    }
  }
  return prod;
}
__device__ __forceinline__ float2 ring_prod2(const float2* rf, unsigned long long m0,
                                             unsigned long long m1, int base, int comp,
                                             int rmask) {
  float2 prod = f2(1.f, 1.f);
  while (m0 | m1) {
    float2 v[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      int idx = -1;
      if (m0) {
        idx = base + __ffsll((long long)m0) - 1;
        m0 &= m0 - 1;
      } else if (m1) {
        idx = base + 64 + __ffsll((long long)m1) - 1;
        m1 &= m1 - 1;
      }
      v[t] = idx >= 0 ? rf[RS2(idx, comp, rmask)] : f2(1.f, 1.f);
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) prod = mul2(prod, v[t]);
  }
  return prod;
}

// EXC = false: the instantiation for renders without uncertain depth pairs (no ring, no
// exception metadata): every exception branch of the walk folds away at compile time
template <int NV, bool EXC>
__global__ void __launch_bounds__(T2, KT2_MINB) k_tile2(TileArgs A) {
  if (A.ovf && *A.ovf) return;  // sizes outgrown: the render is repeated
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_work;
  __shared__ unsigned s_skip[8];
  __shared__ int s_F[2];
  const int ts = A.ts;
  const int nsbx = ts / B2;
  const int nsub = nsbx * nsbx;
  const int BS = A.bs;
  SRec2<NV>* srec = reinterpret_cast<SRec2<NV>*>(smem_raw);
  double* cx2 = reinterpret_cast<double*>(srec + BS);  // [BS][16] per column
  double* cy2 = cx2 + (size_t)BS * B2;                 // [BS][16] per row
  FinS* fins = reinterpret_cast<FinS*>(cy2 + (size_t)BS * B2);  // [FB]
  // raw per-Gaussian records of the next batch, gathered by the bulk-copy engine while the
  // current batch is walked (one mbarrier phase per batch)
  HotRec<NV>* raw = reinterpret_cast<HotRec<NV>*>(fins + FB);     // [BS]
  __shared__ __align__(8) unsigned long long s_bar;
  const bool has_exc = EXC && A.pm != nullptr;
  const int tid = threadIdx.x;
  float2* rf = has_exc ? reinterpret_cast<float2*>(A.ring) + (size_t)blockIdx.x * A.R * 4 * T2 + tid
                       : nullptr;
  constexpr unsigned HSZ = sizeof(HotRec<NV>);
  const HotRec<NV>* hot = reinterpret_cast<const HotRec<NV>*>(A.hot);
  if (tid == 0) mbar_init(&s_bar, 1);
  fence_proxy_async();
  __syncthreads();
  unsigned phase = 0;
  const int lx = v2_x(tid), ly = v2_y(tid);
  // pixel centres in the block (minus each record's form centre in the walk)
  const float lxh = (float)lx + 0.5f;
  const float2 LYH = f2((float)ly + 0.5f, (float)ly + 4.5f);
  unsigned active = 0;
  const int nwork = A.n_items * nsub;
#ifdef KT2_PROF
  long long pr_bar = 0, pr_mbar = 0, pr_stage = 0, pr_walk = 0, pr_t = 0;
#endif

  for (;;) {
    if (tid == 0) s_work = atomicAdd(A.counter, 1);
    __syncthreads();
    const int w = s_work;
    __syncthreads();
    if (w >= nwork) break;
    const int islot = A.order[w / nsub];
    const int sub = w % nsub;
    const int4 it = A.items[islot];
    if (it.x < 0) continue;
    const int tile = it.x, pbeg = it.y, pend = it.z, iflags = it.w;
    const int4 it2 = A.items2[islot];
    const int scan0 = it2.x, scan1 = it2.y, anext = it2.z;
    const int rmask = (1 << ((iflags >> 8) & 0xff)) - 1;
    DCHECK(islot >= 0 && islot < A.n_items && tile >= 0 && tile < A.ntiles);
    DCHECK(0 <= scan0 && scan0 <= pbeg && pbeg <= pend && pend <= scan1);
    DCHECK(A.tbegin[tile] + scan1 <= A.tend[tile] && rmask < A.R);
    const int tx = tile % A.ntx, ty = tile / A.ntx;
    const int ox = tx * ts + (sub % nsbx) * B2, oy = ty * ts + (sub / nsbx) * B2;
    const int64_t tb = A.tbegin[tile];
    const double ucx = ox + 0.5 * B2, ucy = oy + 0.5 * B2;
    const bool iexc = has_exc && (iflags & IT_EXC);
    const double bx0 = ox + 0.5, bx1 = fmin((double)(ox + B2), (double)A.W) - 0.5;
    const double by0 = oy + 0.5, by1 = fmin((double)(oy + B2), (double)A.H) - 0.5;
    const bool block_live = ox < A.W && oy < A.H;
    float2 Tb = f2(1.f, 1.f), Tl = f2(1.f, 1.f);
    float2 ahc[3] = {f2(0.f, 0.f), f2(0.f, 0.f), f2(0.f, 0.f)};
    float2 alc[3] = {f2(0.f, 0.f), f2(0.f, 0.f), f2(0.f, 0.f)};
    float2 recb = f2(1.f, 1.f), recl = f2(1.f, 1.f);
    bool rec = false;
    // gather the item's first batch (later batches are prefetched during the previous walk)
    if (scan0 < scan1) {
      const int nb0 = min(BS, scan1 - scan0);
      if (tid < nb0) {
        const int32_t g = A.vals[tb + scan0 + tid];
        fence_proxy_async();
        bulk_g2s(raw + tid, hot + g, HSZ, &s_bar);
      }
      if (tid == 0) mbar_expect_tx(&s_bar, nb0 * HSZ);
    }

    for (int b0 = scan0; b0 < scan1; b0 += BS) {
      const int nb = min(BS, scan1 - b0);
      const int nbn = min(BS, scan1 - (b0 + nb));  // next batch (0: none)
      int f0l = 0, f1l = 0;
      if (tid == 0 && iexc) {
        f0l = A.finstart[tb + b0];
        f1l = A.finstart[tb + b0 + nb];
      }
      // the next batch's Gaussian ids, loaded now so the copies can be issued right after
      // this batch's records are staged
      const int32_t gnext = tid < nbn ? A.vals[tb + b0 + nb + tid] : 0;
#ifdef KT2_PROF
      // profiling order: the bulk-copy wait first (per thread), then the barrier
      pr_t = clock64();
      mbar_wait(&s_bar, phase);
      { const long long t = clock64(); pr_mbar += t - pr_t; pr_t = t; }
      __syncthreads();
      { volatile int dep = s_work; (void)dep; const long long t = clock64(); pr_bar += t - pr_t; pr_t = t; }
      phase ^= 1u;
#else
      __syncthreads();
      mbar_wait(&s_bar, phase);  // this batch's raw records have landed
      phase ^= 1u;
#endif
      // ---- phase A: metadata + cull tables (one thread per Gaussian, highest ids) and
      //      staging (NPART threads per Gaussian), as in k_tile
      for (int j = T2 - 1 - tid; j < nb; j += T2) {
        const int64_t gp = tb + b0 + j;
        DCHECK(gp >= 0 && gp < A.M);
        const HotRec<NV>* H = raw + j;
        SRec2<NV>& S = srec[j];
        const double mxl = H->mu[0], myl = H->mu[1], mxh = H->mu[2], myh = H->mu[3];
        const double r2 = H->r2;
        bool skip;
        {
          const double dx = fmax(0.0, fmax(__dsub_rn(mxl, bx1), __dsub_rn(bx0, mxh)));
          const double dy = fmax(0.0, fmax(__dsub_rn(myl, by1), __dsub_rn(by0, myh)));
          skip = !block_live || __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)) > r2;
        }
        const int bit = (b0 + j) & 255;
        if (skip)
          atomicOr(&s_skip[bit >> 5], 1u << (bit & 31));
        else
          atomicAnd(&s_skip[bit >> 5], ~(1u << (bit & 31)));
        int pmf = 0;
        if (iexc) {
          const int4 m = A.pm[gp];
          pmf = m.x;
          S.ph = m.y;
          S.pg = m.z;
          S.pnF = m.w;
          S.pnG = A.nG[gp];
          S.peoff = A.eoff[gp];
          S.pfb = A.finstart[gp];
          S.pfe = A.finstart[gp + 1];
          const ulonglong2 mf = A.mF[gp];
          S.mf0 = mf.x;
          S.mf1 = mf.y;
        } else {
          S.pfb = S.pfe = 0;
        }
        S.tmode = 0;
        S.nT = 0;
        S.pmf = pmf;
        S.flags = H->flags | (skip ? F_SKIP : 0);
        // finite radius: an infinite cull-table entry (pixel outside the image) then always
        // fails the walk's test, which needs no per-pixel in-image flag (r2 = inf or NaN keeps
        // every in-image pixel either way)
        S.r2 = fmin(r2, DBL_MAX);
        S.o[0] = H->o[0];
        S.o[1] = H->o[1];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          S.clo[c] = H->clo[c];
          S.chi[c] = H->chi[c];
        }
        if (!skip) {
#pragma unroll
          for (int l = 0; l < B2; ++l) {
            const double x = ox + l + 0.5;
            const double dx = fmax(0.0, fmax(__dsub_rn(mxl, x), __dsub_rn(x, mxh)));
            cx2[j * B2 + l] = ox + l < A.W ? __dmul_rn(dx, dx) : (double)INFINITY;
            const double y = oy + l + 0.5;
            const double dy = fmax(0.0, fmax(__dsub_rn(myl, y), __dsub_rn(y, myh)));
            cy2[j * B2 + l] = oy + l < A.H ? __dmul_rn(dy, dy) : (double)INFINITY;
          }
        }
      }
      for (int jj = tid; jj < NPART * nb; jj += T2) {
        const int j = jj / NPART, part = jj % NPART;
        const HotRec<NV>* H = raw + j;
        bool skip;
        {
          const double dx = fmax(0.0, fmax(__dsub_rn(H->mu[0], bx1), __dsub_rn(bx0, H->mu[2])));
          const double dy = fmax(0.0, fmax(__dsub_rn(H->mu[1], by1), __dsub_rn(by0, H->mu[3])));
          skip = !block_live || __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)) > H->r2;
        }
        if (!skip) stage_forms2<NV>(srec[j], H, ucx, ucy, part);
      }
      if (tid == 0) {
        s_F[0] = f0l;
        s_F[1] = f1l;
      }
      __syncthreads();
      // raw records consumed: gather the next batch's while this one is walked
      if (tid < nbn) {
        fence_proxy_async();
        bulk_g2s(raw + tid, hot + gnext, HSZ, &s_bar);
      }
      if (tid == 0 && nbn > 0) mbar_expect_tx(&s_bar, nbn * HSZ);
      // ---- phase B: T_hi window operand lists (warp 0) and staged finalisation records
      if (iexc) {
        for (int j = tid < 32 ? tid : nb; j < nb; j += 32) {
          SRec2<NV>& S = srec[j];
          const int pmf = S.pmf, qpos = b0 + j;
          if (!(pmf & PM_EF) || (S.flags & F_SKIP) || qpos < pbeg || qpos >= pend || (pmf & PM_OVF))
            continue;
          const int h = S.ph, wlen = qpos - h;
          const unsigned long long v0 = wlen >= 64 ? ~0ull : ((1ull << wlen) - 1ull);
          const unsigned long long v1 =
              wlen <= 64 ? 0ull : (wlen >= 128 ? ~0ull : ((1ull << (wlen - 64)) - 1ull));
          unsigned long long k0, k1;
          skip_win(s_skip, h, k0, k1);
          const unsigned long long e0 = S.mf0 & ~k0, e1 = S.mf1 & ~k1;
          const unsigned long long g0 = ~S.mf0 & ~k0 & v0, g1 = ~S.mf1 & ~k1 & v1;
          const int nef = __popcll(e0) + __popcll(e1), nkept = __popcll(g0) + __popcll(g1);
          const bool dense = !(nkept > nef + 2);
          unsigned long long m0 = dense ? g0 : e0;
          unsigned long long m1 = dense ? g1 : e1;
          const int cnt = dense ? nkept : nef;
          int nT = 0;
          if (cnt <= TL8) {
            S.tmode = dense ? 1 : 2;
            for (; m0; m0 &= m0 - 1) S.tlo[nT++] = (unsigned char)(__ffsll((long long)m0) - 1);
            for (; m1; m1 &= m1 - 1) S.tlo[nT++] = (unsigned char)(64 + __ffsll((long long)m1) - 1);
          } else {
            S.tmode = 3;
            if (A.dbg) atomicAdd(A.dbg + DBG_TMODE3, 1ull);
          }
          S.nT = nT;
        }
      }
      const int F0 = s_F[0];
      for (int t = tid - 32; EXC && t < min(s_F[1] - F0, FB); t += T2 - 32) {
        if (t < 0) break;
        const FinRec fr = A.fin_rec[F0 + t];
        FinS& F = fins[t];
        const int qq = fr.qq;
        F.clo[0] = fr.clo[0];
        F.clo[1] = fr.clo[1];
        F.clo[2] = fr.clo[2];
        F.qq = -1;
        F.n = 0;
        if (qq < pbeg || qq >= pend) continue;
        if (fr.flags & PM_OVF) {
          F.qq = qq;
          F.n = -1;
          continue;
        }
        const int qb = qq & 255;
        if ((s_skip[qb >> 5] >> (qb & 31)) & 1u) continue;
        F.qq = qq;
        unsigned long long k0, k1;
        skip_win(s_skip, qq + 1, k0, k1);
        unsigned long long g0 = fr.mg.x & ~k0, g1 = fr.mg.y;
        if (g1) {
          g1 &= ~(1ull << (63 - __clzll((long long)g1)));
          g1 &= ~k1;
        } else {
          g0 &= ~(1ull << (63 - __clzll((long long)fr.mg.x)));
        }
        if (__popcll(g0) + __popcll(g1) > EG8) {
          F.n = -1;
          continue;
        }
        int n = 0;
        for (; g0; g0 &= g0 - 1) F.off[n++] = (unsigned char)__ffsll((long long)g0);
        for (; g1; g1 &= g1 - 1) F.off[n++] = (unsigned char)(64 + __ffsll((long long)g1));
        F.n = (short)n;
      }
      __syncthreads();
#ifdef KT2_PROF
      { const long long t = clock64(); pr_stage += t - pr_t; pr_t = t; }
#endif
      // ---- walk the batch in (kappa, index) order, two pixels per thread
      for (int j = 0; j < nb; ++j) {
        const SRec2<NV>& R = srec[j];
        const int flags = R.flags, pmf = EXC ? R.pmf : 0;
        const int qpos = b0 + j;
        if (qpos == anext) {
          recb = Tb;
          recl = Tl;
          rec = true;
        }
        if ((flags & F_SKIP) && pmf == 0) continue;
        const bool main = qpos >= pbeg && qpos < pend;
        // the first finalisation record's deferred term, loaded before the opacity so its
        // latency hides behind it (slot qq is not rewritten before the use: qpos - qq < R)
        const int fr0 = R.pfb - F0;
        float2 tl0 = f2(0.f, 0.f);
        if (EXC && fr0 < R.pfe - F0 && fr0 < FB) {
          const int q0 = fins[fr0].qq;
          if (q0 >= 0) tl0 = rf[RS2(q0, 3, rmask)];
        }
        float2 alo = f2(0.f, 0.f), ahi = f2(0.f, 0.f);
        bool kA = false, kB = false;
        if (!(flags & F_SKIP)) {
          const double cx = cx2[j * B2 + lx];
          kA = !(__dadd_rn(cx, cy2[j * B2 + ly]) > R.r2);
          kB = !(__dadd_rn(cx, cy2[j * B2 + ly + 4]) > R.r2);
          if (__any_sync(FULLM, kA || kB)) {
            if (flags & F_FAIL) {
              ahi = f2(kA ? R.o[1] : 0.f, kB ? R.o[1] : 0.f);
            } else {
              float2 l, h;
              // offsets from the record's form centre (exact)
              opacity2<NV>(R, lxh - R.ctr[0], f2(LYH.x - R.ctr[1], LYH.y - R.ctr[1]), l, h);
              const bool st = flags & F_STRADDLE;
              alo = f2(kA && !st ? l.x : 0.f, kB && !st ? l.y : 0.f);
              ahi = f2(kA ? h.x : 0.f, kB ? h.y : 0.f);
            }
          }
        }
        active += main ? (unsigned)kA + (unsigned)kB : 0u;
        if (pmf & PM_STORE) {
          const int rs = RS2(qpos, 0, rmask);
          DCHECK(rf != nullptr);
          if (pmf & PM_HSTART) rf[rs] = Tb;
          rf[rs + T2] = f2(1.f - alo.x, 1.f - alo.y);
          if (pmf & PM_EF) rf[rs + 2 * T2] = f2(1.f - ahi.x, 1.f - ahi.y);
          if (pmf & PM_EG) rf[rs + 3 * T2] = mul2(Tl, alo);
        }
        float2 tbv = Tb;
        if (main && (pmf & PM_EF) && !(flags & F_SKIP) && (ahi.x > 0.f || ahi.y > 0.f)) {
          const int wlen = qpos - R.ph;
          DCHECK(wlen > 0 && wlen <= rmask && R.ph >= scan0);
          DCHECK(!(pmf & PM_OVF) || (R.peoff >= 0 && R.peoff + R.pnF <= A.nexc));
          if (!(pmf & PM_OVF)) {
            bool done = false;
            if (R.tmode == 1) {
              float2 pr = rf[RS2(R.ph, 0, rmask)];
#pragma unroll 4
              for (int t = 0; t < R.nT; ++t) pr = mul2(pr, rf[RS2(R.ph + R.tlo[t], 1, rmask)]);
              tbv = pr;
              done = true;
            } else if (R.tmode == 2) {
              float2 dfac = f2(1.f, 1.f);
#pragma unroll 4
              for (int t = 0; t < R.nT; ++t) dfac = mul2(dfac, rf[RS2(R.ph + R.tlo[t], 1, rmask)]);
              if (dfac.x >= 1e-20f && dfac.y >= 1e-20f && Tb.x >= 1e-25f && Tb.y >= 1e-25f) {
                tbv = f2(Tb.x / dfac.x, Tb.y / dfac.y);
                done = true;
              } else if (A.dbg) {
                atomicAdd(A.dbg + DBG_THI_DIV_UNSAFE, 1ull);
              }
            }
            if (!done) {
              if (A.dbg) atomicAdd(A.dbg + DBG_THI_BITS, 1ull);
              const unsigned long long v0 = wlen >= 64 ? ~0ull : ((1ull << wlen) - 1ull);
              const unsigned long long v1 =
                  wlen <= 64 ? 0ull : (wlen >= 128 ? ~0ull : ((1ull << (wlen - 64)) - 1ull));
              tbv = mul2(rf[RS2(R.ph, 0, rmask)],
                         ring_prod2(rf, ~R.mf0 & v0, ~R.mf1 & v1, R.ph, 1, rmask));
            }
          } else {
            if (A.dbg) atomicAdd(A.dbg + DBG_THI_OVF, 1ull);
            bool done = false;
            if (wlen > 2 * R.pnF + 8) {
              const float2 dfac = exc_prod2(rf, A.exc + R.peoff, R.pnF, 1, rmask);
              if (dfac.x >= 1e-20f && dfac.y >= 1e-20f && Tb.x >= 1e-25f && Tb.y >= 1e-25f) {
                tbv = f2(Tb.x / dfac.x, Tb.y / dfac.y);
                done = true;
              }
            }
            if (!done && A.dbg) atomicAdd(A.dbg + DBG_THI_OVF_WINDOW, 1ull);
            if (!done)
              tbv = mul2(rf[RS2(R.ph, 0, rmask)],
                         window_prod2(rf, R.ph, qpos, A.exc + R.peoff, R.pnF, rmask));
          }
        }
        // (unc_only: the interval terms of uncertain positions only, O20)
        const float2 wb = (main && (!A.unc_only || (pmf & (PM_EF | PM_EG)))) ? mul2(tbv, ahi)
                                                                            : f2(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < 3; ++c) ahc[c] = __ffma2_rn(wb, bc(R.chi[c]), ahc[c]);
        if (main && !(pmf & PM_EG) && (!A.unc_only || (pmf & PM_EF))) {
          const float2 wl = mul2(Tl, alo);
#pragma unroll
          for (int c = 0; c < 3; ++c) alc[c] = __ffma2_rn(wl, bc(R.clo[c]), alc[c]);
        }
        Tb = __ffma2_rn(f2(-Tb.x, -Tb.y), alo, Tb);
        Tl = __ffma2_rn(f2(-Tl.x, -Tl.y), ahi, Tl);
        for (int f = R.pfb - F0; EXC && f < R.pfe - F0; ++f) {
          float2 tl;
          const float* clo;
          if (f < FB) {
            const FinS& F = fins[f];
            if (F.qq < 0) continue;
            DCHECK(qpos - F.qq > 0 && qpos - F.qq <= rmask && F.qq >= scan0);
            clo = F.clo;
            tl = f == fr0 ? tl0 : rf[RS2(F.qq, 3, rmask)];
            if (tl.x == 0.f && tl.y == 0.f) continue;
            if (F.n >= 0) {
              tl = mul2(tl, f2(1.f - ahi.x, 1.f - ahi.y));
#pragma unroll 4
              for (int e = 0; e < F.n; ++e) tl = mul2(tl, rf[RS2(F.qq + F.off[e], 2, rmask)]);
            } else {
              if (A.dbg) atomicAdd(A.dbg + DBG_FIN_SLOW, 1ull);
              const FinRec& fr = A.fin_rec[F0 + f];
              if (!(fr.flags & PM_OVF)) {
                tl = mul2(tl, ring_prod2(rf, fr.mg.x, fr.mg.y, fr.qq + 1, 2, rmask));
              } else {
                if (A.dbg) atomicAdd(A.dbg + DBG_FIN_OVF, 1ull);
                tl = mul2(tl, exc_prod2(rf, A.exc + fr.eoff + fr.nF, fr.nG, 2, rmask));
              }
            }
          } else {
            const FinRec& fr = A.fin_rec[F0 + f];
            if (fr.qq < pbeg || fr.qq >= pend) continue;
            if (A.dbg) atomicAdd(A.dbg + DBG_FIN_UNSTAGED, 1ull);
            DCHECK(qpos - fr.qq > 0 && qpos - fr.qq <= rmask && fr.qq >= scan0);
            DCHECK(!(fr.flags & PM_OVF) || fr.eoff + fr.nF + fr.nG <= A.nexc);
            clo = fr.clo;
            tl = rf[RS2(fr.qq, 3, rmask)];
            if (tl.x == 0.f && tl.y == 0.f) continue;
            if (!(fr.flags & PM_OVF)) {
              tl = mul2(tl, ring_prod2(rf, fr.mg.x, fr.mg.y, fr.qq + 1, 2, rmask));
            } else {
              if (A.dbg) atomicAdd(A.dbg + DBG_FIN_OVF, 1ull);
              tl = mul2(tl, exc_prod2(rf, A.exc + fr.eoff + fr.nF, fr.nG, 2, rmask));
            }
          }
#pragma unroll
          for (int c = 0; c < 3; ++c) alc[c] = __ffma2_rn(tl, bc(clo[c]), alc[c]);
        }
      }
#ifdef KT2_PROF
      { const long long t = clock64(); pr_walk += t - pr_t; pr_t = t; }
#endif
    }
    // ---- epilogue (both pixels)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int py = oy + ly + 4 * e, px = ox + lx;
      const bool in = (px < A.W) && (py < A.H);
      const float hc[3] = {e ? ahc[0].y : ahc[0].x, e ? ahc[1].y : ahc[1].x, e ? ahc[2].y : ahc[2].x};
      const float lc[3] = {e ? alc[0].y : alc[0].x, e ? alc[1].y : alc[1].x, e ? alc[2].y : alc[2].x};
      if (iflags & IT_SINGLE) {
        int64_t o = -1;
        if (A.tile_slot) {
          o = ((int64_t)A.tile_slot[tile] * ts * ts + (int64_t)(py - ty * ts) * ts + (px - tx * ts)) * 3;
        } else if (in) {
          o = ((int64_t)py * A.W + px) * 3;
        }
        if (o >= 0) {
          DCHECK(o + 3 <= A.n_out);
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            float l = fminf(fmaxf(lc[c] - A.ntau, 0.f), 1.f);
            float h = fminf(fmaxf(hc[c] + A.ntau, 0.f), 1.f);
            if (A.unc_only) {
              l = lc[c];
              h = hc[c];
            }
            if (!in) l = h = 0.f;
            if (A.first) {
              A.lo[o + c] = l;
              A.hi[o + c] = h;
            } else {
              A.lo[o + c] = fminf(A.lo[o + c], l);
              A.hi[o + c] = fmaxf(A.hi[o + c], h);
            }
          }
        }
      } else {
        const float2 rb = rec ? recb : Tb, rl = rec ? recl : Tl;
        const int pix = (ly + 4 * e) * B2 + lx;
        DCHECK((int64_t)(((size_t)islot * nsub + sub) * P2 + pix) * 8 + 8 <= A.n_partial);
        float4* dst = reinterpret_cast<float4*>(A.partial + (((size_t)islot * nsub + sub) * P2 + pix) * 8);
        dst[0] = make_float4(hc[0], hc[1], hc[2], e ? rb.y : rb.x);
        dst[1] = make_float4(lc[0], lc[1], lc[2], e ? rl.y : rl.x);
      }
    }
  }
#ifdef KT2_PROF
  if ((tid & 31) == 0 && A.dbg) {
    atomicAdd(A.dbg + 0, (unsigned long long)pr_bar);
    atomicAdd(A.dbg + 1, (unsigned long long)pr_mbar);
    atomicAdd(A.dbg + 2, (unsigned long long)pr_stage);
    atomicAdd(A.dbg + 3, (unsigned long long)pr_walk);
  }
#endif
  unsigned v = active;
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(FULLM, v, s);
  if ((tid & 31) == 0 && v) atomicAdd(A.active, (unsigned long long)v);
}

// ---------------------------------------------------------------- NEXT-1 linear blend
// One CTA per (exception-free tile, 8x8 block), one thread per pixel: BlendInd with linear
// relations along the sorted fold (Alg. 3; oracle blend_linear):
//   a = o Exp(-s/2) with Table 2's tangent (lower) / chord (upper) kept linear in xi,
//   pc_c += Mul(T, a) c,  T <- Mul(T, 1 - a)   (R1 McCormick, fp32 forms),
// finalised (+- N tau, clamp) and intersected with the interval bounds already in img.
template <int NV>
__global__ void __launch_bounds__(64) k_tile_lin(TileArgs A, const int32_t* tiles, int n_tiles,
                                                 float* img_lo, float* img_hi,
                                                 const float* unc_lo, const float* unc_hi) {
  constexpr int SBX = 8, SBP = 64, C = NV + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int ts = A.ts, nsb = ts / SBX, nsub = nsb * nsb;
  const int BS = A.bs;
  SRec<NV>* srec = reinterpret_cast<SRec<NV>*>(smem_raw);
  double* cx2 = reinterpret_cast<double*>(srec + BS);
  double* cy2 = cx2 + (size_t)BS * SBX;
  const int w = blockIdx.x;
  if (w >= n_tiles * nsub) return;
  const int tile = tiles[w / nsub], sub = w % nsub;
  const int pix = threadIdx.x, lx = pix & 7, ly = pix >> 3;
  const int tx = tile % A.ntx, ty = tile / A.ntx;
  const int ox = tx * ts + (sub % nsb) * SBX, oy = ty * ts + (sub / nsb) * SBY;
  const double ucx = ox + 0.5 * SBX, ucy = oy + 0.5 * SBY;
  const bool in_img = (ox + lx < A.W) && (oy + ly < A.H);
  const bool block_live = ox < A.W && oy < A.H;
  const double bx0 = ox + 0.5, bx1 = fmin((double)(ox + SBX), (double)A.W) - 0.5;
  const double by0 = oy + 0.5, by1 = fmin((double)(oy + SBY), (double)A.H) - 0.5;
  const int64_t tb = A.tbegin[tile];
  const int K = (int)(A.tend[tile] - tb);
  float Tl[C], Th[C], pl[3][C], ph[3][C];
#pragma unroll
  for (int k = 0; k < C; ++k) {
    Tl[k] = Th[k] = (k == NV) ? 1.f : 0.f;
#pragma unroll
    for (int c = 0; c < 3; ++c) pl[c][k] = ph[c][k] = 0.f;
  }
  for (int b0 = 0; b0 < K; b0 += BS) {
    const int nb = min(BS, K - b0);
    __syncthreads();
    for (int jj = threadIdx.x; jj < NPART * nb; jj += SBP) {
      const int j = jj / NPART, part = jj % NPART;
      const HotRec<NV>* H = reinterpret_cast<const HotRec<NV>*>(A.hot) + A.vals[tb + b0 + j];
      SRec<NV>& S = srec[j];
      const double mxl = H->mu[0], myl = H->mu[1], mxh = H->mu[2], myh = H->mu[3];
      const double dx = fmax(0.0, fmax(__dsub_rn(mxl, bx1), __dsub_rn(bx0, mxh)));
      const double dy = fmax(0.0, fmax(__dsub_rn(myl, by1), __dsub_rn(by0, myh)));
      const bool skip = !block_live || __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)) > H->r2;
      if (part == NPART - 1) {
        S.flags = H->flags | (skip ? F_SKIP : 0);
        S.pmf = A.pm ? A.pm[tb + b0 + j].x : 0;  // uncertain partners (O20)
        S.r2 = H->r2;
        S.o[0] = H->o[0];
        S.o[1] = H->o[1];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          S.clo[c] = H->clo[c];
          S.chi[c] = H->chi[c];
        }
        if (!skip) {
#pragma unroll
          for (int l = 0; l < SBX; ++l) {
            const double x = ox + l + 0.5, y = oy + l + 0.5;
            const double ddx = fmax(0.0, fmax(__dsub_rn(mxl, x), __dsub_rn(x, mxh)));
            const double ddy = fmax(0.0, fmax(__dsub_rn(myl, y), __dsub_rn(y, myh)));
            cx2[j * SBX + l] = __dmul_rn(ddx, ddx);
            cy2[j * SBY + l] = __dmul_rn(ddy, ddy);
          }
        }
      }
      if (!skip) stage_forms<NV>(S, H, ucx, ucy, 0.5 * SBX, 0.5 * SBY, part);
    }
    __syncthreads();
    for (int j = 0; j < nb; ++j) {
      const SRec<NV>& R = srec[j];
      const int flags = R.flags;
      if (flags & F_SKIP) continue;
      const bool keep = in_img && !(__dadd_rn(cx2[j * SBX + lx], cy2[j * SBY + ly]) > R.r2);
      if (!keep) continue;  // a = 0 at this pixel: T unchanged, no contribution
      float al[C], ah[C];
      if (flags & F_FAIL) {
#pragma unroll
        for (int k = 0; k < C; ++k) al[k] = ah[k] = 0.f;
        ah[NV] = R.o[1];
      } else {
        float sl[C], sh[C];
        opacity_sforms<NV>(R, (float)lx + 0.5f - R.ctr[0], (float)ly + 0.5f - R.ctr[1], sl, sh);
        float smin = sl[NV], smax = sh[NV];
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          smin -= fabsf(sl[k]);
          smax += fabsf(sh[k]);
        }
        smin = fmaxf(smin, 0.f);
        const float zl = -0.5f * smax, zh = -0.5f * smin;
        const float el = expf(zl), eh = expf(zh);
        const float m = zh > zl ? (eh - el) / (zh - zl) : eh;
        const float cl = R.o[0] * el, ch = R.o[1] * m;
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          al[k] = cl * (-0.5f * sh[k]);
          ah[k] = ch * (-0.5f * sl[k]);
        }
        al[NV] = cl * (-0.5f * sh[NV] + 1.f - zl);
        ah[NV] = R.o[1] * fmaf(m, -0.5f * sl[NV] - zl, el);
        if (flags & F_STRADDLE) {
#pragma unroll
          for (int k = 0; k < C; ++k) al[k] = 0.f;
        }
      }
      if (!(R.pmf & (PM_EF | PM_EG))) {  // certain position: Mul(T, a) c (uncertain: unc_*)
        float tal[C], tah[C];
        form_mul<NV>(Tl, Th, al, ah, tal, tah);
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int k = 0; k < C; ++k) {
            pl[c][k] = fmaf(R.clo[c], tal[k], pl[c][k]);
            ph[c][k] = fmaf(R.chi[c], tah[k], ph[c][k]);
          }
      }
      float oml[C], omh[C];  // 1 - a
#pragma unroll
      for (int k = 0; k < C; ++k) {
        oml[k] = -ah[k];
        omh[k] = -al[k];
      }
      oml[NV] += 1.f;
      omh[NV] += 1.f;
      float nl[C], nh[C];
      form_mul<NV>(Tl, Th, oml, omh, nl, nh);
#pragma unroll
      for (int k = 0; k < C; ++k) {
        Tl[k] = nl[k];
        Th[k] = nh[k];
      }
    }
  }
  if (!in_img) return;
  const int64_t o = ((int64_t)(oy + ly) * A.W + (ox + lx)) * 3;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    float l = pl[c][NV], h = ph[c][NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      l -= fabsf(pl[c][k]);
      h += fabsf(ph[c][k]);
    }
    if (unc_lo) {  // the uncertain positions' interval terms (raw sums, O20)
      l += unc_lo[o + c];
      h += unc_hi[o + c];
    }
    l = fminf(fmaxf(l - A.ntau, 0.f), 1.f);
    h = fminf(fmaxf(h + A.ntau, 0.f), 1.f);
    img_lo[o + c] = fmaxf(img_lo[o + c], l);
    img_hi[o + c] = fminf(img_hi[o + c], h);
  }
}

// union of one sub-box image into the result (step 22): copy for the first sub-box
__global__ void k_union(const float* slo, const float* shi, float* lo, float* hi, int64_t n,
                        int first) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  lo[i] = first ? slo[i] : fminf(lo[i], slo[i]);
  hi[i] = first ? shi[i] : fmaxf(hi[i], shi[i]);
}

// front-to-back composition of a tile's chunks: pc = sum_k P(<A_k) S_k with
// P(<A_{k+1}) = P(<A_k) R_k (R_k = chunk k's running product at A_{k+1})
__global__ void k_merge(TileArgs A) {
  if (A.ovf && *A.ovf) return;
  const int tile = blockIdx.x;
  const int n = A.item_cnt[tile];
  if (n <= 1) return;
  const int ts = A.ts, npix = ts * ts;
  // partial layout of the kernel that wrote them: k_tile2 16x16 blocks (row-major pixels),
  // k_tile its 16x8 / 8x8 blocks
  const bool v2 = A.kver == 2;
  const int SBX = v2 ? B2 : block_w(ts), SBH = v2 ? B2 : SBY, SBP = SBX * SBH;
  const int nsbx = ts / SBX, nsub = nsbx * (ts / SBH);
  const int tx = tile % A.ntx, ty = tile / A.ntx;
  for (int tp = threadIdx.x; tp < npix; tp += blockDim.x) {
    const int lx = tp % ts, ly = tp / ts;
    const int sub = (ly / SBH) * nsbx + lx / SBX;
    const int pix = v2 ? (ly % SBH) * SBX + lx % SBX : pix_of(lx % SBX, ly % SBY, SBX);
    float Pb = 1.f, Pl = 1.f, h[3] = {0.f, 0.f, 0.f}, l[3] = {0.f, 0.f, 0.f};
    for (int k = 0; k < n; ++k) {
      const int64_t it = A.item_off[tile] + k;
      DCHECK(it >= 0 && it < A.n_items &&
             (int64_t)(((size_t)it * nsub + sub) * SBP + pix) * 8 + 8 <= A.n_partial);
      const float4* src =
          reinterpret_cast<const float4*>(A.partial + (((size_t)it * nsub + sub) * SBP + pix) * 8);
      const float4 a = src[0], b = src[1];
      h[0] = fmaf(Pb, a.x, h[0]);
      h[1] = fmaf(Pb, a.y, h[1]);
      h[2] = fmaf(Pb, a.z, h[2]);
      l[0] = fmaf(Pl, b.x, l[0]);
      l[1] = fmaf(Pl, b.y, l[1]);
      l[2] = fmaf(Pl, b.z, l[2]);
      Pb *= a.w;
      Pl *= b.w;
    }
    const int px = tx * ts + lx, py = ty * ts + ly;
    const bool inside = px < A.W && py < A.H;
    int64_t o;
    if (A.tile_slot) {
      o = ((int64_t)A.tile_slot[tile] * npix + tp) * 3;
    } else {
      if (!inside) continue;
      o = ((int64_t)py * A.W + px) * 3;
    }
    for (int c = 0; c < 3; ++c) {
      float lv = fminf(fmaxf(l[c] - A.ntau, 0.f), 1.f);
      float hv = fminf(fmaxf(h[c] + A.ntau, 0.f), 1.f);
      if (A.unc_only) {
        lv = l[c];
        hv = h[c];
      }
      if (!inside) lv = hv = 0.f;
      if (A.first) {
        A.lo[o + c] = lv;
        A.hi[o + c] = hv;
      } else {
        A.lo[o + c] = fminf(A.lo[o + c], lv);
        A.hi[o + c] = fmaxf(A.hi[o + c], hv);
      }
    }
  }
}

// kernel version: 2 = k_tile2 (TS >= 16: 16x16 blocks, two pixels per thread), 1 = k_tile
// (TS = 8).  A warp-independent variant (every warp its own 8x8 quadrant work items, no CTA
// barrier) measured 44 ms on C4 against k_tile2's 27.5 ms (4x the staging per pixel, each
// warp waiting on its own record loads) and was removed.
int tile_kernel_version(int ts) { return ts >= B2 ? 2 : 1; }
int tile_threads(int ts) { return tile_kernel_version(ts) == 2 ? T2 : block_w(ts) * SBY; }
int tile_subblocks(int ts) {
  return tile_kernel_version(ts) == 2 ? (ts / B2) * (ts / B2) : (ts / block_w(ts)) * (ts / SBY);
}
size_t tile_ring_slot_bytes(int ts) {  // exception ring bytes per slot per CTA
  return tile_kernel_version(ts) == 2 ? (size_t)4 * T2 * sizeof(float2)
                                      : (size_t)tile_threads(ts) * sizeof(float4);
}
int tile_batch(int nv, int ts, int bs);

template <int NV>
static size_t smem_for(int ts, int bs) {
  if (ts >= B2)
    return (size_t)bs * (sizeof(SRec2<NV>) + 2 * B2 * sizeof(double) + sizeof(HotRec<NV>)) +
           FB * sizeof(FinS);
  return (size_t)bs * (sizeof(SRec<NV>) + (block_w(ts) + SBY) * sizeof(double)) +
         FB * sizeof(FinS);
}

// BS clamped to what fits (<= 96 KB of shared memory) and to 128 (the 256-position skip
// ring covers a batch plus the 128 positions before it)
int tile_batch(int nv, int ts, int bs) {
  bs = std::min(bs, 128);
  if (tile_kernel_version(ts) == 2) {  // k_tile2: as many CTAs per SM as the registers allow
    while (bs > 1 && tile_smem_bytes(nv, ts, bs) > (size_t)(220 / KT2_MINB - 1) * 1024) --bs;
    return bs;
  }
  while (bs > 1 && tile_smem_bytes(nv, ts, bs) > 96 * 1024) bs >>= 1;
  return bs;
}

size_t tile_smem_bytes(int nv, int ts, int bs) {
  switch (nv) {
#define CASE(K) \
  case K:       \
    return smem_for<K>(ts, bs);
    CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9)
#undef CASE
    default:
      return 0;
  }
}

template <int NV, int BX>
static int grid_bx(int ts, int bs) {
  // the dynamic shared-memory opt-in is per device: set it on the current one every time
  // (a host-side attribute write), and report failure as grid 0
  if (cudaFuncSetAttribute(k_tile<NV, BX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           200 * 1024) != cudaSuccess)
    return 0;
  int per_sm = 0, dev = 0, nsm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tile<NV, BX>, BX * SBY,
                                                smem_for<NV>(ts, bs));
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  return std::max(1, per_sm) * nsm;
}
template <int NV>
static int grid_v2(int ts, int bs) {
  if (cudaFuncSetAttribute(k_tile2<NV, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           200 * 1024) != cudaSuccess ||
      cudaFuncSetAttribute(k_tile2<NV, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           200 * 1024) != cudaSuccess)
    return 0;
  int per_sm = 0, dev = 0, nsm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tile2<NV, true>, T2,
                                                smem_for<NV>(ts, bs));
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  return std::max(1, per_sm) * nsm;
}
template <int NV>
static int grid_one(int ts, int bs) {
  if (tile_kernel_version(ts) == 2) return grid_v2<NV>(ts, bs);
  return block_w(ts) == 16 ? grid_bx<NV, 16>(ts, bs) : grid_bx<NV, 8>(ts, bs);
}

int tile_grid(int nv, int ts, int bs) {
  switch (nv) {
#define CASE(K) \
  case K:       \
    return grid_one<K>(ts, bs);
    CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9)
#undef CASE
    default:
      return 0;
  }
}

template <int NV>
static void launch_one(const TileArgs& a, int grid, cudaStream_t st) {
  if (a.kver == 2 && a.pm)
    k_tile2<NV, true><<<grid, T2, smem_for<NV>(a.ts, a.bs), st>>>(a);
  else if (a.kver == 2)
    k_tile2<NV, false><<<grid, T2, smem_for<NV>(a.ts, a.bs), st>>>(a);
  else if (block_w(a.ts) == 16)
    k_tile<NV, 16><<<grid, 16 * SBY, smem_for<NV>(a.ts, a.bs), st>>>(a);
  else
    k_tile<NV, 8><<<grid, 8 * SBY, smem_for<NV>(a.ts, a.bs), st>>>(a);
}

void launch_tile(int nv, const TileArgs& a, int grid, cudaStream_t st) {
  if (a.n_items <= 0 || grid <= 0) return;
  switch (nv) {
#define CASE(K)                    \
  case K:                          \
    launch_one<K>(a, grid, st);    \
    break;
    CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9)
#undef CASE
    default:
      break;
  }
}

template <int NV>
static size_t smem_lin(int bs) {
  return (size_t)bs * (sizeof(SRec<NV>) + 2 * 8 * sizeof(double));
}
void launch_tile_lin(int nv, const TileArgs& a, const int32_t* tiles, int n_tiles, float* lo,
                     float* hi, const float* unc_lo, const float* unc_hi, cudaStream_t st) {
  const int grid = n_tiles * (a.ts / 8) * (a.ts / 8);
  if (grid <= 0) return;
  switch (nv) {
#define CASE(K)                                                                              \
  case K:                                                                                    \
    cudaFuncSetAttribute(k_tile_lin<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,         \
                         200 * 1024);                                                        \
    k_tile_lin<K><<<grid, 64, smem_lin<K>(a.bs), st>>>(a, tiles, n_tiles, lo, hi, unc_lo,     \
                                                       unc_hi);                              \
    break;
    CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9)
#undef CASE
    default:
      break;
  }
}
void launch_union(const float* slo, const float* shi, float* lo, float* hi, int64_t n, bool first,
                  cudaStream_t st) {
  if (n > 0) k_union<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(slo, shi, lo, hi, n, first ? 1 : 0);
}

void launch_merge(const TileArgs& a, cudaStream_t st) {
  k_merge<<<a.ntiles, 256, 0, st>>>(a);
}

}  // namespace absplat
