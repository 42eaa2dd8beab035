// k_bin.cu -- rows a6-a7: tile culling + binning of (tile, Gaussian) pairs in depth order,
// per-tile ranges, and the depth-order abstraction (three-valued Ind with index tie-break,
// Alg. 3 line 1 P:382 with Table 2's Ind relaxation P:222-229, reading G6) restricted to a
// provably sufficient window of the (kappa, index)-sorted list.
#include "internal.cuh"

namespace absplat {

// exact fp64 cull test of a rectangle of pixel centres (no FMA contraction: the decision
// must be reproducible bit for bit, H1 / reading O1)
__device__ __forceinline__ bool rect_culled(const double mu[4], double r2, double x0, double x1,
                                            double y0, double y1) {
  const double dx = fmax(0.0, fmax(__dsub_rn(mu[0], x1), __dsub_rn(x0, mu[2])));
  const double dy = fmax(0.0, fmax(__dsub_rn(mu[1], y1), __dsub_rn(y0, mu[3])));
  return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)) > r2;
}

template <int NV>
__device__ __forceinline__ void footprint(const HotRec<NV>* H, double mu[4], double& r2,
                                          int& flags) {
  flags = H->flags;
#pragma unroll
  for (int k = 0; k < 4; ++k) mu[k] = H->mu[k];
  r2 = H->r2;
}

// candidate tile range (superset) of a footprint
__device__ __forceinline__ void tile_range(const double mu[4], double r2, int ts, int W, int H,
                                           int& tx0, int& tx1, int& ty0, int& ty1) {
  const double R = sqrt(r2) * (1.0 + 1e-9) + 1e-6;
  const double xl = mu[0] - R, xh = mu[2] + R, yl = mu[1] - R, yh = mu[3] + R;
  // pixel centres px + 0.5 in [xl, xh]
  double pxl = floor(xl - 0.5) - 1.0, pxh = ceil(xh - 0.5) + 1.0;
  double pyl = floor(yl - 0.5) - 1.0, pyh = ceil(yh - 0.5) + 1.0;
  pxl = fmax(pxl, 0.0);
  pyl = fmax(pyl, 0.0);
  pxh = fmin(pxh, (double)(W - 1));
  pyh = fmin(pyh, (double)(H - 1));
  if (!(pxl <= pxh) || !(pyl <= pyh)) {
    tx0 = 1;
    tx1 = 0;
    ty0 = 1;
    ty1 = 0;
    return;
  }
  tx0 = (int)pxl / ts;
  tx1 = (int)pxh / ts;
  ty0 = (int)pyl / ts;
  ty1 = (int)pyh / ts;
}

template <int NV, bool EMIT>
__global__ void k_bin(BinArgs A) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= A.N) return;
  const int32_t g = A.order[r];
  const HotRec<NV>* H = reinterpret_cast<const HotRec<NV>*>(A.hot) + g;
  double mu[4], r2;
  int flags;
  footprint<NV>(H, mu, r2, flags);
  int cnt = 0;
  int64_t out = EMIT ? A.offsets[r] : 0;
  if (!(flags & F_DROP)) {
    int tx0, tx1, ty0, ty1;
    tile_range(mu, r2, A.ts, A.W, A.H, tx0, tx1, ty0, ty1);
    for (int ty = ty0; ty <= ty1; ++ty) {
      const double y0 = ty * A.ts + 0.5, y1 = fmin((double)((ty + 1) * A.ts), (double)A.H) - 0.5;
      for (int tx = tx0; tx <= tx1; ++tx) {
        const double x0 = tx * A.ts + 0.5, x1 = fmin((double)((tx + 1) * A.ts), (double)A.W) - 0.5;
        if (rect_culled(mu, r2, x0, x1, y0, y1)) continue;
        const int tile = ty * A.ntx + tx;
        if (A.owner && A.owner[tile] != A.rank) {
          if (!EMIT && A.tile_cost) atomicAdd(&A.tile_cost[tile], 1ull);
          continue;
        }
        if (EMIT) {
          if (out < A.cap) {
            A.keys[out] = (uint32_t)tile;
            A.vals[out] = g;
          }
          ++out;
        } else if (A.tile_cost) {
          atomicAdd(&A.tile_cost[tile], 1ull);
        }
        ++cnt;
      }
    }
  }
  if (!EMIT) A.counts[r] = cnt;
}

#define NV_SWITCH(nv, ...)                                   \
  switch (nv) {                                              \
    case 0: { constexpr int NVc = 0; __VA_ARGS__; } break;   \
    case 1: { constexpr int NVc = 1; __VA_ARGS__; } break;   \
    case 2: { constexpr int NVc = 2; __VA_ARGS__; } break;   \
    case 3: { constexpr int NVc = 3; __VA_ARGS__; } break;   \
    case 4: { constexpr int NVc = 4; __VA_ARGS__; } break;   \
    case 5: { constexpr int NVc = 5; __VA_ARGS__; } break;   \
    case 6: { constexpr int NVc = 6; __VA_ARGS__; } break;   \
    case 7: { constexpr int NVc = 7; __VA_ARGS__; } break;   \
    case 8: { constexpr int NVc = 8; __VA_ARGS__; } break;   \
    case 9: { constexpr int NVc = 9; __VA_ARGS__; } break;   \
    default: break;                                          \
  }

void launch_count(const BinArgs& a, cudaStream_t st) {
  if (a.N <= 0) return;
  const unsigned blocks = (unsigned)((a.N + 127) / 128);
  NV_SWITCH(a.nv, (k_bin<NVc, false><<<blocks, 128, 0, st>>>(a)));
}
void launch_emit(const BinArgs& a, cudaStream_t st) {
  if (a.N <= 0) return;
  const unsigned blocks = (unsigned)((a.N + 127) / 128);
  NV_SWITCH(a.nv, (k_bin<NVc, true><<<blocks, 128, 0, st>>>(a)));
}

__global__ void k_ranges(const uint32_t* keys, int64_t M, int ntiles, int64_t* begin,
                         int64_t* end) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= M) return;
  const uint32_t t = keys[p];
  if (t >= (uint32_t)ntiles) return;  // padding
  if (p == 0 || keys[p - 1] != t) begin[t] = p;
  if (p == M - 1 || keys[p + 1] != t) end[t] = p + 1;
}
void launch_ranges(const uint32_t* keys, int64_t M, int ntiles, int64_t* begin, int64_t* end,
                   cudaStream_t st) {
  cudaMemsetAsync(begin, 0, sizeof(int64_t) * ntiles, st);
  cudaMemsetAsync(end, 0, sizeof(int64_t) * ntiles, st);
  if (M <= 0) return;
  k_ranges<<<(unsigned)((M + 255) / 256), 256, 0, st>>>(keys, M, ntiles, begin, end);
}

// ------------------------------------------------------------------------- pairs (a7)
template <int NV>
__device__ __forceinline__ PairRec<NV> load_pair(const void* base, int32_t g) {
  return reinterpret_cast<const PairRec<NV>*>(base)[g];
}

// depth form of position q from the position-ordered copy (d lower then upper coefficients)
template <int NV>
struct DForm {
  double l[NV + 1], u[NV + 1];
};
// posD is coefficient-major ([2(NV+1)][M]): the window scans of neighbouring positions read
// neighbouring entries, so a warp's load of one coefficient is contiguous
template <int NV>
__device__ __forceinline__ DForm<NV> load_posd(const double* posD, int64_t M, int64_t q) {
  DForm<NV> f;
#pragma unroll
  for (int k = 0; k <= NV; ++k) {
    f.l[k] = posD[(size_t)k * M + q];
    f.u[k] = posD[(size_t)(NV + 1 + k) * M + q];
  }
  return f;
}
// Ind(d_i - d_j) over the box with the index tie-break (G6): 1 = j certainly in front of i,
// 0 = certainly not, -1 = '?'.  Same expression order as the definition (no FMA).  Slots
// k >= ns are private to each Gaussian (NEXT-2): independent, so their slopes add.
template <int NV>
__device__ __forceinline__ int ind_class_d(const DForm<NV>& Pi, int32_t i, const DForm<NV>& Pj,
                                           int32_t j, int ns) {
  double dl = __dsub_rn(Pi.l[NV], Pj.u[NV]);
  double du = __dsub_rn(Pi.u[NV], Pj.l[NV]);
  double s1 = 0.0, s2 = 0.0;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    if (k < ns) {
      s1 = __dadd_rn(s1, fabs(__dsub_rn(Pi.l[k], Pj.u[k])));
      s2 = __dadd_rn(s2, fabs(__dsub_rn(Pi.u[k], Pj.l[k])));
    } else {
      s1 = __dadd_rn(s1, __dadd_rn(fabs(Pi.l[k]), fabs(Pj.u[k])));
      s2 = __dadd_rn(s2, __dadd_rn(fabs(Pi.u[k]), fabs(Pj.l[k])));
    }
  }
  dl = __dsub_rn(dl, s1);
  du = __dadd_rn(du, s2);
  if (i > j) {
    if (dl >= 0.0) return 1;
    if (du < 0.0) return 0;
  } else {
    if (dl > 0.0) return 1;
    if (du <= 0.0) return 0;
  }
  return -1;
}

// Window bound (SURVEY §8(c) step 13 pruning, slope-aware).  For any vector h and
// m_i = g0 + kappa_i h:  |lA_i - uA_j|_1 <= S'_i + |kappa_i - kappa_j| |h|_1 + S'_j with
// S'_i = max(|lA_i - m_i|_1, |uA_i - m_i|_1).  A '?' pair (j before i) needs
// kappa_i - kappa_j <= w_i + w_j + |lA_i - uA_j|_1, hence
// (kappa_i - kappa_j)(1 - |h|_1) <= ws'_i + ws'_j <= ws'_i + M_T (and symmetrically forward).
// h_T = depth slope per unit depth of the rotation variables along the tile's centre ray
// (d = R_2 (P - t) and P - t = d R^T ray), so Gaussians of similar depth in the tile have
// slopes close to m(kappa) and the window shrinks to about the form widths.
__global__ void k_tile_h(PairArgs A) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= A.ntiles) return;
  const PoseDev& P = *A.pose;
  const int tx = t % A.ntx, ty = t / A.ntx;
  const double ray[3] = {((tx + 0.5) * A.ts - A.cx) / A.fx, ((ty + 0.5) * A.ts - A.cy) / A.fy, 1.0};
  // world direction R^T ray with R the centre rotation (mid of the constant terms)
  double wd[3];
  for (int b = 0; b < 3; ++b) {
    double v = 0.0;
    for (int a = 0; a < 3; ++a) v += 0.5 * (P.Rl[3 * a + b][NVMAX] + P.Ru[3 * a + b][NVMAX]) * ray[a];
    wd[b] = v;
  }
  double* h = A.tileh + (size_t)t * (NVMAX + 1);
  double norm = 0.0;
  for (int k = 0; k < NVMAX; ++k) {
    double v = 0.0;
    if (k < P.n)
      for (int b = 0; b < 3; ++b) v += P.Rl[6 + b][k] * wd[b];  // row 2 of R, slope k
    h[k] = v;
    norm += fabs(v);
  }
  h[NVMAX] = (norm < 0.5) ? (1.0 - norm) : 0.0;
  A.tilemax[t] = 0ull;
}

// warp-aggregated atomics over the lanes currently converged (each converged group elects
// its lowest lane): one atomic per warp instead of one per thread
__device__ __forceinline__ void warp_add(unsigned long long* dst, unsigned v) {
  const unsigned mask = __activemask();
  v = __reduce_add_sync(mask, v);
  if ((int)(threadIdx.x & 31) == __ffs(mask) - 1 && v) atomicAdd(dst, (unsigned long long)v);
}
__device__ __forceinline__ void warp_max_u32(unsigned* dst, unsigned v) {
  const unsigned mask = __activemask();
  v = __reduce_max_sync(mask, v);
  if ((int)(threadIdx.x & 31) == __ffs(mask) - 1 && v) atomicMax(dst, v);
}

template <int NV>
__global__ void k_pairs_prep(PairArgs A) {
  const int64_t p0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t p = p0 < A.M ? p0 : A.M - 1;  // dead lanes mirror the last position (no writes)
  const uint32_t t = A.keys[p];
  const bool pad = t >= (uint32_t)A.ntiles;  // padding position: arithmetic on tile 0, no writes
  const bool live = p0 < A.M && !pad;
  const PairRec<NV> Pi = load_pair<NV>(A.pair, A.vals[p]);
  const double* h = A.tileh + (size_t)(pad ? 0u : t) * (NVMAX + 1);
  double s1 = 0.0, s2 = 0.0;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const double m = A.pose->gslope[k] + Pi.kappa * h[k];
    s1 += fabs(Pi.dl[k] - m);
    s2 += fabs(Pi.du[k] - m);
  }
  // >= 0 by construction, clamped: rounding can leave the half-width of a zero-width constant
  // a few ulp negative, and the tile maximum below compares bit patterns (a negative double's
  // pattern orders above every positive one, which made M tiny and the window unsound)
  const double ws = fmax(0.5 * (Pi.du[NV] - Pi.dl[NV]) + fmax(s1, s2), 0.0);
  if (p0 < A.M) {  // E_F accumulators of the forward-only classification (k_pairs PASS 0)
    A.mF[p] = make_ulonglong2(0ull, 0ull);
    A.nF[p] = 0;
    A.hpos[p] = 0x7fffffff;
  }
  if (live) {
    A.wsP[p] = ws;
    A.kapP[p] = Pi.kappa;
    // position-ordered copy of the depth form: the window scans then read neighbours
    // contiguously instead of gathering PairRec by Gaussian id
#pragma unroll
    for (int k = 0; k <= NV; ++k) {
      A.posD[(size_t)k * A.M + p] = Pi.dl[k];
      A.posD[(size_t)(NV + 1 + k) * A.M + p] = Pi.du[k];
    }
  }
  // tile max of ws (ws >= 0, so its bit pattern orders like the value): positions are
  // sorted by tile, so equal keys form runs; reduce each run inside the warp first
  unsigned long long v = (unsigned long long)__double_as_longlong(ws);
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long vo = __shfl_down_sync(0xffffffffu, v, o);
    const uint32_t to = __shfl_down_sync(0xffffffffu, t, o);
    if (lane + o < 32 && to == t) v = max(v, vo);
  }
  const uint32_t tp = __shfl_up_sync(0xffffffffu, t, 1);
  if (live && (lane == 0 || tp != t)) atomicMax(&A.tilemax[t], v);
}

// true when every later/earlier candidate is certainly ordered (the scan can stop)
__device__ __forceinline__ bool beyond(double dk, double factor, double wsi, double M, double ki,
                                       double kj) {
  const double bound = (wsi + M) * (1.0 + 1e-9) + 1e-12 * (fabs(ki) + fabs(kj)) + 1e-300;
  return dk * factor * (1.0 - 1e-9) > bound;
}

// 128-bit helpers (lo, hi halves)
__device__ __forceinline__ void set_bit128(unsigned long long& m0, unsigned long long& m1, int i) {
  if (i < 64)
    m0 |= 1ull << i;
  else
    m1 |= 1ull << (i - 64);
}
__device__ __forceinline__ void shr128(unsigned long long& m0, unsigned long long& m1, int s) {
  if (s >= 128) {
    m0 = m1 = 0;
  } else if (s >= 64) {
    m0 = m1 >> (s - 64);
    m1 = 0;
  } else if (s > 0) {
    m0 = (m0 >> s) | (m1 << (64 - s));
    m1 >>= s;
  }
}

// PASS 0 (every position p): classify the forward window once.  Ind is antisymmetric
// (ind_class_d(q, p) = 1 - ind_class_d(p, q) on certain pairs, '?' on both sides together:
// dl and du swap and negate exactly), so each unordered pair is classified by its earlier
// position only: E_G(p) is kept in registers (bits over (p, p + 128], its count and last
// partner), and p enters E_F(q) of the later partner through one atomic per uncertain pair
// (a bit of q's mask over [q - 128, q), or, further than 128 positions, a far count and the
// far minimum).  k_pairs_post then derives |E_F|, h = min E_F, the masks relative to h and the
// overflow flags.  PASS 1 (PM_OVF positions only: a partner more than 128 positions away)
// fills their explicit E_F / E_G lists by scanning both directions.
template <int NV, int PASS>
__global__ void k_pairs(PairArgs A) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= A.M) return;
  int64_t off = 0, ntp = 0;
  int nFt = 0;
  if (PASS == 1) {
    ntp = A.ntot[p];
    if (ntp == 0) return;  // not an overflow position
    off = A.off[p];
    nFt = A.nF[p];
    if (off + ntp > A.nexc_cap) return;  // no room: the caller renders again
  }
  const uint32_t t = A.keys[p];
  if (t >= (uint32_t)A.ntiles) {  // padding position: no partners
    if (PASS == 0) {
      A.nG[p] = 0;
      A.gpos[p] = 0;
      A.ntot[p] = 0;
      A.mG[p] = make_ulonglong2(0ull, 0ull);
    }
    return;
  }
  const int64_t b = A.tbegin[t], e = A.tend[t];
  const int32_t gi = A.vals[p];
  const DForm<NV> Pi = load_posd<NV>(A.posD, A.M, p);
  const double ki = A.kapP[p];
  const double M = __longlong_as_double((long long)A.tilemax[t]);
  const double factor = A.tileh[(size_t)t * (NVMAX + 1) + NVMAX];
  const double wsi = A.wsP[p];
  if (PASS == 1) {
    // backward: earlier positions (expected Ind in {1, ?}), E_F in ascending order
    int nF = 0;
    for (int64_t q = p - 1; q >= b; --q) {
      const double kj = A.kapP[q];
      if (beyond(ki - kj, factor, wsi, M, ki, kj)) break;
      const int c = ind_class_d<NV>(Pi, gi, load_posd<NV>(A.posD, A.M, q), A.vals[q], A.ns);
      if ((c == -1 || c == 0) && nF < nFt) A.exc[off + nFt - 1 - nF++] = (int32_t)(q - b);
    }
  }
  // forward: later positions (expected Ind in {0, ?})
  int nG = 0, viol = 0;
  int gmax = (int)(p - b);
  unsigned long long g0 = 0, g1 = 0;  // E_G rel. p + 1
  bool far = false;
  for (int64_t q = p + 1; q < e; ++q) {
    const double kj = A.kapP[q];
    if (beyond(kj - ki, factor, wsi, M, ki, kj)) break;
    const int32_t gj = A.vals[q];
    const int c = ind_class_d<NV>(Pi, gi, load_posd<NV>(A.posD, A.M, q), gj, A.ns);
    if (c == -1 || c == 1) {  // c == 1 contradicts the order: counted, treated as '?'
      if (PASS == 1 && nFt + nG < ntp) A.exc[off + nFt + nG] = (int32_t)(q - b);
      if (PASS == 0) {
        if (c == 1) ++viol;
        const int d = (int)(q - p);
        if (d <= 128) {
          set_bit128(g0, g1, d - 1);
          const int k = 128 - d;  // p as a bit of q's E_F mask over [q - 128, q)
          if (k < 64)
            atomicOr(&A.mF[q].x, 1ull << k);
          else
            atomicOr(&A.mF[q].y, 1ull << (k - 64));
        } else {
          far = true;
          atomicAdd(&A.nF[q], 1);
          atomicMin(&A.hpos[q], (int)(p - b));
        }
      }
      gmax = (int)(q - b);
      ++nG;
    }
  }
  if (PASS == 0) {
    A.nG[p] = nG;
    A.gpos[p] = gmax;
    A.ntot[p] = far ? 1 : 0;  // provisional: E_G past 128 (k_pairs_post completes it)
    A.mG[p] = make_ulonglong2(g0, g1);
    warp_add(&A.counters[0], (unsigned)nG);
    warp_add(&A.counters[1], (unsigned)viol);
    warp_add(A.subunc, (unsigned)nG);
  }
}

// Completes PASS 0 per position: |E_F| = mask bits + far count, h = min E_F (the far minimum
// when there is one, else the lowest mask bit, else p itself), PM_OVF positions (a partner
// more than 128 positions away on either side) get ntot = |E_F| + |E_G| and no masks, the
// others their E_F mask shifted to start at h.
__global__ void k_pairs_post(PairArgs A) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= A.M) return;
  const uint32_t t = A.keys[p];
  if (t >= (uint32_t)A.ntiles) {  // padding: prep zeroed nF / mF; h is unused
    A.hpos[p] = 0;
    return;
  }
  const int loc = (int)(p - A.tbegin[t]);
  unsigned long long f0 = A.mF[p].x, f1 = A.mF[p].y;
  const int nfar = A.nF[p];
  const int nF = __popcll(f0) + __popcll(f1) + nfar;
  int h = loc;
  if (nfar > 0) {
    h = A.hpos[p];
  } else if (f0 | f1) {
    const int kmin = f0 ? __ffsll((long long)f0) - 1 : 64 + __ffsll((long long)f1) - 1;
    h = loc - 128 + kmin;
    shr128(f0, f1, kmin);
  }
  const bool ovf = nfar > 0 || A.ntot[p] != 0;
  A.nF[p] = nF;
  A.hpos[p] = h;
  A.ntot[p] = ovf ? nF + A.nG[p] : 0;
  A.mF[p] = ovf ? make_ulonglong2(0ull, 0ull) : make_ulonglong2(f0, f1);
  if (ovf) A.mG[p] = make_ulonglong2(0ull, 0ull);
}

void launch_pairs_prep(const PairArgs& a, cudaStream_t st) {
  if (a.M <= 0) return;
  k_tile_h<<<(a.ntiles + 127) / 128, 128, 0, st>>>(a);
  const unsigned blocks = (unsigned)((a.M + 255) / 256);
  NV_SWITCH(a.nv, (k_pairs_prep<NVc><<<blocks, 256, 0, st>>>(a)));
}

void launch_pairs_count(const PairArgs& a, cudaStream_t st) {
  if (a.M <= 0) return;
  const unsigned blocks = (unsigned)((a.M + 127) / 128);
  NV_SWITCH(a.nv, (k_pairs<NVc, 0><<<blocks, 128, 0, st>>>(a)));
  k_pairs_post<<<(unsigned)((a.M + 255) / 256), 256, 0, st>>>(a);
}
void launch_pairs_fill(const PairArgs& a, cudaStream_t st) {
  if (a.M <= 0) return;
  const unsigned blocks = (unsigned)((a.M + 127) / 128);
  NV_SWITCH(a.nv, (k_pairs<NVc, 1><<<blocks, 128, 0, st>>>(a)));
}

// Exception metadata (a7 -> a9).  For a position p with uncertain partners:
//   * its T_hi window [h_p, p] (h_p = min E_F(p), or p) must be kept in the ring: every
//     position inside some window is flagged PM_STORE (difference array `dstore`);
//   * a chunk boundary between b-1 and b must not separate an uncertain pair (q < b <= p):
//     positions b in (h_p, p] are flagged PM_NOCUT (difference array `dcut`);
//   * the window start h_p itself is flagged PM_HSTART (the only positions whose running
//     T_hi the ring must keep).
__global__ void k_mark(PairArgs A, int32_t* dstore, int32_t* dcut, int32_t* hstart) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= A.M) return;
  const int nF = A.nF[p], nG = A.nG[p];
  if (nF + nG == 0) return;
  const int64_t b = A.tbegin[A.keys[p]];
  const int h = A.hpos[p];
  atomicAdd(&dstore[b + h], 1);
  atomicAdd(&dstore[p + 1], -1);
  if (nF > 0) {
    hstart[b + h] = 1;
    atomicAdd(&dcut[b + h + 1], 1);
    atomicAdd(&dcut[p + 1], -1);
  }
}
void launch_mark(const PairArgs& a, int32_t* dstore, int32_t* dcut, int32_t* hstart,
                 cudaStream_t st) {
  if (a.M <= 0) return;
  k_mark<<<(unsigned)((a.M + 255) / 256), 256, 0, st>>>(a, dstore, dcut, hstart);
}

// per-position metadata for the tile kernel: {flags, h, g, nF}; max window -> wmax;
// E_F(p) as a 128-bit mask over [h, h+128) and E_G(p) over (p, p+128] (PM_OVF if longer)
__global__ void k_meta(PairArgs A, const int32_t* cstore, const int32_t* ccut,
                       const int32_t* hstart, int4* pm, unsigned int* wmax, uint32_t* finkey,
                       int32_t* finval) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= A.M) return;
  if (A.keys[p] >= (uint32_t)A.ntiles) {  // padding position
    pm[p] = make_int4(0, 0, 0, 0);
    finkey[p] = (uint32_t)A.M;
    finval[p] = (int32_t)p;
    return;
  }
  const int nF = A.nF[p], nG = A.nG[p];
  const int64_t b = A.tbegin[A.keys[p]];
  const int loc = (int)(p - b);
  const int h = A.hpos[p], g = A.gpos[p];
  const bool ovf = (loc - h) > 128 || (g - loc) > 128;
  int fl = (nF ? PM_EF : 0) | (nG ? PM_EG : 0) | (cstore[p] > 0 ? PM_STORE : 0) |
           (ccut[p] > 0 ? PM_NOCUT : 0) | (ovf ? PM_OVF : 0) | (hstart[p] ? PM_HSTART : 0);
  pm[p] = make_int4(fl, h, g, nF);
  warp_max_u32(wmax, (unsigned)max(loc - h, g - loc));
  // deferred lower contribution of p is finalised at its last later partner b + g
  finkey[p] = nG ? (uint32_t)(b + g) : (uint32_t)A.M;  // no finalisation: sorts last
  finval[p] = (int32_t)p;
}
void launch_meta(const PairArgs& a, const int32_t* cstore, const int32_t* ccut,
                 const int32_t* hstart, int4* pm, unsigned int* wmax, uint32_t* finkey,
                 int32_t* finval, cudaStream_t st) {
  if (a.M <= 0) return;
  k_meta<<<(unsigned)((a.M + 255) / 256), 256, 0, st>>>(a, cstore, ccut, hstart, pm, wmax, finkey,
                                                          finval);
}

// finalisation records in sorted order: everything the tile kernel needs about q'
template <int NV>
__global__ void k_finrec(const uint32_t* key, const int32_t* val, PairArgs A, const int4* pm,
                         const ulonglong2* mG, const void* hot, FinRec* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.M) return;
  if (key[i] >= (uint32_t)A.M) return;
  const int32_t gq = val[i];
  const int64_t b = A.tbegin[A.keys[gq]];
  const int4 m = pm[gq];
  const HotRec<NV>* H = reinterpret_cast<const HotRec<NV>*>(hot) + A.vals[gq];
  FinRec r;
  r.qq = (int)(gq - b);
  r.nF = m.w;
  r.nG = A.nG[gq];
  r.flags = m.x;
  r.eoff = A.off[gq];
  r.mg = mG[gq];
  r.clo[0] = H->clo[0];
  r.clo[1] = H->clo[1];
  r.clo[2] = H->clo[2];
  r.pad = 0.f;
  out[i] = r;
}
void launch_finrec(const uint32_t* key, const int32_t* val, const PairArgs& a, const int4* pm,
                   const ulonglong2* mG, const void* hot, FinRec* out, cudaStream_t st) {
  if (a.M <= 0) return;
  const unsigned blocks = (unsigned)((a.M + 255) / 256);
  NV_SWITCH(a.nv, (k_finrec<NVc><<<blocks, 256, 0, st>>>(key, val, a, pm, mG, hot, out)));
}

// ------------------------------------------------------------------------- work items
// Split every tile's list into chunks of `target` positions.  A chunk [s, e) is scanned
// over [A, L): the lookback [A, s) covers the E_F windows of its positions (A = min h_p)
// and the lookahead [e, L) their E_G partners (L = max g_p + 1); those margin positions
// only feed the chunk's transmittance and exception factors.  Chunks then compose front
// to back with multiplications only:  pc = sum_k P(<A_k) S_k,  P(<A_{k+1}) = P(<A_k) Rk,
// where S_k is the chunk's sum relative to A_k and Rk its running product at A_{k+1}
// (A is made non-decreasing, A_k <= A_{k+1}, so A_{k+1} lies inside chunk k's scan
// [A_k, L_k) for any chunk length).  One warp per tile.
//   items[i]  = {tile, s, e, flags | log2(ring length) << 8}
//   items2[i] = {A, L, A_next, 0}
__device__ __forceinline__ int chunk_target(const ChunkTarget& g) {
  if (g.over > 0) return max(g.over, g.bs);
  const int64_t t = *g.M * g.nsub / ((int64_t)g.grid * 6) + 1;
  // long windows: finer chunks balance the few expensive tiles, but every chunk rescans its
  // lookback window; two batches is the measured optimum on C5 (1.82 ms vs 2.17 at one batch,
  // 2.61 at four)
  if (g.wmax && *g.wmax > 128u) return (int)(t / 6 > 2 * g.bs ? t / 6 : 2 * (int64_t)g.bs);
  const int64_t u = t > 2 * (int64_t)g.bs ? t : 2 * (int64_t)g.bs;
  return (int)(u < (1 << 30) ? u : (1 << 30));
}
__global__ void k_item_caps(const int64_t* tbegin, const int64_t* tend, int ntiles,
                            ChunkTarget tg, int64_t* caps) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntiles) return;
  const int target = chunk_target(tg);
  const int64_t K = tend[t] - tbegin[t];
  caps[t] = K > 0 ? (K + target - 1) / target : 1;
}
void launch_item_caps(const int64_t* tbegin, const int64_t* tend, int ntiles, ChunkTarget tg,
                      int64_t* caps, cudaStream_t st) {
  k_item_caps<<<(ntiles + 255) / 256, 256, 0, st>>>(tbegin, tend, ntiles, tg, caps);
}
// Chunk statistics in parallel (warp per work item): the lookback / lookahead margins a, l
// of the chunk's exception windows, its longest window and whether it has any exception.
__global__ void k_chunk_stats(const int64_t* tbegin, const int64_t* tend, const int4* pm,
                              const int64_t* item_off, int ntiles, int64_t n_items,
                              ChunkTarget tg, const int32_t* owner, int rank, int4* stats) {
  const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= n_items) return;
  const int target = chunk_target(tg);
  int lo = 0, hi = ntiles - 1;  // tile t with item_off[t] <= j < item_off[t + 1]
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (item_off[mid] <= j) lo = mid; else hi = mid - 1;
  }
  const int t = lo;
  const int64_t b = tbegin[t];
  const int K = (int)(tend[t] - b);
  const bool mine = owner == nullptr || owner[t] == rank;
  const int k = (int)(j - item_off[t]);
  const int s = k * target, e = min(K, s + target);
  int a = s, l = e, wl = 0;
  bool ex = false;
  if (mine && pm) {
#pragma unroll 4
    for (int i = s + lane; i < e; i += 32) {
      const int4 m = pm[b + i];
      if (m.x != 0) {
        ex = true;
        if (m.x & PM_EF) a = min(a, m.y);
        if (m.x & PM_EG) l = max(l, m.z + 1);
        wl = max(wl, max(i - m.y, m.z - i));
      }
    }
    for (int sh = 16; sh > 0; sh >>= 1) {
      a = min(a, __shfl_xor_sync(0xffffffffu, a, sh));
      l = max(l, __shfl_xor_sync(0xffffffffu, l, sh));
      wl = max(wl, __shfl_xor_sync(0xffffffffu, wl, sh));
    }
    ex = __any_sync(0xffffffffu, ex);
  }
  if (lane == 0) stats[j] = make_int4(a, l, wl, ex ? 1 : 0);
}
// per tile, back to front (A_next known, scan starts non-decreasing): the work items
__global__ void k_chunk_items(const int64_t* tbegin, const int64_t* tend, const int4* pm,
                              const int64_t* item_off, int ntiles, int64_t n_items,
                              ChunkTarget tg, int R, const int32_t* owner, int rank,
                              const int4* stats, int4* items, int4* items2, int32_t* item_cnt,
                              uint32_t* item_key, unsigned long long* ovf) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntiles) return;
  const int target = chunk_target(tg);
  const int K = (int)(tend[t] - tbegin[t]);
  const int64_t o = item_off[t];
  const int64_t cap = item_off[t + 1] - o;
  const bool mine = owner == nullptr || owner[t] == rank;
  const int n = mine ? (K > 0 ? (K + target - 1) / target : 1) : 0;
  if (o + (cap > n ? cap : (int64_t)n) > n_items) {  // no room for this tile's items
    atomicOr(ovf, 1ull);
    for (int64_t j = o; j < n_items; ++j) {  // its slots inside the buffer: empty
      items[j] = make_int4(-1, 0, 0, 0);
      items2[j] = make_int4(0, 0, 0, 0);
      item_key[j] = 0;
    }
    item_cnt[t] = 0;
    return;
  }
  int prevA = 0;
  for (int k = n - 1; k >= 0; --k) {
    const int s = k * target, e = min(K, s + target);
    const int4 st = stats[o + k];
    int A = min(s, st.x);
    const int L = max(e, st.y);
    int lr = 0;
    while ((1 << lr) <= st.z) ++lr;
    if ((1 << lr) > R) {  // window longer than the ring: clamped, the caller renders again
      atomicOr(ovf, 2ull);
      lr = 0;
      while ((2 << lr) <= R) ++lr;
    }
    const int Anext = (k == n - 1) ? e : prevA;
    if (k < n - 1) A = min(A, prevA);
    const int fl = ((pm && st.w) ? IT_EXC : 0) | (n == 1 ? IT_SINGLE : 0) | (lr << 8);
    items[o + k] = make_int4(t, s, e, fl);
    items2[o + k] = make_int4(A, L, Anext, 0);
    item_key[o + k] = (uint32_t)(L - A);
    prevA = A;
  }
  for (int64_t jj = n; jj < cap; ++jj) {  // unused slots: empty items, sorted last
    items[o + jj] = make_int4(-1, 0, 0, 0);
    items2[o + jj] = make_int4(0, 0, 0, 0);
    item_key[o + jj] = 0;
  }
  item_cnt[t] = n;
}
void launch_chunks(const int64_t* tbegin, const int64_t* tend, const int4* pm,
                   const int64_t* item_off, int ntiles, int64_t n_items, ChunkTarget tg, int R,
                   const int32_t* owner, int rank, int4* stats, int4* items, int4* items2,
                   int32_t* item_cnt, uint32_t* item_key, unsigned long long* ovf,
                   cudaStream_t st) {
  if (n_items > 0)
    k_chunk_stats<<<(unsigned)((n_items + 3) / 4), 128, 0, st>>>(
        tbegin, tend, pm, item_off, ntiles, n_items, tg, owner, rank, stats);
  k_chunk_items<<<(ntiles + 127) / 128, 128, 0, st>>>(tbegin, tend, pm, item_off, ntiles, n_items,
                                                      tg, R, owner, rank, stats, items, items2,
                                                      item_cnt, item_key, ovf);
}

// ------------------------------------------------------------------------- untile (a11)
__global__ void k_untile(const float* lo_tm, const float* hi_tm, const int32_t* slot_of_tile,
                         int ts, int ntx, int W, int H, float* lo, float* hi) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)W * H) return;
  const int px = (int)(idx % W), py = (int)(idx / W);
  const int tile = (py / ts) * ntx + px / ts;
  const int64_t s = slot_of_tile[tile];
  const int64_t src = (s * ts * ts + (int64_t)(py % ts) * ts + (px % ts)) * 3;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    lo[3 * idx + c] = lo_tm[src + c];
    hi[3 * idx + c] = hi_tm[src + c];
  }
}
void launch_untile(const float* lo_tm, const float* hi_tm, const int32_t* slot_of_tile, int ts,
                   int ntx, int nty, int W, int H, float* lo, float* hi, cudaStream_t st) {
  (void)nty;
  const int64_t n = (int64_t)W * H;
  if (n <= 0) return;
  k_untile<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(lo_tm, hi_tm, slot_of_tile, ts, ntx, W, H,
                                                        lo, hi);
}

}  // namespace absplat
