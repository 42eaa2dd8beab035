// k_tile.cu -- rows a8-a10, the hot loop: per (pixel, Gaussian) opacity bounds (Alg. 1 lines
// 9-10 lifted: x = d^2 u - d up, q = x W, s = q q^T, a = o exp(-s/2)) and the
// transmittance scan + bounded blend (Alg. 3, interval reading O7), with the
// finalise/union epilogue.
//
// One CTA per image tile (TS x TS pixels, 1 or 4 pixels per thread), tiles launched in
// descending Gaussian-count order.  The tile's Gaussian list (sorted by (kappa, index)) is
// streamed through shared memory in batches of BS: the staging step turns each Gaussian's
// fp64 record into tile-centred fp32 forms (B = u_c D2 - DU at the tile centre u_c, so the
// per-pixel x = B + (u - u_c) D2 avoids the d^2 u - d up cancellation; H2) and
// fp64 per-row / per-column squared distances for the exact per-pixel cull (reading O1).
// Every thread then walks the batch for its pixel(s) in order: FP32 on CUDA cores.
//
// Work is a list of (tile, chunk) items, longest first, pulled by persistent CTAs from an
// atomic counter (load balance).  A chunk ends only where no uncertain depth
// pair is split, so chunks of one tile compose front to back in k_merge.
//
// Uncertain depth pairs (rotation / scene boxes; step 13) are handled in the walk itself
// with a per-CTA ring in global memory (L2-resident): position q writes (T_hi before q,
// 1 - a_lo, 1 - a_hi, deferred T_lo a_lo) for its pixel; T_hi of a position with earlier
// uncertain partners is re-multiplied over its window [h, q) skipping E_F (no division,
// H3); the lower contribution of a position with later uncertain partners is deferred and
// finalised at g = max E_G, when all of E_G's (1 - a_hi) are known.
#include <algorithm>
#include <cstdio>

#include "internal.cuh"

namespace absplat {

namespace {
constexpr unsigned FULLM = 0xffffffffu;
constexpr float LOG2E_HALF = 0.72134752044448170368f;  // log2(e) / 2

template <int NV>
struct alignas(16) SRec {
  static constexpr int C = NV + 1;
  float xb[2][2][C];  // [a][lo/hi][k]: tile-centred constant part of x_a's forms
  float d2[2][C];     // [lo/hi][k]
  float w[6][2][C];   // [a*3+c][lo/hi][k]
  float wc[6][2];
  float o[2];
  float clo[3], chi[3];
  int flags;                // F_* of the Gaussian
  int pmf, ph, pg, pnF, pnG;  // position metadata (PM_*, h, g, |E_F|, |E_G|)
  int pfb, pfe;             // finalisation list range
  long long peoff;          // offset of E_F(p) then E_G(p) in exc[]
  double r2;
};

__device__ __forceinline__ float sel(bool c, float a, float b) { return c ? a : b; }

// steps 14-17 for one pixel: returns (a_lo, a_hi)
template <int NV>
__device__ __forceinline__ void opacity(const SRec<NV>& R, float du0, float du1, float& alo,
                                        float& ahi) {
  constexpr int C = NV + 1;
  // 14: x_a = Add(Mul(d,d,u_a), -Mul(d, up_a)) in tile-centred form
  float xl0[C], xh0[C], xl1[C], xh1[C];
#pragma unroll
  for (int k = 0; k < C; ++k) {
    xl0[k] = fmaf(du0, R.d2[0][k], R.xb[0][0][k]);
    xh0[k] = fmaf(du0, R.d2[1][k], R.xb[0][1][k]);
    xl1[k] = fmaf(du1, R.d2[0][k], R.xb[1][0][k]);
    xh1[k] = fmaf(du1, R.d2[1][k], R.xb[1][1][k]);
  }
  float x0l = xl0[NV], x0h = xh0[NV], x1l = xl1[NV], x1h = xh1[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    x0l -= fabsf(xl0[k]);
    x0h += fabsf(xh0[k]);
    x1l -= fabsf(xl1[k]);
    x1h += fabsf(xh1[k]);
  }
  (void)x0h;
  (void)x1h;
  // 15-16: q_c = mul(x0, W_0c) + mul(x1, W_1c); s = sum_c sq(q_c)
  float sl[C], sh[C];
#pragma unroll
  for (int k = 0; k < C; ++k) sl[k] = sh[k] = 0.f;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    float ql[C], qh[C];
    const float w0l = R.wc[c][0], w0h = R.wc[c][1];
    const float w1l = R.wc[3 + c][0], w1h = R.wc[3 + c][1];
    const bool a0 = w0l >= 0.f, b0 = x0l >= 0.f, c0 = w0h >= 0.f;
    const bool a1 = w1l >= 0.f, b1 = x1l >= 0.f, c1 = w1h >= 0.f;
#pragma unroll
    for (int k = 0; k < C; ++k) {
      float lo = w0l * sel(a0, xl0[k], xh0[k]);
      lo = fmaf(x0l, sel(b0, R.w[c][0][k], R.w[c][1][k]), lo);
      lo = fmaf(w1l, sel(a1, xl1[k], xh1[k]), lo);
      lo = fmaf(x1l, sel(b1, R.w[3 + c][0][k], R.w[3 + c][1][k]), lo);
      float hi = w0h * sel(c0, xh0[k], xl0[k]);
      hi = fmaf(x0l, sel(b0, R.w[c][1][k], R.w[c][0][k]), hi);
      hi = fmaf(w1h, sel(c1, xh1[k], xl1[k]), hi);
      hi = fmaf(x1l, sel(b1, R.w[3 + c][1][k], R.w[3 + c][0][k]), hi);
      ql[k] = lo;
      qh[k] = hi;
    }
    ql[NV] -= fmaf(x0l, w0l, x1l * w1l);
    qh[NV] -= fmaf(x0l, w0h, x1l * w1h);
    float qmin = ql[NV], qmax = qh[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      qmin -= fabsf(ql[k]);
      qmax += fabsf(qh[k]);
    }
    const float p = fminf(fmaxf(0.f, qmin), qmax);
    const float tp = 2.f * p, sm = qmin + qmax;
    const bool pa = tp >= 0.f, pb = sm >= 0.f;
#pragma unroll
    for (int k = 0; k < C; ++k) {
      sl[k] = fmaf(tp, sel(pa, ql[k], qh[k]), sl[k]);
      sh[k] = fmaf(sm, sel(pb, qh[k], ql[k]), sh[k]);
    }
    sl[NV] -= p * p;
    sh[NV] -= qmin * qmax;
  }
  float smin = sl[NV], smax = sh[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    smin -= fabsf(sl[k]);
    smax += fabsf(sh[k]);
  }
  smin = fmaxf(smin, 0.f);
  // 17: a = o * Exp(-s/2) concretised (O11)
  alo = R.o[0] * exp2f(-LOG2E_HALF * smax);
  ahi = R.o[1] * exp2f(-LOG2E_HALF * smin);
}
}  // namespace

template <int NV, int PPT>
__global__ void __launch_bounds__(256) k_tile(TileArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_item;
  const int ts = A.ts;
  const int npix = ts * ts;
  const int nthr = blockDim.x;
  const int BS = A.bs;
  SRec<NV>* srec = reinterpret_cast<SRec<NV>*>(smem_raw);
  double* cx2 = reinterpret_cast<double*>(srec + BS);  // [BS][ts]
  double* cy2 = cx2 + (size_t)BS * ts;                 // [BS][ts]
  const bool has_exc = A.pm != nullptr;
  float4* ring = has_exc ? A.ring + (size_t)blockIdx.x * A.R * npix : nullptr;
  const int rmask = A.R - 1;
  unsigned active = 0;

  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(A.counter, 1);
    __syncthreads();
    const int iidx = s_item;
    __syncthreads();
    if (iidx >= A.n_items) break;
    const int islot = A.order[iidx];
    const int4 it = A.items[islot];
    if (it.x < 0) continue;  // padding
    const int tile = it.x, pbeg = it.y, pend = it.z, iflags = it.w;
    const int tx = tile % A.ntx, ty = tile / A.ntx;
    const int64_t tb = A.tbegin[tile];
    const double ucx = tx * ts + 0.5 * ts, ucy = ty * ts + 0.5 * ts;  // tile centre
    const bool iexc = has_exc && (iflags & IT_EXC);

    int lx[PPT], ly[PPT];
    bool in_img[PPT];
    float du0[PPT], du1[PPT];
    float Tb[PPT], Tl[PPT], ahc[PPT][3], alc[PPT][3];
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const int l = threadIdx.x + q * nthr;
      lx[q] = l % ts;
      ly[q] = l / ts;
      in_img[q] = (tx * ts + lx[q] < A.W) && (ty * ts + ly[q] < A.H);
      du0[q] = (float)lx[q] + 0.5f - 0.5f * ts;
      du1[q] = (float)ly[q] + 0.5f - 0.5f * ts;
      Tb[q] = Tl[q] = 1.f;
      ahc[q][0] = ahc[q][1] = ahc[q][2] = 0.f;
      alc[q][0] = alc[q][1] = alc[q][2] = 0.f;
    }

    for (int b0 = pbeg; b0 < pend; b0 += BS) {
      const int nb = min(BS, pend - b0);
      __syncthreads();
      // ---- staging: fp64 record -> tile-centred fp32 forms + cull tables + metadata
      for (int j = threadIdx.x; j < nb; j += nthr) {
        const int64_t gp = tb + b0 + j;
        const int32_t g = A.vals[gp];
        const HotRec<NV>* H = reinterpret_cast<const HotRec<NV>*>(A.hot) + g;
        SRec<NV>& S = srec[j];
#pragma unroll
        for (int k = 0; k <= NV; ++k) {
          const double d2l = H->d2[0][k], d2h = H->d2[1][k];
          // x_a lower = u_a D2_lo - DU_a,hi ; upper = u_a D2_hi - DU_a,lo  (u_a > 0)
          S.xb[0][0][k] = (float)(ucx * d2l - H->du[0][1][k]);
          S.xb[0][1][k] = (float)(ucx * d2h - H->du[0][0][k]);
          S.xb[1][0][k] = (float)(ucy * d2l - H->du[1][1][k]);
          S.xb[1][1][k] = (float)(ucy * d2h - H->du[1][0][k]);
          S.d2[0][k] = (float)d2l;
          S.d2[1][k] = (float)d2h;
        }
#pragma unroll
        for (int e = 0; e < 6; ++e) {
#pragma unroll
          for (int k = 0; k <= NV; ++k) {
            S.w[e][0][k] = H->w[e][0][k];
            S.w[e][1][k] = H->w[e][1][k];
          }
          S.wc[e][0] = H->wc[e][0];
          S.wc[e][1] = H->wc[e][1];
        }
        S.o[0] = H->o[0];
        S.o[1] = H->o[1];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          S.clo[c] = H->clo[c];
          S.chi[c] = H->chi[c];
        }
        S.flags = H->flags;
        if (iexc) {
          const int4 m = A.pm[gp];
          S.pmf = m.x;
          S.ph = m.y;
          S.pg = m.z;
          S.pnF = m.w;
          S.pnG = A.nG[gp];
          S.peoff = A.eoff[gp];
          S.pfb = A.fin_b[gp];
          S.pfe = A.fin_e[gp];
        } else {
          S.pmf = 0;
          S.pfb = S.pfe = 0;
        }
        S.r2 = H->r2;
        const double mxl = H->mu[0], myl = H->mu[1], mxh = H->mu[2], myh = H->mu[3];
        for (int l = 0; l < ts; ++l) {
          const double x = tx * ts + l + 0.5, y = ty * ts + l + 0.5;
          const double dx = fmax(0.0, fmax(__dsub_rn(mxl, x), __dsub_rn(x, mxh)));
          const double dy = fmax(0.0, fmax(__dsub_rn(myl, y), __dsub_rn(y, myh)));
          cx2[j * ts + l] = __dmul_rn(dx, dx);
          cy2[j * ts + l] = __dmul_rn(dy, dy);
        }
      }
      __syncthreads();
      // ---- walk the batch in (kappa, index) order
      for (int j = 0; j < nb; ++j) {
        const SRec<NV>& R = srec[j];
        const int flags = R.flags, pmf = R.pmf;
        const int qpos = b0 + j;  // tile-local position
        float alo[PPT], ahi[PPT];
        bool keep[PPT];
        bool any = false;
#pragma unroll
        for (int q = 0; q < PPT; ++q) {
          keep[q] = in_img[q] && !(__dadd_rn(cx2[j * ts + lx[q]], cy2[j * ts + ly[q]]) > R.r2);
          any |= keep[q];
          alo[q] = ahi[q] = 0.f;
        }
        if (__any_sync(FULLM, any)) {
          if (flags & F_FAIL) {
#pragma unroll
            for (int q = 0; q < PPT; ++q) {
              alo[q] = 0.f;
              ahi[q] = keep[q] ? R.o[1] : 0.f;
            }
          } else {
#pragma unroll
            for (int q = 0; q < PPT; ++q) {
              float l, h;
              opacity<NV>(R, du0[q], du1[q], l, h);
              alo[q] = keep[q] ? ((flags & F_STRADDLE) ? 0.f : l) : 0.f;
              ahi[q] = keep[q] ? h : 0.f;
            }
          }
        }
#pragma unroll
        for (int q = 0; q < PPT; ++q) {
          active += keep[q] ? 1u : 0u;
          const int pix = threadIdx.x + q * nthr;
          if (pmf & PM_STORE)
            ring[(size_t)(qpos & rmask) * npix + pix] =
                make_float4(Tb[q], 1.f - alo[q], 1.f - ahi[q], (pmf & PM_EG) ? Tl[q] * alo[q] : 0.f);
          // upper: T_hi over before(q) \ E_F(q).  Dense windows (mostly E_F): multiply the
          // window [h, q) skipping E_F.  Sparse windows: divide the running product by the
          // E_F factors when that is numerically safe (both products far from underflow),
          // else fall back to the window product (H3).
          float tbv = Tb[q];
          if (pmf & PM_EF) {
            bool done = false;
            const int wlen = qpos - R.ph;
            if (wlen > 2 * R.pnF + 8) {
              float dfac = 1.f;
              for (int e = 0; e < R.pnF; ++e)
                dfac *= ring[(size_t)(A.exc[R.peoff + e] & rmask) * npix + pix].y;
              if (dfac >= 1e-20f && Tb[q] >= 1e-25f) {
                tbv = Tb[q] / dfac;
                done = true;
              }
            }
            if (!done) {
              tbv = ring[(size_t)(R.ph & rmask) * npix + pix].x;
              int e = 0;
              for (int r = R.ph; r < qpos; ++r) {
                if (e < R.pnF && A.exc[R.peoff + e] == r) {
                  ++e;
                  continue;
                }
                tbv *= ring[(size_t)(r & rmask) * npix + pix].y;
              }
            }
          }
          const float wb = tbv * ahi[q];
#pragma unroll
          for (int c = 0; c < 3; ++c) ahc[q][c] = fmaf(wb, R.chi[c], ahc[q][c]);
          // lower: T_lo over before(q) (E_G(q) empty) or deferred to max E_G(q)
          if (!(pmf & PM_EG)) {
            const float wl = Tl[q] * alo[q];
#pragma unroll
            for (int c = 0; c < 3; ++c) alc[q][c] = fmaf(wl, R.clo[c], alc[q][c]);
          }
          Tb[q] = fmaf(-Tb[q], alo[q], Tb[q]);
          Tl[q] = fmaf(-Tl[q], ahi[q], Tl[q]);
          // finalise deferred lower contributions of earlier partners whose last later
          // partner is q:  T_lo(q') = T_lo,before(q') prod_{r in E_G(q')} (1 - a_hi,r)
          for (int f = R.pfb; f < R.pfe; ++f) {
            const int gq = A.fin_val[f];
            const int qq = (int)(gq - tb);
            const int4 m = A.pm[gq];
            float tl = ring[(size_t)(qq & rmask) * npix + pix].w;
            const int64_t o2 = A.eoff[gq] + m.w;
            const int ng2 = A.nG[gq];
            for (int e = 0; e < ng2; ++e) {
              const int r = A.exc[o2 + e];
              tl *= ring[(size_t)(r & rmask) * npix + pix].z;
            }
            const HotRec<NV>* H2 = reinterpret_cast<const HotRec<NV>*>(A.hot) + A.vals[gq];
#pragma unroll
            for (int c = 0; c < 3; ++c) alc[q][c] = fmaf(tl, H2->clo[c], alc[q][c]);
          }
        }
      }
    }
    // ---- epilogue
    if (iflags & IT_SINGLE) {
      // +- N tau, clamp to [0,1], union over sub-boxes (steps 20-22)
#pragma unroll
      for (int q = 0; q < PPT; ++q) {
        const int px = tx * ts + lx[q], py = ty * ts + ly[q];
        int64_t o;
        if (A.tile_slot) {
          o = ((int64_t)A.tile_slot[tile] * npix + (int64_t)ly[q] * ts + lx[q]) * 3;
        } else {
          if (!in_img[q]) continue;
          o = ((int64_t)py * A.W + px) * 3;
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          float l = fminf(fmaxf(alc[q][c] - A.ntau, 0.f), 1.f);
          float h = fminf(fmaxf(ahc[q][c] + A.ntau, 0.f), 1.f);
          if (!in_img[q]) l = h = 0.f;
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
#pragma unroll
      for (int q = 0; q < PPT; ++q) {
        const int pix = threadIdx.x + q * nthr;
        float4* dst = reinterpret_cast<float4*>(A.partial + ((size_t)islot * npix + pix) * 8);
        dst[0] = make_float4(ahc[q][0], ahc[q][1], ahc[q][2], Tb[q]);
        dst[1] = make_float4(alc[q][0], alc[q][1], alc[q][2], Tl[q]);
      }
    }
  }
  // active (pixel, Gaussian) pairs
  unsigned v = active;
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(FULLM, v, s);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(A.active, (unsigned long long)v);
}

// front-to-back composition of a tile's chunks: pc = sum_k (prod_{m<k} P_m) S_k
__global__ void k_merge(TileArgs A) {
  const int tile = blockIdx.x;
  const int n = A.item_cnt[tile];
  if (n <= 1) return;
  const int ts = A.ts, npix = ts * ts;
  const int tx = tile % A.ntx, ty = tile / A.ntx;
  for (int pix = threadIdx.x; pix < npix; pix += blockDim.x) {
    float Pb = 1.f, Pl = 1.f, h[3] = {0.f, 0.f, 0.f}, l[3] = {0.f, 0.f, 0.f};
    for (int k = 0; k < n; ++k) {
      const int64_t it = A.item_off[tile] + k;
      const float4* src = reinterpret_cast<const float4*>(A.partial + ((size_t)it * npix + pix) * 8);
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
    const int lx = pix % ts, ly = pix / ts;
    const int px = tx * ts + lx, py = ty * ts + ly;
    const bool inside = px < A.W && py < A.H;
    int64_t o;
    if (A.tile_slot) {
      o = ((int64_t)A.tile_slot[tile] * npix + pix) * 3;
    } else {
      if (!inside) continue;
      o = ((int64_t)py * A.W + px) * 3;
    }
    for (int c = 0; c < 3; ++c) {
      float lv = fminf(fmaxf(l[c] - A.ntau, 0.f), 1.f);
      float hv = fminf(fmaxf(h[c] + A.ntau, 0.f), 1.f);
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

int tile_threads(int ts) { return ts <= 16 ? ts * ts : 256; }

template <int NV>
static size_t smem_for(int ts, int bs) {
  return (size_t)bs * (sizeof(SRec<NV>) + 2 * ts * sizeof(double));
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

template <int NV, int PPT>
static int grid_one(int ts, int bs) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_tile<NV, PPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured = true;
  }
  int per_sm = 0, dev = 0, nsm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tile<NV, PPT>, tile_threads(ts),
                                                smem_for<NV>(ts, bs));
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  return std::max(1, per_sm) * nsm;
}

int tile_grid(int nv, int ts, int bs) {
  const bool four = ts == 32;
  switch (nv) {
#define CASE(K) \
  case K:       \
    return four ? grid_one<K, 4>(ts, bs) : grid_one<K, 1>(ts, bs);
    CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9)
#undef CASE
    default:
      return 0;
  }
}

void launch_tile(int nv, const TileArgs& a, int grid, cudaStream_t st) {
  if (a.n_items <= 0 || grid <= 0) return;
  const bool four = a.ts == 32;
  switch (nv) {
#define CASE(K)                                                                          \
  case K:                                                                                \
    if (four)                                                                            \
      k_tile<K, 4><<<grid, tile_threads(a.ts), smem_for<K>(a.ts, a.bs), st>>>(a);        \
    else                                                                                 \
      k_tile<K, 1><<<grid, tile_threads(a.ts), smem_for<K>(a.ts, a.bs), st>>>(a);        \
    break;
    CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9)
#undef CASE
    default:
      break;
  }
}

void launch_merge(const TileArgs& a, cudaStream_t st) {
  k_merge<<<a.ntiles, 256, 0, st>>>(a);
}

}  // namespace absplat
