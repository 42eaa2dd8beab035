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
// Uncertain depth pairs (rotation / scene boxes): positions flagged P_STORE write
// (a_lo, a_hi, T_hi-before, T_lo-before) per pixel to a scratch slot; positions flagged
// P_EXC are left out of the running sums and added after the walk from their exception
// windows (T_hi over before(i) minus E_F(i), T_lo over before(i) plus E_G(i)) without any
// division (H3).
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
  int flags, pflag, slot, pad;
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
  const int ts = A.ts;
  const int nthr = blockDim.x;
  const int BS = A.bs;
  SRec<NV>* srec = reinterpret_cast<SRec<NV>*>(smem_raw);
  double* cx2 = reinterpret_cast<double*>(srec + BS);  // [BS][ts]
  double* cy2 = cx2 + (size_t)BS * ts;                 // [BS][ts]

  const int tile = A.tile_list[blockIdx.x];
  const int tx = tile % A.ntx, ty = tile / A.ntx;
  const int64_t tb = A.tbegin[tile], te = A.tend[tile];
  const int K = (int)(te - tb);
  const double ucx = tx * ts + 0.5 * ts, ucy = ty * ts + 0.5 * ts;  // tile centre

  // my pixels
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
  unsigned active = 0;
  const bool has_exc = A.pflag != nullptr;

  for (int b0 = 0; b0 < K; b0 += BS) {
    const int nb = min(BS, K - b0);
    __syncthreads();
    // ---- staging: fp64 record -> tile-centred fp32 forms + cull tables
    for (int j = threadIdx.x; j < nb; j += nthr) {
      const int32_t g = A.vals[tb + b0 + j];
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
      S.pflag = has_exc ? A.pflag[tb + b0 + j] : 0;
      S.slot = has_exc ? A.slot[tb + b0 + j] : 0;
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
      const int flags = R.flags, pflag = R.pflag;
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
        if (pflag & P_STORE) {
          const int64_t si = (int64_t)R.slot * ts * ts + threadIdx.x + q * nthr;
          A.scratch[si] = make_float4(alo[q], ahi[q], Tb[q], Tl[q]);
        }
        if (!(pflag & P_EXC)) {
          const float wb = Tb[q] * ahi[q], wl = Tl[q] * alo[q];
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            ahc[q][c] = fmaf(wb, R.chi[c], ahc[q][c]);
            alc[q][c] = fmaf(wl, R.clo[c], alc[q][c]);
          }
        }
        Tb[q] = fmaf(-Tb[q], alo[q], Tb[q]);
        Tl[q] = fmaf(-Tl[q], ahi[q], Tl[q]);
      }
    }
  }
  // ---- exception post-pass (positions with uncertain depth partners)
  if (has_exc) {
    for (int p = 0; p < K; ++p) {
      const int64_t gp = tb + p;
      if (!(A.pflag[gp] & P_EXC)) continue;
      const int nF = A.nF[gp], nG = A.nG[gp];
      const int64_t off = A.eoff[gp];
      const int h = A.hpos[gp];
      const HotRec<NV>* H = reinterpret_cast<const HotRec<NV>*>(A.hot) + A.vals[gp];
      float clo[3], chi[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        clo[c] = H->clo[c];
        chi[c] = H->chi[c];
      }
      const int64_t sp = (int64_t)A.slot[gp] * ts * ts;
      const int64_t sh = (int64_t)A.slot[tb + h] * ts * ts;
#pragma unroll
      for (int q = 0; q < PPT; ++q) {
        const int pix = threadIdx.x + q * nthr;
        const float4 me = A.scratch[sp + pix];
        float tbv, tlv = me.w;
        if (nF == 0) {
          tbv = me.z;
        } else {
          tbv = A.scratch[sh + pix].z;
          int e = 0;
          for (int r = h; r < p; ++r) {
            if (e < nF && A.exc[off + e] == r) {
              ++e;
              continue;
            }
            tbv = fmaf(-tbv, A.scratch[(int64_t)A.slot[tb + r] * ts * ts + pix].x, tbv);
          }
        }
        for (int e = 0; e < nG; ++e) {
          const int r = A.exc[off + nF + e];
          tlv = fmaf(-tlv, A.scratch[(int64_t)A.slot[tb + r] * ts * ts + pix].y, tlv);
        }
        const float wb = tbv * me.y, wl = tlv * me.x;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          ahc[q][c] = fmaf(wb, chi[c], ahc[q][c]);
          alc[q][c] = fmaf(wl, clo[c], alc[q][c]);
        }
      }
    }
  }
  // ---- epilogue: +- N tau, clamp to [0,1], union over sub-boxes (steps 20-22)
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    const int px = tx * ts + lx[q], py = ty * ts + ly[q];
    const bool inside = px < A.W && py < A.H;
    int64_t o;
    if (A.tile_slot) {
      o = ((int64_t)A.tile_slot[tile] * ts * ts + (int64_t)ly[q] * ts + lx[q]) * 3;
    } else {
      if (!inside) continue;
      o = ((int64_t)py * A.W + px) * 3;
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      float l = fminf(fmaxf(alc[q][c] - A.ntau, 0.f), 1.f);
      float h = fminf(fmaxf(ahc[q][c] + A.ntau, 0.f), 1.f);
      if (!inside) {
        l = 0.f;
        h = 0.f;
      }
      if (A.first) {
        A.lo[o + c] = l;
        A.hi[o + c] = h;
      } else {
        A.lo[o + c] = fminf(A.lo[o + c], l);
        A.hi[o + c] = fmaxf(A.hi[o + c], h);
      }
    }
  }
  // active (pixel, Gaussian) pairs
  unsigned v = active;
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(FULLM, v, s);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(A.active, (unsigned long long)v);
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
static void launch_one(const TileArgs& a, cudaStream_t st) {
  const size_t smem = smem_for<NV>(a.ts, a.bs);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_tile<NV, PPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured = true;
  }
  k_tile<NV, PPT><<<a.n_list, tile_threads(a.ts), smem, st>>>(a);
}

void launch_tile(int nv, const TileArgs& a, cudaStream_t st) {
  if (a.n_list <= 0) return;
  const bool four = a.ts == 32;
  switch (nv) {
#define CASE(K)                     \
  case K:                           \
    if (four)                       \
      launch_one<K, 4>(a, st);      \
    else                            \
      launch_one<K, 1>(a, st);      \
    break;
    CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9)
#undef CASE
    default:
      break;
  }
}

}  // namespace absplat
