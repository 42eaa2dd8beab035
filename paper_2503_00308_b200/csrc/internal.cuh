// internal.cuh -- device-side data layout and affine-form arithmetic of libabsplat.
//
// B200 (sm_100a) implementation of the AbstractSplat hot path (arXiv 2503.00308).  This
// header is private to the CUDA sources in this directory; it shares nothing with oracle/.
//
// Affine forms (D7): y(xi) in [lo(xi), hi(xi)] over xi in [-1,1]^NV, stored as
// coefficient arrays c[0..NV-1] (slopes) and c[NV] (constant).  Per-Gaussian setup runs in
// fp64 (all discontinuous decisions are taken on fp64 data, H1); the per-pixel hot
// loop runs in fp32 on tile-centred forms (H2).
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../../include/absplat.h"

namespace absplat {

constexpr int NVMAX = AS_MAX_VARS;

// Device-side invariant checks of the checked build (-DABSPLAT_CHECKS, libabsplat_checked.so):
// index bounds of every gathered / ring / list access in the tile kernels, trapping on the
// first violation.  compute-sanitizer is closed on this GPU pool; the parity suite runs
// against the checked build instead (tools/checked_build.sh).
#ifdef ABSPLAT_CHECKS
#define DCHECK(cond)                                                                     \
  do {                                                                                   \
    if (!(cond)) {                                                                       \
      printf("DCHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                         \
      __trap();                                                                          \
    }                                                                                    \
  } while (0)
#else
#define DCHECK(cond) \
  do {               \
  } while (0)
#endif
constexpr double TAU = 1e-12;   // per-pixel cull threshold on a (G12)
constexpr double DMIN = 0.01;   // near plane (G8)
constexpr int KTAYLOR = 8;      // MatrixInv order
constexpr double WCAP = 1e12;   // |W| guard -> FAIL (reading O3)

enum : int { F_DROP = 1, F_STRADDLE = 2, F_FAIL = 4, F_SKIP = 8 };  // F_SKIP: staging-only
// per list-position flags (exceptions, a9) and work-item flags
enum : int { PM_EF = 1, PM_EG = 2, PM_STORE = 4, PM_NOCUT = 8, PM_OVF = 16, PM_HSTART = 32 };
enum : int { IT_EXC = 1, IT_SINGLE = 2 };

// ------------------------------------------------------------------------- pose / box
// One sub-box: the perturbed axes in canonical order with their centre and radius.
struct SubBoxDev {
  int n;
  int axis[NVMAX];
  double c[NVMAX], r[NVMAX];
  double fixed[9];  // parameter value of every axis at xi = 0
};

struct BoxParams {  // kernel-argument copy of the box (a0)
  double lo[9], hi[9];
  int parts[9];
  int n_sub;
  const double* sub;  // explicit partition [n_sub][9][2] (device), or nullptr: uniform grid
  int t_frame;
  double euler0[3], t0[3];
  double dir[3][3];
};

// Pose forms of one sub-box (a1): R (world->camera, row-major 3x3), t, group shifts,
// all as forms over NVMAX+1 coefficients (only the first n slopes are meaningful), plus
// the common depth slope g used to bound the pair-classification window.
struct PoseDev {
  double Rl[9][NVMAX + 1], Ru[9][NVMAX + 1];
  double t[3][NVMAX + 1];  // exact affine
  double g[3][NVMAX + 1];  // exact affine
  double gslope[NVMAX];
  double Rcl[9];  // concretised lower bound of each R form (uniform over the Gaussians)
  int n;
};

// ------------------------------------------------------------------------- records
// Hot record of one Gaussian for one sub-box, read by the tile kernel's staging step.
// Layout (AoS, 16-byte aligned, NV-dependent size):
//   double d2[2][NV+1]        D2 = d^2 lower / upper coefficients
//   double du[2][2][NV+1]     DU_a = d*up_a  [a][lo/hi][coef]
//   double mu[4]              mu-rect x_lo, y_lo, x_hi, y_hi (footprint, step 11)
//   double r2                 s_cut * lambda_bar
//   double pad
//   float  w[6][2][NV+1]      W_ac = (Conic Mp)_ac  [a*3+c][lo/hi][coef]
//   float  wc[6][2]           concretised W (lo, hi)
//   float  o[2], clo[3], chi[3]
//   int    flags, pad
template <int NV>
struct alignas(16) HotRec {
  static constexpr int C = NV + 1;
  double d2[2][C];
  double du[2][2][C];
  double mu[4];
  double r2;
  double pad0;
  float w[6][2][C];
  float wc[6][2];
  float o[2];
  float clo[3], chi[3];
  int flags;
};

// Pair record (decisions): depth form and the window half-width w + S (a7).
template <int NV>
struct PairRec {
  double dl[NV + 1], du[NV + 1];
  double kappa;
  double ws;
};

// ------------------------------------------------------------------------- fp64 forms
template <int NV>
struct DF {
  double l[NV + 1], u[NV + 1];
};

template <int NV>
__device__ __forceinline__ DF<NV> df_const(double v) {
  DF<NV> f;
#pragma unroll
  for (int k = 0; k < NV; ++k) f.l[k] = f.u[k] = 0.0;
  f.l[NV] = f.u[NV] = v;
  return f;
}
template <int NV>
__device__ __forceinline__ double df_min(const DF<NV>& f) {
  double v = f.l[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) v -= fabs(f.l[k]);
  return v;
}
template <int NV>
__device__ __forceinline__ double df_max(const DF<NV>& f) {
  double v = f.u[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) v += fabs(f.u[k]);
  return v;
}
template <int NV>
__device__ __forceinline__ void df_addto(DF<NV>& a, const DF<NV>& b) {
#pragma unroll
  for (int k = 0; k <= NV; ++k) {
    a.l[k] += b.l[k];
    a.u[k] += b.u[k];
  }
}
// c * f, exact (sides swap for c < 0)
template <int NV>
__device__ __forceinline__ DF<NV> df_scale(const DF<NV>& f, double c) {
  DF<NV> r;
  if (c >= 0) {
#pragma unroll
    for (int k = 0; k <= NV; ++k) {
      r.l[k] = c * f.l[k];
      r.u[k] = c * f.u[k];
    }
  } else {
#pragma unroll
    for (int k = 0; k <= NV; ++k) {
      r.l[k] = c * f.u[k];
      r.u[k] = c * f.l[k];
    }
  }
  return r;
}
// acc += c * f
template <int NV>
__device__ __forceinline__ void df_axpy(DF<NV>& acc, const DF<NV>& f, double c) {
  if (c >= 0) {
#pragma unroll
    for (int k = 0; k <= NV; ++k) {
      acc.l[k] += c * f.l[k];
      acc.u[k] += c * f.u[k];
    }
  } else {
#pragma unroll
    for (int k = 0; k <= NV; ++k) {
      acc.l[k] += c * f.u[k];
      acc.u[k] += c * f.l[k];
    }
  }
}
// acc += x*y under fixed McCormick planes (G1):
//   lower: y_lo*x + x_lo*y - x_lo*y_lo,  upper: y_hi*x + x_lo*y - x_lo*y_hi
template <int NV>
__device__ __forceinline__ void df_mul_acc(DF<NV>& acc, const DF<NV>& x, const DF<NV>& y) {
  const double xl = df_min(x), yl = df_min(y), yh = df_max(y);
  const bool a = yl >= 0, b = xl >= 0, c = yh >= 0;
#pragma unroll
  for (int k = 0; k <= NV; ++k) {
    acc.l[k] += yl * (a ? x.l[k] : x.u[k]) + xl * (b ? y.l[k] : y.u[k]);
    acc.u[k] += yh * (c ? x.u[k] : x.l[k]) + xl * (b ? y.u[k] : y.l[k]);
  }
  acc.l[NV] -= xl * yl;
  acc.u[NV] -= xl * yh;
}
// acc += x*x: tangent at p = clamp(0, x_lo, x_hi) (lower), chord (upper) (G2)
template <int NV>
__device__ __forceinline__ void df_sq_acc(DF<NV>& acc, const DF<NV>& x) {
  const double xl = df_min(x), xh = df_max(x);
  const double p = fmin(fmax(0.0, xl), xh);
  const double tp = 2.0 * p, sh = xl + xh;
  const bool a = tp >= 0, b = sh >= 0;
#pragma unroll
  for (int k = 0; k <= NV; ++k) {
    acc.l[k] += tp * (a ? x.l[k] : x.u[k]);
    acc.u[k] += sh * (b ? x.u[k] : x.l[k]);
  }
  acc.l[NV] -= p * p;
  acc.u[NV] -= xl * xh;
}

// monotone uint64 image of a double (for radix sorting by kappa)
__device__ __forceinline__ unsigned long long key_of_double(double v) {
  unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

// ------------------------------------------------------------------------- launch plumbing
struct LaunchCounter {
  int64_t* counter;
};

// host-side launchers implemented in the .cu files (all enqueue on `st`)
struct SetupArgs {
  const float* mean;
  const float* chol;
  const float* opacity;
  const float* color;
  const int32_t* group_of;
  const float* col_lo;
  const float* col_hi;
  const float* op_lo;
  const float* op_hi;
  int64_t N;
  double fx, fy, cx, cy;
  double dir[3][3];           // group shift directions
  const PoseDev* pose;        // device pointer (one sub-box)
  void* hot;                  // HotRec<NV>[N]
  void* pair;                 // PairRec<NV>[N]
  unsigned long long* kkey;   // [N] sort keys (kappa)
  int32_t* kval;              // [N] Gaussian index
  unsigned long long* wsmax;  // max over kept Gaussians of w+S (as ordered bits)
  unsigned long long* counters;  // [4]: fails, straddles, dropped, spare
  double k_tol;               // adaptive MatrixInv order (P:470 (3)): > 0 enables
  int k_max;
  const float* priv_lo;       // [N][3] private mean offsets (NEXT-2) or nullptr
  const float* priv_hi;
  int ns;                     // shared variables (privates are ns .. ns+2)
  int inv_backward;           // NEXT-4: conic bounds by back-substitution
};

void launch_pose(const BoxParams& bp, PoseDev* out, cudaStream_t st);
void launch_setup(int nv, const SetupArgs& a, cudaStream_t st);

struct BinArgs {
  const int32_t* order;  // [N] Gaussians in (kappa, index) order
  int64_t N;
  const void* hot;
  int nv;
  int ts, ntx, nty, W, H;
  const int32_t* owner;  // [ntiles] or nullptr
  int rank;
  int64_t* counts;       // [N+1]
  const int64_t* offsets;  // [N+1]
  uint32_t* keys;        // [M] tile id
  int32_t* vals;         // [M] Gaussian index
  unsigned long long* tile_cost;  // [ntiles] or nullptr
  int64_t cap;           // room in keys / vals: pairs beyond it are not written (the caller
                         // detects the overflow from offsets[N] and renders again)
};
void launch_count(const BinArgs& a, cudaStream_t st);
void launch_emit(const BinArgs& a, cudaStream_t st);
// keys >= ntiles are padding (sorted last) and ignored
void launch_ranges(const uint32_t* keys, int64_t M, int ntiles, int64_t* begin, int64_t* end,
                   cudaStream_t st);

struct PairArgs {
  const uint32_t* keys;   // [M] sorted tile ids; ids >= ntiles are padding positions (empty)
  const int32_t* vals;    // [M] Gaussian ids
  const int64_t* tbegin;  // [ntiles]
  const int64_t* tend;
  int64_t M;              // positions, padding included (row stride of posD)
  int64_t nexc_cap;       // room in exc: lists past it are not written (caller re-renders)
  const void* pair;       // PairRec<NV>[N]
  int nv;
  // slope-aware window (a7): per tile the depth slope model m(kappa) = g0 + kappa h_T
  const PoseDev* pose;    // sub-box pose forms (R slopes, translation slope g0)
  double fx, fy, cx, cy;
  int ts, ntx, ntiles;
  double* tileh;          // [ntiles][NVMAX+1]: h_T and, at [NVMAX], 1 - |h_T|_1 (0 = no pruning)
  unsigned long long* tilemax;  // [ntiles] max over the tile's list of w + S' (ordered bits)
  double* wsP;            // [M] w + S' of the Gaussian at each position
  double* kapP;           // [M] kappa at each position
  double* posD;           // [2(NV+1)][M] depth form at each position (coefficient-major)
  int32_t* nF;            // [M] |E_F| (during k_pairs PASS 0: the count of partners > 128 back)
  int32_t* nG;            // [M]
  int64_t* ntot;          // [M+1] nF + nG of PM_OVF positions, else 0 (scanned into off)
  const int64_t* off;     // [M+1] exclusive scan of nF+nG
  int32_t* exc;           // [total] tile-local positions: E_F ascending then E_G ascending
  int32_t* hpos;          // [M] first position of E_F (tile-local) or own position (during
                          //     PASS 0: the minimum over partners > 128 back)
  int32_t* gpos;          // [M] last position of E_G (tile-local) or own position
  ulonglong2* mF;         // [M] E_F bits over [h, h+128) (0 for PM_OVF positions; during
                          //     PASS 0: bits over [p-128, p), set by the earlier partners)
  ulonglong2* mG;         // [M] E_G bits over (p, p+128] (0 for PM_OVF positions)
  unsigned long long* subunc;  // uncertain (position, partner) entries of this sub-box
  int ns;                 // shared variables; slots ns.. are per-Gaussian private (NEXT-2)
  unsigned long long* counters;  // [0] uncertain pairs, [1] order violations
};
void launch_pairs_prep(const PairArgs& a, cudaStream_t st);
void launch_pairs_count(const PairArgs& a, cudaStream_t st);
void launch_pairs_fill(const PairArgs& a, cudaStream_t st);
void launch_mark(const PairArgs& a, int32_t* dstore, int32_t* dcut, int32_t* hstart,
                 cudaStream_t st);
// finalisation record of a position q' with later uncertain partners (sorted by max E_G)
struct alignas(16) FinRec {
  int qq, nF, nG, flags;   // tile-local position, |E_F|, |E_G|, PM_* flags
  long long eoff;          // exc[] offset (E_F then E_G), for PM_OVF
  long long pad0;
  ulonglong2 mg;           // E_G(q') as bits over (q', q'+128]
  float clo[3], pad;       // lower colour of q'
};
void launch_meta(const PairArgs& a, const int32_t* cstore, const int32_t* ccut,
                 const int32_t* hstart, int4* pm, unsigned int* wmax, uint32_t* finkey,
                 int32_t* finval, cudaStream_t st);
void launch_finrec(const uint32_t* key, const int32_t* val, const PairArgs& a, const int4* pm,
                   const ulonglong2* mG, const void* hot, FinRec* out, cudaStream_t st);
// chunk length, decided on the device from the sub-box's own pair count and longest window
// (so a render sized from remembered capacities cuts exactly the chunks a probed one does):
// `over` > 0 is as_set_chunk_target's value; otherwise about six chunks per CTA of `grid`,
// six times finer (but at least two batches) when a window passes the 128-position masks
struct ChunkTarget {
  const int64_t* M;        // device: pairs of this sub-box
  const unsigned* wmax;    // device: longest exception window, or nullptr (no exceptions)
  int nsub, grid, bs, over;
};
void launch_item_caps(const int64_t* tbegin, const int64_t* tend, int ntiles, ChunkTarget tg,
                      int64_t* caps, cudaStream_t st);
// items beyond n_items (room) are not written and a ring longer than R is clamped: both set
// *ovf, and the caller renders again with larger buffers
void launch_chunks(const int64_t* tbegin, const int64_t* tend, const int4* pm,
                   const int64_t* item_off, int ntiles, int64_t n_items, ChunkTarget tg, int R,
                   const int32_t* owner, int rank, int4* stats, int4* items, int4* items2,
                   int32_t* item_cnt, uint32_t* item_key, unsigned long long* ovf,
                   cudaStream_t st);

struct TileArgs {
  const void* hot;            // HotRec<NV>[N]
  const int32_t* vals;        // [M] Gaussian ids in (tile, kappa, index) order
  const int64_t* tbegin;
  const int64_t* tend;
  // work items: {tile, begin, end (tile-local positions), flags}, processed in `order`
  const int4* items;
  const int4* items2;         // {A (scan start), L (scan end), A_next, 0}
  const int32_t* order;       // item indices, longest first
  int n_items;
  int* counter;               // dynamic work counter (zeroed before the launch)
  const int64_t* item_off;    // [ntiles+1] first item of each tile
  const int32_t* item_cnt;    // [ntiles] items per tile
  const int32_t* tile_slot;   // output slot of each tile id (tile-major) or nullptr
  int ntiles;
  int ts, ntx, W, H;
  int bs;
  int first;                  // first sub-box: store instead of union
  float ntau;                 // N * tau slack
  // exceptions (nullptr when the sub-box has no uncertain pair)
  const int4* pm;             // [M] {flags, h, g, nF} (tile-local positions)
  const int32_t* nG;          // [M]
  const int64_t* eoff;        // [M+1]
  const int32_t* exc;         // E_F ascending then E_G ascending, tile-local
  const int32_t* finstart;    // [M+1] fin_rec[finstart[p] .. finstart[p+1]) finalise at p
  const FinRec* fin_rec;
  const ulonglong2* mF;       // [M] E_F bits over [h, h+128)
  float4* ring;               // [gridDim][R][ts*ts] (T_hi before, 1-a_lo, 1-a_hi, deferred)
  int R;                      // ring length (power of two > max window)
  float* partial;             // [items][sub-blocks][64][8] chunk partials (multi-chunk tiles)
  // outputs
  float* lo;                  // row-major [H][W][3] (tile_slot == nullptr) or tile-major
  float* hi;
  unsigned long long* active; // active pair counter
  unsigned long long* dbg;    // [DBG_N] rare-path counters (as_debug_counters) or nullptr
  int kver;                   // tile kernel version (tile_kernel_version): partial layout
  int64_t M;                  // pairs (positions) of the sub-box: bound of the per-position arrays
  int64_t nexc;               // entries of exc[]
  int64_t n_partial;          // floats of partial[]
  int64_t n_out;              // floats of lo / hi (row-major image or tile-major slots)
  // NEXT-1 (reading O20): 1 = sum the interval terms of the uncertain positions only (E_F or
  // E_G non-empty) and write the raw sums (no +- N tau, no clamp) -- the linear blend adds them
  int unc_only;
  // sync-free renders: set on the device when a size outgrew its remembered capacity; the
  // tile kernels and the merge then do nothing (the render is repeated) -- nullptr: never
  const unsigned long long* ovf;
};
// rare-path counters of the tile kernel (as_debug_counters): evidence that every slow path
// of the exception machinery runs in some parity case
enum { DBG_THI_BITS = 0, DBG_THI_DIV_UNSAFE = 1, DBG_THI_OVF = 2, DBG_THI_OVF_WINDOW = 3,
       DBG_FIN_SLOW = 4, DBG_FIN_UNSTAGED = 5, DBG_FIN_OVF = 6, DBG_TMODE3 = 7, DBG_N = 8 };
void launch_tile(int nv, const TileArgs& a, int grid, cudaStream_t st);
void launch_merge(const TileArgs& a, cudaStream_t st);
// NEXT-1 linear blend (n <= 9, reading O20): intersect every tile's bounds in lo / hi
constexpr int NV_LINEAR_MAX = 9;
void launch_tile_lin(int nv, const TileArgs& a, const int32_t* tiles, int n_tiles, float* lo,
                     float* hi, const float* unc_lo, const float* unc_hi, cudaStream_t st);
void launch_union(const float* slo, const float* shi, float* lo, float* hi, int64_t n, bool first,
                  cudaStream_t st);
int tile_threads(int ts);
size_t tile_ring_slot_bytes(int ts);
int tile_kernel_version(int ts);
int tile_batch(int nv, int ts, int bs);
int tile_subblocks(int ts);
int tile_grid(int nv, int ts, int bs);
size_t tile_smem_bytes(int nv, int ts, int bs);

// concrete renderer (tests)
struct ConcreteArgs {
  const float* mean;
  const float* chol;
  const float* opacity;
  const float* color;
  const int32_t* group_of;
  int64_t N;
  double R[9], t[3], shift[3][3];  // world->camera R, camera centre, shift vector per group
  double fx, fy, cx, cy;
  int W, H;
  double* gdata;                   // [N][8] scratch: mu, conic-like, depth, opacity
  unsigned long long* key;         // [N]
  int32_t* val;                    // [N]
  const int32_t* order;            // [N] after sort
  float* img;
};
void launch_concrete_setup(const ConcreteArgs& a, cudaStream_t st);
void launch_concrete_render(const ConcreteArgs& a, cudaStream_t st);

void launch_untile(const float* lo_tm, const float* hi_tm, const int32_t* slot_of_tile,
                   int ts, int ntx, int nty, int W, int H, float* lo, float* hi,
                   cudaStream_t st);

}  // namespace absplat
