// absplat.cu -- C ABI (include/absplat.h) and host orchestration of the B200 abstract-
// rendering path: context, device buffers, per-sub-box pipeline (pose -> setup -> depth
// sort -> bin -> tile sort -> pair classification -> tile kernel), tile sharding (LPT owner
// map, compact tile-major outputs, untile), and the concrete renderer used by tests.
#include <cub/cub.cuh>
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "internal.cuh"

using namespace absplat;

namespace {

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  as_free_fn free_fn = nullptr;  // allocator that produced p (nullptr = cudaMalloc)
  void* user = nullptr;
};

struct Err {
  as_status st;
};

}  // namespace

struct as_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  // scene
  int64_t N = -1;
  DevBuf mean, chol, opacity, color;
  DevBuf st_mean, st_chol, st_opacity, st_color;  // as_load_scene staging (validated, swapped)
  // scene box
  int n_groups = 0;
  double dir[3][3] = {};
  double shift_lo[3] = {}, shift_hi[3] = {};
  int gparts[3] = {1, 1, 1};
  DevBuf group_of, col_lo, col_hi, op_lo, op_hi, priv_lo, priv_hi;
  bool has_group = false, has_col = false, has_op = false, has_priv = false;
  // camera / box
  as_camera cam{};
  as_pose_box box{};
  bool have_cam = false, have_box = false;
  // work buffers
  DevBuf pose, hot, pair, kkey, kkey2, kval, order, counts, offsets, cub_tmp;
  DevBuf keys, keys2, vals, vals2, tbegin, tend, tcost, tkey, tkey2, tids, tlist, tslot, owner;
  DevBuf nF, nG, ntot, eoff, exc, hpos, gpos, diff, cover, pflag, is_store, slot, scratch;
  DevBuf tileh, tilemax, wsP, kapP, posD;
  DevBuf item_off, items, items2, item_key, item_key2, item_idx, item_order, item_cnt, partial, work_counter;
  DevBuf finkey, finkey2, finval, finval2, finstart, finrec, maskF, maskG;
  DevBuf img_lo, img_hi, counters, conc_g, untile_map;
  size_t bytes = 0, peak_bytes = 0;
  int64_t launches = 0;
  int last_items = 0, last_grid = 0, last_R = 1, last_wmax = 0;
  int host_syncs = 0;  // blocking device -> host reads inside the current render
  cudaEvent_t ev[8] = {};
  bool events = false;
  // explicit partition (as_set_subboxes): host copy [n][9][2] and its device mirror
  std::vector<double> sub_host;
  DevBuf subs;
  int chunk_target = 0;  // as_set_chunk_target (0 = automatic)
  double k_tol = 0.0;  // as_set_matrixinv (adaptive Taylor order)
  int k_max = 8;
  int inv_backward = 0;  // as_set_inverse_mode (NEXT-4 back-substitution)
  int blend_mode = 0;  // as_set_blend: 0 interval, 1 + linear on exception-free tiles
  bool debug = false;  // as_debug_counters: rare-path counters of the tile kernel
  DevBuf dbg;
  // multi-GPU (as_comm_init): NCCL communicator of this rank, shard axis, gather buffers,
  // the device owner map / slots of the LPT assignment
  void* comm = nullptr;  // ncclComm_t
  int rank = 0, world = 1;
  int shard_axis = 0;    // as_set_shard_axis: 0 auto, 1 tiles, 2 sub-boxes
  DevBuf gsend, grecv, lptkey, lptkey2, lptid, lptid2, tslot_all, nown, chunk_stats;
  double last_gather_ms = 0.0;
  int64_t last_nexc = 0;
  int last_out_tiles = 0;  // tile-major output capacity (checked build bounds)
  int last_n_owned = 0;
  bool last_has_exc = false;
  DevBuf tmp_lo, tmp_hi, lin_tiles, unc_lo, unc_hi;
  bool last_unc = false;  // unc_lo / unc_hi hold the last sub-box's uncertain terms
  // Sync-free renders: the sizes a render would otherwise read back mid-pipeline (pairs,
  // exception-list length, ring length, work items), remembered from the last probed render
  // with the same tile / batch / box dimension.  spec_on: this render sizes from `spec`
  // (buffers padded, kernels skip padding) and is verified once at its end; `probe`
  // collects the maxima while a probing render reads them.
  struct Sizes {
    bool valid = false, exc = false;
    int ts = 0, bs = 0, nv = -1, R = 1;
    int64_t M = 0, nexc = 0, items = 0;
  } spec, probe;
  bool spec_on = false;
  int64_t spec_redo = 0;  // renders repeated after a failed verification (stats)
  // as_render_shard's remembered sizes, per (tile, batch, box dimension, world, rank): emulated
  // ranks run in turn on one context, each with its own pair and item counts
  std::map<uint64_t, Sizes> shard_spec;
  Sizes* cur_spec = &spec;  // the sizes a sync-free render_subbox takes (render or shard cache)
  // as_render_shard's owner map (LPT over the cost pass's per-tile pair counts) is a function of
  // the state: kept while gen, tile, world and the per-rank capacity are unchanged
  bool lpt_valid = false;
  uint64_t lpt_gen = 0;
  int lpt_tile = 0, lpt_world = 0, lpt_cap = 0, lpt_s0 = 0, lpt_s1 = 0;
  // CUDA graph of the sync-free pipeline: captured on the render after a sync-free one that
  // allocated nothing, replayed while the key holds.  gen counts every state-changing API
  // call, alloc_gen every (re)allocation; both are part of the key.
  struct GraphKey {
    int tile = 0, batch = 0, s0 = 0, s1 = 0;
    const float* lo = nullptr;
    const float* hi = nullptr;
    bool timed = false, exc = false;
    uint64_t gen = 0, alloc_gen = 0;
    int64_t M = 0, nexc = 0, items = 0;
    int R = 0;
    bool operator==(const GraphKey& o) const {
      return tile == o.tile && batch == o.batch && s0 == o.s0 && s1 == o.s1 && lo == o.lo &&
             hi == o.hi && timed == o.timed && exc == o.exc && gen == o.gen &&
             alloc_gen == o.alloc_gen && M == o.M && nexc == o.nexc && items == o.items &&
             R == o.R;
    }
  } gkey, gready;
  bool gready_ok = false;
  cudaGraphExec_t gexec = nullptr;
  // graphs are captured on / launched into a private non-blocking stream (the caller's may be
  // the legacy default stream, which cannot be captured), ordered after and before the
  // caller's stream by two events
  cudaStream_t gstream = nullptr;
  cudaEvent_t gev_in = nullptr, gev_out = nullptr;
  int64_t glaunches = 0;
  uint64_t gen = 0, alloc_gen = 0;
  bool use_graphs = true;
  // per sub-box phase events (collected after the render's single synchronisation)
  std::vector<cudaEvent_t> sbev;
  as_alloc_fn alloc_fn = nullptr;  // as_set_allocator hook (nullptr = cudaMalloc)
  as_free_fn free_fn = nullptr;
  void* alloc_user = nullptr;
};

namespace {

void set_err(as_ctx* c, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  c->err = buf;
}

#define CK(call)                                                                     \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess) {                                                         \
      set_err(ctx, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
              __LINE__);                                                             \
      throw Err{e_ == cudaErrorMemoryAllocation ? AS_E_OOM : AS_E_CUDA};             \
    }                                                                                \
  } while (0)

#define LAUNCHED(ctx, n)                                                                    \
  do {                                                                                      \
    (ctx)->launches += (n);                                                                 \
    cudaError_t e_ = cudaGetLastError();                                                    \
    if (e_ != cudaSuccess) {                                                                \
      set_err(ctx, "kernel launch failed: %s (%s:%d)", cudaGetErrorString(e_), __FILE__, \
              __LINE__);                                                                    \
      throw Err{AS_E_CUDA};                                                                 \
    }                                                                                       \
  } while (0)

void free_buf(as_ctx* ctx, DevBuf& b) {
  if (!b.p) return;
  ++ctx->alloc_gen;
  if (b.free_fn)
    b.free_fn(b.user, b.p, b.cap, ctx->stream);
  else
    cudaFree(b.p);
  ctx->bytes -= b.cap;
  b.p = nullptr;
  b.cap = 0;
  b.free_fn = nullptr;
  b.user = nullptr;
}
void ensure(as_ctx* ctx, DevBuf& b, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (b.cap >= bytes) return;
  free_buf(ctx, b);
  size_t want = bytes + bytes / 4;
  if (ctx->alloc_fn) {
    b.p = ctx->alloc_fn(ctx->alloc_user, want, ctx->stream);
    if (!b.p) {
      set_err(ctx, "allocator hook returned NULL for %zu bytes", want);
      throw Err{AS_E_OOM};
    }
    b.free_fn = ctx->free_fn;
    b.user = ctx->alloc_user;
  } else {
    CK(cudaMalloc(&b.p, want));
  }
  b.cap = want;
  ++ctx->alloc_gen;
  ctx->bytes += want;
  ctx->peak_bytes = std::max(ctx->peak_bytes, ctx->bytes);
}
void release(as_ctx* ctx, DevBuf& b) { free_buf(ctx, b); }

template <typename T>
T* P(DevBuf& b) {
  return reinterpret_cast<T*>(b.p);
}

size_t hot_size(int nv) {
  switch (nv) {
#define CASE(K) \
  case K:       \
    return sizeof(HotRec<K>);
    CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9)
#undef CASE
  }
  return 0;
}
size_t pair_size(int nv) { return sizeof(double) * (2 * (nv + 1) + 2); }


// ---------------------------------------------------------------- box (a0)
struct BoxInfo {
  BoxParams bp;
  int n_sub;
  int n_vars;    // form variables: shared + private (3 with per-Gaussian mean offsets)
  int n_shared;  // pose axes and group shifts
  // full-box variables (for as_render_concrete)
  int axis[NVMAX];
  double c[NVMAX], r[NVMAX];
};

as_status make_box(as_ctx* ctx, BoxInfo& bi) {
  BoxParams& bp = bi.bp;
  std::memset(&bp, 0, sizeof bp);
  const as_pose_box& b = ctx->box;
  for (int a = 0; a < 3; ++a) {
    if (!(b.eps_t[a] >= 0) || !(b.eps_R[a] >= 0) || !std::isfinite(b.eps_t[a]) ||
        !std::isfinite(b.eps_R[a]) || !std::isfinite(b.t_off[a]) || !std::isfinite(b.R_off[a])) {
      set_err(ctx, "pose box: half-widths must be finite and >= 0");
      return AS_E_ARG;
    }
    bp.lo[a] = b.t_off[a] - b.eps_t[a];
    bp.hi[a] = b.t_off[a] + b.eps_t[a];
    bp.lo[3 + a] = b.R_off[a] - b.eps_R[a];
    bp.hi[3 + a] = b.R_off[a] + b.eps_R[a];
    bp.parts[a] = b.parts[a];
    bp.parts[3 + a] = b.parts[3 + a];
  }
  for (int g = 0; g < 3; ++g) {
    if (g < ctx->n_groups) {
      bp.lo[6 + g] = ctx->shift_lo[g];
      bp.hi[6 + g] = ctx->shift_hi[g];
      bp.parts[6 + g] = ctx->gparts[g];
      for (int k = 0; k < 3; ++k) bp.dir[g][k] = ctx->dir[g][k];
    } else {
      bp.lo[6 + g] = bp.hi[6 + g] = 0.0;
      bp.parts[6 + g] = 1;
    }
  }
  long long nsub = 1;
  int nv = 0;
  for (int a = 0; a < 9; ++a) {
    if (bp.parts[a] < 1) {
      set_err(ctx, "parts must be >= 1");
      return AS_E_ARG;
    }
    const bool var = bp.hi[a] > bp.lo[a];
    if (!var && bp.parts[a] != 1) {
      set_err(ctx, "parts > 1 on an unperturbed axis %d", a);
      return AS_E_ARG;
    }
    if (var) {
      bi.axis[nv] = a;
      bi.c[nv] = 0.5 * (bp.lo[a] + bp.hi[a]);
      bi.r[nv] = 0.5 * (bp.hi[a] - bp.lo[a]);
      ++nv;
    }
    nsub *= bp.parts[a];
  }
  if (!ctx->sub_host.empty()) {  // explicit partition: each sub-box inside the box
    const int ne = (int)(ctx->sub_host.size() / 18);
    for (int s = 0; s < ne; ++s)
      for (int a = 0; a < 9; ++a) {
        const double lo = ctx->sub_host[(s * 9 + a) * 2], hi = ctx->sub_host[(s * 9 + a) * 2 + 1];
        if (!(lo <= hi) || lo < bp.lo[a] || hi > bp.hi[a]) {
          set_err(ctx, "explicit sub-box %d axis %d [%g, %g] outside the box [%g, %g]", s, a, lo,
                  hi, bp.lo[a], bp.hi[a]);
          return AS_E_ARG;
        }
      }
    nsub = ne;
    bp.sub = P<double>(ctx->subs);
  }
  if (nsub > 1000000) {
    set_err(ctx, "too many sub-boxes (%lld)", nsub);
    return AS_E_ARG;
  }
  bp.n_sub = (int)nsub;
  bp.t_frame = b.t_frame;
  for (int k = 0; k < 3; ++k) {
    bp.euler0[k] = ctx->cam.euler[k];
    bp.t0[k] = ctx->cam.t[k];
  }
  bi.n_sub = (int)nsub;
  bi.n_shared = nv;
  bi.n_vars = nv + (ctx->has_priv ? 3 : 0);
  if (bi.n_vars > NVMAX) {
    set_err(ctx, "too many box variables (%d shared + 3 private > %d)", nv, NVMAX);
    return AS_E_ARG;
  }
  return AS_OK;
}

struct Geometry {
  int ts, ntx, nty, ntiles;
};

// ---------------------------------------------------------------- per sub-box pipeline
void run_setup(as_ctx* ctx, const BoxInfo& bi, int s) {
  SetupArgs a{};
  a.mean = P<float>(ctx->mean);
  a.chol = P<float>(ctx->chol);
  a.opacity = P<float>(ctx->opacity);
  a.color = P<float>(ctx->color);
  a.group_of = ctx->has_group ? P<int32_t>(ctx->group_of) : nullptr;
  a.col_lo = ctx->has_col ? P<float>(ctx->col_lo) : nullptr;
  a.col_hi = ctx->has_col ? P<float>(ctx->col_hi) : nullptr;
  a.op_lo = ctx->has_op ? P<float>(ctx->op_lo) : nullptr;
  a.op_hi = ctx->has_op ? P<float>(ctx->op_hi) : nullptr;
  a.priv_lo = ctx->has_priv ? P<float>(ctx->priv_lo) : nullptr;
  a.priv_hi = ctx->has_priv ? P<float>(ctx->priv_hi) : nullptr;
  a.ns = bi.n_shared;
  a.N = ctx->N;
  a.fx = ctx->cam.fx;
  a.fy = ctx->cam.fy;
  a.cx = ctx->cam.cx;
  a.cy = ctx->cam.cy;
  for (int g = 0; g < 3; ++g)
    for (int k = 0; k < 3; ++k) a.dir[g][k] = ctx->dir[g][k];
  a.pose = P<PoseDev>(ctx->pose) + s;
  a.hot = ctx->hot.p;
  a.pair = ctx->pair.p;
  a.kkey = P<unsigned long long>(ctx->kkey);
  a.kval = P<int32_t>(ctx->kval);
  a.k_tol = ctx->k_tol;
  a.k_max = ctx->k_max;
  a.inv_backward = ctx->inv_backward;
  a.wsmax = P<unsigned long long>(ctx->counters) + 4;
  a.counters = P<unsigned long long>(ctx->counters);
  launch_setup(bi.n_vars, a, ctx->stream);
  LAUNCHED(ctx, 1);
}

void cub_sort_keys64(as_ctx* ctx, unsigned long long* kin, unsigned long long* kout,
                     int32_t* vin, int32_t* vout, int64_t n, int end_bit) {
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, vout, (int)n, 0, end_bit,
                                  ctx->stream);
  ensure(ctx, ctx->cub_tmp, tmp);
  CK(cub::DeviceRadixSort::SortPairs(ctx->cub_tmp.p, tmp, kin, kout, vin, vout, (int)n, 0,
                                     end_bit, ctx->stream));
  LAUNCHED(ctx, 1);
}
void cub_sort_keys32(as_ctx* ctx, uint32_t* kin, uint32_t* kout, int32_t* vin, int32_t* vout,
                     int64_t n, int end_bit, bool descending) {
  size_t tmp = 0;
  if (descending)
    cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp, kin, kout, vin, vout, (int)n, 0,
                                              end_bit, ctx->stream);
  else
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, vout, (int)n, 0, end_bit,
                                    ctx->stream);
  ensure(ctx, ctx->cub_tmp, tmp);
  if (descending)
    CK(cub::DeviceRadixSort::SortPairsDescending(ctx->cub_tmp.p, tmp, kin, kout, vin, vout,
                                                 (int)n, 0, end_bit, ctx->stream));
  else
    CK(cub::DeviceRadixSort::SortPairs(ctx->cub_tmp.p, tmp, kin, kout, vin, vout, (int)n, 0,
                                       end_bit, ctx->stream));
  LAUNCHED(ctx, 1);
}
template <typename TI, typename TO>
void cub_exclusive_sum(as_ctx* ctx, TI* in, TO* out, int64_t n) {
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, (int)n, ctx->stream);
  ensure(ctx, ctx->cub_tmp, tmp);
  CK(cub::DeviceScan::ExclusiveSum(ctx->cub_tmp.p, tmp, in, out, (int)n, ctx->stream));
  LAUNCHED(ctx, 1);
}
template <typename T>
void cub_inclusive_sum(as_ctx* ctx, T* in, T* out, int64_t n) {
  size_t tmp = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tmp, in, out, (int)n, ctx->stream);
  ensure(ctx, ctx->cub_tmp, tmp);
  CK(cub::DeviceScan::InclusiveSum(ctx->cub_tmp.p, tmp, in, out, (int)n, ctx->stream));
  LAUNCHED(ctx, 1);
}

int bits_for(int64_t v) {
  int b = 1;
  while ((1ll << b) <= v) ++b;
  return b;
}

__global__ void k_seq(int32_t* v, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = i;
}
// longest tile list (out[0]) and the number of non-empty tiles (nonempty)
__global__ void k_tile_max(const int64_t* tb, const int64_t* te, int n, unsigned long long* out,
                           unsigned long long* nonempty) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const int64_t k = te[i] - tb[i];
    if (k > 0) {
      atomicMax(out, (unsigned long long)k);
      atomicAdd(nonempty, 1ull);
    }
  }
}

// counters layout (unsigned long long[16])
enum { C_FAIL = 0, C_STRAD = 1, C_DROP = 2, C_PAIRS = 3, C_WSMAX = 4, C_KMAX = 5, C_ACTIVE = 6,
       C_MMAX = 7, C_UNC = 8, C_VIOL = 9, C_WMAX = 10, C_SUBUNC = 11, C_SCENE = 12,
       C_NEXCMAX = 13, C_ITEMSMAX = 14, C_WMAXALL = 15, C_OVF = 16, C_NONEMPTY = 17,
       C_NCOUNTERS = 24 };

// per-position count of the finalisation records (keys >= M: none)
__global__ void k_fin_hist(const uint32_t* key, int64_t M, int32_t* cnt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < M && key[i] < (uint64_t)M) atomicAdd(&cnt[key[i]], 1);
}

// sizes the render needs on the device only: max (and sum) over the render's sub-boxes
__global__ void k_note(const int64_t* v, unsigned long long* mx, unsigned long long* sum) {
  const unsigned long long x = (unsigned long long)(*v > 0 ? *v : 0);
  if (mx) atomicMax(mx, x);
  if (sum) atomicAdd(sum, x);
}
// a size past its remembered capacity: flag it (the tile kernels then skip their work)
__global__ void k_cap_check(const int64_t* v, int64_t cap, unsigned long long* ovf,
                            unsigned long long bit) {
  if (*v > cap) atomicOr(ovf, bit);
}
__global__ void k_note32(const unsigned* v, unsigned long long* mx) {
  atomicMax(mx, (unsigned long long)*v);
}
// padding of a buffer sized from remembered capacities: positions [*n, cap) get a tile id
// past the last tile (sorted last, skipped by every later kernel)
__global__ void k_pad_pairs(uint32_t* keys, int32_t* vals, const int64_t* n, int64_t cap,
                            uint32_t sentinel) {
  for (int64_t p = *n + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < cap;
       p += (int64_t)gridDim.x * blockDim.x) {
    keys[p] = sentinel;
    vals[p] = 0;
  }
}
// work items [*n, cap): empty (tile -1), sorted last
__global__ void k_pad_items(int4* items, int4* items2, uint32_t* key, const int64_t* n,
                            int64_t cap) {
  for (int64_t j = *n + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < cap;
       j += (int64_t)gridDim.x * blockDim.x) {
    items[j] = make_int4(-1, 0, 0, 0);
    items2[j] = make_int4(0, 0, 0, 0);
    key[j] = 0;
  }
}

// a timing event: recorded for real inside a captured graph too (an event record node; a
// plain record would only mark a capture dependency)
cudaError_t timing_record(cudaEvent_t e, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  const cudaError_t r = cudaStreamIsCapturing(st, &cs);
  if (r != cudaSuccess) return r;
  return cs == cudaStreamCaptureStatusActive
             ? cudaEventRecordWithFlags(e, st, cudaEventRecordExternal)
             : cudaEventRecord(e, st);
}

// a blocking read of a device value (a host synchronisation inside the pipeline)
template <typename T>
T read_dev(as_ctx* ctx, const T* dptr) {
  T v{};
  CK(cudaMemcpyAsync(&v, dptr, sizeof v, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ++ctx->host_syncs;
  return v;
}
int64_t read_i64(as_ctx* ctx, const int64_t* dptr) { return read_dev(ctx, dptr); }

struct PhaseTimes {
  double setup = 0, bin = 0, pairs = 0, tile = 0, sort = 0, merge = 0;
};

// Render one sub-box (rows a2-a10) into row-major (tslot == nullptr) or compact tile-major
// outputs.  tlist: device list of n_list tiles to render; owner: device owner map or null.
// Sizes: a probing render reads each size back when it is known (a host synchronisation);
// a sync-free one (ctx->spec_on) takes the remembered capacity, pads up to it on the device and
// leaves the check to the end of the render (verify_sizes).  The kernels compute the same
// chunks and results either way.
int64_t size_or_cap(as_ctx* ctx, const int64_t* dptr, int64_t cap, int64_t& probe_max) {
  if (ctx->spec_on) return cap;
  const int64_t v = read_i64(ctx, dptr);
  probe_max = std::max(probe_max, v);
  return v;
}

// ev: SUB_EVENTS events of this sub-box for the phase times (nullptr: none)
void render_subbox(as_ctx* ctx, const BoxInfo& bi, int s, bool do_setup, const Geometry& G,
                   int bs, const int32_t* owner, int rank, const int32_t* tlist, int n_list,
                   const int32_t* tslot, float* lo, float* hi, bool first, cudaEvent_t* ev) {
  cudaStream_t st = ctx->stream;
  const bool spec = ctx->spec_on;
  ctx->last_has_exc = false;
  const int64_t N = ctx->N;
  const int nv = bi.n_vars;
  unsigned long long* ctr = P<unsigned long long>(ctx->counters);
  // BS is a performance knob: clamp it to what fits in shared memory at this n, and to 128
  // (k_tile's 256-position skip ring covers a batch plus the 128 positions before it)
  bs = tile_batch(nv, G.ts, bs);
  if (ev) CK(timing_record(ev[0], st));
  nvtxRangePushA("absplat.setup");
  if (do_setup) {
    CK(cudaMemsetAsync(ctr + C_WSMAX, 0, sizeof(unsigned long long), st));
    run_setup(ctx, bi, s);
  }
  if (ev) CK(timing_record(ev[1], st));
  nvtxRangePop();
  nvtxRangePushA("absplat.bin");
  // ---- a6: depth order (stable radix sort by kappa: ties keep ascending index, G6)
  if (ev) CK(timing_record(ev[6], st));
  cub_sort_keys64(ctx, P<unsigned long long>(ctx->kkey), P<unsigned long long>(ctx->kkey2),
                  P<int32_t>(ctx->kval), P<int32_t>(ctx->order), N, 64);
  if (ev) CK(timing_record(ev[7], st));
  // ---- a6: count overlapped tiles per Gaussian, scan, emit in depth order
  BinArgs ba{};
  ba.order = P<int32_t>(ctx->order);
  ba.N = N;
  ba.hot = ctx->hot.p;
  ba.nv = nv;
  ba.ts = G.ts;
  ba.ntx = G.ntx;
  ba.nty = G.nty;
  ba.W = ctx->cam.W;
  ba.H = ctx->cam.H;
  ba.owner = owner;
  ba.rank = rank;
  ba.counts = P<int64_t>(ctx->counts);
  ba.offsets = P<int64_t>(ctx->offsets);
  ba.tile_cost = nullptr;
  CK(cudaMemsetAsync(ba.counts + N, 0, sizeof(int64_t), st));
  launch_count(ba, st);
  LAUNCHED(ctx, 1);
  cub_exclusive_sum(ctx, ba.counts, P<int64_t>(ctx->offsets), N + 1);
  const int64_t* Mdev = P<int64_t>(ctx->offsets) + N;
  k_note<<<1, 1, 0, st>>>(Mdev, ctr + C_MMAX, ctr + C_PAIRS);
  LAUNCHED(ctx, 1);
  const int64_t M = size_or_cap(ctx, Mdev, ctx->cur_spec->M, ctx->probe.M);
  if (spec) {
    k_cap_check<<<1, 1, 0, st>>>(Mdev, M, ctr + C_OVF, 4ull);
    LAUNCHED(ctx, 1);
  }
  ensure(ctx, ctx->keys, sizeof(uint32_t) * (M + 1));
  ensure(ctx, ctx->keys2, sizeof(uint32_t) * (M + 1));
  ensure(ctx, ctx->vals, sizeof(int32_t) * (M + 1));
  ensure(ctx, ctx->vals2, sizeof(int32_t) * (M + 1));
  ba.keys = P<uint32_t>(ctx->keys);
  ba.vals = P<int32_t>(ctx->vals);
  ba.cap = M;
  launch_emit(ba, st);
  LAUNCHED(ctx, 1);
  if (spec && M > 0) {
    k_pad_pairs<<<148, 256, 0, st>>>(ba.keys, ba.vals, Mdev, M, (uint32_t)G.ntiles);
    LAUNCHED(ctx, 1);
  }
  // stable sort by tile id: within a tile the depth order of emission is kept (padding ids
  // = ntiles fit the sorted bits and go last)
  if (ev) CK(timing_record(ev[8], st));
  if (M > 0)
    cub_sort_keys32(ctx, P<uint32_t>(ctx->keys), P<uint32_t>(ctx->keys2), P<int32_t>(ctx->vals),
                    P<int32_t>(ctx->vals2), M, bits_for(G.ntiles), false);
  if (ev) CK(timing_record(ev[9], st));
  const uint32_t* skeys = P<uint32_t>(ctx->keys2);
  const int32_t* svals = P<int32_t>(ctx->vals2);
  launch_ranges(skeys, M, G.ntiles, P<int64_t>(ctx->tbegin), P<int64_t>(ctx->tend), st);
  LAUNCHED(ctx, 1);
  k_tile_max<<<(G.ntiles + 255) / 256, 256, 0, st>>>(P<int64_t>(ctx->tbegin),
                                                     P<int64_t>(ctx->tend), G.ntiles, ctr + C_KMAX,
                                                     ctr + C_NONEMPTY);
  LAUNCHED(ctx, 1);
  if (ev) CK(timing_record(ev[2], st));
  nvtxRangePop();
  nvtxRangePushA("absplat.pairs");
  // ---- a7: depth-order abstraction (uncertain pairs + exception windows)
  TileArgs ta{};
  bool has_exc = false;
  int R = 1;
  ctx->last_wmax = 0;
  if (nv > 0 && M > 0) {
    ensure(ctx, ctx->nF, sizeof(int32_t) * M);
    ensure(ctx, ctx->nG, sizeof(int32_t) * M);
    ensure(ctx, ctx->ntot, sizeof(int64_t) * (M + 1));
    ensure(ctx, ctx->eoff, sizeof(int64_t) * (M + 1));
    ensure(ctx, ctx->wsP, sizeof(double) * M);
    ensure(ctx, ctx->kapP, sizeof(double) * M);
    ensure(ctx, ctx->posD, sizeof(double) * 2 * (nv + 1) * M);
    ensure(ctx, ctx->tileh, sizeof(double) * (NVMAX + 1) * G.ntiles);
    ensure(ctx, ctx->tilemax, sizeof(unsigned long long) * G.ntiles);
    PairArgs pa{};
    pa.keys = skeys;
    pa.vals = svals;
    pa.tbegin = P<int64_t>(ctx->tbegin);
    pa.tend = P<int64_t>(ctx->tend);
    pa.M = M;
    pa.nexc_cap = 0;
    pa.pair = ctx->pair.p;
    pa.nv = nv;
    pa.pose = P<PoseDev>(ctx->pose) + s;
    pa.fx = ctx->cam.fx;
    pa.fy = ctx->cam.fy;
    pa.cx = ctx->cam.cx;
    pa.cy = ctx->cam.cy;
    pa.ts = G.ts;
    pa.ntx = G.ntx;
    pa.ntiles = G.ntiles;
    pa.tileh = P<double>(ctx->tileh);
    pa.tilemax = P<unsigned long long>(ctx->tilemax);
    pa.wsP = P<double>(ctx->wsP);
    pa.kapP = P<double>(ctx->kapP);
    pa.posD = P<double>(ctx->posD);
    pa.nF = P<int32_t>(ctx->nF);
    pa.nG = P<int32_t>(ctx->nG);
    pa.ntot = P<int64_t>(ctx->ntot);
    pa.counters = ctr + C_UNC;
    CK(cudaMemsetAsync(pa.ntot + M, 0, sizeof(int64_t), st));
    ensure(ctx, ctx->hpos, sizeof(int32_t) * M);
    ensure(ctx, ctx->gpos, sizeof(int32_t) * M);
    ensure(ctx, ctx->maskF, sizeof(ulonglong2) * M);
    ensure(ctx, ctx->maskG, sizeof(ulonglong2) * M);
    pa.hpos = P<int32_t>(ctx->hpos);
    pa.gpos = P<int32_t>(ctx->gpos);
    pa.mF = P<ulonglong2>(ctx->maskF);
    pa.mG = P<ulonglong2>(ctx->maskG);
    pa.subunc = ctr + C_SUBUNC;
    pa.ns = bi.n_shared;
    CK(cudaMemsetAsync(pa.subunc, 0, sizeof(unsigned long long), st));
    launch_pairs_prep(pa, st);
    LAUNCHED(ctx, 2);
    launch_pairs_count(pa, st);  // forward-only classification + completion: counts, h, g, masks
    LAUNCHED(ctx, 2);
    bool any_unc = ctx->cur_spec->exc;  // sync-free: the remembered answer (checked at the end)
    if (!spec) {
      any_unc = read_dev(ctx, pa.subunc) > 0;
      ctx->probe.exc = ctx->probe.exc || any_unc;
    }
    if (any_unc) {
      // explicit lists only for positions with a partner more than 128 positions away
      cub_exclusive_sum(ctx, pa.ntot, P<int64_t>(ctx->eoff), M + 1);
      k_note<<<1, 1, 0, st>>>(P<int64_t>(ctx->eoff) + M, ctr + C_NEXCMAX, nullptr);
      LAUNCHED(ctx, 1);
      const int64_t nexc = size_or_cap(ctx, P<int64_t>(ctx->eoff) + M, ctx->cur_spec->nexc,
                                       ctx->probe.nexc);
      if (spec) {
        k_cap_check<<<1, 1, 0, st>>>(P<int64_t>(ctx->eoff) + M, nexc, ctr + C_OVF, 8ull);
        LAUNCHED(ctx, 1);
      }
      ctx->last_nexc = nexc;
      pa.off = P<int64_t>(ctx->eoff);
      pa.nexc_cap = nexc;
      ensure(ctx, ctx->exc, sizeof(int32_t) * std::max<int64_t>(nexc, 1));
      pa.exc = P<int32_t>(ctx->exc);
      if (nexc > 0) {
        launch_pairs_fill(pa, st);
        LAUNCHED(ctx, 1);
      }
      ensure(ctx, ctx->diff, sizeof(int32_t) * 3 * (M + 1));
      ensure(ctx, ctx->cover, sizeof(int32_t) * 2 * (M + 1));
      ensure(ctx, ctx->pflag, sizeof(int4) * M);
      int32_t* dstore = P<int32_t>(ctx->diff);
      int32_t* dcut = dstore + (M + 1);
      int32_t* hstart = dcut + (M + 1);
      int32_t* cstore = P<int32_t>(ctx->cover);
      int32_t* ccut = cstore + (M + 1);
      CK(cudaMemsetAsync(dstore, 0, sizeof(int32_t) * 3 * (M + 1), st));
      launch_mark(pa, dstore, dcut, hstart, st);
      LAUNCHED(ctx, 1);
      cub_inclusive_sum(ctx, dstore, cstore, M + 1);
      cub_inclusive_sum(ctx, dcut, ccut, M + 1);
      unsigned int* wmax = reinterpret_cast<unsigned int*>(ctr + C_WMAX);
      CK(cudaMemsetAsync(wmax, 0, sizeof(unsigned long long), st));
      ensure(ctx, ctx->finkey, sizeof(uint32_t) * M);
      ensure(ctx, ctx->finkey2, sizeof(uint32_t) * M);
      ensure(ctx, ctx->finval, sizeof(int32_t) * M);
      ensure(ctx, ctx->finval2, sizeof(int32_t) * M);
      ensure(ctx, ctx->finstart, sizeof(int32_t) * (M + 1));
      ensure(ctx, ctx->finrec, sizeof(FinRec) * M);
      launch_meta(pa, cstore, ccut, hstart, P<int4>(ctx->pflag), wmax, P<uint32_t>(ctx->finkey),
                  P<int32_t>(ctx->finval), st);
      LAUNCHED(ctx, 1);
      cub_sort_keys32(ctx, P<uint32_t>(ctx->finkey), P<uint32_t>(ctx->finkey2),
                      P<int32_t>(ctx->finval), P<int32_t>(ctx->finval2), M, bits_for(M), false);
      // CSR start of the finalisation lists over all positions: fs = exclusive scan of the
      // per-position record counts (the keys' histogram; `cover` is free after k_meta)
      int32_t* fcnt = P<int32_t>(ctx->cover);
      CK(cudaMemsetAsync(fcnt, 0, sizeof(int32_t) * (M + 1), st));
      k_fin_hist<<<(unsigned)((M + 255) / 256), 256, 0, st>>>(P<uint32_t>(ctx->finkey2), M, fcnt);
      LAUNCHED(ctx, 1);
      cub_exclusive_sum(ctx, fcnt, P<int32_t>(ctx->finstart), M + 1);
      launch_finrec(P<uint32_t>(ctx->finkey2), P<int32_t>(ctx->finval2), pa, P<int4>(ctx->pflag),
                    P<ulonglong2>(ctx->maskG), ctx->hot.p, P<FinRec>(ctx->finrec), st);
      LAUNCHED(ctx, 1);
      ta.finstart = P<int32_t>(ctx->finstart);
      ta.fin_rec = P<FinRec>(ctx->finrec);
      ta.mF = P<ulonglong2>(ctx->maskF);
      k_note32<<<1, 1, 0, st>>>(wmax, ctr + C_WMAXALL);
      LAUNCHED(ctx, 1);
      if (spec) {
        R = ctx->cur_spec->R;
      } else {
        const unsigned hw = read_dev(ctx, wmax);
        while (R <= (int)hw) R <<= 1;
        ctx->probe.R = std::max(ctx->probe.R, R);
        ctx->last_wmax = (int)hw;
      }
      has_exc = true;
      ctx->last_has_exc = true;
      ta.pm = P<int4>(ctx->pflag);
      ta.nG = P<int32_t>(ctx->nG);
      ta.eoff = P<int64_t>(ctx->eoff);
      ta.exc = P<int32_t>(ctx->exc);
    }
  }
  if (ev) CK(timing_record(ev[3], st));
  nvtxRangePop();
  nvtxRangePushA("absplat.items");
  // ---- work items: (tile, chunk) cut where no uncertain pair is split, longest first
  const int grid0 = tile_grid(nv, G.ts, bs);
  int grid = grid0;
  if (grid <= 0) {
    (void)cudaGetLastError();
    set_err(ctx, "tile kernel: shared-memory opt-in / occupancy query failed (n=%d, TS=%d, BS=%d)",
            nv, G.ts, bs);
    throw Err{AS_E_CUDA};
  }
  const size_t npix = (size_t)G.ts * G.ts;
  if (has_exc) {  // ring memory: grid x R x threads float4 (cap the total at ~8 GB)
    const size_t per = (size_t)R * tile_ring_slot_bytes(G.ts);
    const size_t budget = (size_t)8 << 30;
    if ((size_t)grid * per > budget) grid = std::max<int>(1, (int)(budget / per));
    ensure(ctx, ctx->scratch, (size_t)grid * per);
  }
  // automatic chunk length (about six chunks per CTA; with windows beyond the 128-position
  // masks six times more but at least two batches, so the few expensive tiles split finely
  // enough to balance without rescanning long lookbacks too often: C5 14.4 -> 5.3 ms in round
  // 1, 2.17 -> 1.82 ms with the two-batch floor), decided on the device from this sub-box's
  // pair count and longest window
  ChunkTarget tg;
  tg.M = Mdev;
  tg.wmax = has_exc ? reinterpret_cast<const unsigned*>(ctr + C_WMAX) : nullptr;
  tg.nsub = tile_subblocks(G.ts);
  tg.grid = grid0;
  tg.bs = bs;
  tg.over = ctx->chunk_target;
  int64_t* caps = P<int64_t>(ctx->ntot);  // reuse: int64 [ntiles+1]
  ensure(ctx, ctx->ntot, sizeof(int64_t) * (std::max<int64_t>(M, G.ntiles) + 1));
  caps = P<int64_t>(ctx->ntot);
  ensure(ctx, ctx->item_off, sizeof(int64_t) * (G.ntiles + 1));
  launch_item_caps(P<int64_t>(ctx->tbegin), P<int64_t>(ctx->tend), G.ntiles, tg, caps, st);
  LAUNCHED(ctx, 1);
  CK(cudaMemsetAsync(caps + G.ntiles, 0, sizeof(int64_t), st));
  cub_exclusive_sum(ctx, caps, P<int64_t>(ctx->item_off), G.ntiles + 1);
  const int64_t* NIdev = P<int64_t>(ctx->item_off) + G.ntiles;
  k_note<<<1, 1, 0, st>>>(NIdev, ctr + C_ITEMSMAX, nullptr);
  LAUNCHED(ctx, 1);
  const int64_t n_items = size_or_cap(ctx, NIdev, ctx->cur_spec->items, ctx->probe.items);
  ensure(ctx, ctx->items, sizeof(int4) * n_items);
  ensure(ctx, ctx->items2, sizeof(int4) * n_items);
  ensure(ctx, ctx->item_key, sizeof(uint32_t) * n_items);
  ensure(ctx, ctx->item_key2, sizeof(uint32_t) * n_items);
  ensure(ctx, ctx->item_idx, sizeof(int32_t) * n_items);
  ensure(ctx, ctx->item_order, sizeof(int32_t) * n_items);
  ensure(ctx, ctx->item_cnt, sizeof(int32_t) * G.ntiles);
  ensure(ctx, ctx->partial, sizeof(float) * 8 * npix * n_items);
  ensure(ctx, ctx->chunk_stats, sizeof(int4) * n_items);
  launch_chunks(P<int64_t>(ctx->tbegin), P<int64_t>(ctx->tend), has_exc ? P<int4>(ctx->pflag) : nullptr,
                P<int64_t>(ctx->item_off), G.ntiles, n_items, tg, R, owner, rank,
                P<int4>(ctx->chunk_stats), P<int4>(ctx->items), P<int4>(ctx->items2),
                P<int32_t>(ctx->item_cnt), P<uint32_t>(ctx->item_key), ctr + C_OVF, st);
  LAUNCHED(ctx, 2);
  if (spec && n_items > 0) {
    k_pad_items<<<148, 256, 0, st>>>(P<int4>(ctx->items), P<int4>(ctx->items2),
                                     P<uint32_t>(ctx->item_key), NIdev, n_items);
    LAUNCHED(ctx, 1);
  }
  if (n_items > 0) {
    k_seq<<<(unsigned)((n_items + 255) / 256), 256, 0, st>>>(P<int32_t>(ctx->item_idx), (int)n_items);
    LAUNCHED(ctx, 1);
  }
  cub_sort_keys32(ctx, P<uint32_t>(ctx->item_key), P<uint32_t>(ctx->item_key2),
                  P<int32_t>(ctx->item_idx), P<int32_t>(ctx->item_order), n_items, 32, true);
  ensure(ctx, ctx->work_counter, sizeof(int));
  CK(cudaMemsetAsync(ctx->work_counter.p, 0, sizeof(int), st));
  // ---- a8-a10: the tile kernel (+ merge of split tiles)
  ta.hot = ctx->hot.p;
  ta.vals = svals;
  ta.tbegin = P<int64_t>(ctx->tbegin);
  ta.tend = P<int64_t>(ctx->tend);
  ta.items = P<int4>(ctx->items);
  ta.items2 = P<int4>(ctx->items2);
  ta.order = P<int32_t>(ctx->item_order);
  ta.n_items = (int)n_items;
  ta.counter = P<int>(ctx->work_counter);
  ta.item_off = P<int64_t>(ctx->item_off);
  ta.item_cnt = P<int32_t>(ctx->item_cnt);
  ta.tile_slot = tslot;
  ta.ntiles = G.ntiles;
  ta.ts = G.ts;
  ta.ntx = G.ntx;
  ta.W = ctx->cam.W;
  ta.H = ctx->cam.H;
  ta.bs = bs;
  ta.first = first ? 1 : 0;
  ta.ntau = (float)((double)N * TAU);
  ta.ring = has_exc ? P<float4>(ctx->scratch) : nullptr;
  ta.R = R;
  ta.partial = P<float>(ctx->partial);
  ta.lo = lo;
  ta.hi = hi;
  ta.active = ctr + C_ACTIVE;
  ta.dbg = ctx->debug ? P<unsigned long long>(ctx->dbg) : nullptr;
  ta.ovf = spec ? ctr + C_OVF : nullptr;
  ta.kver = tile_kernel_version(G.ts);
  ta.M = M;
  ta.nexc = has_exc ? ctx->last_nexc : 0;
  ta.n_partial = (int64_t)(8 * npix * n_items);
  ta.n_out = tslot ? (int64_t)ctx->last_out_tiles * G.ts * G.ts * 3 : (int64_t)ctx->cam.W * ctx->cam.H * 3;
  ctx->last_items = (int)n_items;
  ctx->last_grid = grid;
  ctx->last_R = R;
  if (ev) CK(timing_record(ev[4], st));
  nvtxRangePop();
  nvtxRangePushA("absplat.tile");
  launch_tile(nv, ta, grid, st);
  LAUNCHED(ctx, 1);
  if (ev) CK(timing_record(ev[5], st));
  nvtxRangePop();
  nvtxRangePushA("absplat.merge");
  launch_merge(ta, st);
  LAUNCHED(ctx, 1);
  if (ev) CK(timing_record(ev[10], st));
  nvtxRangePop();
  // NEXT-1 (O20): the uncertain positions' interval terms as raw per-pixel sums, for the
  // linear blend that follows (full-image renders only)
  ctx->last_unc = false;
  if (ctx->blend_mode == 1 && has_exc && !tslot) {
    const size_t img = (size_t)ctx->cam.W * ctx->cam.H * 3;
    ensure(ctx, ctx->unc_lo, sizeof(float) * img);
    ensure(ctx, ctx->unc_hi, sizeof(float) * img);
    TileArgs tu = ta;
    tu.unc_only = 1;
    tu.first = 1;
    tu.lo = P<float>(ctx->unc_lo);
    tu.hi = P<float>(ctx->unc_hi);
    tu.active = ctr + C_SCENE;  // scratch: the active pairs were counted by the first pass
    tu.dbg = nullptr;
    CK(cudaMemsetAsync(ctx->work_counter.p, 0, sizeof(int), st));
    launch_tile(nv, tu, grid, st);
    launch_merge(tu, st);
    LAUNCHED(ctx, 2);
    ctx->last_unc = true;
  }
  (void)tlist;
  (void)n_list;
}

// the phase events of the k-th sub-box of a render (pooled): [0] start, [1] after setup,
// [2] after binning, [3] after pair classification, [4] before / [5] after the tile kernel,
// [6]/[7] around the kappa sort, [8]/[9] around the pair sort, [10] after the chunk merge
constexpr int SUB_EVENTS = 11;
cudaEvent_t* sub_events(as_ctx* ctx, int k) {
  while ((int)ctx->sbev.size() < SUB_EVENTS * (k + 1)) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    ctx->sbev.push_back(e);
  }
  return ctx->sbev.data() + SUB_EVENTS * k;
}
// phase times of n sub-boxes (after the render's synchronisation)
void collect_phases(as_ctx* ctx, int n, PhaseTimes* pt) {
  for (int k = 0; k < n; ++k) {
    cudaEvent_t* e = ctx->sbev.data() + SUB_EVENTS * k;
    float a = 0, b = 0, c = 0, d = 0, f = 0, s1 = 0, s2 = 0, m = 0;
    CK(cudaEventElapsedTime(&a, e[0], e[1]));
    CK(cudaEventElapsedTime(&b, e[1], e[2]));
    CK(cudaEventElapsedTime(&c, e[2], e[3]));
    CK(cudaEventElapsedTime(&f, e[3], e[4]));
    CK(cudaEventElapsedTime(&d, e[4], e[5]));
    CK(cudaEventElapsedTime(&s1, e[6], e[7]));
    CK(cudaEventElapsedTime(&s2, e[8], e[9]));
    CK(cudaEventElapsedTime(&m, e[5], e[10]));
    pt->setup += a;
    pt->bin += b + f;
    pt->pairs += c;
    pt->tile += d;
    pt->sort += s1 + s2;
    pt->merge += m;
  }
}

as_status check_ready(as_ctx* ctx) {
  if (!ctx) return AS_E_ARG;
  if (ctx->N < 0) {
    set_err(ctx, "no scene loaded (as_load_scene)");
    return AS_E_STATE;
  }
  if (!ctx->have_cam) {
    set_err(ctx, "no camera (as_set_camera)");
    return AS_E_STATE;
  }
  if (!ctx->have_box) {
    set_err(ctx, "no pose box (as_set_pose_box)");
    return AS_E_STATE;
  }
  return AS_OK;
}

as_status check_tile_args(as_ctx* ctx, int tile, int batch, int nv) {
  if (tile != 8 && tile != 16 && tile != 32) {
    set_err(ctx, "tile must be 8, 16 or 32 (got %d)", tile);
    return AS_E_ARG;
  }
  if (batch < 1 || batch > 256) {
    set_err(ctx, "batch must be in [1, 256] (got %d)", batch);
    return AS_E_ARG;
  }
  return AS_OK;
}

void prepare_common(as_ctx* ctx, const BoxInfo& bi, const Geometry& G) {
  const int64_t N = ctx->N;
  const int nv = bi.n_vars;
  ensure(ctx, ctx->hot, hot_size(nv) * (size_t)std::max<int64_t>(N, 1));
  ensure(ctx, ctx->pair, pair_size(nv) * (size_t)std::max<int64_t>(N, 1));
  ensure(ctx, ctx->kkey, sizeof(unsigned long long) * (N + 1));
  ensure(ctx, ctx->kkey2, sizeof(unsigned long long) * (N + 1));
  ensure(ctx, ctx->kval, sizeof(int32_t) * (N + 1));
  ensure(ctx, ctx->order, sizeof(int32_t) * (N + 1));
  ensure(ctx, ctx->counts, sizeof(int64_t) * (N + 1));
  ensure(ctx, ctx->offsets, sizeof(int64_t) * (N + 1));
  ensure(ctx, ctx->counters, sizeof(unsigned long long) * C_NCOUNTERS);
  ensure(ctx, ctx->pose, sizeof(PoseDev) * bi.n_sub);
  ensure(ctx, ctx->tbegin, sizeof(int64_t) * G.ntiles);
  ensure(ctx, ctx->tend, sizeof(int64_t) * G.ntiles);
  ensure(ctx, ctx->tcost, sizeof(unsigned long long) * G.ntiles);
  ensure(ctx, ctx->tkey, sizeof(uint32_t) * G.ntiles);
  ensure(ctx, ctx->tkey2, sizeof(uint32_t) * G.ntiles);
  ensure(ctx, ctx->tids, sizeof(int32_t) * G.ntiles);
  ensure(ctx, ctx->tlist, sizeof(int32_t) * G.ntiles);
  ensure(ctx, ctx->tslot, sizeof(int32_t) * G.ntiles);
  ensure(ctx, ctx->owner, sizeof(int32_t) * G.ntiles);
  CK(cudaMemsetAsync(ctx->counters.p, 0, sizeof(unsigned long long) * C_NCOUNTERS, ctx->stream));
  if (ctx->debug) {
    ensure(ctx, ctx->dbg, sizeof(unsigned long long) * DBG_N);
    CK(cudaMemsetAsync(ctx->dbg.p, 0, sizeof(unsigned long long) * DBG_N, ctx->stream));
  }
  launch_pose(bi.bp, P<PoseDev>(ctx->pose), ctx->stream);
  LAUNCHED(ctx, 1);
}

Geometry geometry(const as_ctx* ctx, int tile) {
  Geometry G;
  G.ts = tile;
  G.ntx = (ctx->cam.W + tile - 1) / tile;
  G.nty = (ctx->cam.H + tile - 1) / tile;
  G.ntiles = G.ntx * G.nty;
  return G;
}

void read_counters(as_ctx* ctx, unsigned long long* h) {
  CK(cudaMemcpyAsync(h, ctx->counters.p, sizeof(unsigned long long) * C_NCOUNTERS,
                     cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
}

// hc: the counters when already read after the render (nullptr: read them here)
void fill_stats(as_ctx* ctx, const BoxInfo& bi, const Geometry& G, int n_tiles_rendered,
                const PhaseTimes& pt, double total_ms, as_stats* out,
                const unsigned long long* hc = nullptr) {
  unsigned long long h[C_NCOUNTERS];
  if (hc)
    std::memcpy(h, hc, sizeof h);
  else
    read_counters(ctx, h);
  std::memset(out, 0, sizeof *out);
  out->pairs = (int64_t)h[C_PAIRS];
  out->active_pairs = (int64_t)h[C_ACTIVE];
  out->uncertain_pairs = (int64_t)h[C_UNC];
  out->fails = (int64_t)h[C_FAIL];
  out->straddles = (int64_t)h[C_STRAD];
  out->dropped = (int64_t)h[C_DROP];
  out->order_violations = (int64_t)h[C_VIOL];
  out->launches = ctx->launches;
  out->kmax = (int32_t)h[C_KMAX];
  out->n_sub = bi.n_sub;
  out->n_vars = bi.n_vars;
  out->n_tiles = n_tiles_rendered;
  out->ms_setup = pt.setup;
  out->ms_bin = pt.bin;
  out->ms_pairs = pt.pairs;
  out->ms_tile = pt.tile;
  out->tile_kernel_ms = pt.tile;
  out->ms_total = total_ms;
  out->device_bytes = ctx->bytes;
  out->n_items = (int32_t)h[C_ITEMSMAX];
  out->grid = ctx->last_grid;
  out->ring_len = ctx->last_R;
  out->max_window = (int32_t)h[C_WMAXALL];
  out->host_syncs = ctx->host_syncs;
  out->ms_sort = pt.sort;
  out->ms_merge = pt.merge;
  out->kmean = h[C_NONEMPTY] ? (double)h[C_PAIRS] / (double)h[C_NONEMPTY] : 0.0;
  out->ms_gather = ctx->last_gather_ms;
  out->world = ctx->world;
  out->n_owned = n_tiles_rendered;
  out->peak_bytes = ctx->peak_bytes;
  (void)G;
}

void lpt(int n, const int64_t* costs, int world, int cap, int32_t* owner) {
  std::vector<int> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return costs[a] > costs[b]; });
  std::vector<int64_t> load(world, 0);
  std::vector<int> cnt(world, 0);
  for (int t : idx) {
    int best = -1;
    for (int r = 0; r < world; ++r) {
      if (cnt[r] >= cap) continue;
      if (best < 0 || load[r] < load[best]) best = r;
    }
    owner[t] = best;
    load[best] += costs[t] + 1;
    ++cnt[best];
  }
}


// ---------------------------------------------------------------- device owner map (a11)
// Longest-processing-time assignment on the device, identical to lpt() above: tiles in
// descending cost (ties: lower id first, the stable radix order), each to the least-loaded
// rank with room (ties: lower rank).  One warp: lane r holds ranks r, r + 32; the argmin is
// a warp min over (load << 7 | rank).  Then the ranks' slots in ascending tile id
// (__match_any over each 32-tile chunk) and the per-rank counts.
constexpr int LPT_CHUNK = 2048;  // sorted (cost, id) entries staged in shared memory at a time
__global__ void __launch_bounds__(256) k_lpt(const int32_t* ids, const unsigned long long* nkeys,
                                             int n, int world, int cap, int32_t* owner,
                                             int32_t* slot, int32_t* nown) {
  __shared__ int sbase[128];
  __shared__ unsigned long long skey[LPT_CHUNK];
  __shared__ int sid[LPT_CHUNK];
  const int lane = threadIdx.x & 31;
  const bool w0 = threadIdx.x < 32;
  unsigned long long load[4] = {0, 0, 0, 0};
  int cnt[4] = {0, 0, 0, 0};
  for (int c0 = 0; c0 < n; c0 += LPT_CHUNK) {
    const int m = min(LPT_CHUNK, n - c0);
    __syncthreads();
    for (int k = threadIdx.x; k < m; k += blockDim.x) {  // coalesced staging by the block
      skey[k] = nkeys[c0 + k];
      sid[k] = ids[c0 + k];
    }
    __syncthreads();
    if (!w0) continue;
  for (int i = 0; i < m; ++i) {
    const unsigned long long cost = ~skey[i];
    const int t = sid[i];
    int r;
    if (world <= 32 && __all_sync(0xffffffffu, load[0] < 0x80000000ull)) {
      // one rank per lane, loads below 2^31: a warp min (REDUX) and the lowest lane holding it
      const unsigned v = (lane < world && cnt[0] < cap) ? (unsigned)load[0] : 0xffffffffu;
      const unsigned mn = __reduce_min_sync(0xffffffffu, v);
      r = __ffs(__ballot_sync(0xffffffffu, v == mn)) - 1;
    } else {
      unsigned long long best = ~0ull;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int rr = lane + 32 * q;
        if (rr < world && cnt[q] < cap) best = min(best, (load[q] << 7) | (unsigned long long)rr);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
      r = (int)(best & 127ull);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (lane + 32 * q == r) {
        load[q] += cost + 1;
        ++cnt[q];
      }
    if (lane == 0) owner[t] = r;
  }
  }
  __syncthreads();
  if (!w0) return;
  for (int r = lane; r < 128; r += 32) sbase[r] = 0;
  __syncwarp();
  for (int c0 = 0; c0 < n; c0 += 32) {
    const int t = c0 + lane;
    const bool ok = t < n;
    const int r = ok ? owner[t] : -1;
    const unsigned act = __ballot_sync(0xffffffffu, ok);
    const unsigned peers = __match_any_sync(0xffffffffu, r) & act;
    const int base = ok ? sbase[r] : 0;
    __syncwarp();
    if (ok) {
      slot[t] = base + __popc(peers & ((1u << lane) - 1u));
      if ((peers & ((1u << lane) - 1u)) == 0) sbase[r] = base + __popc(peers);
    }
    __syncwarp();
  }
  for (int r = lane; r < world; r += 32) nown[r] = sbase[r];
}
// this rank's tile -> compact slot map (-1: another rank's), and the gathered-buffer slot map
// of every tile (rank-major [world][2][cap] layout: lo block then hi block per rank)
__global__ void k_slot_maps(const int32_t* owner, const int32_t* slot, int n, int rank, int cap,
                            int32_t* tslot, int32_t* gslot) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int r = owner[t];
  if (tslot) tslot[t] = r == rank ? slot[t] : -1;
  if (gslot) gslot[t] = r * 2 * cap + slot[t];
}
__global__ void k_cost_key(const unsigned long long* cost, int n, unsigned long long* key,
                           int32_t* id) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) {
    key[t] = ~cost[t];  // ascending ~cost == descending cost, stable ties keep the id order
    id[t] = t;
  }
}

// per-tile costs (pairs summed over the sub-boxes [s0, s1)) into ctx->tcost, no host sync;
// with a single sub-box its setup is left in place for the render to reuse
void tile_costs_dev(as_ctx* ctx, const BoxInfo& bi, const Geometry& G, int s0, int s1) {
  cudaStream_t st = ctx->stream;
  CK(cudaMemsetAsync(ctx->tcost.p, 0, sizeof(unsigned long long) * G.ntiles, st));
  unsigned long long* ctr = P<unsigned long long>(ctx->counters);
  for (int s = s0; s < s1; ++s) {
    CK(cudaMemsetAsync(ctr + C_WSMAX, 0, sizeof(unsigned long long), st));
    run_setup(ctx, bi, s);
    BinArgs ba{};
    ba.order = P<int32_t>(ctx->kval);  // identity order suffices for counting
    ba.N = ctx->N;
    ba.hot = ctx->hot.p;
    ba.nv = bi.n_vars;
    ba.ts = G.ts;
    ba.ntx = G.ntx;
    ba.nty = G.nty;
    ba.W = ctx->cam.W;
    ba.H = ctx->cam.H;
    ba.owner = nullptr;
    ba.counts = P<int64_t>(ctx->counts);
    ba.tile_cost = P<unsigned long long>(ctx->tcost);
    launch_count(ba, st);
    LAUNCHED(ctx, 1);
  }
  if (s1 - s0 != 1) CK(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long) * C_WSMAX, st));
  else CK(cudaMemsetAsync(ctr + C_DROP + 1, 0, sizeof(unsigned long long) * (C_WSMAX - C_DROP - 1), st));
  CK(cudaMemsetAsync(ctr + C_WSMAX + 1, 0, sizeof(unsigned long long) * (C_NCOUNTERS - C_WSMAX - 1),
                     st));
}

// device LPT owner map of the current costs (ctx->tcost): ctx->owner, ctx->tslot_all (slot of
// every tile in its owner's compact list), ctx->nown (tiles per rank)
void device_lpt(as_ctx* ctx, const Geometry& G, int world, int cap) {
  cudaStream_t st = ctx->stream;
  const int n = G.ntiles;
  ensure(ctx, ctx->lptkey, sizeof(unsigned long long) * n);
  ensure(ctx, ctx->lptkey2, sizeof(unsigned long long) * n);
  ensure(ctx, ctx->lptid, sizeof(int32_t) * n);
  ensure(ctx, ctx->lptid2, sizeof(int32_t) * n);
  ensure(ctx, ctx->tslot_all, sizeof(int32_t) * n);
  ensure(ctx, ctx->nown, sizeof(int32_t) * 128);
  k_cost_key<<<(n + 255) / 256, 256, 0, st>>>(P<unsigned long long>(ctx->tcost), n,
                                               P<unsigned long long>(ctx->lptkey),
                                               P<int32_t>(ctx->lptid));
  LAUNCHED(ctx, 1);
  cub_sort_keys64(ctx, P<unsigned long long>(ctx->lptkey), P<unsigned long long>(ctx->lptkey2),
                  P<int32_t>(ctx->lptid), P<int32_t>(ctx->lptid2), n, 64);
  k_lpt<<<1, 256, 0, st>>>(P<int32_t>(ctx->lptid2), P<unsigned long long>(ctx->lptkey2), n, world,
                          cap, P<int32_t>(ctx->owner), P<int32_t>(ctx->tslot_all),
                          P<int32_t>(ctx->nown));
  LAUNCHED(ctx, 1);
}

// ---------------------------------------------------------------- NCCL (loaded at run time)
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};
// the process's NCCL (the one torch already loaded, if any: same soname), resolved once
const NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return;
    }
    api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.allGather = reinterpret_cast<decltype(api.allGather)>(dlsym(h, "ncclAllGather"));
    api.allReduce = reinterpret_cast<decltype(api.allReduce)>(dlsym(h, "ncclAllReduce"));
    api.errorString = reinterpret_cast<decltype(api.errorString)>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.allGather &&
             api.allReduce && api.errorString;
    if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
  });
  return api;
}

#define NCK(call)                                                                        \
  do {                                                                                   \
    ncclResult_t r_ = (call);                                                            \
    if (r_ != ncclSuccess) {                                                             \
      set_err(ctx, "%s failed: %s (%s:%d)", #call, nccl_api().errorString(r_), __FILE__, \
              __LINE__);                                                                 \
      throw Err{AS_E_COMM};                                                              \
    }                                                                                    \
  } while (0)

void rot_c2w_host(const double e[3], double R[9]) {
  const double c0 = std::cos(e[0]), s0 = std::sin(e[0]), c1 = std::cos(e[1]), s1 = std::sin(e[1]);
  const double c2 = std::cos(e[2]), s2 = std::sin(e[2]);
  const double X[9] = {1, 0, 0, 0, c0, -s0, 0, s0, c0};
  const double Y[9] = {c1, 0, s1, 0, 1, 0, -s1, 0, c1};
  const double Z[9] = {c2, -s2, 0, s2, c2, 0, 0, 0, 1};
  double T[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) T[3 * i + j] = Z[3 * i] * Y[j] + Z[3 * i + 1] * Y[3 + j] + Z[3 * i + 2] * Y[6 + j];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) R[3 * i + j] = T[3 * i] * X[j] + T[3 * i + 1] * X[3 + j] + T[3 * i + 2] * X[6 + j];
}

}  // namespace

// ======================================================================== C ABI
extern "C" {

int32_t as_version(void) { return ABSPLAT_VERSION; }

const char* as_last_error(const as_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

as_status as_create(as_ctx** out, int32_t device, void* cuda_stream) {
  if (!out) return AS_E_ARG;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) return AS_E_CUDA;
  if (cudaSetDevice(device) != cudaSuccess) return AS_E_CUDA;
  as_ctx* c = new as_ctx();
  c->device = device;
  c->stream = reinterpret_cast<cudaStream_t>(cuda_stream);
  for (int k = 0; k < 8; ++k)
    if (cudaEventCreate(&c->ev[k]) != cudaSuccess) {
      delete c;
      return AS_E_CUDA;
    }
  *out = c;
  return AS_OK;
}

as_status as_destroy(as_ctx* ctx) {
  if (!ctx) return AS_E_ARG;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  DevBuf* bufs[] = {&ctx->mean, &ctx->chol, &ctx->opacity, &ctx->color, &ctx->st_mean,
                    &ctx->st_chol, &ctx->st_opacity, &ctx->st_color, &ctx->group_of,
                    &ctx->col_lo, &ctx->col_hi, &ctx->op_lo, &ctx->op_hi, &ctx->priv_lo, &ctx->priv_hi, &ctx->subs, &ctx->tmp_lo, &ctx->tmp_hi, &ctx->lin_tiles, &ctx->unc_lo, &ctx->unc_hi, &ctx->pose, &ctx->hot,
                    &ctx->pair, &ctx->kkey, &ctx->kkey2, &ctx->kval, &ctx->order, &ctx->counts,
                    &ctx->offsets, &ctx->cub_tmp, &ctx->keys, &ctx->keys2, &ctx->vals,
                    &ctx->vals2, &ctx->tbegin, &ctx->tend, &ctx->tcost, &ctx->tkey, &ctx->tkey2,
                    &ctx->tids, &ctx->tlist, &ctx->tslot, &ctx->owner, &ctx->nF, &ctx->nG,
                    &ctx->ntot, &ctx->eoff, &ctx->exc, &ctx->hpos, &ctx->gpos, &ctx->diff, &ctx->cover,
                    &ctx->pflag, &ctx->is_store, &ctx->slot, &ctx->scratch, &ctx->img_lo,
                    &ctx->img_hi, &ctx->counters, &ctx->conc_g, &ctx->untile_map, &ctx->tileh,
                    &ctx->tilemax, &ctx->wsP, &ctx->kapP, &ctx->posD, &ctx->item_off, &ctx->items, &ctx->items2,
                    &ctx->item_key, &ctx->item_key2, &ctx->item_idx, &ctx->item_order,
                    &ctx->item_cnt, &ctx->partial, &ctx->work_counter, &ctx->finkey,
                    &ctx->finkey2, &ctx->finval, &ctx->finval2, &ctx->finstart, &ctx->finrec, &ctx->maskF,
                    &ctx->maskG, &ctx->dbg, &ctx->gsend, &ctx->grecv, &ctx->lptkey,
                    &ctx->lptkey2, &ctx->lptid, &ctx->lptid2, &ctx->tslot_all, &ctx->nown,
                    &ctx->chunk_stats};
  for (DevBuf* b : bufs) release(ctx, *b);
  if (ctx->comm && nccl_api().ok) nccl_api().commDestroy((ncclComm_t)ctx->comm);
  for (int k = 0; k < 8; ++k)
    if (ctx->ev[k]) cudaEventDestroy(ctx->ev[k]);
  for (cudaEvent_t e : ctx->sbev) cudaEventDestroy(e);
  if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
  if (ctx->gev_in) cudaEventDestroy(ctx->gev_in);
  if (ctx->gev_out) cudaEventDestroy(ctx->gev_out);
  if (ctx->gstream) cudaStreamDestroy(ctx->gstream);
  delete ctx;
  return AS_OK;
}

as_status as_nccl_id(uint8_t id[128]) {
  if (!id) return AS_E_ARG;
  const NcclApi& api = nccl_api();
  if (!api.ok) return AS_E_COMM;
  ncclUniqueId u;
  if (api.getUniqueId(&u) != ncclSuccess) return AS_E_COMM;
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
  std::memcpy(id, &u, 128);
  return AS_OK;
}

as_status as_comm_init(as_ctx* ctx, int32_t rank, int32_t world, const uint8_t id[128]) {
  if (ctx) ++ctx->gen;  // state (or buffers) may change: no stale graph replay
  if (!ctx) return AS_E_ARG;
  if (!id || world < 1 || world > 128 || rank < 0 || rank >= world) {
    set_err(ctx, "as_comm_init: bad arguments (rank %d, world %d)", rank, world);
    return AS_E_ARG;
  }
  const NcclApi& api = nccl_api();
  if (!api.ok) {
    set_err(ctx, "as_comm_init: %s", api.why.c_str());
    return AS_E_COMM;
  }
  try {
    cudaSetDevice(ctx->device);
    if (ctx->comm) {
      api.commDestroy((ncclComm_t)ctx->comm);
      ctx->comm = nullptr;
    }
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    ncclComm_t c = nullptr;
    NCK(api.commInitRank(&c, world, u, rank));
    ctx->comm = c;
    ctx->rank = rank;
    ctx->world = world;
    return AS_OK;
  } catch (const Err& e) {
    ctx->rank = 0;
    ctx->world = 1;
    return e.st;
  }
}

as_status as_set_shard_axis(as_ctx* ctx, int32_t axis) {
  if (ctx) ++ctx->gen;  // state (or buffers) may change: no stale graph replay
  if (!ctx) return AS_E_ARG;
  if (axis < 0 || axis > 2) {
    set_err(ctx, "as_set_shard_axis: axis must be 0 (auto), 1 (tiles) or 2 (sub-boxes)");
    return AS_E_ARG;
  }
  ctx->shard_axis = axis;
  return AS_OK;
}

as_status as_debug_counters(as_ctx* ctx, int32_t enable, uint64_t* out) {
  if (ctx) ++ctx->gen;  // state (or buffers) may change: no stale graph replay
  if (!ctx) return AS_E_ARG;
  try {
    cudaSetDevice(ctx->device);
    if (out) {
      std::memset(out, 0, sizeof(uint64_t) * AS_DBG_N);
      if (ctx->debug && ctx->dbg.p) {
        CK(cudaMemcpyAsync(out, ctx->dbg.p, sizeof(uint64_t) * DBG_N, cudaMemcpyDeviceToHost,
                           ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
      }
    }
    if (enable >= 0) ctx->debug = enable != 0;
    return AS_OK;
  } catch (const Err& e) {
    return e.st;
  }
}

as_status as_set_allocator(as_ctx* ctx, as_alloc_fn alloc, as_free_fn free_fn, void* user) {
  if (ctx) ++ctx->gen;  // state (or buffers) may change: no stale graph replay
  if (!ctx) return AS_E_ARG;
  if ((alloc == nullptr) != (free_fn == nullptr)) {
    set_err(ctx, "as_set_allocator: alloc and free must both be set or both be NULL");
    return AS_E_ARG;
  }
  ctx->alloc_fn = alloc;
  ctx->free_fn = free_fn;
  ctx->alloc_user = alloc ? user : nullptr;
  return AS_OK;
}

namespace {
// scene validation on the device: the smallest invalid Gaussian index and its reason
// (1 mean / colour not finite or colour outside [0,1], 2 chol not finite, 3 chol diagonal
// <= 0, 4 opacity outside [0,1]) packed as index * 8 + reason into an atomicMin
// scene box (as_set_scene_box), on the device: lowest bad index * 8 + reason into *bad
__global__ void k_validate_sbox(int64_t N, const int32_t* group_of, int n_groups,
                                const float* col_lo, const float* col_hi, const float* op_lo,
                                const float* op_hi, const float* priv_lo, const float* priv_hi,
                                unsigned long long* bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  int why = 0;
  if (group_of && (group_of[i] < -1 || group_of[i] >= n_groups)) why = 1;
  if (!why && col_lo)
    for (int k = 0; k < 3; ++k) {
      const float l = col_lo[3 * i + k], h = col_hi[3 * i + k];
      if (!(l >= 0.f) || !(l <= h) || !(h <= 1.f)) why = 2;
    }
  if (!why && op_lo) {
    const float l = op_lo[i], h = op_hi[i];
    if (!(l >= 0.f) || !(l <= h) || !(h <= 1.f)) why = 3;
  }
  if (!why && priv_lo)
    for (int k = 0; k < 3; ++k) {
      const float l = priv_lo[3 * i + k], h = priv_hi[3 * i + k];
      if (!isfinite(l) || !isfinite(h) || !(l <= h)) why = 4;
    }
  if (why) atomicMin(bad, (unsigned long long)i * 8ull + (unsigned long long)why);
}

__global__ void k_validate(int64_t N, const float* m, const float* c, const float* o,
                           const float* col, unsigned long long* bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  int why = 0;
  for (int k = 0; k < 3 && !why; ++k)
    if (!isfinite(m[3 * i + k]) || !isfinite(col[3 * i + k]) || !(col[3 * i + k] >= 0.f) ||
        !(col[3 * i + k] <= 1.f))
      why = 1;
  for (int k = 0; k < 6 && !why; ++k)
    if (!isfinite(c[6 * i + k])) why = 2;
  if (!why && (!(c[6 * i] > 0.f) || !(c[6 * i + 2] > 0.f) || !(c[6 * i + 5] > 0.f))) why = 3;
  if (!why && (!(o[i] >= 0.f) || !(o[i] <= 1.f))) why = 4;
  if (why) atomicMin(bad, (unsigned long long)i * 8ull + (unsigned long long)why);
}
}  // namespace

as_status as_load_scene(as_ctx* ctx, int64_t N, const float* mean, const float* chol,
                        const float* opacity, const float* color, int32_t flags) {
  if (ctx) ++ctx->gen;  // state (or buffers) may change: no stale graph replay
  if (!ctx) return AS_E_ARG;
  if (N < 0 || (N > 0 && (!mean || !chol || !opacity || !color))) {
    set_err(ctx, "as_load_scene: bad arguments");
    return AS_E_ARG;
  }
  if (N > (int64_t)INT32_MAX / 16) {
    set_err(ctx, "as_load_scene: N too large");
    return AS_E_ARG;
  }
  try {
    cudaSetDevice(ctx->device);
    cudaStream_t st = ctx->stream;
    const bool dev = flags & AS_PTR_DEVICE;
    // copy into staging buffers, validate there, and only then replace the scene (no partial
    // writes on error)
    DevBuf &sm = ctx->st_mean, &sc = ctx->st_chol, &so = ctx->st_opacity, &scol = ctx->st_color;
    const size_t n1 = (size_t)std::max<int64_t>(N, 1);
    ensure(ctx, sm, 12 * n1);
    ensure(ctx, sc, 24 * n1);
    ensure(ctx, so, 4 * n1);
    ensure(ctx, scol, 12 * n1);
    ensure(ctx, ctx->counters, sizeof(unsigned long long) * C_NCOUNTERS);
    const cudaMemcpyKind kind = dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    unsigned long long bad = ~0ull;
    try {
      if (N > 0) {
        CK(cudaMemcpyAsync(sm.p, mean, 12 * N, kind, st));
        CK(cudaMemcpyAsync(sc.p, chol, 24 * N, kind, st));
        CK(cudaMemcpyAsync(so.p, opacity, 4 * N, kind, st));
        CK(cudaMemcpyAsync(scol.p, color, 12 * N, kind, st));
        unsigned long long* dbad = P<unsigned long long>(ctx->counters) + C_SCENE;
        CK(cudaMemcpyAsync(dbad, &bad, sizeof bad, cudaMemcpyHostToDevice, st));
        k_validate<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(N, P<float>(sm), P<float>(sc),
                                                                 P<float>(so), P<float>(scol), dbad);
        LAUNCHED(ctx, 1);
        CK(cudaMemcpyAsync(&bad, dbad, sizeof bad, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
      }
    } catch (const Err&) {
      throw;
    }
    if (bad != ~0ull) {
      const long long gi = (long long)(bad >> 3);
      switch ((int)(bad & 7)) {
        case 1: set_err(ctx, "Gaussian %lld: mean/colour not finite or colour outside [0,1]", gi); break;
        case 2: set_err(ctx, "Gaussian %lld: chol not finite", gi); break;
        case 3: set_err(ctx, "Gaussian %lld: chol diagonal must be > 0", gi); break;
        default: set_err(ctx, "Gaussian %lld: opacity outside [0,1]", gi); break;
      }
      return AS_E_SCENE;
    }
    std::swap(ctx->mean, sm);  // the previous scene becomes the next staging area
    std::swap(ctx->chol, sc);
    std::swap(ctx->opacity, so);
    std::swap(ctx->color, scol);
    ctx->N = N;
    ctx->n_groups = 0;
    ctx->has_group = ctx->has_col = ctx->has_op = ctx->has_priv = false;
    return AS_OK;
  } catch (const Err& e) {
    return e.st;
  }
}

as_status as_set_camera(as_ctx* ctx, const as_camera* cam) {
  if (ctx) ++ctx->gen;  // state (or buffers) may change: no stale graph replay
  if (!ctx) return AS_E_ARG;
  if (!cam || cam->W <= 0 || cam->H <= 0 || cam->W > 65536 || cam->H > 65536 ||
      !(cam->fx > 0) || !(cam->fy > 0) || !std::isfinite(cam->cx) || !std::isfinite(cam->cy)) {
    set_err(ctx, "as_set_camera: invalid camera");
    return AS_E_ARG;
  }
  for (int k = 0; k < 3; ++k)
    if (!std::isfinite(cam->euler[k]) || !std::isfinite(cam->t[k])) {
      set_err(ctx, "as_set_camera: non-finite pose");
      return AS_E_ARG;
    }
  ctx->cam = *cam;
  ctx->have_cam = true;
  return AS_OK;
}

as_status as_set_subboxes(as_ctx* ctx, int32_t n, const double* bounds) {
  if (ctx) ++ctx->gen;  // state (or buffers) may change: no stale graph replay
  if (!ctx) return AS_E_ARG;
  if (n < 0 || (n > 0 && !bounds) || n > 1000000) {
    set_err(ctx, "as_set_subboxes: bad arguments (n = %d)", n);
    return AS_E_ARG;
  }
  std::vector<double> saved;
  saved.swap(ctx->sub_host);
  ctx->sub_host.assign(bounds, bounds + (size_t)n * 18);
  if (ctx->have_box) {
    BoxInfo bi;
    const as_status st = make_box(ctx, bi);
    if (st != AS_OK) {
      ctx->sub_host.swap(saved);
      return st;
    }
  }
  try {
    if (n > 0) {
      cudaSetDevice(ctx->device);
      ensure(ctx, ctx->subs, sizeof(double) * 18 * (size_t)n);
      CK(cudaMemcpyAsync(ctx->subs.p, ctx->sub_host.data(), sizeof(double) * 18 * (size_t)n,
                         cudaMemcpyHostToDevice, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
    }
  } catch (const Err& e) {
    ctx->sub_host.swap(saved);
    return e.st;
  }
  return AS_OK;
}

as_status as_set_blend(as_ctx* ctx, int32_t mode) {
  if (ctx) ++ctx->gen;  // state (or buffers) may change: no stale graph replay
  if (!ctx) return AS_E_ARG;
  if (mode != 0 && mode != 1) {
    set_err(ctx, "as_set_blend: mode 0 (interval) or 1 (interval + linear)");
    return AS_E_ARG;
  }
  ctx->blend_mode = mode;
  return AS_OK;
}

as_status as_set_chunk_target(as_ctx* ctx, int32_t target) {
  if (ctx) ++ctx->gen;  // state (or buffers) may change: no stale graph replay
  if (!ctx) return AS_E_ARG;
  if (target < 0) {
    set_err(ctx, "as_set_chunk_target: target >= 0 (0 = automatic), got %d", target);
    return AS_E_ARG;
  }
  ctx->chunk_target = target;
  return AS_OK;
}

as_status as_set_inverse_mode(as_ctx* ctx, int32_t backward) {
  if (ctx) ++ctx->gen;  // state (or buffers) may change: no stale graph replay
  if (!ctx) return AS_E_ARG;
  if (backward != 0 && backward != 1) {
    set_err(ctx, "as_set_inverse_mode: 0 (forward) or 1 (back-substitution)");
    return AS_E_ARG;
  }
  if (backward && ctx->k_tol > 0 && ctx->k_max > 32) {
    set_err(ctx, "as_set_inverse_mode: back-substitution supports k_max <= 32");
    return AS_E_ARG;
  }
  ctx->inv_backward = backward;
  return AS_OK;
}

as_status as_set_matrixinv(as_ctx* ctx, double k_tol, int32_t k_max) {
  if (ctx) ++ctx->gen;  // state (or buffers) may change: no stale graph replay
  if (!ctx) return AS_E_ARG;
  if (!std::isfinite(k_tol) || (k_tol > 0 && (k_max < 8 || k_max > 64))) {
    set_err(ctx, "as_set_matrixinv: k_tol finite, k_max in [8, 64] (got %g, %d)", k_tol, k_max);
    return AS_E_ARG;
  }
  if (ctx->inv_backward && k_tol > 0 && k_max > 32) {
    set_err(ctx, "as_set_matrixinv: back-substitution mode supports k_max <= 32");
    return AS_E_ARG;
  }
  ctx->k_tol = k_tol > 0 ? k_tol : 0.0;
  ctx->k_max = k_tol > 0 ? k_max : 8;
  return AS_OK;
}

as_status as_subbox_fails(as_ctx* ctx, int32_t n, int64_t* fails) {
  if (ctx) ++ctx->gen;  // state (or buffers) may change: no stale graph replay
  as_status st = check_ready(ctx);
  if (st != AS_OK) return st;
  BoxInfo bi;
  if ((st = make_box(ctx, bi)) != AS_OK) return st;
  if (!fails || n < bi.n_sub) {
    set_err(ctx, "as_subbox_fails: need room for %d counts", bi.n_sub);
    return AS_E_ARG;
  }
  try {
    cudaSetDevice(ctx->device);
    prepare_common(ctx, bi, geometry(ctx, 16));
    unsigned long long* ctr = P<unsigned long long>(ctx->counters);
    for (int s = 0; s < bi.n_sub; ++s) {
      CK(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long) * C_NCOUNTERS, ctx->stream));
      run_setup(ctx, bi, s);
      unsigned long long h = 0;
      CK(cudaMemcpyAsync(&h, ctr + C_FAIL, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      fails[s] = (int64_t)h;
    }
    CK(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long) * C_NCOUNTERS, ctx->stream));
    return AS_OK;
  } catch (const Err& e) {
    return e.st;
  }
}

as_status as_set_pose_box(as_ctx* ctx, const as_pose_box* box) {
  if (ctx) ++ctx->gen;  // state (or buffers) may change: no stale graph replay
  if (!ctx) return AS_E_ARG;
  if (!box) {
    set_err(ctx, "as_set_pose_box: NULL");
    return AS_E_ARG;
  }
  as_pose_box saved = ctx->box;
  const bool had = ctx->have_box;
  ctx->box = *box;
  std::vector<double> saved_sub;
  saved_sub.swap(ctx->sub_host);  // a new box clears an explicit partition
  BoxInfo bi;
  as_status st = make_box(ctx, bi);
  if (st != AS_OK) {
    ctx->box = saved;
    ctx->have_box = had;
    ctx->sub_host.swap(saved_sub);
    return st;
  }
  if (box->t_frame != 0 && box->t_frame != 1) {
    ctx->box = saved;
    ctx->sub_host.swap(saved_sub);
    set_err(ctx, "t_frame must be 0 or 1");
    return AS_E_ARG;
  }
  ctx->have_box = true;
  return AS_OK;
}

as_status as_set_scene_box(as_ctx* ctx, const as_scene_box* sb) {
  if (ctx) ++ctx->gen;  // state (or buffers) may change: no stale graph replay
  if (!ctx) return AS_E_ARG;
  if (ctx->N < 0) {
    set_err(ctx, "as_set_scene_box before as_load_scene");
    return AS_E_STATE;
  }
  if (!sb) {
    ctx->n_groups = 0;
    ctx->has_group = ctx->has_col = ctx->has_op = ctx->has_priv = false;
    return AS_OK;
  }
  const int64_t N = ctx->N;
  if (sb->n_groups < 0 || sb->n_groups > 3 || (sb->n_groups > 0 && (!sb->group_of || !sb->dir ||
                                                                     !sb->shift_lo || !sb->shift_hi))) {
    set_err(ctx, "as_set_scene_box: bad group arguments");
    return AS_E_ARG;
  }
  if ((sb->col_lo == nullptr) != (sb->col_hi == nullptr) ||
      (sb->op_lo == nullptr) != (sb->op_hi == nullptr) ||
      (sb->priv_lo == nullptr) != (sb->priv_hi == nullptr)) {
    set_err(ctx, "as_set_scene_box: lo/hi must both be given");
    return AS_E_ARG;
  }
  for (int g = 0; g < sb->n_groups; ++g) {
    if (!(sb->shift_hi[g] >= sb->shift_lo[g]) || !std::isfinite(sb->shift_lo[g]) ||
        !std::isfinite(sb->shift_hi[g]) || sb->parts[g] < 1) {
      set_err(ctx, "as_set_scene_box: bad shift range of group %d", g);
      return AS_E_ARG;
    }
  }
  try {
    cudaSetDevice(ctx->device);
    ctx->n_groups = sb->n_groups;
    for (int g = 0; g < 3; ++g) {
      ctx->gparts[g] = g < sb->n_groups ? sb->parts[g] : 1;
      ctx->shift_lo[g] = g < sb->n_groups ? sb->shift_lo[g] : 0.0;
      ctx->shift_hi[g] = g < sb->n_groups ? sb->shift_hi[g] : 0.0;
      for (int k = 0; k < 3; ++k) ctx->dir[g][k] = g < sb->n_groups ? sb->dir[3 * g + k] : 0.0;
    }
    ctx->has_group = sb->n_groups > 0;
    if (ctx->has_group) {
      ensure(ctx, ctx->group_of, 4 * std::max<int64_t>(N, 1));
      CK(cudaMemcpyAsync(ctx->group_of.p, sb->group_of, 4 * N, cudaMemcpyHostToDevice, ctx->stream));
    }
    ctx->has_col = sb->col_lo != nullptr;
    if (ctx->has_col) {
      ensure(ctx, ctx->col_lo, 12 * std::max<int64_t>(N, 1));
      ensure(ctx, ctx->col_hi, 12 * std::max<int64_t>(N, 1));
      CK(cudaMemcpyAsync(ctx->col_lo.p, sb->col_lo, 12 * N, cudaMemcpyHostToDevice, ctx->stream));
      CK(cudaMemcpyAsync(ctx->col_hi.p, sb->col_hi, 12 * N, cudaMemcpyHostToDevice, ctx->stream));
    }
    ctx->has_op = sb->op_lo != nullptr;
    if (ctx->has_op) {
      ensure(ctx, ctx->op_lo, 4 * std::max<int64_t>(N, 1));
      ensure(ctx, ctx->op_hi, 4 * std::max<int64_t>(N, 1));
      CK(cudaMemcpyAsync(ctx->op_lo.p, sb->op_lo, 4 * N, cudaMemcpyHostToDevice, ctx->stream));
      CK(cudaMemcpyAsync(ctx->op_hi.p, sb->op_hi, 4 * N, cudaMemcpyHostToDevice, ctx->stream));
    }
    ctx->has_priv = sb->priv_lo != nullptr;
    if (ctx->has_priv) {
      ensure(ctx, ctx->priv_lo, 12 * std::max<int64_t>(N, 1));
      ensure(ctx, ctx->priv_hi, 12 * std::max<int64_t>(N, 1));
      CK(cudaMemcpyAsync(ctx->priv_lo.p, sb->priv_lo, 12 * N, cudaMemcpyHostToDevice, ctx->stream));
      CK(cudaMemcpyAsync(ctx->priv_hi.p, sb->priv_hi, 12 * N, cudaMemcpyHostToDevice, ctx->stream));
    }
    // validated on the device (copies first, one check): a bad entry clears the scene box
    unsigned long long bad = ~0ull;
    ensure(ctx, ctx->counters, sizeof(unsigned long long) * C_NCOUNTERS);
    unsigned long long* dbad = P<unsigned long long>(ctx->counters) + C_SCENE;
    CK(cudaMemcpyAsync(dbad, &bad, sizeof bad, cudaMemcpyHostToDevice, ctx->stream));
    if (N > 0) {
      k_validate_sbox<<<(unsigned)((N + 255) / 256), 256, 0, ctx->stream>>>(
          N, ctx->has_group ? P<int32_t>(ctx->group_of) : nullptr, sb->n_groups,
          ctx->has_col ? P<float>(ctx->col_lo) : nullptr, ctx->has_col ? P<float>(ctx->col_hi) : nullptr,
          ctx->has_op ? P<float>(ctx->op_lo) : nullptr, ctx->has_op ? P<float>(ctx->op_hi) : nullptr,
          ctx->has_priv ? P<float>(ctx->priv_lo) : nullptr,
          ctx->has_priv ? P<float>(ctx->priv_hi) : nullptr, dbad);
      LAUNCHED(ctx, 1);
    }
    CK(cudaMemcpyAsync(&bad, dbad, sizeof bad, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));  // host sources may be freed after return
    if (bad != ~0ull) {
      ctx->n_groups = 0;
      ctx->has_group = ctx->has_col = ctx->has_op = ctx->has_priv = false;
      const long long gi = (long long)(bad >> 3);
      switch ((int)(bad & 7)) {
        case 1:
          set_err(ctx, "group_of[%lld] out of range", gi);
          return AS_E_ARG;
        case 2:
          set_err(ctx, "colour interval of Gaussian %lld invalid", gi);
          return AS_E_SCENE;
        case 3:
          set_err(ctx, "opacity interval of Gaussian %lld invalid", gi);
          return AS_E_SCENE;
        default:
          set_err(ctx, "private mean interval of Gaussian %lld invalid", gi);
          return AS_E_SCENE;
      }
    }
    return AS_OK;
  } catch (const Err& e) {
    return e.st;
  }
}

namespace {
// NEXT-1: after the interval render of one sub-box into (lo, hi), intersect the exception-free
// tiles with the linear-relation blend
void linear_pass(as_ctx* ctx, const BoxInfo& bi, const Geometry& G, int batch, float* lo,
                 float* hi) {
  // NEXT-1 (O20): every non-empty tile, longest lists first (blocks are scheduled roughly in
  // launch order, so the long tiles do not form the tail); certain positions through the
  // linear fold, uncertain ones through the interval terms of the pass in render_subbox
  cudaStream_t st = ctx->stream;
  ensure(ctx, ctx->lin_tiles, sizeof(int32_t) * G.ntiles);
  std::vector<int64_t> tb(G.ntiles), te(G.ntiles);
  CK(cudaMemcpyAsync(tb.data(), ctx->tbegin.p, sizeof(int64_t) * G.ntiles, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(te.data(), ctx->tend.p, sizeof(int64_t) * G.ntiles, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  ++ctx->host_syncs;
  std::vector<int32_t> list;
  for (int t = 0; t < G.ntiles; ++t)
    if (te[t] > tb[t]) list.push_back(t);
  if (list.empty()) return;
  std::stable_sort(list.begin(), list.end(),
                   [&](int32_t a, int32_t b) { return te[a] - tb[a] > te[b] - tb[b]; });
  CK(cudaMemcpyAsync(ctx->lin_tiles.p, list.data(), sizeof(int32_t) * list.size(),
                     cudaMemcpyHostToDevice, st));
  TileArgs ta{};
  ta.hot = ctx->hot.p;
  ta.vals = P<int32_t>(ctx->vals2);
  ta.tbegin = P<int64_t>(ctx->tbegin);
  ta.tend = P<int64_t>(ctx->tend);
  ta.pm = ctx->last_unc ? P<int4>(ctx->pflag) : nullptr;
  ta.ts = G.ts;
  ta.ntx = G.ntx;
  ta.W = ctx->cam.W;
  ta.H = ctx->cam.H;
  ta.bs = std::min(batch, 16);
  ta.ntau = (float)((double)ctx->N * TAU);
  launch_tile_lin(bi.n_vars, ta, P<int32_t>(ctx->lin_tiles), (int)list.size(), lo, hi,
                  ctx->last_unc ? P<float>(ctx->unc_lo) : nullptr,
                  ctx->last_unc ? P<float>(ctx->unc_hi) : nullptr, st);
  LAUNCHED(ctx, 1);
  CK(cudaStreamSynchronize(st));  // list (host) must outlive the copy above
}

__global__ void k_fill2(float* a, float va, float* b, float vb, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    a[i] = va;
    b[i] = vb;
  }
}
as_status render_range(as_ctx* ctx, int32_t tile, int32_t batch, int32_t s0, int32_t s1,
                       float* lo, float* hi, int32_t flags, as_stats* stats);
}  // namespace

as_status as_render_bounds(as_ctx* ctx, int32_t tile, int32_t batch, float* lo, float* hi,
                           int32_t flags, as_stats* stats) {
  return render_range(ctx, tile, batch, 0, -1, lo, hi, flags, stats);
}

as_status as_render_subboxes(as_ctx* ctx, int32_t tile, int32_t batch, int32_t sub_begin,
                             int32_t sub_end, float* lo, float* hi, int32_t flags,
                             as_stats* stats) {
  if (sub_begin < 0 || sub_end < sub_begin) {
    if (ctx) set_err(ctx, "as_render_subboxes: bad range [%d, %d)", sub_begin, sub_end);
    return AS_E_ARG;
  }
  return render_range(ctx, tile, batch, sub_begin, sub_end, lo, hi, flags, stats);
}

as_status as_subbox_count(as_ctx* ctx, int32_t* n_sub) {
  as_status st = check_ready(ctx);
  if (st != AS_OK) return st;
  if (!n_sub) return AS_E_ARG;
  BoxInfo bi;
  if ((st = make_box(ctx, bi)) != AS_OK) return st;
  *n_sub = bi.n_sub;
  return AS_OK;
}

namespace {
// union over the sub-boxes [b, e) on this GPU into device images dlo / dhi (identities for an
// empty range); the single-GPU body of a render
void render_local(as_ctx* ctx, const BoxInfo& bi, const Geometry& G, int32_t batch, int b, int e,
                  float* dlo, float* dhi, bool timed) {
  cudaStream_t s = ctx->stream;
  const size_t img = (size_t)ctx->cam.W * ctx->cam.H * 3;
  k_seq<<<(G.ntiles + 255) / 256, 256, 0, s>>>(P<int32_t>(ctx->tlist), G.ntiles);
  LAUNCHED(ctx, 1);
  if (b >= e) {  // empty union: the identities of min / max (step 22)
    k_fill2<<<(unsigned)((img + 255) / 256), 256, 0, s>>>(dlo, 1.f, dhi, 0.f, (int64_t)img);
    LAUNCHED(ctx, 1);
  }
  const bool linear = ctx->blend_mode == 1;
  if (linear) {
    ensure(ctx, ctx->tmp_lo, sizeof(float) * img);
    ensure(ctx, ctx->tmp_hi, sizeof(float) * img);
  }
  for (int sb = b; sb < e; ++sb) {
    cudaEvent_t* ev = timed ? sub_events(ctx, sb - b) : nullptr;
    if (!linear) {
      render_subbox(ctx, bi, sb, true, G, batch, nullptr, 0, P<int32_t>(ctx->tlist), G.ntiles,
                    nullptr, dlo, dhi, sb == b, ev);
    } else {  // intersection per sub-box, then the union (step 22)
      float* tl = P<float>(ctx->tmp_lo);
      float* th = P<float>(ctx->tmp_hi);
      render_subbox(ctx, bi, sb, true, G, batch, nullptr, 0, P<int32_t>(ctx->tlist), G.ntiles,
                    nullptr, tl, th, true, ev);
      linear_pass(ctx, bi, G, batch, tl, th);
      launch_union(tl, th, dlo, dhi, (int64_t)img, sb == b, s);
      LAUNCHED(ctx, 1);
    }
  }
}

as_status render_range(as_ctx* ctx, int32_t tile, int32_t batch, int32_t s0, int32_t s1,
                       float* lo, float* hi, int32_t flags, as_stats* stats) {
  as_status st = check_ready(ctx);
  if (st != AS_OK) return st;
  if (!lo || !hi) {
    set_err(ctx, "as_render_bounds: NULL output");
    return AS_E_ARG;
  }
  BoxInfo bi;
  if ((st = make_box(ctx, bi)) != AS_OK) return st;
  if (s1 < 0) s1 = bi.n_sub;
  if (s1 > bi.n_sub) {
    set_err(ctx, "sub-box range [%d, %d) beyond the %d sub-boxes", s0, s1, bi.n_sub);
    return AS_E_ARG;
  }
  if ((st = check_tile_args(ctx, tile, batch, bi.n_vars)) != AS_OK) return st;
  if (ctx->blend_mode == 1 && bi.n_vars > NV_LINEAR_MAX) {
    set_err(ctx, "linear blend supports boxes with at most %d variables (got %d)", NV_LINEAR_MAX,
            bi.n_vars);
    return AS_E_ARG;
  }
  if ((flags & AS_ASYNC) && !(flags & AS_PTR_DEVICE)) {
    set_err(ctx, "AS_ASYNC requires device outputs");
    return AS_E_ARG;
  }
  // multi-GPU axis: 0 none, 1 image tiles (all-gather), 2 sub-boxes (all-reduce min / max)
  const int world = ctx->world, rank = ctx->rank;
  int axis = 0;
  if (ctx->comm && (world > 1 || ctx->shard_axis != 0))
    axis = ctx->shard_axis != 0 ? ctx->shard_axis : (s1 - s0 >= world ? 2 : 1);
  if (axis == 1 && ctx->blend_mode != 0) {
    set_err(ctx, "tile sharding: the linear blend is available on the sub-box axis only");
    return AS_E_ARG;
  }
  try {
    cudaSetDevice(ctx->device);
    cudaStream_t s = ctx->stream;
    const Geometry G = geometry(ctx, tile);
    // Sync-free when this shape's sizes are remembered (single GPU, interval blend, a call
    // that synchronises at its end anyway): no host read inside the pipeline, one check of
    // the sizes at the end; if they outgrew the remembered ones the render runs again,
    // probing (reading each size back), and the new sizes are remembered.
    as_ctx::Sizes& sp = ctx->spec;
    const bool can_spec = axis == 0 && ctx->blend_mode == 0 && !(flags & AS_ASYNC);
    bool spec = can_spec && sp.valid && sp.ts == tile && sp.bs == batch && sp.nv == bi.n_vars;
    bool resized = false;
    const size_t img = (size_t)ctx->cam.W * ctx->cam.H * 3;
    float *dlo = lo, *dhi = hi;
    int n_done = 0, n_timed = 0;
    if (!(flags & AS_PTR_DEVICE)) {
      ensure(ctx, ctx->img_lo, sizeof(float) * img);
      ensure(ctx, ctx->img_hi, sizeof(float) * img);
      dlo = P<float>(ctx->img_lo);
      dhi = P<float>(ctx->img_hi);
    }
    bool replayed = false;
    unsigned long long hfinal[C_NCOUNTERS];
    bool have_h = false;
    for (;;) {
      have_h = false;
      ctx->spec_on = spec;
      ctx->cur_spec = &ctx->spec;
      ctx->probe = as_ctx::Sizes{};
      ctx->host_syncs = 0;
      ctx->launches = 0;
      ctx->last_gather_ms = 0.0;
      ctx->last_n_owned = G.ntiles;
      // the whole pipeline, enqueued on the stream (captured into a graph when sync-free)
      auto enqueue = [&]() {
        if (stats) CK(timing_record(ctx->ev[0], s));
        prepare_common(ctx, bi, G);
        n_done = s1 > s0 ? s1 - s0 : 0;  // sub-boxes rendered by this rank
        n_timed = n_done;
        if (axis == 2) {
          // rank r: contiguous balanced range of [s0, s1); an empty range gives the identities
          const int ns = s1 - s0, q = ns / world, rm = ns % world;
          const int b = s0 + rank * q + std::min(rank, rm), e = b + q + (rank < rm ? 1 : 0);
          n_done = n_timed = e - b;
          render_local(ctx, bi, G, batch, b, e, dlo, dhi, stats != nullptr);
          CK(timing_record(ctx->ev[3], s));
          NCK(nccl_api().allReduce(dlo, dlo, img, ncclFloat, ncclMin, (ncclComm_t)ctx->comm, s));
          NCK(nccl_api().allReduce(dhi, dhi, img, ncclFloat, ncclMax, (ncclComm_t)ctx->comm, s));
          CK(timing_record(ctx->ev[4], s));
        } else if (axis == 1) {
          // every rank: setup + per-tile costs, the same device LPT owner map, its own tiles
          // into a compact tile-major buffer, ONE all-gather, the untile on the device
          const int per = (G.ntiles + world - 1) / world;
          const int cap = per + std::max(1, per / 4);
          // the owner map of an unchanged state is kept (no cost pass on repeated renders;
          // every rank takes the same decision: same calls, same state)
          const bool reuse_lpt = ctx->lpt_valid && ctx->lpt_gen == ctx->gen &&
                                 ctx->lpt_tile == tile && ctx->lpt_world == world &&
                                 ctx->lpt_cap == cap && ctx->lpt_s0 == s0 && ctx->lpt_s1 == s1;
          if (!reuse_lpt) {
            tile_costs_dev(ctx, bi, G, s0, s1);
            device_lpt(ctx, G, world, cap);
            ctx->lpt_valid = true;
            ctx->lpt_gen = ctx->gen;
            ctx->lpt_tile = tile;
            ctx->lpt_world = world;
            ctx->lpt_cap = cap;
            ctx->lpt_s0 = s0;
            ctx->lpt_s1 = s1;
          }
          ensure(ctx, ctx->untile_map, sizeof(int32_t) * G.ntiles);
          k_slot_maps<<<(G.ntiles + 255) / 256, 256, 0, s>>>(
              P<int32_t>(ctx->owner), P<int32_t>(ctx->tslot_all), G.ntiles, rank, cap,
              P<int32_t>(ctx->tslot), P<int32_t>(ctx->untile_map));
          LAUNCHED(ctx, 1);
          const size_t tm = (size_t)cap * tile * tile * 3;
          ensure(ctx, ctx->gsend, sizeof(float) * 2 * tm);
          ensure(ctx, ctx->grecv, sizeof(float) * 2 * tm * world);
          float* slo = P<float>(ctx->gsend);
          float* shi = slo + tm;
          // tiles a rank owns but that no Gaussian touches are never written by the tile kernel
          k_fill2<<<(unsigned)((2 * tm + 255) / 256), 256, 0, s>>>(slo, 0.f, shi, 0.f, (int64_t)tm);
          LAUNCHED(ctx, 1);
          ctx->last_out_tiles = cap;
          for (int sb = s0; sb < s1; ++sb)
            render_subbox(ctx, bi, sb, s1 - s0 != 1 || reuse_lpt, G, batch,
                          P<int32_t>(ctx->owner), rank,
                          P<int32_t>(ctx->tlist), 0, P<int32_t>(ctx->tslot), slo, shi, sb == s0,
                          stats ? sub_events(ctx, sb - s0) : nullptr);
          CK(timing_record(ctx->ev[3], s));
          NCK(nccl_api().allGather(slo, P<float>(ctx->grecv), 2 * tm, ncclFloat,
                                   (ncclComm_t)ctx->comm, s));
          const float* rl = P<float>(ctx->grecv);
          launch_untile(rl, rl + tm, P<int32_t>(ctx->untile_map), tile, G.ntx, G.nty, ctx->cam.W,
                        ctx->cam.H, dlo, dhi, s);
          LAUNCHED(ctx, 1);
          CK(timing_record(ctx->ev[4], s));
        } else {
          render_local(ctx, bi, G, batch, s0, s1, dlo, dhi, stats != nullptr);
        }
      };
      auto key = [&]() {
        as_ctx::GraphKey k;
        k.tile = tile;
        k.batch = batch;
        k.s0 = s0;
        k.s1 = s1;
        k.lo = dlo;
        k.hi = dhi;
        k.timed = stats != nullptr;
        k.exc = sp.exc;
        k.gen = ctx->gen;
        k.alloc_gen = ctx->alloc_gen;
        k.M = sp.M;
        k.nexc = sp.nexc;
        k.items = sp.items;
        k.R = sp.R;
        return k;
      };
      bool done = false;
      replayed = false;
      if (spec && ctx->use_graphs) {
        const as_ctx::GraphKey k = key();
        auto launch_graph = [&]() {  // the graph between two events of the caller's stream
          CK(cudaEventRecord(ctx->gev_in, s));
          CK(cudaStreamWaitEvent(ctx->gstream, ctx->gev_in, 0));
          CK(cudaGraphLaunch(ctx->gexec, ctx->gstream));
          CK(cudaEventRecord(ctx->gev_out, ctx->gstream));
          CK(cudaStreamWaitEvent(s, ctx->gev_out, 0));
        };
        if (ctx->gexec && ctx->gkey == k) {  // replay
          n_done = n_timed = s1 > s0 ? s1 - s0 : 0;
          nvtxRangePushA("absplat.graph_replay");
          launch_graph();
          nvtxRangePop();
          ctx->launches = ctx->glaunches;
          done = replayed = true;
        } else if (ctx->gready_ok && ctx->gready == k) {
          // the last render of this key ran sync-free and allocated nothing: capture it
          if (ctx->gexec) {
            cudaGraphExecDestroy(ctx->gexec);
            ctx->gexec = nullptr;
          }
          if (!ctx->gstream) {
            CK(cudaStreamCreateWithFlags(&ctx->gstream, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&ctx->gev_in, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ctx->gev_out, cudaEventDisableTiming));
          }
          cudaGraph_t g = nullptr;
          const cudaStream_t user = s;
          s = ctx->stream = ctx->gstream;  // everything below enqueues on the capture stream
          try {
            CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
            try {
              enqueue();
            } catch (...) {
              cudaStreamEndCapture(s, &g);
              if (g) cudaGraphDestroy(g);
              throw;
            }
            CK(cudaStreamEndCapture(s, &g));
          } catch (...) {
            s = ctx->stream = user;
            throw;
          }
          s = ctx->stream = user;
          if (ctx->alloc_gen == k.alloc_gen &&
              cudaGraphInstantiate(&ctx->gexec, g, 0ull) != cudaSuccess) {
            (void)cudaGetLastError();
            ctx->gexec = nullptr;
          }
          cudaGraphDestroy(g);
          ctx->gready_ok = false;
          if (ctx->gexec) {
            ctx->gkey = k;
            ctx->glaunches = ctx->launches;
            launch_graph();
            done = replayed = true;
          } else {  // not capturable this time: plain sync-free launches
            ctx->launches = 0;
            enqueue();
            done = true;
          }
        }
      }
      if (!done) {
        const uint64_t ag = ctx->alloc_gen;
        enqueue();
        ctx->gready_ok = spec && ctx->alloc_gen == ag;
        if (ctx->gready_ok) ctx->gready = key();
      }
      if (!(flags & AS_PTR_DEVICE)) {  // queued before the check: one synchronisation for both
        CK(cudaMemcpyAsync(lo, dlo, sizeof(float) * img, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(hi, dhi, sizeof(float) * img, cudaMemcpyDeviceToHost, s));
      }
      if (stats) CK(cudaEventRecord(ctx->ev[6], s));
      if (spec) {  // the one check of a sync-free render
        unsigned long long* h = hfinal;
        read_counters(ctx, h);
        have_h = true;
        const bool fits = h[C_OVF] == 0 && (int64_t)h[C_MMAX] <= sp.M &&
                          (h[C_UNC] == 0 || sp.exc) && (int64_t)h[C_NEXCMAX] <= sp.nexc &&
                          (int64_t)h[C_WMAXALL] < sp.R && (int64_t)h[C_ITEMSMAX] <= sp.items;
        if (!fits) {
          sp.valid = false;
          spec = false;
          resized = true;
          ++ctx->spec_redo;
          continue;
        }
        if (2 * (int64_t)h[C_MMAX] < sp.M) sp.valid = false;  // far smaller: re-probe next time
      } else if (can_spec && n_done > 0) {  // (an empty range measures nothing)
        sp = ctx->probe;
        sp.valid = true;
        sp.ts = tile;
        sp.bs = batch;
        sp.nv = bi.n_vars;
      }
      break;
    }
    ctx->spec_on = false;
    if (stats) {
      CK(cudaEventSynchronize(ctx->ev[6]));
      float tot = 0;
      CK(cudaEventElapsedTime(&tot, ctx->ev[0], ctx->ev[6]));
      if (axis != 0) {
        float g = 0;
        CK(cudaEventElapsedTime(&g, ctx->ev[3], ctx->ev[4]));
        ctx->last_gather_ms = g;
      }
      if (axis == 1) {
        int32_t no = 0;
        CK(cudaMemcpy(&no, P<int32_t>(ctx->nown) + rank, sizeof no, cudaMemcpyDeviceToHost));
        ctx->last_n_owned = no;
      }
      PhaseTimes pt;
      collect_phases(ctx, n_timed, &pt);
      BoxInfo br = bi;
      br.n_sub = n_done;
      fill_stats(ctx, br, G, ctx->last_n_owned, pt, tot, stats, have_h ? hfinal : nullptr);
      stats->resized = resized ? 1 : 0;
      stats->graph_replay = replayed ? 1 : 0;
    }
    if (!(flags & AS_ASYNC)) CK(cudaStreamSynchronize(s));
    return AS_OK;
  } catch (const Err& e) {
    ctx->spec_on = false;
    return e.st;
  }
}
}  // namespace

as_status as_lpt_assign(int32_t n_tiles, const int64_t* costs, int32_t world, int32_t cap,
                        int32_t* owner) {
  if (n_tiles < 0 || world < 1 || !owner || (n_tiles > 0 && !costs)) return AS_E_ARG;
  if ((int64_t)cap * world < n_tiles) return AS_E_ARG;
  lpt(n_tiles, costs, world, cap, owner);
  return AS_OK;
}

as_status as_tile_owners(as_ctx* ctx, int32_t tile, int32_t world, int32_t max_tiles,
                         int32_t* owner, int64_t* costs) {
  if (ctx) ++ctx->gen;  // state (or buffers) may change: no stale graph replay
  as_status st = check_ready(ctx);
  if (st != AS_OK) return st;
  BoxInfo bi;
  if ((st = make_box(ctx, bi)) != AS_OK) return st;
  if ((st = check_tile_args(ctx, tile, 1, bi.n_vars)) != AS_OK) return st;
  if (world < 1 || !owner) {
    set_err(ctx, "as_tile_owners: bad arguments");
    return AS_E_ARG;
  }
  try {
    cudaSetDevice(ctx->device);
    const Geometry G = geometry(ctx, tile);
    if ((int64_t)max_tiles * world < G.ntiles) {
      set_err(ctx, "max_tiles * world < n_tiles");
      return AS_E_ARG;
    }
    prepare_common(ctx, bi, G);
    tile_costs_dev(ctx, bi, G, 0, bi.n_sub);
    device_lpt(ctx, G, world, max_tiles);
    ctx->lpt_valid = false;
    CK(cudaMemcpyAsync(owner, ctx->owner.p, sizeof(int32_t) * G.ntiles, cudaMemcpyDeviceToHost,
                       ctx->stream));
    std::vector<unsigned long long> c(G.ntiles);
    CK(cudaMemcpyAsync(c.data(), ctx->tcost.p, sizeof(unsigned long long) * G.ntiles,
                       cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (costs) std::copy(c.begin(), c.end(), costs);
    return AS_OK;
  } catch (const Err& e) {
    return e.st;
  }
}

as_status as_render_shard(as_ctx* ctx, int32_t tile, int32_t batch, int32_t rank, int32_t world,
                          float* lo_tm, float* hi_tm, int32_t max_tiles, int32_t* owned,
                          int32_t* n_owned, int32_t flags, as_stats* stats) {
  // (no generation bump: a shard render changes no state a render graph depends on; any
  // reallocation moves alloc_gen)
  as_status st = check_ready(ctx);
  if (st != AS_OK) return st;
  BoxInfo bi;
  if ((st = make_box(ctx, bi)) != AS_OK) return st;
  if ((st = check_tile_args(ctx, tile, batch, bi.n_vars)) != AS_OK) return st;
  if (world < 1 || rank < 0 || rank >= world || !lo_tm || !hi_tm || !owned || !n_owned) {
    set_err(ctx, "as_render_shard: bad arguments");
    return AS_E_ARG;
  }
  if (ctx->blend_mode != 0) {
    set_err(ctx, "as_render_shard: the linear blend is available for full-image renders only");
    return AS_E_ARG;
  }
  try {
    cudaSetDevice(ctx->device);
    cudaStream_t s = ctx->stream;
    const Geometry G = geometry(ctx, tile);
    if ((int64_t)max_tiles * world < G.ntiles) {
      set_err(ctx, "max_tiles * world < n_tiles");
      return AS_E_ARG;
    }
    // sync-free after the first render of this (shape, world, rank): sizes remembered and
    // checked once, with the owner map, at the end (as in render_range)
    const uint64_t skey = ((uint64_t)tile << 52) ^ ((uint64_t)batch << 40) ^
                          ((uint64_t)bi.n_vars << 32) ^ ((uint64_t)world << 16) ^ (uint64_t)rank;
    as_ctx::Sizes& sp = ctx->shard_spec[skey];
    bool spec = sp.valid && !(flags & AS_ASYNC);
    bool resized = false;
    std::vector<int32_t> own(G.ntiles);
    unsigned long long hc[C_NCOUNTERS];
    float *dlo = lo_tm, *dhi = hi_tm;
    for (;;) {
    ctx->launches = 0;
    ctx->host_syncs = 0;
    ctx->spec_on = spec;
    ctx->cur_spec = &sp;
    ctx->probe = as_ctx::Sizes{};
    if (stats) CK(cudaEventRecord(ctx->ev[0], s));
    prepare_common(ctx, bi, G);
    // ---- owner map (identical on every rank): LPT over per-tile pair counts, on the device;
    // unchanged state: the map of the previous call (no cost pass)
    const bool reuse_lpt = world > 1 && ctx->lpt_valid && ctx->lpt_gen == ctx->gen &&
                           ctx->lpt_tile == tile && ctx->lpt_world == world &&
                           ctx->lpt_cap == max_tiles && ctx->lpt_s0 == 0 &&
                           ctx->lpt_s1 == bi.n_sub;
    if (world > 1 && !reuse_lpt) {
      tile_costs_dev(ctx, bi, G, 0, bi.n_sub);
      device_lpt(ctx, G, world, max_tiles);
      ctx->lpt_valid = true;
      ctx->lpt_gen = ctx->gen;
      ctx->lpt_tile = tile;
      ctx->lpt_world = world;
      ctx->lpt_cap = max_tiles;
      ctx->lpt_s0 = 0;
      ctx->lpt_s1 = bi.n_sub;
    } else if (world == 1) {
      ctx->lpt_valid = false;  // the owner map is overwritten
      ensure(ctx, ctx->tslot_all, sizeof(int32_t) * G.ntiles);
      CK(cudaMemsetAsync(ctx->owner.p, 0, sizeof(int32_t) * G.ntiles, s));
      k_seq<<<(G.ntiles + 255) / 256, 256, 0, s>>>(P<int32_t>(ctx->tslot_all), G.ntiles);
      LAUNCHED(ctx, 1);
    }
    k_slot_maps<<<(G.ntiles + 255) / 256, 256, 0, s>>>(P<int32_t>(ctx->owner),
                                                        P<int32_t>(ctx->tslot_all), G.ntiles,
                                                        rank, max_tiles, P<int32_t>(ctx->tslot),
                                                        nullptr);
    LAUNCHED(ctx, 1);
    const size_t tmax = (size_t)max_tiles * tile * tile * 3;
    if (!(flags & AS_PTR_DEVICE)) {
      ensure(ctx, ctx->img_lo, sizeof(float) * tmax);
      ensure(ctx, ctx->img_hi, sizeof(float) * tmax);
      dlo = P<float>(ctx->img_lo);
      dhi = P<float>(ctx->img_hi);
    }
    ctx->last_out_tiles = max_tiles;
    for (int sb = 0; sb < bi.n_sub; ++sb) {
      const bool need_setup = !(world > 1 && bi.n_sub == 1 && !reuse_lpt);  // cost pass left it
      render_subbox(ctx, bi, sb, need_setup, G, batch, P<int32_t>(ctx->owner), rank,
                    P<int32_t>(ctx->tlist), 0, P<int32_t>(ctx->tslot), dlo, dhi, sb == 0,
                    stats ? sub_events(ctx, sb) : nullptr);
    }
    // the owned tile ids (host output) and the counters come back in one synchronisation
    CK(cudaMemcpyAsync(own.data(), ctx->owner.p, sizeof(int32_t) * G.ntiles,
                       cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hc, ctx->counters.p, sizeof hc, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (spec) {
      const bool fits = hc[C_OVF] == 0 && (int64_t)hc[C_MMAX] <= sp.M &&
                        (hc[C_UNC] == 0 || sp.exc) && (int64_t)hc[C_NEXCMAX] <= sp.nexc &&
                        (int64_t)hc[C_WMAXALL] < sp.R && (int64_t)hc[C_ITEMSMAX] <= sp.items;
      if (!fits) {
        sp.valid = false;
        spec = false;
        resized = true;
        ++ctx->spec_redo;
        continue;
      }
      if (2 * (int64_t)hc[C_MMAX] < sp.M) sp.valid = false;
    } else {
      sp = ctx->probe;
      sp.valid = true;
    }
    break;
    }
    ctx->spec_on = false;
    int nm = 0;
    for (int t = 0; t < G.ntiles; ++t)
      if (own[t] == rank) {
        if (nm >= max_tiles) {
          set_err(ctx, "as_render_shard: more than max_tiles tiles assigned");
          return AS_E_ARG;
        }
        owned[nm++] = t;
      }
    *n_owned = nm;
    if (!(flags & AS_PTR_DEVICE) && nm > 0) {
      CK(cudaMemcpyAsync(lo_tm, dlo, sizeof(float) * nm * tile * tile * 3, cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(hi_tm, dhi, sizeof(float) * nm * tile * tile * 3, cudaMemcpyDeviceToHost, s));
    }
    if (stats) {
      CK(cudaEventRecord(ctx->ev[6], s));
      CK(cudaEventSynchronize(ctx->ev[6]));
      float tot = 0;
      CK(cudaEventElapsedTime(&tot, ctx->ev[0], ctx->ev[6]));
      PhaseTimes pt;
      collect_phases(ctx, bi.n_sub, &pt);
      fill_stats(ctx, bi, G, nm, pt, tot, stats, hc);
      stats->resized = resized ? 1 : 0;
    }
    if (!(flags & AS_ASYNC)) CK(cudaStreamSynchronize(s));
    return AS_OK;
  } catch (const Err& e) {
    ctx->spec_on = false;
    return e.st;
  }
}

as_status as_untile(as_ctx* ctx, int32_t W, int32_t H, int32_t tile, int32_t world,
                    int32_t max_tiles, const int32_t* owned, const int32_t* n_owned,
                    const float* lo_tm, const float* hi_tm, float* lo, float* hi, int32_t flags) {
  if (ctx) ++ctx->gen;  // state (or buffers) may change: no stale graph replay
  const bool dev = flags & AS_PTR_DEVICE;
  if (dev && !ctx) return AS_E_ARG;
  if ((tile != 8 && tile != 16 && tile != 32) || W <= 0 || H <= 0 || world < 1 ||
      max_tiles < 1 || !owned || !n_owned || !lo_tm || !hi_tm || !lo || !hi) {
    if (ctx) set_err(ctx, "as_untile: bad arguments");
    return AS_E_ARG;
  }
  Geometry G;
  G.ts = tile;
  G.ntx = (W + tile - 1) / tile;
  G.nty = (H + tile - 1) / tile;
  G.ntiles = G.ntx * G.nty;
  std::vector<int32_t> slot_of(G.ntiles, -1);
  for (int r = 0; r < world; ++r) {
    if (n_owned[r] < 0 || n_owned[r] > max_tiles) {
      if (ctx) set_err(ctx, "as_untile: n_owned[%d] out of range", r);
      return AS_E_ARG;
    }
    for (int k = 0; k < n_owned[r]; ++k) {
      const int t = owned[(size_t)r * max_tiles + k];
      if (t < 0 || t >= G.ntiles || slot_of[t] != -1) {
        if (ctx) set_err(ctx, "as_untile: tile %d invalid or owned twice", t);
        return AS_E_ARG;
      }
      slot_of[t] = r * max_tiles + k;
    }
  }
  for (int t = 0; t < G.ntiles; ++t)
    if (slot_of[t] < 0) {
      if (ctx) set_err(ctx, "as_untile: tile %d not owned by any rank", t);
      return AS_E_ARG;
    }
  const int ts = tile;
  if (!dev) {  // host assembly (plain index arithmetic)
    for (int py = 0; py < H; ++py)
      for (int px = 0; px < W; ++px) {
        const int t = (py / ts) * G.ntx + px / ts;
        const size_t src = ((size_t)slot_of[t] * ts * ts + (size_t)(py % ts) * ts + (px % ts)) * 3;
        const size_t dst = ((size_t)py * W + px) * 3;
        for (int c = 0; c < 3; ++c) {
          lo[dst + c] = lo_tm[src + c];
          hi[dst + c] = hi_tm[src + c];
        }
      }
    return AS_OK;
  }
  try {
    cudaSetDevice(ctx->device);
    ensure(ctx, ctx->untile_map, sizeof(int32_t) * G.ntiles);
    CK(cudaMemcpyAsync(ctx->untile_map.p, slot_of.data(), sizeof(int32_t) * G.ntiles,
                       cudaMemcpyHostToDevice, ctx->stream));
    launch_untile(lo_tm, hi_tm, P<int32_t>(ctx->untile_map), ts, G.ntx, G.nty, W, H, lo, hi,
                  ctx->stream);
    LAUNCHED(ctx, 1);
    if (!(flags & AS_ASYNC)) CK(cudaStreamSynchronize(ctx->stream));
    return AS_OK;
  } catch (const Err& e) {
    return e.st;
  }
}

as_status as_render_concrete(as_ctx* ctx, const double* xi, float* img, int32_t flags) {
  if (ctx) ++ctx->gen;  // state (or buffers) may change: no stale graph replay
  as_status st = check_ready(ctx);
  if (st != AS_OK) return st;
  BoxInfo bi;
  if ((st = make_box(ctx, bi)) != AS_OK) return st;
  if (!img || (bi.n_vars > 0 && !xi)) {
    set_err(ctx, "as_render_concrete: bad arguments");
    return AS_E_ARG;
  }
  if (ctx->has_priv) {
    set_err(ctx, "as_render_concrete: private mean offsets set (load the offset means instead)");
    return AS_E_ARG;
  }
  double param[9];
  for (int a = 0; a < 9; ++a) param[a] = bi.bp.lo[a];
  for (int i = 0; i < bi.n_vars; ++i) {
    if (!(xi[i] >= -1.0 && xi[i] <= 1.0)) {
      set_err(ctx, "xi[%d] outside [-1,1]", i);
      return AS_E_ARG;
    }
    param[bi.axis[i]] = bi.c[i] + bi.r[i] * xi[i];
  }
  try {
    cudaSetDevice(ctx->device);
    cudaStream_t s = ctx->stream;
    ConcreteArgs a{};
    double e[3], Rc[9], Mf[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    for (int k = 0; k < 3; ++k) e[k] = ctx->cam.euler[k] + param[3 + k];
    rot_c2w_host(e, Rc);
    if (ctx->box.t_frame == 1) rot_c2w_host(ctx->cam.euler, Mf);
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) a.R[3 * r + c] = Rc[3 * c + r];
    for (int k = 0; k < 3; ++k)
      a.t[k] = ctx->cam.t[k] + Mf[3 * k] * param[0] + Mf[3 * k + 1] * param[1] + Mf[3 * k + 2] * param[2];
    for (int g = 0; g < 3; ++g)
      for (int k = 0; k < 3; ++k) a.shift[g][k] = (g < ctx->n_groups) ? param[6 + g] * ctx->dir[g][k] : 0.0;
    const int64_t N = ctx->N;
    ensure(ctx, ctx->conc_g, sizeof(double) * 8 * std::max<int64_t>(N, 1));
    ensure(ctx, ctx->kkey, sizeof(unsigned long long) * (N + 1));
    ensure(ctx, ctx->kkey2, sizeof(unsigned long long) * (N + 1));
    ensure(ctx, ctx->kval, sizeof(int32_t) * (N + 1));
    ensure(ctx, ctx->order, sizeof(int32_t) * (N + 1));
    a.mean = P<float>(ctx->mean);
    a.chol = P<float>(ctx->chol);
    a.opacity = P<float>(ctx->opacity);
    a.color = P<float>(ctx->color);
    a.group_of = ctx->has_group ? P<int32_t>(ctx->group_of) : nullptr;
    a.N = N;
    a.fx = ctx->cam.fx;
    a.fy = ctx->cam.fy;
    a.cx = ctx->cam.cx;
    a.cy = ctx->cam.cy;
    a.W = ctx->cam.W;
    a.H = ctx->cam.H;
    a.gdata = P<double>(ctx->conc_g);
    a.key = P<unsigned long long>(ctx->kkey);
    a.val = P<int32_t>(ctx->kval);
    launch_concrete_setup(a, s);
    LAUNCHED(ctx, 1);
    if (N > 0)
      cub_sort_keys64(ctx, P<unsigned long long>(ctx->kkey), P<unsigned long long>(ctx->kkey2),
                      P<int32_t>(ctx->kval), P<int32_t>(ctx->order), N, 64);
    a.order = P<int32_t>(ctx->order);
    const size_t n = (size_t)a.W * a.H * 3;
    float* dimg = img;
    if (!(flags & AS_PTR_DEVICE)) {
      ensure(ctx, ctx->img_lo, sizeof(float) * n);
      dimg = P<float>(ctx->img_lo);
    }
    a.img = dimg;
    launch_concrete_render(a, s);
    LAUNCHED(ctx, 1);
    if (!(flags & AS_PTR_DEVICE))
      CK(cudaMemcpyAsync(img, dimg, sizeof(float) * n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return AS_OK;
  } catch (const Err& e) {
    return e.st;
  }
}

}  // extern "C"


