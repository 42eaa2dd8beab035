// pipebench.cu -- issue-rate microbenchmark of the instruction classes the k_tile opacity
// block is made of (FFMA / FFMA2 / FADD / FADD2 with |.| modifiers / LDS broadcast / mixes),
// measured with clock64 per CTA: warp instructions per SMSP per cycle.  Informs DESIGN.md §6.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipebench tools/pipebench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITER = 256;
constexpr int CH = 8;

template <int OP>
__global__ void __launch_bounds__(1024, 1) kb(float* out, long long* cyc, float s0, float s1) {
  __shared__ float4 sm[64];
  if (threadIdx.x < 64) sm[threadIdx.x] = make_float4(s0 + threadIdx.x, s1, s0, s1 * threadIdx.x);
  __syncthreads();
  float a[CH];
  float2 p[CH];
  int ia[CH];
  double d[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    a[i] = s0 * (threadIdx.x + i);
    p[i] = make_float2(s0 * i, s1 * threadIdx.x);
    ia[i] = threadIdx.x * (i + 3);
    d[i] = (double)s0 * i;
  }
  const float2 b2 = make_float2(s1, s0), c2 = make_float2(s0 * 0.5f, s1 * 0.25f);
  const float b = s1, c = s0 * 0.5f;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      if constexpr (OP == 0) a[i] = fmaf(a[i], b, c);
      if constexpr (OP == 1) p[i] = __ffma2_rn(p[i], b2, c2);
      if constexpr (OP == 2) p[i] = __ffma2_rn(make_float2(a[i], a[i]), b2, p[i]);
      if constexpr (OP == 3) a[i] = a[i] + b;
      if constexpr (OP == 4) p[i] = __fadd2_rn(p[i], b2);
      if constexpr (OP == 5) {
        const float2 q = p[(i + 1) % CH];
        p[i] = __fadd2_rn(p[i], make_float2(-fabsf(q.x), fabsf(q.y)));
      }
      if constexpr (OP == 6) a[i] = fmaxf(a[i], b);
      if constexpr (OP == 7) {
        p[i] = __ffma2_rn(p[i], b2, c2);
        const float2 q = p[(i + 3) % CH];
        p[i] = __fadd2_rn(p[i], make_float2(-fabsf(q.x), fabsf(q.y)));
      }
      if constexpr (OP == 8) {
        p[i] = __ffma2_rn(p[i], b2, c2);
        a[i] = a[i] - fabsf(a[(i + 1) % CH]);
      }
      if constexpr (OP == 9) {
        p[i] = __ffma2_rn(p[i], b2, c2);
        ia[i] = (ia[i] ^ ia[(i + 1) % CH]) + 7;
      }
      if constexpr (OP == 10) {
        const float4 v = sm[(it + i) & 63];
        p[i] = __ffma2_rn(p[i], make_float2(v.x, v.y), make_float2(v.z, v.w));
      }
      if constexpr (OP == 11) d[i] = fma(d[i], (double)b, (double)c);
      if constexpr (OP == 12) a[i] = exp2f(a[i]);
      if constexpr (OP == 13) p[i] = __fmul2_rn(p[i], b2);
      if constexpr (OP == 14) {
        p[i] = __ffma2_rn(p[i], b2, c2);
        p[i] = __ffma2_rn(p[i], c2, b2);
        a[i] = a[i] - fabsf(a[(i + 1) % CH]);
      }
      if constexpr (OP == 15) {  // FFMA2 with a scalar-broadcast first operand
        p[i] = __ffma2_rn(make_float2(a[(i + 1) % CH], a[(i + 1) % CH]), p[i], b2);
      }
      if constexpr (OP == 16) d[i] = d[i] + (double)b;
      if constexpr (OP == 18) {  // LDS.32 broadcast + FFMA
        const float v = reinterpret_cast<const float*>(sm)[(it * 8 + i) & 255];
        a[i] = fmaf(a[i], v, c);
      }
      if constexpr (OP == 19) {  // LDS.64 broadcast + FFMA2
        const float2 v = reinterpret_cast<const float2*>(sm)[(it * 8 + i) & 127];
        p[i] = __ffma2_rn(p[i], v, c2);
      }
      if constexpr (OP == 20) {  // LDS.128 per-lane distinct (conflict-free) + FFMA2
        const float4 v = sm[(it + i + threadIdx.x) & 63];
        p[i] = __ffma2_rn(p[i], make_float2(v.x, v.y), make_float2(v.z, v.w));
      }
      if constexpr (OP == 21) {  // LDS.128 bcast feeding 4 FFMA2 (register reuse)
        const float4 v = sm[(it + i) & 63];
        p[i] = __ffma2_rn(p[i], make_float2(v.x, v.y), make_float2(v.z, v.w));
        p[(i + 1) % CH] = __ffma2_rn(p[(i + 1) % CH], make_float2(v.z, v.w), make_float2(v.x, v.y));
      }
      if constexpr (OP == 22) {  // FFMA2 with broadcast addend
        p[i] = __ffma2_rn(p[i], b2, make_float2(a[(i + 1) % CH], a[(i + 1) % CH]));
      }
      if constexpr (OP == 17) {  // FADD2 (m - r, m + r) from two broadcasts
        const float m = p[i].x, r = p[(i + 1) % CH].y;
        p[i] = __fadd2_rn(make_float2(m, m), make_float2(-r, r));
      }
    }
  }
  long long t1 = clock64();
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < CH; ++i) acc += a[i] + p[i].x + p[i].y + (float)ia[i] + (float)d[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int ipc, int nsm, float* out, long long* cyc) {
  // ipc = SASS instructions per (i) step of the inner loop (checked against cuobjdump)
  const int threads = 1024;
  kb<OP><<<nsm, threads>>>(out, cyc, 1.0001f, 0.9999f);
  kb<OP><<<nsm, threads>>>(out, cyc, 1.0001f, 0.9999f);
  cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, cyc, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < nsm; ++i) mx = h[i] > mx ? h[i] : mx;
  const double warp_instr_per_smsp = (double)ITER * CH * ipc * (threads / 32) / 4.0;
  printf("%-34s %6.3f warp-instr/SMSP/clk  (%.0f cycles)\n", name, warp_instr_per_smsp / mx, mx);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  long long* cyc;
  cudaMalloc(&out, nsm * 1024 * sizeof(float));
  cudaMalloc(&cyc, nsm * sizeof(long long));
  printf("SMs %d\n", nsm);
  run<0>("FFMA (3 reg)", 1, nsm, out, cyc);
  run<1>("FFMA2 (3 pairs)", 1, nsm, out, cyc);
  run<2>("FFMA2 (bcast op)", 1, nsm, out, cyc);
  run<15>("FFMA2 (bcast op, varying)", 1, nsm, out, cyc);
  run<3>("FADD", 1, nsm, out, cyc);
  run<4>("FADD2", 1, nsm, out, cyc);
  run<5>("FADD2 -|x|.NP", 1, nsm, out, cyc);
  run<17>("FADD2 (m-r, m+r)", 1, nsm, out, cyc);
  run<13>("FMUL2", 1, nsm, out, cyc);
  run<6>("FMNMX", 1, nsm, out, cyc);
  run<7>("FFMA2+FADD2 (2 instr)", 2, nsm, out, cyc);
  run<8>("FFMA2+FADD|x| (2 instr)", 2, nsm, out, cyc);
  run<14>("2 FFMA2+FADD|x| (3 instr)", 3, nsm, out, cyc);
  run<9>("FFMA2+LOP3/IADD (3 instr?)", 3, nsm, out, cyc);
  run<10>("LDS.128 bcast+FFMA2 (2 instr)", 2, nsm, out, cyc);
  run<18>("LDS.32 bcast+FFMA (2+ instr)", 2, nsm, out, cyc);
  run<19>("LDS.64 bcast+FFMA2 (2+ instr)", 2, nsm, out, cyc);
  run<20>("LDS.128 distinct+FFMA2 (2+ instr)", 2, nsm, out, cyc);
  run<21>("LDS.128 bcast+2 FFMA2 (3+ instr)", 3, nsm, out, cyc);
  run<22>("FFMA2 bcast addend", 1, nsm, out, cyc);
  run<11>("DFMA", 1, nsm, out, cyc);
  run<16>("DADD", 1, nsm, out, cyc);
  run<12>("MUFU.EX2 (+FMUL?)", 1, nsm, out, cyc);
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
