// k_concrete.cu -- concrete GaussianSplat (Alg. 1 + BlendSort) at one pose, used
// by the soundness tests to sample renders inside the box on scenes too large for the CPU.
// fp64 throughout; depth cull d <= d_min (G8); ties in depth ordered by index (G6).
// Effective opacity uses the textbook form o exp(-1/2 (u-mu)^T Sigma_2D^-1 (u-mu)), equal to
// Alg. 1 l.9-10 by the d^4 identity (pinned in tests/test_oracle_pipeline.py).
#include "internal.cuh"

namespace absplat {

// gdata per Gaussian: mu_x, mu_y, A, B, C (Sigma^-1 = [[A,B],[B,C]]), opacity, depth, pad
__global__ void k_concrete_setup(ConcreteArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.N) return;
  const int grp = a.group_of ? a.group_of[i] : -1;
  double uw[3];
  for (int b = 0; b < 3; ++b)
    uw[b] = (double)a.mean[3 * i + b] + (grp >= 0 && grp < 3 ? a.shift[grp][b] : 0.0);
  double uc[3];
  for (int r = 0; r < 3; ++r)
    uc[r] = a.R[3 * r] * (uw[0] - a.t[0]) + a.R[3 * r + 1] * (uw[1] - a.t[1]) +
            a.R[3 * r + 2] * (uw[2] - a.t[2]);
  const float* ch = a.chol + 6 * i;
  const double Mw[9] = {ch[0], 0, 0, ch[1], ch[2], 0, ch[3], ch[4], ch[5]};
  double Mc[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      Mc[3 * r + c] = a.R[3 * r] * Mw[c] + a.R[3 * r + 1] * Mw[3 + c] + a.R[3 * r + 2] * Mw[6 + c];
  const double z = uc[2];
  double* g = a.gdata + 8 * i;
  if (!(z > DMIN)) {
    a.key[i] = ~0ull;
    a.val[i] = (int32_t)i;
    g[5] = 0.0;
    return;
  }
  const double J[6] = {a.fx / z, 0.0, -a.fx * uc[0] / (z * z), 0.0, a.fy / z, -a.fy * uc[1] / (z * z)};
  double JM[6];
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 3; ++c)
      JM[3 * r + c] = J[3 * r] * Mc[c] + J[3 * r + 1] * Mc[3 + c] + J[3 * r + 2] * Mc[6 + c];
  const double S00 = JM[0] * JM[0] + JM[1] * JM[1] + JM[2] * JM[2];
  const double S01 = JM[0] * JM[3] + JM[1] * JM[4] + JM[2] * JM[5];
  const double S11 = JM[3] * JM[3] + JM[4] * JM[4] + JM[5] * JM[5];
  const double det = S00 * S11 - S01 * S01;
  g[0] = a.fx * uc[0] / z + a.cx;
  g[1] = a.fy * uc[1] / z + a.cy;
  g[2] = S11 / det;
  g[3] = -S01 / det;
  g[4] = S00 / det;
  g[5] = (det > 0) ? (double)a.opacity[i] : 0.0;
  g[6] = z;
  g[7] = 0.0;
  a.key[i] = key_of_double(z);
  a.val[i] = (int32_t)i;
}

__global__ void __launch_bounds__(256) k_concrete_render(ConcreteArgs a) {
  __shared__ double sg[128][8];
  __shared__ float sc[128][3];
  const int64_t pix = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool inside = pix < (int64_t)a.W * a.H;
  const double ux = inside ? (double)(pix % a.W) + 0.5 : 0.0;
  const double uy = inside ? (double)(pix / a.W) + 0.5 : 0.0;
  double T = 1.0, pc[3] = {0.0, 0.0, 0.0};
  for (int64_t b0 = 0; b0 < a.N; b0 += 128) {
    const int nb = (int)((a.N - b0) < 128 ? (a.N - b0) : 128);
    __syncthreads();
    for (int j = threadIdx.x; j < nb; j += blockDim.x) {
      const int32_t g = a.order[b0 + j];
      for (int k = 0; k < 8; ++k) sg[j][k] = a.gdata[8 * (int64_t)g + k];
      for (int c = 0; c < 3; ++c) sc[j][c] = a.color[3 * (int64_t)g + c];
    }
    __syncthreads();
    for (int j = 0; j < nb; ++j) {
      const double o = sg[j][5];
      if (o == 0.0) continue;
      const double dx = ux - sg[j][0], dy = uy - sg[j][1];
      const double q = sg[j][2] * dx * dx + 2.0 * sg[j][3] * dx * dy + sg[j][4] * dy * dy;
      const double al = o * exp(-0.5 * q);
      for (int c = 0; c < 3; ++c) pc[c] += T * al * (double)sc[j][c];
      T *= 1.0 - al;
    }
  }
  if (inside)
    for (int c = 0; c < 3; ++c) a.img[3 * pix + c] = (float)pc[c];
}

void launch_concrete_setup(const ConcreteArgs& a, cudaStream_t st) {
  if (a.N <= 0) return;
  k_concrete_setup<<<(unsigned)((a.N + 127) / 128), 128, 0, st>>>(a);
}
void launch_concrete_render(const ConcreteArgs& a, cudaStream_t st) {
  const int64_t n = (int64_t)a.W * a.H;
  k_concrete_render<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(a);
}

}  // namespace absplat
