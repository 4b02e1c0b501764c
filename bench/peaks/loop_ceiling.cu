// Ceiling of the K2 inner sweep alone (no layers, no barriers, no LPT): every
// warp sweeps 1024 splits for its 32 columns REPS times over shared-memory rows.
// Reports cells/clk/SM against the 42.67 ALU-pipe bound (3 ALU cycles per cell).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../include \
//        -I../../paper_2603_28101_b200/csrc -o loop_ceiling loop_ceiling.cu
#include <cstdio>
#include "dp_batched.cuh"
using namespace hp;

constexpr int NN = 1024, REPS = 64;

// MODE 0: interleaved sweep (R=4, 8 column lanes x 4 split lanes, 2 G loads / step)
// MODE 1: sliding window, R columns per lane, CL column lanes, 32/CL split lanes each
//         owning a contiguous quarter of the split range
template <int WARPS, int MODE, int R, int CL>
__global__ void __launch_bounds__(32 * WARPS) kern(float* sink, long long* cyc) {
  __shared__ __align__(16) float sG[kGPad + NN + kGTail + 8];
  __shared__ __align__(16) float sG2[kGPad + NN + kGTail + 8];
  __shared__ __align__(16) float sL[NN + kLPad];
  __shared__ __align__(16) float sdp[NN + kLPad];
  for (int t = threadIdx.x; t < kGPad + NN + kGTail + 8; t += blockDim.x) {
    sG[t] = 1.0f + 0.001f * t;
    sG2[t] = 1.0f + 0.001f * (t + 1);
  }
  for (int t = threadIdx.x; t < NN + kLPad; t += blockDim.x) { sL[t] = 2000.f - t; sdp[t] = 0.5f * t; }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float tot = 0.f;
  long long t0 = clock64();
  for (int rep = 0; rep < REPS; ++rep) {
    const int cb = ((warp * 7 + rep * 3) % 7) * 64 + 528;  // column block in [528, 912]: no triangle
    if (MODE == 0) {
      const int cl = lane & 7, kg = lane >> 3;
      const int c = cb + 4 * cl;
      float acc[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
      int arg[4], klo[4] = {0, 0, 0, 0};
      sweep<HEDDLE_F32, HEDDLE_MINMAX, false, false>(sL, sdp, sG + kGPad + c, 0, 512, kg, acc, arg, klo);
      for (int r = 0; r < 4; ++r) tot += acc[r];
    } else {
      constexpr int KG = 32 / CL;
      const int cl = lane % CL, kg = lane / CL;
      const int c = cb + R * cl;
      float acc[R];
      int arg[R], klo[R];
      for (int r = 0; r < R; ++r) { acc[r] = INFINITY; klo[r] = 0; }
      const int iters = 512 / 4 / KG;
      if (MODE == 1)
        sweep_slide<HEDDLE_F32, HEDDLE_MINMAX, false, false, R>(sL, sdp, sG + kGPad + c, sG2 + kGPad + c,
                                                               4 * iters * kg, iters, acc, arg, klo);
      else   // generic path (no FMUL2), for comparison
        sweep_slide<HEDDLE_F32, HEDDLE_MINMAX, false, true, R>(sL, sdp, sG + kGPad + c, sG2 + kGPad + c,
                                                              4 * iters * kg, iters, acc, arg, klo);
      for (int r = 0; r < R; ++r) tot += acc[r];
    }
  }
  long long t1 = clock64();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = tot;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int WARPS, int CTAS, int MODE, int R, int CL>
void run() {
  const int blocks = 148 * CTAS;
  float* sink; long long* cyc;
  cudaMalloc(&sink, sizeof(float) * blocks * 32 * WARPS);
  cudaMalloc(&cyc, sizeof(long long) * blocks);
  for (int w = 0; w < 3; ++w) kern<WARPS, MODE, R, CL><<<blocks, 32 * WARPS>>>(sink, cyc);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int w = 0; w < 10; ++w) kern<WARPS, MODE, R, CL><<<blocks, 32 * WARPS>>>(sink, cyc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double cells = 10.0 * blocks * WARPS * REPS * 32.0 * (MODE == 0 ? 4 : R) * 512 / (MODE == 0 ? 4 : 32 / CL) ;   // executed (state, split) pairs
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double per_sm_clk = cells / (ms * 1e-3) / 148 / (clk * 1e3);
  printf("{\"mode\": %d, \"R\": %d, \"CL\": %d, \"warps\": %d, \"ctas_per_sm\": %d, \"ms\": %.3f, \"cells_per_sm_clk_at_max\": %.2f, \"frac_of_42.67\": %.3f, \"err\": \"%s\"}\n",
         MODE, R, CL, WARPS, CTAS, ms, per_sm_clk, per_sm_clk / 42.667, cudaGetErrorString(cudaGetLastError()));
  cudaFree(sink); cudaFree(cyc);
}

int main() {
  run<8, 4, 0, 4, 8>();
  run<8, 4, 2, 4, 8>();
  run<8, 4, 1, 4, 8>(); run<16, 2, 1, 4, 8>(); run<8, 6, 1, 4, 8>();
  run<8, 4, 1, 8, 4>(); run<16, 2, 1, 8, 4>();
  run<8, 4, 1, 8, 8>(); run<16, 2, 1, 8, 8>();
  run<8, 4, 1, 4, 32>();
  run<8, 3, 1, 12, 4>(); run<16, 2, 1, 16, 2>();
  return 0;
}
