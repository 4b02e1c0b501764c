// Shared-memory lane mapping of the K2 sweep (F32 min-max, R = 8 columns x 8 column lanes x
// 4 split quarters).  LDS.128 is served per quarter-warp (8 lanes = 128 B): with the natural
// mapping lane = 8*kg + cl the 8 lanes of a phase read G at 32-byte strides (2-way conflict),
// and the dp / L broadcasts of the 4 quarters collide whenever the quarter length Q is a
// multiple of 32 splits.  MAP 1 puts two column quads x two split quarters in each phase
// (lane bits: b0,b1 -> cl 0..1, b2 -> kg bit 0, b3 -> cl bit 2, b4 -> kg bit 1); with Q/4 odd
// every phase then touches 8 distinct 16-byte bank groups.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../include \
//        -I../../paper_2603_28101_b200/csrc -o smem_map smem_map.cu
#include <cstdio>
#include "dp_batched.cuh"
using namespace hp;

constexpr int NN = 1024, REPS = 64;

template <int MAP>
__device__ __forceinline__ void lane_map(int lane, int& cl, int& kg) {
  if (MAP == 0) { cl = lane & 7; kg = lane >> 3; }
  else { cl = (lane & 3) | (((lane >> 3) & 1) << 2); kg = ((lane >> 2) & 1) | ((lane >> 4) << 1); }
}

template <int WARPS, int MAP, int ITERS>
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
  int cl, kg;
  lane_map<MAP>(lane, cl, kg);
  float tot = 0.f;
  long long t0 = clock64();
  for (int rep = 0; rep < REPS; ++rep) {
    const int cb = ((warp * 7 + rep * 3) % 7) * 64 + 536;   // no triangle: splits < 4*4*ITERS <= 536
    const int c = cb + 8 * cl;
    float acc[8];
    int arg[8], klo[8];
    for (int r = 0; r < 8; ++r) { acc[r] = INFINITY; klo[r] = 0; }
    sweep_slide<HEDDLE_F32, HEDDLE_MINMAX, false, false, 8>(sL, sdp, sG + kGPad + c, sG2 + kGPad + c,
                                                           4 * ITERS * kg, ITERS, acc, arg, klo);
    for (int r = 0; r < 8; ++r) tot += acc[r];
  }
  long long t1 = clock64();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = tot;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int WARPS, int CTAS, int MAP, int ITERS>
void run() {
  const int blocks = 148 * CTAS;
  float* sink; long long* cyc;
  cudaMalloc(&sink, sizeof(float) * blocks * 32 * WARPS);
  cudaMalloc(&cyc, sizeof(long long) * blocks);
  for (int w = 0; w < 3; ++w) kern<WARPS, MAP, ITERS><<<blocks, 32 * WARPS>>>(sink, cyc);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int w = 0; w < 10; ++w) kern<WARPS, MAP, ITERS><<<blocks, 32 * WARPS>>>(sink, cyc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  // executed (state, split) cells: per warp and rep, 64 columns x 4 quarters x 4*ITERS splits
  double cells = 10.0 * blocks * WARPS * REPS * 64.0 * 4 * 4 * ITERS;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double per_sm_clk = cells / (ms * 1e-3) / 148 / (clk * 1e3);
  printf("{\"map\": %d, \"q\": %d, \"warps\": %d, \"ctas_per_sm\": %d, \"ms\": %.3f, \"cells_per_sm_clk_at_max\": %.2f, "
         "\"frac_of_42.67\": %.3f, \"err\": \"%s\"}\n",
         MAP, ITERS, WARPS, CTAS, ms, per_sm_clk, per_sm_clk / 42.667, cudaGetErrorString(cudaGetLastError()));
  cudaFree(sink); cudaFree(cyc);
}

int main() {
  run<4, 7, 0, 32>();   // K2 today: 4-warp CTAs, 7 per SM, quarter length a multiple of 32 splits
  run<4, 7, 0, 33>();
  run<4, 7, 1, 32>();
  run<4, 7, 1, 33>();   // conflict-free
  run<8, 4, 0, 32>();
  run<8, 4, 1, 33>();
  return 0;
}
