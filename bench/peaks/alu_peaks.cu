// ALU-pipe peak microbenchmark for the presorted-DP roofline.
// Measures warp-instruction throughput per SM per clock of the instructions the
// DP inner loop is made of: FMNMX (2-input), FMNMX3 (3-input min), FMUL, IMAD,
// VIMNMX (u32), and the fused "transition" pattern min(acc, max(a, x*y)).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o alu_peaks alu_peaks.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int ILP = 8;
constexpr int ITERS = 1 << 16;

__device__ unsigned long long g_clk[1024];

template <int OP>
__global__ void __launch_bounds__(256) kern(float* out, float seed, long long* cyc) {
  float a[ILP], b[ILP];
#pragma unroll
  for (int q = 0; q < ILP; ++q) { a[q] = seed + threadIdx.x * 0.001f + q; b[q] = seed * 0.5f + q; }
  long long t0 = clock64();
  unsigned long long g0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int q = 0; q < ILP; ++q) {
      if (OP == 0) {        // FMNMX (2-input max)
        asm volatile("max.f32 %0, %0, %1;" : "+f"(a[q]) : "f"(b[q]));
      } else if (OP == 1) { // FMNMX3 (3-input min)
        asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(a[q]) : "f"(b[q]), "f"(b[(q + 1) % ILP]));
      } else if (OP == 2) { // FMUL
        asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(a[q]) : "f"(b[q]));
      } else if (OP == 3) { // IMAD u32
        unsigned x = __float_as_uint(a[q]);
        asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(x) : "r"(__float_as_uint(b[q])));
        a[q] = __uint_as_float(x);
      } else if (OP == 4) { // VIMNMX u32
        unsigned x = __float_as_uint(a[q]);
        asm volatile("max.u32 %0, %0, %1;" : "+r"(x) : "r"(__float_as_uint(b[q])));
        a[q] = __uint_as_float(x);
      } else if (OP == 6) { // FMNMX + FMUL, independent, 1:1
        asm volatile("max.f32 %0, %0, %1;" : "+f"(a[q]) : "f"(b[q]));
        asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(b[(q + 4) % ILP]) : "f"(b[q]));
      } else if (OP == 7) { // FMNMX3 + FMUL 1:1
        asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(a[q]) : "f"(b[q]), "f"(b[(q + 1) % ILP]));
        asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(b[(q + 4) % ILP]) : "f"(b[(q + 2) % ILP]));
      } else if (OP == 8) { // cell with 2-input min: FMUL + FMNMX(max) + FMNMX(min)
        float c0, v0;
        asm volatile("mul.rn.f32 %0, %1, %2;" : "=f"(c0) : "f"(b[q]), "f"(a[(q + 1) % ILP]));
        asm volatile("max.f32 %0, %1, %2;" : "=f"(v0) : "f"(c0), "f"(b[(q + 4) % ILP]));
        asm volatile("min.f32 %0, %0, %1;" : "+f"(a[q]) : "f"(v0));
      } else if (OP == 9) { // argmin step: FSETP + FSEL + SEL
        float v = b[q];
        unsigned idx = (unsigned)q;
        asm volatile("{ .reg .pred p; setp.lt.f32 p, %2, %0; selp.f32 %0, %2, %0, p; selp.u32 %1, %3, %1, p; }"
                     : "+f"(a[q]), "+r"(idx) : "f"(v), "r"((unsigned)it));
        b[q] = __uint_as_float(idx) * 0.f + b[q];
      } else if (OP == 5) { // transition pair: 2x FMUL, 2x FMNMX, 1x FMNMX3
        float c0, c1, v0, v1;
        asm volatile("mul.rn.f32 %0, %1, %2;" : "=f"(c0) : "f"(b[q]), "f"(a[(q + 1) % ILP]));
        asm volatile("mul.rn.f32 %0, %1, %2;" : "=f"(c1) : "f"(b[(q + 2) % ILP]), "f"(a[(q + 3) % ILP]));
        asm volatile("max.f32 %0, %1, %2;" : "=f"(v0) : "f"(c0), "f"(b[(q + 4) % ILP]));
        asm volatile("max.f32 %0, %1, %2;" : "=f"(v1) : "f"(c1), "f"(b[(q + 5) % ILP]));
        asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(a[q]) : "f"(v0), "f"(v1));
      }
    }
  }
  long long t1 = clock64();
  unsigned long long g1; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  float s = 0.f;
#pragma unroll
  for (int q = 0; q < ILP; ++q) s += a[q];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) { cyc[2 * blockIdx.x] = t1 - t0; cyc[2 * blockIdx.x + 1] = (long long)(g1 - g0); }
}

template <int OP>
int run(const char* name, double instr_per_inner, int nsm) {
  const int blocks = nsm * 8, threads = 256;
  float* out; long long* cyc;
  CK(cudaMalloc(&out, sizeof(float) * blocks * threads));
  CK(cudaMalloc(&cyc, 2 * sizeof(long long) * blocks));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) kern<OP><<<blocks, threads>>>(out, 1.0f, cyc);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  kern<OP><<<blocks, threads>>>(out, 1.0f, cyc);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long* hc = new long long[2 * blocks];
  CK(cudaMemcpy(hc, cyc, 2 * sizeof(long long) * blocks, cudaMemcpyDeviceToHost));
  double sc = 0, sg = 0; for (int i = 0; i < blocks; ++i) { sc += hc[2 * i]; sg += hc[2 * i + 1]; }
  double clk_ghz = sc / sg;                     // SM cycles per ns, averaged over blocks
  double avgc = ms * 1e6 * clk_ghz;             // kernel span in SM cycles
  double warp_instr = (double)blocks * (threads / 32) * ITERS * ILP * instr_per_inner;
  double per_sm_per_clk = warp_instr / nsm / avgc;
  double lanes_per_sm_clk = per_sm_per_clk * 32;
  printf("{\"op\": \"%s\", \"ms\": %.4f, \"span_cycles\": %.0f, \"est_clk_ghz\": %.3f, "
         "\"warp_instr_per_sm_clk\": %.3f, \"lane_ops_per_sm_clk\": %.2f}\n",
         name, ms, avgc, clk_ghz, per_sm_per_clk, lanes_per_sm_clk);
  delete[] hc; cudaFree(out); cudaFree(cyc);
  return 0;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int nsm = p.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\"}\n", p.name, nsm, p.major, p.minor);
  run<0>("FMNMX", 1, nsm);
  run<1>("FMNMX3", 1, nsm);
  run<2>("FMUL", 1, nsm);
  run<3>("IMAD", 1, nsm);
  run<4>("VIMNMX.U32", 1, nsm);
  // transition pattern: 5 instructions for 2 transitions; report instr/sm/clk
  run<5>("PAIR(2xFMUL+2xFMNMX+FMNMX3)", 5, nsm);
  run<6>("FMNMX+FMUL", 2, nsm);
  run<7>("FMNMX3+FMUL", 2, nsm);
  run<8>("CELL(FMUL+FMNMX+FMNMX)", 3, nsm);
  run<9>("ARGMIN(FSETP+FSEL+SEL)", 3, nsm);
  return 0;
}
