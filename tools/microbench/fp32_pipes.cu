// Microbenchmark: per-SM per-clock throughput of FFMA, FFMA2, FADD2, FMNMX, FSETP
// on sm_100a.  Used once to fix the FP32-issue roofline denominator.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
typedef unsigned long long u64;

template <int KIND>
__global__ void __launch_bounds__(1024, 1) bench(float* out, long long* cyc, float seed) {
  float a[8]; u64 p[8];
  #pragma unroll
  for (int i = 0; i < 8; i++) { a[i] = seed + threadIdx.x * 1e-7f + i; float lo = a[i], hi = a[i] + 1.f;
    asm("mov.b64 %0, {%1,%2};" : "=l"(p[i]) : "f"(lo), "f"(hi)); }
  float b = 0.999f, c = 1e-3f; u64 pb, pc;
  asm("mov.b64 %0, {%1,%1};" : "=l"(pb) : "f"(b)); asm("mov.b64 %0, {%1,%1};" : "=l"(pc) : "f"(c));
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
    #pragma unroll
    for (int i = 0; i < 8; i++) {
      if (KIND == 0) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(b), "f"(c));
      if (KIND == 1) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(pb), "l"(pc));
      if (KIND == 2) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(pc));
      if (KIND == 3) asm volatile("min.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b));
      if (KIND == 4) asm volatile("{.reg .pred q; setp.le.f32 q, %0, %1; @q add.f32 %0, %0, %2;}" : "+f"(a[i]) : "f"(b), "f"(c));
      if (KIND == 5) { asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(pb), "l"(pc));
                       asm volatile("min.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b)); }
      if (KIND == 6) { asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(b), "f"(c));
                       asm volatile("min.f32 %0, %0, %1;" : "+f"(a[(i+4)&7]) : "f"(c)); }
      if (KIND == 7) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(c));
    }
  }
  long long t1 = clock64();
  float s = 0.f;
  #pragma unroll
  for (int i = 0; i < 8; i++) { float lo, hi; asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(p[i])); s += a[i] + lo + hi; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int KIND> void run(const char* name, double lane_ops_per_inner) {
  int nsm = 148; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* out; long long* cyc; cudaMalloc(&out, nsm * 1024 * 4); cudaMalloc(&cyc, nsm * 8);
  bench<KIND><<<nsm, 1024>>>(out, cyc, 1.f); cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); bench<KIND><<<nsm, 1024>>>(out, cyc, 1.f); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long h[1024]; cudaMemcpy(h, cyc, nsm * 8, cudaMemcpyDeviceToHost);
  double mx = 0; for (int i = 0; i < nsm; i++) mx = h[i] > mx ? h[i] : mx;
  double lane_ops = 1024.0 * ITERS * 8 * lane_ops_per_inner;  // per SM
  printf("%-28s lane-ops/clk/SM = %7.1f   (%.3f ms, implied clock %.0f MHz, %.2f Tlane-op/s chip)\n", name,
         lane_ops / mx, ms, mx / (ms * 1e3), lane_ops * nsm / (ms * 1e-3) / 1e12);
  cudaFree(out); cudaFree(cyc);
}

int main() {
  run<0>("FFMA", 1); run<1>("FFMA2 (2 lane-ops)", 2); run<2>("FADD2 (2 lane-ops)", 2);
  run<3>("FMNMX", 1); run<4>("FSETP+@P FADD (2 instr)", 2); run<5>("FFMA2+FMNMX (3 lane-ops)", 3);
  run<6>("FFMA+FMNMX (2 lane-ops)", 2); run<7>("FADD", 1);
  return 0;
}
