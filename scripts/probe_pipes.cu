// Pipe-throughput probe (sm_100a): warp-instructions per clock per SM for
// FFMA, FFMA2, FADD2, FMNMX, MUFU.EX2, LEA/IADD, F2FP e2m1. Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe_pipes scripts/probe_pipes.cu && /tmp/probe_pipes
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

#define ITERS 4096
template <int OP>
__global__ void k(float* out, float a, float b, long long* clk) {
  float x[8];
  float2 y[8];
  uint32_t u[8];
  for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x * 0.001f + i; y[i] = make_float2(x[i], x[i] + 1); u[i] = threadIdx.x + i; }
  long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) x[i] = fmaf(x[i], a, b);                                              // FFMA
      if (OP == 1) y[i] = __ffma2_rn(y[i], make_float2(a, a), make_float2(b, b));         // FFMA2
      if (OP == 2) y[i] = __fadd2_rn(y[i], make_float2(b, b));                            // FADD2
      if (OP == 3) x[i] = fmaxf(x[(i + 1) & 7], -x[(i + 3) & 7]);                           // FMNMX
      if (OP == 4) { float r; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x[i])); x[i] = r; }  // MUFU
      if (OP == 5) u[i] = (u[i] << 23) + u[(i + 1) & 7];                                 // LEA-ish
      if (OP == 6) { uint16_t c; asm volatile("{.reg .b8 t; cvt.rn.satfinite.e2m1x2.f32 t, %1, %2; cvt.u16.u8 %0, t;}" : "=h"(c) : "f"(x[i]), "f"(a)); x[i] = __int_as_float(c | 0x3f800000u); }
      if (OP == 7) x[i] = fmaf(x[i], 1.0001f, 0.5f);                                     // FFMA imm
      if (OP == 8) { uint32_t r; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(r) : "r"(u[i])); u[i] = r; }  // 2x MUFU.EX2.F16
      if (OP == 9) { uint32_t r; asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(r) : "r"(u[i])); u[i] = r; }
      if (OP == 10) { float r; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x[i])); x[i] = r; }
      if (OP == 11) { uint16_t r; asm volatile("ex2.approx.f16 %0, %1;" : "=h"(r) : "h"((uint16_t)u[i])); u[i] = r; }
    }
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i] + y[i].x + y[i].y + u[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

template <int OP>
void run(const char* name, int warps) {
  float* out; long long* clk;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&clk, 8);
  k<OP><<<148, warps * 32>>>(out, 0.999f, 0.001f, clk);
  cudaDeviceSynchronize();
  long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
  double instr = double(ITERS) * 8 * warps;  // warp-instructions per SM
  printf("%-8s warps/SM %2d: %.3f warp-instr/clk/SM (%.2f clk per warp-instr per SMSP)\n", name, warps, instr / c, 4.0 * c / instr);
  cudaFree(out); cudaFree(clk);
}
int main() {
  for (int w : {8, 16, 32}) {
    run<0>("FFMA", w); run<7>("FFMAimm", w); run<1>("FFMA2", w); run<2>("FADD2", w); run<3>("FMNMX", w);
    run<4>("MUFUEX2", w); run<5>("SHL+ADD", w); run<6>("F2FPe2m1", w);
    run<8>("EX2f16x2", w); run<9>("EX2bf16x2", w); run<10>("RCP", w); run<11>("EX2f16", w);
  }
}
