// Issue-rate microbenchmark of the instruction classes in the selu/sigmoid epilogue on sm_100a:
// warp-instructions per cycle per SM for long streams of independent ops (8 chains per thread).
#include <cstdio>
#include <cstdint>
#define CH 8
#define ITERS 4096
template <int OP>
__global__ void k(float* out, int seed, long long* cyc) {
  float a[CH];
  uint32_t u[CH];
  uint64_t v[CH];
  for (int i = 0; i < CH; i++) { a[i] = threadIdx.x * 1e-3f + i + seed; u[i] = threadIdx.x + i * 77 + seed; v[i] = ((uint64_t)u[i] << 32) | u[i]; }
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) {
      if (OP == 0) asm volatile("fma.rn.f32 %0, %0, 0f3F800001, 0f3A000000;" : "+f"(a[i]));                 // FFMA imm
      if (OP == 1) { float b = __int_as_float(u[i]); asm volatile("fma.rn.f32 %0, %0, %1, %0;" : "+f"(a[i]) : "f"(b)); }  // FFMA reg
      if (OP == 2) asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(v[i]));                               // FFMA2
      if (OP == 3) asm volatile("mad.lo.u32 %0, %0, %1, 12345;" : "+r"(u[i]) : "r"(seed));                  // IMAD
      if (OP == 4) asm volatile("{.reg .u32 t; shl.b32 t, %0, 23; add.u32 %0, t, 12345;}" : "+r"(u[i]));   // LEA
      if (OP == 5) asm volatile("max.f32 %0, %0, 0fC2A00000;" : "+f"(a[i]));                                // FMNMX
      if (OP == 6) asm volatile("{.reg .pred p; setp.gt.f32 p, %0, 0f00000000; selp.f32 %0, %0, 0f3F800000, p;}" : "+f"(a[i]));  // FSETP+FSEL
      if (OP == 7) asm volatile("{.reg .b32 h; cvt.rn.f16x2.f32 h, %0, %0; mov.b32 %0, h;}" : "+f"(a[i]));  // F2FP
      if (OP == 8) asm volatile("add.rn.f32x2 %0, %0, %0;" : "+l"(v[i]));                                   // FADD2
      if (OP == 9) asm volatile("lop3.b32 %0, %0, %1, 0x55, 0x96;" : "+r"(u[i]) : "r"(seed));               // LOP3
      if (OP == 10) asm volatile("prmt.b32 %0, %0, %1, 0x3210;" : "+r"(u[i]) : "r"(seed + 1));              // PRMT
    }
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < CH; i++) s += a[i] + __uint_as_float(u[i]) + __uint_as_float((uint32_t)v[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int OP>
void run(const char* name, int warps) {
  float* o; long long* c; cudaMalloc(&o, 148 * 1024 * 4); cudaMallocManaged(&c, 8);
  k<OP><<<148, warps * 32>>>(o, 1, c); cudaDeviceSynchronize();
  k<OP><<<148, warps * 32>>>(o, 1, c); cudaDeviceSynchronize();
  const double instr = (double)ITERS * CH * warps;   // warp-instructions per SM
  printf("%-14s warps/SM %2d: %.3f warp-instr/clk/SM (%.3f per SMSP)\n", name, warps, instr / *c, instr / *c / 4);
  cudaFree(o); cudaFree(c);
}
int main() {
  for (int w : {16, 32}) {
    run<0>("FFMA imm", w); run<1>("FFMA reg", w); run<2>("FFMA2", w); run<8>("FADD2", w); run<3>("IMAD", w);
    run<4>("LEA", w); run<5>("FMNMX", w); run<6>("FSETP+FSEL", w); run<7>("F2FP", w); run<9>("LOP3", w); run<10>("PRMT", w);
  }
  return 0;
}
