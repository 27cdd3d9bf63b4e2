// Which epilogue instruction classes share an issue pipe on sm_100a: each thread runs 8 independent
// chains, even chains one op class, odd chains another; 32 warps per SM.  Two classes on different
// pipes reach ~2x the single-class rate (0.5 warp-instr/clk/SMSP for the half-rate classes).
#include <cstdio>
#include <cstdint>
#define CH 8
#define ITERS 4096
template <int OP>
__device__ __forceinline__ void op(float& a, uint32_t& u, uint64_t& v, int seed) {
  if (OP == 0) asm volatile("fma.rn.f32 %0, %0, 0f3F800001, 0f3A000000;" : "+f"(a));
  if (OP == 2) asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(v));
  if (OP == 3) asm volatile("mad.lo.u32 %0, %0, %1, 12345;" : "+r"(u) : "r"(seed));
  if (OP == 4) asm volatile("{.reg .u32 t; shl.b32 t, %0, 23; add.u32 %0, t, 12345;}" : "+r"(u));
  if (OP == 5) asm volatile("max.f32 %0, %0, 0fC2A00000;" : "+f"(a));
  if (OP == 6) asm volatile("{.reg .pred p; setp.gt.f32 p, %0, 0f00000000; selp.f32 %0, %0, 0f3F800000, p;}" : "+f"(a));
  if (OP == 7) asm volatile("{.reg .b32 h; cvt.rn.f16x2.f32 h, %0, %0; mov.b32 %0, h;}" : "+f"(a));
  if (OP == 9) asm volatile("lop3.b32 %0, %0, %1, 0x55, 0x96;" : "+r"(u) : "r"(seed));
  if (OP == 11) asm volatile("mul.rn.f32 %0, %0, 0f3F800001;" : "+f"(a));
  if (OP == 12) asm volatile("add.rn.f32 %0, %0, 0f3F800001;" : "+f"(a));
  if (OP == 13) asm volatile("{.reg .pred p; setp.gt.f32 p, %0, 0f00000000; selp.u32 %1, 1, 0, p;}" : "+f"(a), "+r"(u));  // FSETP (+SEL on u)
  if (OP == 14) asm volatile("{.reg .pred p; setp.ne.u32 p, %1, 0; selp.f32 %0, %0, 0f3F800000, p;}" : "+f"(a) : "r"(seed));  // FSEL (p hoistable)
  if (OP == 15) asm volatile("slct.f32.f32 %0, %0, 0f3F800000, %0;" : "+f"(a));
}
template <int A, int B>
__global__ void k(float* out, int seed, long long* cyc) {
  float a[CH]; uint32_t u[CH]; uint64_t v[CH];
  for (int i = 0; i < CH; i++) { a[i] = threadIdx.x * 1e-3f + i + seed; u[i] = threadIdx.x + i * 77 + seed; v[i] = ((uint64_t)u[i] << 32) | u[i]; }
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) { if (i & 1) op<B>(a[i], u[i], v[i], seed); else op<A>(a[i], u[i], v[i], seed); }
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < CH; i++) s += a[i] + __uint_as_float(u[i]) + __uint_as_float((uint32_t)v[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int A, int B>
void run(const char* name) {
  float* o; long long* c; cudaMalloc(&o, 148 * 1024 * 4); cudaMallocManaged(&c, 8);
  const int warps = 32;
  k<A, B><<<148, warps * 32>>>(o, 1, c); cudaDeviceSynchronize();
  k<A, B><<<148, warps * 32>>>(o, 1, c); cudaDeviceSynchronize();
  const double n = (double)ITERS * CH * warps;
  printf("%-16s %.3f warp-instr/clk/SMSP\n", name, n / *c / 4);
  cudaFree(o); cudaFree(c);
}
int main() {
  run<13, 13>("FSETP/SEL*"); run<14, 14>("FSEL"); run<2, 14>("FFMA2+FSEL"); run<5, 14>("FMNMX+FSEL");
  run<3, 14>("IMAD+FSEL"); run<2, 13>("FFMA2+FSETP*"); run<5, 13>("FMNMX+FSETP*"); run<6, 5>("SETP/SEL+FMNMX");
  run<15, 15>("SLCT"); run<2, 15>("FFMA2+SLCT"); run<5, 15>("FMNMX+SLCT");
  return 0;
}
