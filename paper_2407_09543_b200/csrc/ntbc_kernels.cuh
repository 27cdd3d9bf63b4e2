// ntbc_kernels.cuh -- the sm_100a kernels of the NTBC inference hot path:
//   (0) dequant_grids_kernel ("prep"): Eq.2 grid dequantization + the fused kernel's shared-memory prefix image;
//   (1) fused_decode_kernel: multi-resolution bilinear sampling (rows a1-a2), endpoint and colour MLPs on
//       tcgen05 tensor cores with TMEM accumulators (a3-a4; contract H, SPLIT contract F or HALF contract P), endpoint
//       quantization, palettes, per-texel argmax, bit packing (a5-a8);
//   (2) pack_kernel_bt (default) / pack_kernel: rows a5-a8 standalone, fed fp32 MLP outputs (HBM-bound:
//       0.7 of the measured bandwidth for pack_kernel_bt);
//   (3) decode_bc_kernel: BC1/BC4 -> fp32 texels (row a9, verification).
// Plus mma_probe_kernel (pins the tensor-core summation, R10).
#pragma once
#include <cstdint>
#include <cuda_fp16.h>

#include "bc_device.cuh"
#include "sm100.cuh"

namespace ntbc {

// NTBC_CHECKS=1: the checked build (libntbc_checked.so, tests/test_gpu_checked.py) -- bounds checks of every
// computed shared-memory, TMEM and global index of the fused and pack kernels (a failed check traps the
// kernel) and shared memory poisoned with NaN patterns before use, so a read of an unwritten location
// corrupts the result the oracle comparison then rejects.  Stands in for compute-sanitizer, which this
// GPU pool refuses (profiles/r02c_compute_sanitizer_refused.log).
#ifndef NTBC_CHECKS
#define NTBC_CHECKS 0
#endif
#ifndef NTBC_PINGPONG
#define NTBC_PINGPONG 0    // 1: H = 64 models run 4 work groups of two colour tiles each, ping-ponged: each slot's
                           // MMAs overlap the other slot's epilogue (correct -- 28 parity tests incl. the
                           // full-size digests -- but slower, A/B r02j: 2.575 vs 2.201 ms: 16 warps per SM
                           // hide less latency than 32)
#endif
#ifndef NTBC_EPI_JOBS
#define NTBC_EPI_JOBS 1    // colour tile's index selection + packing: 0 = every thread its texel of every texture
                           // (round 1); 1 = (texture, block, half) jobs after a group barrier (A/B r02x: 2.174 vs
                           // 2.201 ms); 2 = warp-local jobs without the barrier (r02y: 2.250, slower)
#endif
#ifndef NTBC_TMEM_PF8
#define NTBC_TMEM_PF8 0    // 1: hidden epilogue loads TMEM in 8-column chunks with the next chunk in flight (same
                           // registers as the x16 loads; A/B r02l: 2.214 vs 2.197 ms, slower -- the TMEM load
                           // latency is not what the warps wait for)
#endif
#ifndef NTBC_WARP_POLL
#define NTBC_WARP_POLL 0   // 1: after a layer's MMAs every warp's lane 0 waits on the MMA mbarrier instead of one
                           // thread + a 128-thread barrier (A/B r02g: 2.242 vs 2.201 ms, slower)
#endif
#if NTBC_CHECKS
#define NTBC_CHECK(c)                                                                                  \
  do {                                                                                                 \
    if (!(c)) {                                                                                        \
      printf("NTBC_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c, blockIdx.x, \
             threadIdx.x);                                                                             \
      __trap();                                                                                        \
    }                                                                                                  \
  } while (0)
#else
#define NTBC_CHECK(c) do { } while (0)
#endif
__device__ __forceinline__ uint32_t dyn_smem_bytes() {
  uint32_t v;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(v));
  return v;
}

constexpr int kMaxTex = 8;
constexpr int kMaxLevels = 8;
constexpr int kUnitBlocks = 128;  // block positions per work unit = rows of one endpoint MMA tile
constexpr int kFmtBC1 = 1;

constexpr int kOnesBytes = 256;    // the bias MMA's ones tile: one 8-row group, read with SBO = 0
constexpr int kUnormBytes = 1536;  // 352 fp32 UNORM expansion values (q/31, q/63, q/255) + 32 BC4 weights

struct GridLevel {
  uint32_t offset;  // byte offset of the level's dequantized fp32 [res][res][2] in the weight slot
  int res;
  float rm1;        // (float)(res - 1), the lattice scale of R1
  float s;          // Eq.2 scale (applied by dequant_grids_kernel)
  int z;            // Eq.2 zero point
};

struct NetLayout {
  uint32_t img_bytes;     // shared-memory operand image of this net (built by the fused kernel)
  uint32_t layer_off[4];  // byte offset of layer l's B operand [N_l][K_l] inside the net image
  uint32_t w_off[4], b_off[4];  // blob byte offsets of layer l's fp16 W [in][out] and bias [out]
  int kin[4], nout[4];    // layer l's input / output widths
  int n_out, n_out16;
};

struct FusedParams {
  const uint8_t* blob;    // device copy of the .ntbc blob (grid payloads are read from here)
  const uint8_t* prefix;  // the shared-memory prefix image built by dequant_grids_kernel (16-B aligned)
  GridLevel lv[2][kMaxLevels];
  int levels[2];
  NetLayout net[2];
  int W, H, BW, BH, row_begin, row_end, units_per_row, n_units;
  int n_tex;
  int fmt[kMaxTex], ep_off[kMaxTex], col_off[kMaxTex];
  uint64_t* out[kMaxTex];
  float* dump_ep;   // DUMP mode: [rows][BW][N_e]
  float* dump_col;  // DUMP mode: [rows*4][W][N_c]
  uint32_t a_bytes, pal_bytes;  // per-work-group shared memory regions
  uint32_t debug_flags;         // bit 1: grid-feature dump (ntbc_debug_features)
  unsigned long long* progress; // optional: per-chunk count of finished units (pipelined D2H, see ntbc_api.cu)
  int chunk_rows;               // block rows per progress chunk before tail_row0 ...
  int tail_row0, tail_rows;     // ... and per (smaller) chunk from tail_row0 on (local rows)
  int* next_unit;               // optional: dynamic unit counter (zeroed before the launch)
  int naive;                    // 1: the texel net outputs one weight per texture (naive approach)
  int pal_off[kMaxTex];         // per texture: float offset of its palette in a block's palette record
  int pal_stride;               // floats per block palette record (BC1 12, BC4 8 per texture)
  uint32_t tpal_off;            // byte offset of the colour tile's palettes inside a work group's region
  int vec16;                    // every out pointer 16-B aligned and BW even: a warp's two adjacent blocks'
                                // words leave as one 16-byte store (else one 8-byte store per block)
  int split;                    // contract F (host side; the kernel's SPLIT template parameter follows it)
  int half;                     // contract P: binary16 selu arithmetic (host side; template parameter HALF)
  int n_bc1, n_bc4;             // the texture indices of each format, in head order
  int tex_bc1[kMaxTex], tex_bc4[kMaxTex];
};

// One fused launch: CTAs [0, split) run model m[0], CTAs [split, grid) run m[1] (the conservative pair,
// P:377-381, in one persistent launch; each CTA holds only its own model's operand images).
struct FusedLaunch {
  FusedParams m[2];
  int split;
};

// ---------------------------------------------------------------- a2 at model upload: Eq.2 dequantization
// Every grid level's uint8 codes become fp32 values v = RN(s (q - z)) (Eq.2; R6: one binary32
// multiply of the exact integer q - z), stored [res][res][2] in the weight slot after the blob, once per
// upload.  The decode kernel then reads 8-byte (f0, f1) vertices and only interpolates.
struct DequantParams {
  uint8_t* slot;                    // weight slot: blob at 0, fp32 grids at dst_off
  int n_levels;                     // block-grid levels then texel-grid levels (<= 2 x kMaxLevels)
  unsigned long long src_off[2 * kMaxLevels], dst_off[2 * kMaxLevels];
  long long end[2 * kMaxLevels];    // cumulative count of 4-code groups, ceil(res^2 x 2 / 4), through level i
  float s[2 * kMaxLevels];
  int z[2 * kMaxLevels];
  unsigned long long zero_off;      // zero block (unused levels read it)
  int zero_n;
  // the fused kernel's shared-memory prefix, built here in global memory (img_off in the slot) and
  // bulk-copied by every CTA's prologue (TMA engine): both nets' tcgen05 B-operand images, the ones tile
  // of the bias MMA, the UNORM expansion tables and BC4 weights -- byte for byte the smem layout
  NetLayout net[2];
  int H;
  unsigned long long img_off;
};
// The shared-memory prefix of the fused kernel: per net and layer the tcgen05 B operand
// B[N_pad][K_in16 + 16] (row n = output n, K-major core-matrix layout, bias at k = K_in16, read against
// the ones tile), then the ones tile (one 8-row group, column 0 = 1.0), then the exact UNORM quotients
// q/31, q/63, q/255 (R12, R13) and the BC4 interpolation weights.  Written with generic stores by
// threads [tid0, tid0 + nthr) of whoever calls it (the prep kernel into global memory).
__device__ __forceinline__ uint32_t prefix_bytes(const NetLayout* net) {
  return net[0].img_bytes + net[1].img_bytes + kOnesBytes + kUnormBytes;
}
__device__ inline void build_smem_prefix(uint8_t* dst0, const uint8_t* blob, const NetLayout* net, int H, int tid0,
                                         int nthr) {
  uint8_t* img = dst0;
  for (int n = 0; n < 2; n++) {
    for (int l = 0; l < 4; l++) {
      const NetLayout& L = net[n];
      const int kin = L.kin[l], nout = L.nout[l], kin16 = l == 0 ? 16 : H, npad = l < 3 ? H : L.n_out16;
      const int K_B = kin16 + 16;
      const __half* W = reinterpret_cast<const __half*>(blob + L.w_off[l]);
      const __half* bias = reinterpret_cast<const __half*>(blob + L.b_off[l]);
      uint8_t* dst = img + L.layer_off[l];
      for (int t = tid0; t < npad * K_B; t += nthr) {
        const int k = t / npad, o = t - k * npad;   // o fastest: coalesced reads of W[k][o]
        __half v = __ushort_as_half((unsigned short)0);
        if (o < nout && k < kin) v = W[(size_t)k * nout + o];
        else if (o < nout && k == kin16) v = bias[o];
        *reinterpret_cast<__half*>(dst + kmajor_offset(o, k, K_B)) = v;
      }
    }
    img += net[n].img_bytes;
  }
  if (tid0 < 8) {  // the constant ones tile used to fold the bias into the MMA (all 16 row groups read it)
    const uint4 c0 = make_uint4(0x3C00u, 0u, 0u, 0u), z = make_uint4(0u, 0u, 0u, 0u);
    *reinterpret_cast<uint4*>(img + kmajor_offset(tid0, 0, 16)) = c0;
    *reinterpret_cast<uint4*>(img + kmajor_offset(tid0, 8, 16)) = z;
  }
  float* unorm = reinterpret_cast<float*>(img + kOnesBytes);
  for (int i = tid0; i < 352; i += nthr)  // UNORM expansion tables: the exact quotients of R12/R13
    unorm[i] = i < 32 ? __fdiv_rn((float)i, 31.0f) : i < 96 ? __fdiv_rn((float)(i - 32), 63.0f)
                                                             : __fdiv_rn((float)(i - 96), 255.0f);
  for (int i = tid0; i < 32; i += nthr) unorm[352 + i] = bc4_weight(i);   // BC4 interpolation weights per mode
}

// four codes per thread: one 4-byte load, one 16-byte store.  A level whose code count res^2 x 2 is not a
// multiple of 4 (odd coarsest resolution) ends with a partial group: its extra codes come from the 16-B
// padding that follows every level in the blob and land in the 16-B padding of the level's fp32 region
// (never read), so every level starts a fresh group.
__global__ void __launch_bounds__(256) dequant_grids_kernel(const __grid_constant__ DequantParams d) {
  const long long total4 = d.end[d.n_levels - 1];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total4; i += (long long)gridDim.x * blockDim.x) {
    int l = 0;
    while (i >= d.end[l]) l++;
    const long long j = i - (l ? d.end[l - 1] : 0);
    const uint32_t q4 = __ldg(reinterpret_cast<const uint32_t*>(d.slot + d.src_off[l]) + j);
    const float s = d.s[l];
    const int z = d.z[l];
    reinterpret_cast<float4*>(d.slot + d.dst_off[l])[j] =
        make_float4(__fmul_rn(s, (float)((int)(q4 & 0xFFu) - z)), __fmul_rn(s, (float)((int)((q4 >> 8) & 0xFFu) - z)),
                    __fmul_rn(s, (float)((int)((q4 >> 16) & 0xFFu) - z)), __fmul_rn(s, (float)((int)(q4 >> 24) - z)));
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d.zero_n; i += gridDim.x * blockDim.x)
    reinterpret_cast<float*>(d.slot + d.zero_off)[i] = 0.0f;
  build_smem_prefix(d.slot + d.img_off, d.slot, d.net, d.H, blockIdx.x * blockDim.x + threadIdx.x,
                    gridDim.x * blockDim.x);
}

// ---------------------------------------------------------------- a1-a2: coordinates + grid encode
// Vertex-centred bilinear lookup of one level (R1) of the dequantized grid (R6), lerp = fma(t, b-a, a),
// both features of a vertex as one fp32x2 pair (one 8-byte load per vertex).
// The reading's clamp i0 = min(floor(X), res-2) never binds here: callers pass p in (0, 1) (rows past
// the texture edge are clamped to the last valid block/texel), so X = RN(p (res-1)) < res - 1.
__device__ __forceinline__ uint64_t level_lookup2(const uint8_t* blob, const GridLevel& L, float pu, float pv) {
  const float X = __fmul_rn(pu, L.rm1), Y = __fmul_rn(pv, L.rm1);
  const int i0 = __float2int_rd(X), j0 = __float2int_rd(Y);
  float fx, fy;
  f2unpack(sub2(f2pack(X, Y), f2pack((float)i0, (float)j0)), fx, fy);
  NTBC_CHECK(i0 >= 0 && j0 >= 0 && i0 <= L.res - 2 && j0 <= L.res - 2);
  const unsigned long long* g = reinterpret_cast<const unsigned long long*>(blob + L.offset) + (j0 * L.res + i0);
  const uint64_t v00 = __ldg(g), v10 = __ldg(g + 1), v01 = __ldg(g + L.res), v11 = __ldg(g + L.res + 1);
  const uint64_t FX = f2pack(fx, fx), FY = f2pack(fy, fy);
  const uint64_t top = fma2(FX, sub2(v10, v00), v00), bot = fma2(FX, sub2(v11, v01), v01);
  return fma2(FY, sub2(bot, top), top);
}

// ---------------------------------------------------------------- TMEM load helper (x16 columns)
__device__ __forceinline__ void tmem_ld16p(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld8p(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld8(uint32_t* r) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7])
               :
               : "memory");
}

__device__ __forceinline__ void tmem_ld2(uint32_t taddr, uint32_t& a, uint32_t& b) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(a), "=r"(b) : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(a), "+r"(b)::"memory");
}

// tcgen05.wait::ld that also "touches" the 16 destination registers, so the compiler cannot move their
// uses above the wait (the registers are undefined until the asynchronous load completes).
__device__ __forceinline__ void tmem_wait_ld16(uint32_t* r) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
               :
               : "memory");
}

// Issue one layer of the MLP for the 128 rows of a work group (called by ONE thread):
// bias chunk first (A = ones tile, B = bias column; overwrites D), then the K/16 activation chunks
// in increasing k (accumulate) -- the summation order pinned by R10.
// SPLIT (contract F): A holds each 16-wide K chunk c of the activations as two physical chunks, hi at 2c and
// lo at 2c + 1; both are multiplied by the same B chunk, hi first (the order the oracle's F mode pins).
template <bool SPLIT = false>
__device__ __forceinline__ void issue_layer(uint32_t tmem_d, uint32_t a_base, int K_A, uint32_t ones_base,
                                            uint32_t b_base, int kin16, int N) {
  const int K_B = kin16 + 16;
  const uint32_t idesc = idesc_f16_f32(128, N);
  mma_f16(tmem_d, smem_desc(ones_base, 128, 0), smem_desc(b_base + (kin16 / 16) * 256, 128, K_B * 16), idesc, 0u);
  for (int c = 0; c < kin16 / 16; c++) {
    const uint64_t bd = smem_desc(b_base + c * 256, 128, K_B * 16);
    mma_f16(tmem_d, smem_desc(a_base + (SPLIT ? 2 * c : c) * 256, 128, K_A * 16), bd, idesc, 1u);
    if (SPLIT) mma_f16(tmem_d, smem_desc(a_base + (2 * c + 1) * 256, 128, K_A * 16), bd, idesc, 1u);
  }
}

// ---------------------------------------------------------------- kernel (1): fused decode
// One CTA per SM, NWG independent 128-thread work groups (8 for H = 64: 64 registers per thread, all
// 512 TMEM columns); each work group owns 64 TMEM columns, an A-operand buffer and the BC word headers
// of its unit, and loops over work units of 128 block positions of one block row: one endpoint tile
// (128 blocks) then up to 16 colour tiles (8 blocks = 128 texels).  More independent groups per SM
// hide more of the dependent epilogue latency.  Units are claimed from a global
// counter (dynamic scheduling) so they finish in row order (pipelined copy-back, ntbc_api.cu).
template <int H, int NWG, bool DUMP, bool NAIVE, bool SPLIT = false, bool HALF = false>
__global__ void __launch_bounds__(NWG * 128, 1) fused_decode_kernel(const __grid_constant__ FusedLaunch L) {
  constexpr int KA = SPLIT ? 2 * H : H;   // K width (fp16 columns) of the A operand rows
  extern __shared__ __align__(1024) uint8_t smem[];
  const int sel = (int)blockIdx.x >= L.split;          // which model this CTA decodes
  const FusedParams& p = L.m[sel];
  const int cta = (int)blockIdx.x - (sel ? L.split : 0), ncta = sel ? (int)gridDim.x - L.split : L.split;
  const int tid = threadIdx.x, wg = tid >> 7, r = tid & 127, warp = tid >> 5, lane = tid & 31;
  // PP: two colour tiles per work group in flight (slots 0 / 1: A operand, TMEM accumulator, mbarrier), the
  // MMAs of one slot overlapping the epilogue of the other (NTBC_PINGPONG, 4 work groups, H = 64)
  constexpr bool PP = NTBC_PINGPONG && NWG == 4 && H == 64 && !DUMP && !SPLIT;
  constexpr int SL = PP ? 2 : 1;

  // ---- carve shared memory
  uint8_t* img_e = smem;                                          // endpoint net operand image
  uint8_t* img_c = smem + p.net[0].img_bytes;                     // colour net operand image
  uint8_t* ones = img_c + p.net[1].img_bytes;                     // [8][16] K-major, column 0 = 1.0
  float* unorm = reinterpret_cast<float*>(ones + kOnesBytes);           // q/31 [32], q/63 [64], q/255 [256], BC4 weights
  uint8_t* wg_base = ones + kOnesBytes + kUnormBytes + wg * (SL * p.a_bytes + p.pal_bytes);
  uint8_t* A = wg_base;                                           // [128][H] K-major fp16 / fp32 staging
  float* stage = reinterpret_cast<float*>(A);                     // [ch][128] fp32 (after the last MMA)
  uint32_t* hdrs = reinterpret_cast<uint32_t*>(wg_base + SL * p.a_bytes);  // [tex][128 blocks] BC word low bits
  uint8_t* swp = reinterpret_cast<uint8_t*>(hdrs + p.n_tex * 128);   // [tex][128 blocks] BC1 endpoint swap (naive)
  float* tpal = reinterpret_cast<float*>(wg_base + SL * p.a_bytes + p.tpal_off);   // [8 SL blocks][pal_stride] tile palettes
  uint64_t* bars = reinterpret_cast<uint64_t*>(ones + kOnesBytes + kUnormBytes + NWG * (SL * p.a_bytes + p.pal_bytes));
  uint64_t* bar_mma = bars + SL * wg;                             // this work group's MMA completion (per slot)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + SL * NWG + 1);
  int* next_slot = reinterpret_cast<int*>(tmem_slot + 1) + wg;    // dynamic scheduling: this group's next unit

#if NTBC_CHECKS
  NTBC_CHECK((uint32_t)(reinterpret_cast<uint8_t*>(next_slot + NWG - wg) - smem) <= dyn_smem_bytes());
  NTBC_CHECK(p.a_bytes >= 128u * KA * 2u && p.tpal_off >= (uint32_t)p.n_tex * 128u * 4u &&
             p.pal_bytes >= p.tpal_off + 8u * SL * p.pal_stride * 4u);
  for (uint32_t i = tid; i < (uint32_t)(reinterpret_cast<uint8_t*>(bars) - smem) / 4; i += NWG * 128)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x7FC17FC1u;   // poison: fp32 and fp16 NaN
  fence_async_smem();
  __syncthreads();
#endif
  // ---- the shared-memory prefix (operand images of both nets, ones tile, UNORM tables), prebuilt in global
  //      memory by the prep kernel: one bulk asynchronous copy (TMA engine) per 32 KB, completing on bar_img
  uint64_t* bar_img = bars + SL * NWG;
  if (tid == 0) {
    for (int g = 0; g <= SL * NWG; g++) mbar_init(bars + g, 1);
    fence_mbar_init();
    const uint32_t total = prefix_bytes(p.net);
    mbar_arrive_expect_tx(bar_img, total);
    for (uint32_t o = 0; o < total; o += 32768u)
      bulk_g2s(smem + o, p.prefix + o, min(32768u, total - o), bar_img);
  }
  constexpr uint32_t kTmemCols = SL * NWG <= 2 ? 128 : SL * NWG <= 4 ? 256 : 512;
  if (warp == 0) tmem_alloc(tmem_slot, kTmemCols);
  __syncthreads();
  mbar_wait(bar_img, 0);   // the copy's writes are visible to this thread (generic reads of the tables) and to
                           // the tensor core (async-proxy reads of the operand images)
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const uint32_t tm = tmem_base + (uint32_t)(wg * 64 * SL);               // D columns of this group (slot 0)
  NTBC_CHECK((tm & 0xFFFFu) + 64u * SL <= kTmemCols);
  const uint32_t tm_row = tm + ((uint32_t)(32 * (warp & 3)) << 16);       // this warp's TMEM lanes
  const uint32_t a_base = smem_u32(A), ones_base = smem_u32(ones);
  const uint32_t img_base[2] = {smem_u32(img_e), smem_u32(img_c)};
  const int bar_id = 1 + wg;
  // the thread that issues this group's MMAs: lane 0 of warp (wg mod 4) of the group, so the issuing
  // warps are spread over the four SM sub-partitions (warp w runs on SMSP w mod 4; measured: all eight
  // on SMSP 0 made each MMA cost ~275 issue cycles on the group's critical path, 2.25 -> 2.15 ms)
  const int issuer = 32 * (wg & 3);

  uint32_t phase[SL];
  for (int q = 0; q < SL; q++) phase[q] = 0;

  // 16 grid features of row r (levels coarse->fine, 2 per level, R3) -> fp16 -> A columns 0..15 of slot sl
  auto features = [&](int g, float pu, float pv, float* dump, int sl) {
    uint32_t hv[kMaxLevels], lv[kMaxLevels];
#pragma unroll
    for (int l = 0; l < kMaxLevels; l++) {
      float f0, f1;   // all levels unconditionally: unused ones are set up to return +0 (launch_fused)
      f2unpack(level_lookup2(p.blob, p.lv[g][l], pu, pv), f0, f1);
      if (dump) { dump[2 * l] = f0; dump[2 * l + 1] = f1; }
      if (SPLIT) {
        split_h2(f0, f1, hv[l], lv[l]);
      } else {
        const __half2 v = __floats2half2_rn(f0, f1);
        hv[l] = *reinterpret_cast<const uint32_t*>(&v);
      }
    }
    uint8_t* As = A + sl * p.a_bytes;
    *reinterpret_cast<uint4*>(As + kmajor_offset(r, 0, KA)) = make_uint4(hv[0], hv[1], hv[2], hv[3]);
    *reinterpret_cast<uint4*>(As + kmajor_offset(r, 8, KA)) = make_uint4(hv[4], hv[5], hv[6], hv[7]);
    if (SPLIT) {
      *reinterpret_cast<uint4*>(As + kmajor_offset(r, 16, KA)) = make_uint4(lv[0], lv[1], lv[2], lv[3]);
      *reinterpret_cast<uint4*>(As + kmajor_offset(r, 24, KA)) = make_uint4(lv[4], lv[5], lv[6], lv[7]);
    }
  };

  // layer l of net n on slot sl: the group's A rows are complete (barrier), one thread issues the MMAs
  auto issue_l = [&](int n, int l, int sl) {
    fence_async_smem();
    tc_fence_before();
    named_bar_sync(bar_id, 128);
    if (r == issuer) {
      tc_fence_after();
      const int kin16 = l == 0 ? 16 : H;
      const int N = l < 3 ? H : p.net[n].n_out16;
      issue_layer<SPLIT>(tm + sl * 64, a_base + sl * p.a_bytes, KA, ones_base, img_base[n] + p.net[n].layer_off[l], kin16, N);
      mma_commit(bar_mma + sl);
    }
  };
  // wait for slot sl's MMAs.  One slot: one thread polls, the others park on bar.sync (measured faster than
  // per-warp polling there); ping-pong: the MMAs ran during the other slot's epilogue, every warp polls once
  auto wait_s = [&](int sl) {
    if (PP || NTBC_WARP_POLL) {
      if (lane == 0) mbar_wait(bar_mma + sl, phase[sl]);
      __syncwarp();
    } else {
      if (r == issuer) mbar_wait(bar_mma + sl, phase[sl]);
      named_bar_sync(bar_id, 128);
    }
    phase[sl] ^= 1u;
    tc_fence_after();
  };
  // hidden layer epilogue of slot sl: selu -> fp16 -> next A operand row (R8-R10), 16 columns at a time
  auto hidden_epi = [&](int sl) {
    constexpr bool PF = NWG <= 4;   // prefetch the next chunk (16 more registers than NWG 8 has)
    const uint32_t tr = tm_row + sl * 64;
    uint8_t* As = A + sl * p.a_bytes;
    if (NTBC_TMEM_PF8 && !PF && !SPLIT) {     // 8-column chunks, the next chunk's load in flight during this chunk's selu
      uint32_t b8[2][8];
      tmem_ld8p(tr, b8[0]);
      tmem_wait_ld8(b8[0]);
#pragma unroll
      for (int c = 0; c < H / 8; c++) {
        if (c + 1 < H / 8) tmem_ld8p(tr + (c + 1) * 8, b8[(c + 1) & 1]);
        uint32_t hv[4];
#pragma unroll
        for (int j = 0; j < 4; j++)
          hv[j] = HALF ? selu2_h16(__uint_as_float(b8[c & 1][2 * j]), __uint_as_float(b8[c & 1][2 * j + 1]))
                       : selu2_h2(__uint_as_float(b8[c & 1][2 * j]), __uint_as_float(b8[c & 1][2 * j + 1]));
        *reinterpret_cast<uint4*>(As + kmajor_offset(r, c * 8, H)) = make_uint4(hv[0], hv[1], hv[2], hv[3]);
        if (c + 1 < H / 8) tmem_wait_ld8(b8[(c + 1) & 1]);
      }
      return;
    }
    uint32_t buf[2][16];
    tmem_ld16p(tr, buf[0]);
    tmem_wait_ld16(buf[0]);
#pragma unroll
    for (int c = 0; c < H / 16; c++) {
      if (!PF && c > 0) {
        tmem_ld16p(tr + c * 16, buf[c & 1]);
        tmem_wait_ld16(buf[c & 1]);
      }
      if (PF && c + 1 < H / 16) tmem_ld16p(tr + (c + 1) * 16, buf[(c + 1) & 1]);
      uint32_t hv[8];
      if (SPLIT) {   // contract F: binary32 selu, hi chunk at physical 2c, lo chunk at 2c + 1
        uint32_t lv[8];
#pragma unroll
        for (int j = 0; j < 8; j++)
          selu2_split(__uint_as_float(buf[c & 1][2 * j]), __uint_as_float(buf[c & 1][2 * j + 1]), hv[j], lv[j]);
        *reinterpret_cast<uint4*>(As + kmajor_offset(r, c * 32, KA)) = make_uint4(hv[0], hv[1], hv[2], hv[3]);
        *reinterpret_cast<uint4*>(As + kmajor_offset(r, c * 32 + 8, KA)) = make_uint4(hv[4], hv[5], hv[6], hv[7]);
        *reinterpret_cast<uint4*>(As + kmajor_offset(r, c * 32 + 16, KA)) = make_uint4(lv[0], lv[1], lv[2], lv[3]);
        *reinterpret_cast<uint4*>(As + kmajor_offset(r, c * 32 + 24, KA)) = make_uint4(lv[4], lv[5], lv[6], lv[7]);
      } else {
#pragma unroll
        for (int j = 0; j < 8; j++)
          hv[j] = HALF ? selu2_h16(__uint_as_float(buf[c & 1][2 * j]), __uint_as_float(buf[c & 1][2 * j + 1]))
                       : selu2_h2(__uint_as_float(buf[c & 1][2 * j]), __uint_as_float(buf[c & 1][2 * j + 1]));
        *reinterpret_cast<uint4*>(As + kmajor_offset(r, c * 16, H)) = make_uint4(hv[0], hv[1], hv[2], hv[3]);
        *reinterpret_cast<uint4*>(As + kmajor_offset(r, c * 16 + 8, H)) = make_uint4(hv[4], hv[5], hv[6], hv[7]);
      }
      if (PF && c + 1 < H / 16) tmem_wait_ld16(buf[(c + 1) & 1]);
    }
  };
  // run the 4-layer MLP of net `n` on the A rows already written (slot 0); leaves the output layer in TMEM
  auto run_mlp = [&](int n) {
#pragma unroll 1
    for (int l = 0; l < 4; l++) {
      issue_l(n, l, 0);
      wait_s(0);
      if (l < 3) hidden_epi(0);
    }
  };
  // output layer epilogue of slot sl: sigmoid of the output channels (pairs) -> fp32 staging [ch][128] (in A)
  auto stage_out = [&](int n, int sl) {
    const int no = p.net[n].n_out;
    float* st = reinterpret_cast<float*>(A + sl * p.a_bytes);
#pragma unroll 1
    for (int c16 = 0; c16 < no; c16 += 16) {
      uint32_t v[16];
      tmem_ld16p(tm_row + sl * 64 + c16, v);
      tmem_wait_ld16(v);
#pragma unroll
      for (int j = 0; j < 16; j += 2) {
        const int ch = c16 + j;
        if (ch < no) {
          float s0, s1;
          sigmoid2(__uint_as_float(v[j]), __uint_as_float(v[j + 1]), s0, s1);
          NTBC_CHECK((uint32_t)((ch + 1) * 128 + r) * 4u < p.a_bytes);
          st[ch * 128 + r] = s0;
          st[(ch + 1) * 128 + r] = s1;
        }
      }
    }
  };
  auto stage_outputs = [&](int n) { stage_out(n, 0); };

#pragma unroll 1
  for (int u = cta * NWG + wg; u < p.n_units;) {
    const int by = p.row_begin + u / p.units_per_row;
    const int bx0 = (u % p.units_per_row) * kUnitBlocks;
    const int nvalid = min(kUnitBlocks, p.BW - bx0);
    const size_t out_row = (size_t)(by - p.row_begin) * p.BW;

    // ================= endpoint tile: row r = block (bx0 + r, by)  (rows a1-a3, a5-a6)
    named_bar_sync(bar_id, 128);  // previous tile's readers of A / staging / headers are done
    // dynamic scheduling (p.next_unit): claim the group's next unit now; it is read at the end of this
    // unit, after the MLP's barriers have ordered the store before every reader
    if (p.next_unit && r == 0) *next_slot = atomicAdd(p.next_unit, 1) + ncta * NWG;
    {
      const float s = __fdiv_rn(__fadd_rn((float)min(bx0 + r, p.BW - 1), 0.5f), (float)p.BW);
      const float t = __fdiv_rn(__fadd_rn((float)by, 0.5f), (float)p.BH);
      float* fd = (DUMP && (p.debug_flags & 2) && r < nvalid) ? p.dump_ep + (out_row + bx0 + r) * 16 : nullptr;
      features(0, s, t, fd, 0);
    }
    run_mlp(0);
    stage_outputs(0);
    if (DUMP) {
      if (r < nvalid && !(p.debug_flags & 2))
        for (int ch = 0; ch < p.net[0].n_out; ch++)
          p.dump_ep[(out_row + bx0 + r) * p.net[0].n_out + ch] = stage[ch * 128 + r];
    } else {
      for (int k = 0; k < p.n_tex; k++) {
        const int eo = p.ep_off[k];
        if (p.fmt[k] == kFmtBC1) {  // BC word header after quantization and the 4-colour-mode swap (R11, R12)
          float ep[6];
#pragma unroll
          for (int c = 0; c < 6; c++) ep[c] = stage[(eo + c) * 128 + r];
          bool swapped;
          hdrs[k * 128 + r] = quant_bc1_hdr(ep, swapped);
          if (NAIVE) swp[k * 128 + r] = swapped;
        } else {                    // E0 | E1 << 8 (R13)
          const float ep[2] = {stage[eo * 128 + r], stage[(eo + 1) * 128 + r]};
          hdrs[k * 128 + r] = quant_bc4_hdr(ep);
        }
      }
    }

    // ================= colour tiles: row r = texel (r & 15) of block 8j + (r >> 4)  (a1-a2, a4, a6-a8)
    // index selection + packing of colour tile jt from slot sl's staged outputs (the block palettes at
    // tpal[8 sl + r / 16] were built at the tile start)
    // index selection + packing of colour tile jt by JOBS: thread r takes half h = r & 1 (texels 8h..8h+7) of
    // job r >> 1 = (texture, block) -- BC1 textures first, then BC4, 8 blocks each -- reading the tile's
    // staged outputs of its block (8 consecutive rows: vector loads), the block's palette built at the tile
    // start, and combining the two halves' index fields with one shuffle; the even thread stores the word.
    // Each (block, texture) palette and header is read once per half instead of once per texel (the
    // per-texel form, pack_tile, costs every thread the whole texture loop).
    auto pack_tile_jobs = [&](int jt, int sl) {
      named_bar_sync(bar_id, 128);                       // every row's outputs are staged
      const float* st = reinterpret_cast<const float*>(A + sl * p.a_bytes);
      const int job = r >> 1, h = r & 1;
      const int nj = 8 * p.n_tex;
      const int jj = min(job, nj - 1);                   // idle threads shadow the last job (no store)
      const int ti = jj >> 3, bl = jj & 7;               // texture slot (BC1 list then BC4 list), block
      const bool bc1 = ti < p.n_bc1;
      const int k = bc1 ? p.tex_bc1[ti] : p.tex_bc4[ti - p.n_bc1];
      const int co = p.col_off[k];
      const int b = 8 * jt + bl;
      const uint32_t hdr = hdrs[k * 128 + b];
      const float* tp = tpal + (8 * sl + bl) * p.pal_stride + p.pal_off[k];
      const int row0 = 16 * bl + 8 * h;                  // this half's first texel row in the stage
      uint64_t bits;
      if (bc1) {
        const float2* P = reinterpret_cast<const float2*>(tp);
        const bool degenerate = (hdr & 0xFFFFu) == (hdr >> 16);
        float cr[8], cg[8], cb[8];
        *reinterpret_cast<float4*>(cr) = *reinterpret_cast<const float4*>(st + co * 128 + row0);
        *reinterpret_cast<float4*>(cr + 4) = *reinterpret_cast<const float4*>(st + co * 128 + row0 + 4);
        *reinterpret_cast<float4*>(cg) = *reinterpret_cast<const float4*>(st + (co + 1) * 128 + row0);
        *reinterpret_cast<float4*>(cg + 4) = *reinterpret_cast<const float4*>(st + (co + 1) * 128 + row0 + 4);
        *reinterpret_cast<float4*>(cb) = *reinterpret_cast<const float4*>(st + (co + 2) * 128 + row0);
        *reinterpret_cast<float4*>(cb + 4) = *reinterpret_cast<const float4*>(st + (co + 2) * 128 + row0 + 4);
        uint32_t v = 0;
#pragma unroll
        for (int i = 0; i < 8; i++) {
          const float c[3] = {cr[i], cg[i], cb[i]};
          v |= bc1_code_pairs(c, P, degenerate) << (2 * i);
        }
        const uint32_t o = __shfl_xor_sync(0xFFFFFFFFu, v, 1);
        bits = (uint64_t)(v | (o << 16)) << 32;
      } else {
        const float4 q0 = reinterpret_cast<const float4*>(tp)[0], q1 = reinterpret_cast<const float4*>(tp)[1];
        const float pl[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
        const bool mode8 = (hdr & 0xFFu) > ((hdr >> 8) & 0xFFu);
        float cv[8];
        *reinterpret_cast<float4*>(cv) = *reinterpret_cast<const float4*>(st + co * 128 + row0);
        *reinterpret_cast<float4*>(cv + 4) = *reinterpret_cast<const float4*>(st + co * 128 + row0 + 4);
        uint32_t v = 0;
#pragma unroll
        for (int i = 0; i < 8; i++) v |= bc4_code(cv[i], pl, mode8) << (3 * i);
        const uint32_t o = __shfl_xor_sync(0xFFFFFFFFu, v, 1);
        bits = (uint64_t)(v | ((uint64_t)o << 24)) << 16;
      }
      // 8-byte stores: pairing adjacent blocks' words into 16-byte stores here (a 64-bit shuffle by two
      // lanes) measured +1.3% (A/B r02ac: 2.184 vs 2.156 ms); a warp's stores still cover two 64-byte runs
      if (h == 0 && job < nj && b < nvalid) {
        NTBC_CHECK(bx0 + b < p.BW && by < p.row_end);
        p.out[k][out_row + bx0 + b] = (uint64_t)hdr | bits;
      }
    };
    // the same work by WARP-LOCAL jobs (NTBC_EPI_JOBS=2): warp w of the group staged rows 32w..32w+31 = the
    // texels of blocks 2w and 2w+1 of the tile, so it packs exactly those two blocks -- no group barrier, only
    // __syncwarp.  The BC1 jobs (2 blocks x n_bc1 textures) and then the BC4 jobs (2 x n_bc4) each spread
    // over the warp: lpj = 32 / jobs lanes per job (a power of two), 16 / lpj texels per lane, the job's
    // index field OR-combined over its lanes with shuffles; the job's first lane stores the word.
    auto pack_tile_warp = [&](int jt, int sl) {
      __syncwarp();
      const float* st = reinterpret_cast<const float*>(A + sl * p.a_bytes);
      const int wq = (r >> 5) & 3;                        // warp of the group: blocks 2 wq, 2 wq + 1
      for (int fmt_pass = 0; fmt_pass < 2; fmt_pass++) {
        const bool bc1 = fmt_pass == 0;
        const int ntx = bc1 ? p.n_bc1 : p.n_bc4;
        if (ntx == 0) continue;
        const int nj = 2 * ntx;
        const int lpj = nj <= 2 ? 16 : nj <= 4 ? 8 : nj <= 8 ? 4 : nj <= 16 ? 2 : 1;
        const int tpl = 16 / lpj;
        const int job = lane / lpj, part = lane - job * lpj;
        const int jj = min(job, nj - 1);
        const int ti = jj >> 1, bl = 2 * wq + (jj & 1);
        const int k = bc1 ? p.tex_bc1[ti] : p.tex_bc4[ti];
        const int co = p.col_off[k];
        const int b = 8 * jt + bl;
        const uint32_t hdr = hdrs[k * 128 + b];
        const float* tp = tpal + (8 * sl + bl) * p.pal_stride + p.pal_off[k];
        const int t0 = part * tpl;                         // this lane's first texel of the block
        const float* sr = st + 16 * bl + t0;               // texel t0's row in the stage
        uint64_t bits = 0;
        if (bc1) {
          const float2* P = reinterpret_cast<const float2*>(tp);
          const bool degenerate = (hdr & 0xFFFFu) == (hdr >> 16);
          for (int i = 0; i < tpl; i++) {
            const float c[3] = {sr[co * 128 + i], sr[(co + 1) * 128 + i], sr[(co + 2) * 128 + i]};
            bits |= (uint64_t)bc1_code_pairs(c, P, degenerate) << (2 * (t0 + i));
          }
        } else {
          const float4 q0 = reinterpret_cast<const float4*>(tp)[0], q1 = reinterpret_cast<const float4*>(tp)[1];
          const float pl[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
          const bool mode8 = (hdr & 0xFFu) > ((hdr >> 8) & 0xFFu);
          for (int i = 0; i < tpl; i++) bits |= (uint64_t)bc4_code(sr[co * 128 + i], pl, mode8) << (3 * (t0 + i));
        }
        for (int d = 1; d < lpj; d <<= 1) {                // OR over the job's lanes (disjoint fields)
          const uint32_t lo = __shfl_xor_sync(0xFFFFFFFFu, (uint32_t)bits, d);
          const uint32_t hi = __shfl_xor_sync(0xFFFFFFFFu, (uint32_t)(bits >> 32), d);
          bits |= (uint64_t)hi << 32 | lo;
        }
        if (part == 0 && job < nj && b < nvalid) {
          NTBC_CHECK(bx0 + b < p.BW && by < p.row_end);
          p.out[k][out_row + bx0 + b] = (uint64_t)hdr | (bits << (bc1 ? 32 : 16));
        }
      }
    };
    auto pack_tile = [&](int jt, int sl) {
      const int b = 8 * jt + (r >> 4);
      const int bx = bx0 + b;
      const float* st = reinterpret_cast<const float*>(A + sl * p.a_bytes);
      const float* tp = tpal + (8 * sl + (r >> 4)) * p.pal_stride;
      // lane 0 of each warp writes the words of the warp's two adjacent blocks (b, b + 1; bx even) as one
      // 16-byte store when p.vec16, else lanes 0 and 16 write one 8-byte word each
      const bool pair = p.vec16 && lane == 0 && b + 1 < nvalid;
      const bool single = p.vec16 ? (lane == 0 && b + 1 >= nvalid && b < nvalid) : ((lane & 15) == 0 && b < nvalid);
      // the words of texture k: header | index field << SHIFT, both blocks of the warp (see above)
      auto store = [&](int k, uint32_t hdr, const uint64_t* idx, int shift) {
        uint64_t* dst = p.out[k] + out_row + bx;
        NTBC_CHECK(!(pair || single) || (bx + (pair ? 1 : 0) < p.BW && by < p.row_end && b < kUnitBlocks));
        if (pair) st_words2(dst, (uint64_t)hdr | (idx[0] << shift), (uint64_t)hdrs[k * 128 + b + 1] | (idx[1] << shift));
        else if (single) *dst = (uint64_t)hdr | ((lane < 16 ? idx[0] : idx[1]) << shift);
      };
      if (NAIVE) {
        for (int k = 0; k < p.n_tex; k++) {  // naive approach: nearest palette weight to the predicted weight
          const int co = p.col_off[k];
          const uint32_t hdr = hdrs[k * 128 + b];
          uint64_t idx[2];
          const float w = st[co * 128 + r];
          if (p.fmt[k] == kFmtBC1) {
            const uint32_t c0 = hdr & 0xFFFFu, c1 = hdr >> 16;
            uint32_t n = naive_bc1_index(w);
            if (swp[k * 128 + b]) n = 3u - n;                  // weights follow the predicted endpoint order
            const uint32_t code = c0 == c1 ? 0u : (0x1320u >> (4 * n)) & 3u;   // linear n -> code [0,2,3,1]
            pack_bc1_indices2(code, lane, idx);
            store(k, hdr, idx, 32);
          } else {
            const uint32_t E0 = hdr & 0xFFu, E1 = (hdr >> 8) & 0xFFu;
            const uint32_t n = naive_bc4_index(w, E0 > E1, unorm + 352);
            const uint32_t map = E0 > E1 ? 0x17654320u : 0x71543206u;
            pack_bc4_indices2((map >> (4 * n)) & 7u, lane, idx);
            store(k, hdr, idx, 16);
          }
        }
      } else {
        // BC1 textures, then BC4 textures (launch-uniform lists): no format branch per texture and
        // constant field shifts (A/B r02g: 2.201 vs 2.222 ms)
        for (int t = 0; t < p.n_bc1; t++) {
          const int k = p.tex_bc1[t], co = p.col_off[k];
          const uint32_t hdr = hdrs[k * 128 + b];
          const float2* P = reinterpret_cast<const float2*>(tp + p.pal_off[k]);
          const float c[3] = {st[co * 128 + r], st[(co + 1) * 128 + r], st[(co + 2) * 128 + r]};
          uint64_t idx[2];
          pack_bc1_indices2(bc1_code_pairs(c, P, (hdr & 0xFFFFu) == (hdr >> 16)), lane, idx);
          store(k, hdr, idx, 32);
        }
        for (int t = 0; t < p.n_bc4; t++) {
          const int k = p.tex_bc4[t], co = p.col_off[k];
          const uint32_t hdr = hdrs[k * 128 + b];
          const float4* P = reinterpret_cast<const float4*>(tp + p.pal_off[k]);
          const float4 q0 = P[0], q1 = P[1];
          const float pl[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
          uint64_t idx[2];
          pack_bc4_indices2(bc4_code(st[co * 128 + r], pl, (hdr & 0xFFu) > ((hdr >> 8) & 0xFFu)), lane, idx);
          store(k, hdr, idx, 16);
        }
      }
    };
#pragma unroll 1
    for (int j = 0; j < kUnitBlocks / 8 && 8 * j < nvalid; j += SL) {
      const int ntile = (PP && 8 * (j + 1) < nvalid) ? 2 : 1;
      named_bar_sync(bar_id, 128);
      if (!DUMP && !NAIVE && r < 8 * ntile * p.n_tex) {   // the tiles' block palettes, once per block (Eq.7/8, R18)
        const int bl = r / p.n_tex, k = r - bl * p.n_tex;
        const uint32_t hdr = hdrs[k * 128 + 8 * j + bl];
        float* dst = tpal + bl * p.pal_stride + p.pal_off[k];
        NTBC_CHECK(bl < 8 * SL && k < p.n_tex && 8 * j + bl < kUnitBlocks);
        if (p.fmt[k] == kFmtBC1) {
          const uint32_t c0 = hdr & 0xFFFFu, c1 = hdr >> 16;
          const float e0[3] = {unorm[c0 >> 11], unorm[32 + ((c0 >> 5) & 63)], unorm[c0 & 31]};
          const float e1[3] = {unorm[c1 >> 11], unorm[32 + ((c1 >> 5) & 63)], unorm[c1 & 31]};
          bc1_palette_pairs(e0, e1, dst);
        } else {
          const uint32_t E0 = hdr & 0xFFu, E1 = (hdr >> 8) & 0xFFu;
          bc4_palette_tab(unorm[96 + E0], unorm[96 + E1], E0 > E1, unorm + 352, dst);
        }
      }
      for (int sl = 0; sl < ntile; sl++) {
        const int b = 8 * (j + sl) + (r >> 4), i = r & 15;
        const int bx = bx0 + b, x = 4 * min(bx, p.BW - 1) + (i & 3), y = 4 * by + (i >> 2);
        const float pu = __fdiv_rn(__fadd_rn((float)x, 0.5f), (float)p.W);
        const float pv = __fdiv_rn(__fadd_rn((float)y, 0.5f), (float)p.H);
        float* fd = (DUMP && (p.debug_flags & 2) && b < nvalid)
                        ? p.dump_col + (((size_t)(y - 4 * p.row_begin)) * p.W + x) * 16 : nullptr;
        features(1, pu, pv, fd, sl);
      }
      if (!PP) {
        run_mlp(1);
        stage_outputs(1);
      } else {   // ping-pong: slot 1's MMAs run during slot 0's epilogue and vice versa
        for (int sl = 0; sl < ntile; sl++) issue_l(1, 0, sl);
#pragma unroll 1
        for (int l = 0; l < 4; l++)
          for (int sl = 0; sl < ntile; sl++) {
            wait_s(sl);
            if (l < 3) {
              hidden_epi(sl);
              issue_l(1, l + 1, sl);
            } else {
              stage_out(1, sl);
            }
          }
      }
      if (DUMP) {
        const int b = 8 * j + (r >> 4), i = r & 15;
        const int bx = bx0 + b, x = 4 * min(bx, p.BW - 1) + (i & 3), y = 4 * by + (i >> 2);
        if (b < nvalid && !(p.debug_flags & 2))
          for (int ch = 0; ch < p.net[1].n_out; ch++)
            p.dump_col[(((size_t)(y - 4 * p.row_begin)) * p.W + x) * p.net[1].n_out + ch] = stage[ch * 128 + r];
      } else {
        for (int sl = 0; sl < ntile; sl++) {
          // jobs pay with >= 3 textures (>= 48 busy threads); with 1-2 textures the per-texel form keeps all four
          // warps busy (tab1 r02ev: 2 BC1 textures 2.08 ms with jobs vs 1.99 per texel)
          if (NTBC_EPI_JOBS == 2 && !NAIVE) pack_tile_warp(j + sl, sl);
          else if (NTBC_EPI_JOBS == 1 && !NAIVE && p.n_tex >= 3) pack_tile_jobs(j + sl, sl);
          else pack_tile(j + sl, sl);
        }
      }
    }
    if (!DUMP && p.progress) {  // publish the finished unit: group barrier, then one system-scope release
      named_bar_sync(bar_id, 128);
      if (r == 0) {
        __threadfence_system();   // the consumer is the copy engine (measured: same cost as a gpu fence)
        const int row = u / p.units_per_row;
        const int chunk = row < p.tail_row0 ? row / p.chunk_rows
                                            : p.tail_row0 / p.chunk_rows + (row - p.tail_row0) / p.tail_rows;
        atomicAdd(p.progress + chunk, 1ull);
      }
    }
    u = p.next_unit ? *next_slot : u + ncta * NWG;
  }

  // the BC-word writers (lanes 0 and 16) order their stores at system scope before the kernel ends: the
  // out pointers may be another GPU's memory mapped over NVLink (the fused peer gather, ntbc_peer_open)
  if (!DUMP && (lane & 15) == 0) __threadfence_system();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem_base, kTmemCols);
}

// ---------------------------------------------------------------- kernel (2): standalone pack (a5-a8)
struct PackParams {
  const float* ep;   // [rows][BW][N_e]
  const float* col;  // [rows*4][W][N_c]
  int W, BW, rows, n_e, n_c, n_tex, tiles_per_row, n_tiles;
  int fmt[kMaxTex], ep_off[kMaxTex], col_off[kMaxTex];
  int pal_off[kMaxTex], pal_stride;   // per block: BC1 12 / BC4 8 palette floats per texture
  uint64_t* out[kMaxTex];
  int vec16;   // every out pointer 16-B aligned and BW even: two adjacent blocks' words per 16-byte store
};
#ifndef NTBC_PACK_TILE
#define NTBC_PACK_TILE 64
#endif
constexpr int kPackTileBlocks = NTBC_PACK_TILE;   // block positions per tile (one block row): 4 x kPackTileBlocks texel columns x 4 rows

#ifndef NTBC_PACK_STAGES
#define NTBC_PACK_STAGES 1      // tile buffers in shared memory: 2 = the next tile's loads overlap this tile's math
#endif
#ifndef NTBC_PACK_PAL
#define NTBC_PACK_PAL 0         // 0 = palette rebuilt per texel from the header; 1 = once per block for the whole
                                // tile in shared memory (+12 KB per CTA, measured slower: occupancy 5 -> 3 CTAs);
                                // 2 = once per block by the lanes of the warp that owns it, into a per-warp
                                // scratch of 2 x pal_stride floats (measured slower, r02f: 0.427 vs 0.410 ms --
                                // one lane per (block, texture) diverges on the format and indexes the
                                // parameter bank at run time)
#endif
#ifndef NTBC_PACK_THREADS
#define NTBC_PACK_THREADS 256
#endif
constexpr int kPackStages = NTBC_PACK_STAGES, kPackThreads = NTBC_PACK_THREADS;

// Per tile: the tile's fp32 MLP outputs (4 texel rows x 256 texels x N_c, and 64 x N_e) are staged in
// shared memory with asynchronous copies (cp.async, 16 B where the source is 16-B aligned, else 8 or 4 B;
// every input byte is read once, the only HBM traffic besides the BC words), issued one tile ahead into
// the other of kPackStages buffers when kPackStages = 2 (measured slower than one buffer with more CTAs
// per SM: the kernel is issue-bound); one thread per (block, texture) quantizes the
// endpoints into the BC word header (R11-R13) and builds the block's palette from it and the exact UNORM
// tables (Eq.7/8, R18) in shared memory; then one warp per two blocks, lane = texel, selects indices
// and packs the words with the fused kernel's epilogue functions.
__device__ __forceinline__ void pack_stage(float* dst, const float* src, int n) {
  const uint32_t d = smem_u32(dst);
  if ((((uintptr_t)src) & 15) == 0 && (n & 3) == 0) {
    for (int i = threadIdx.x; i < n / 4; i += blockDim.x)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + 16 * i), "l"(src + 4 * i) : "memory");
  } else if ((((uintptr_t)src) & 7) == 0 && (n & 1) == 0) {
    for (int i = threadIdx.x; i < n / 2; i += blockDim.x)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d + 8 * i), "l"(src + 2 * i) : "memory");
  } else {
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d + 4 * i), "l"(src + i) : "memory");
  }
}

__device__ __forceinline__ void pack_issue(const PackParams& p, int t, float* s_col, float* s_ep, int rs) {
  if (t < p.n_tiles) {
    const int row = t / p.tiles_per_row, bx0 = (t - row * p.tiles_per_row) * kPackTileBlocks;
    const int nb = min(kPackTileBlocks, p.BW - bx0);
    for (int yi = 0; yi < 4; yi++)
      pack_stage(s_col + yi * rs, p.col + ((size_t)(4 * row + yi) * p.W + 4 * bx0) * p.n_c, 4 * nb * p.n_c);
    pack_stage(s_ep, p.ep + ((size_t)row * p.BW + bx0) * p.n_e, nb * p.n_e);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");   // one group per tile (empty past the end)
}

// NT = the texture count as a template parameter (1..kMaxTex): the texture loop unrolls, so each texture's
// format, offsets and output pointer are immediates of the parameter bank instead of indexed loads
template <int NT>
__global__ void __launch_bounds__(kPackThreads) pack_kernel(const __grid_constant__ PackParams p) {
  extern __shared__ __align__(16) float psm[];
  float* s_unorm = psm;                                   // 352 UNORM quotients + 32 BC4 weights
  const int rs = 4 * kPackTileBlocks * p.n_c + 4;         // texel-row stride (+4 floats: rows start 4 banks apart)
  const int stage_floats = 4 * rs + ((kPackTileBlocks * p.n_e + 3) & ~3);
  float* s_pal = psm + 384 + kPackStages * stage_floats;                                   // [64][pal_stride]
  uint32_t* s_hdr = reinterpret_cast<uint32_t*>(s_pal + (NTBC_PACK_PAL == 1 ? kPackTileBlocks * p.pal_stride : 0));   // [64][kMaxTex]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  float* w_pal = reinterpret_cast<float*>(s_hdr + kPackTileBlocks * kMaxTex) + warp * 2 * p.pal_stride;   // [2][pal_stride]
  for (int i = tid; i < 352; i += blockDim.x)
    s_unorm[i] = i < 32 ? __fdiv_rn((float)i, 31.0f) : i < 96 ? __fdiv_rn((float)(i - 32), 63.0f)
                                                            : __fdiv_rn((float)(i - 96), 255.0f);
  if (tid < 32) s_unorm[352 + tid] = bc4_weight(tid);
#if NTBC_CHECKS
  NTBC_CHECK((uint32_t)(reinterpret_cast<uint8_t*>(NTBC_PACK_PAL == 2 ? w_pal + 2 * p.pal_stride
                                                                     : reinterpret_cast<float*>(s_hdr + kPackTileBlocks * kMaxTex)) -
                        reinterpret_cast<uint8_t*>(psm)) <= dyn_smem_bytes());
  for (int i = 384 + tid; i < 384 + kPackStages * stage_floats; i += blockDim.x)
    reinterpret_cast<uint32_t*>(psm)[i] = 0x7FC17FC1u;   // poison the staging buffers
  __syncthreads();
#endif
  int it = 0;
  if (kPackStages > 1) pack_issue(p, blockIdx.x, psm + 384, psm + 384 + 4 * rs, rs);
  for (int t = blockIdx.x; t < p.n_tiles; t += gridDim.x, it++) {
    const int row = t / p.tiles_per_row, bx0 = (t - row * p.tiles_per_row) * kPackTileBlocks;
    const int nb = min(kPackTileBlocks, p.BW - bx0);
    float* s_col = psm + 384 + (it % kPackStages) * stage_floats;   // [4][256 * N_c + 4]
    float* s_ep = s_col + 4 * rs;                                    // [64][N_e]
    __syncthreads();   // previous tile's readers are done (and the tables are written)
    if (kPackStages > 1) {
      float* n_col = psm + 384 + ((it + 1) % kPackStages) * stage_floats;
      pack_issue(p, t + gridDim.x, n_col, n_col + 4 * rs, rs);
      asm volatile("cp.async.wait_group 1;" ::: "memory");   // this tile's copies (issued one tile ago) landed
    } else {
      pack_issue(p, t, s_col, s_ep, rs);
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    for (int bk = tid; bk < nb * p.n_tex; bk += blockDim.x) {   // BC word headers (R11-R13) and palettes
      const int b = bk / p.n_tex, k = bk - b * p.n_tex;
      const float* e = s_ep + b * p.n_e + p.ep_off[k];
      float* dst = s_pal + b * p.pal_stride + p.pal_off[k];
      if (p.fmt[k] == kFmtBC1) {
        float ep6[6];
#pragma unroll
        for (int c = 0; c < 6; c++) ep6[c] = e[c];
        bool swapped;
        const uint32_t hdr = quant_bc1_hdr(ep6, swapped);
        s_hdr[b * kMaxTex + k] = hdr;
        if (NTBC_PACK_PAL == 1) {
          const uint32_t c0 = hdr & 0xFFFFu, c1 = hdr >> 16;
          const float e0[3] = {s_unorm[c0 >> 11], s_unorm[32 + ((c0 >> 5) & 63)], s_unorm[c0 & 31]};
          const float e1[3] = {s_unorm[c1 >> 11], s_unorm[32 + ((c1 >> 5) & 63)], s_unorm[c1 & 31]};
          bc1_palette_pairs(e0, e1, dst);
        }
      } else {
        const float ep2[2] = {e[0], e[1]};
        const uint32_t hdr = quant_bc4_hdr(ep2);
        s_hdr[b * kMaxTex + k] = hdr;
        if (NTBC_PACK_PAL == 1) {
          const uint32_t E0 = hdr & 0xFFu, E1 = (hdr >> 8) & 0xFFu;
          bc4_palette_tab(s_unorm[96 + E0], s_unorm[96 + E1], E0 > E1, s_unorm + 352, dst);
        }
      }
    }
    __syncthreads();
    for (int wb = 2 * warp; wb < nb; wb += 2 * (blockDim.x >> 5)) {   // warp = blocks wb, wb + 1
      const int h = lane >> 4, i = lane & 15, b = min(wb + h, nb - 1);
      const bool valid = wb + h < nb;
      const float* c = s_col + (i >> 2) * rs + (4 * b + (i & 3)) * p.n_c;
      // lane 0 writes both blocks' words as one 16-byte store (p.vec16; wb is even), else lanes 0 / 16
      const bool pair = p.vec16 && lane == 0 && wb + 1 < nb;
      const bool single = p.vec16 ? (lane == 0 && wb + 1 >= nb) : ((lane & 15) == 0 && valid);
      const size_t oidx = (size_t)row * p.BW + bx0 + wb + (p.vec16 ? 0 : h);   // texture-independent word index
      NTBC_CHECK(!(pair || single) || (bx0 + wb + (pair ? 1 : p.vec16 ? 0 : h) < p.BW && row < p.rows));
      if (NTBC_PACK_PAL == 2) {   // the two blocks' palettes, one (block, texture) per lane
        __syncwarp();             // the previous pair's readers are done
        if (lane < 2 * NT) {
          const int hh = lane >= NT, k = lane - hh * NT, bb = min(wb + hh, nb - 1);
          const uint32_t hdr = s_hdr[bb * kMaxTex + k];
          float* dst = w_pal + hh * p.pal_stride + p.pal_off[k];
          if (p.fmt[k] == kFmtBC1) {
            const uint32_t c0 = hdr & 0xFFFFu, c1 = hdr >> 16;
            const float e0[3] = {s_unorm[c0 >> 11], s_unorm[32 + ((c0 >> 5) & 63)], s_unorm[c0 & 31]};
            const float e1[3] = {s_unorm[c1 >> 11], s_unorm[32 + ((c1 >> 5) & 63)], s_unorm[c1 & 31]};
            bc1_palette_pairs(e0, e1, dst);
          } else {
            const uint32_t E0 = hdr & 0xFFu, E1 = (hdr >> 8) & 0xFFu;
            bc4_palette_tab(s_unorm[96 + E0], s_unorm[96 + E1], E0 > E1, s_unorm + 352, dst);
          }
        }
        __syncwarp();
      }
      // the words of texture k: header | index field << SHIFT (lane 0: both blocks, one 16-byte store)
      auto store = [&](int k, uint32_t hdr, const uint64_t* idx, int shift) {
        if (pair) st_words2(p.out[k] + oidx, (uint64_t)hdr | (idx[0] << shift),
                            (uint64_t)s_hdr[(b + 1) * kMaxTex + k] | (idx[1] << shift));
        else if (single) p.out[k][oidx] = (uint64_t)hdr | ((lane < 16 ? idx[0] : idx[1]) << shift);
      };
#pragma unroll
      for (int k = 0; k < NT; k++) {
        const uint32_t hdr = s_hdr[b * kMaxTex + k];
        const int co = p.col_off[k];
        uint64_t idx[2];
        const float* P = NTBC_PACK_PAL == 2 ? w_pal + h * p.pal_stride + p.pal_off[k] : s_pal + b * p.pal_stride + p.pal_off[k];
        // texture loop unrolled over NT: format, offsets and output pointer are parameter-bank immediates
        // (measured faster than BC1-then-BC4 runtime loops over index lists, r02i: 0.410 vs 0.461 ms)
        if (NTBC_PACK_PAL && p.fmt[k] == kFmtBC1) {
          const float cc[3] = {c[co], c[co + 1], c[co + 2]};
          pack_bc1_indices2(bc1_code_pairs(cc, reinterpret_cast<const float2*>(P), (hdr & 0xFFFFu) == (hdr >> 16)), lane, idx);
          store(k, hdr, idx, 32);
        } else if (NTBC_PACK_PAL) {
          const float4 q0 = reinterpret_cast<const float4*>(P)[0], q1 = reinterpret_cast<const float4*>(P)[1];
          const float pl[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
          pack_bc4_indices2(bc4_code(c[co], pl, (hdr & 0xFFu) > ((hdr >> 8) & 0xFFu)), lane, idx);
          store(k, hdr, idx, 16);
        } else if (p.fmt[k] == kFmtBC1) {
          const uint32_t c0 = hdr & 0xFFFFu, c1 = hdr >> 16;
          const float e0[3] = {s_unorm[c0 >> 11], s_unorm[32 + ((c0 >> 5) & 63)], s_unorm[c0 & 31]};
          const float e1[3] = {s_unorm[c1 >> 11], s_unorm[32 + ((c1 >> 5) & 63)], s_unorm[c1 & 31]};
          const float cc[3] = {c[co], c[co + 1], c[co + 2]};
          pack_bc1_indices2(bc1_code(cc, e0, e1, c0 == c1), lane, idx);
          store(k, hdr, idx, 32);
        } else {
          const uint32_t E0 = hdr & 0xFFu, E1 = (hdr >> 8) & 0xFFu;
          float pl[8];
          bc4_palette_tab(s_unorm[96 + E0], s_unorm[96 + E1], E0 > E1, s_unorm + 352, pl);
          pack_bc4_indices2(bc4_code(c[co], pl, E0 > E1), lane, idx);
          store(k, hdr, idx, 16);
        }
      }
    }
  }
}

// Kernel (2), thread-per-(block, texture) form (the default since r02): 64 x NT threads per CTA, thread
// j = k * 64 + b owns texture k of block b of the tile.  It quantizes the block's endpoints (R11-R13), builds
// the palette ONCE in registers (Eq.7/8, R18), then walks the block's 16 texels (argmin of Eq.9-10, R14/R15)
// accumulating the index field with shifts -- no per-texel palette rebuild, no warp reductions -- and stores
// its word; the 32 lanes of a warp hold 32 consecutive blocks of one texture, so the stores are coalesced
// (even lanes write two adjacent words as one 16-byte store when p.vec16).  Same tile staging (cp.async) as
// pack_kernel.
#ifndef NTBC_PACK_BT_THREADS
#define NTBC_PACK_BT_THREADS 1280   // launch-bounds target of resident threads per SM (register budget)
#endif
#ifndef NTBC_PACK_BT_TILE
#define NTBC_PACK_BT_TILE 32    // block positions per tile of pack_kernel_bt (threads = tile x textures); C3 A/B
                                // r02v/w: 32 -> 0.156 ms (0.707 of HBM), 64 -> 0.164, 128 -> 0.174, 16 -> 0.182
#endif
#ifndef NTBC_PACK_BT_STAGES
#define NTBC_PACK_BT_STAGES 1   // 2: the next tile's bulk copies in flight during this tile's work (r02t: slower,
                                // 0.172 vs 0.164 ms -- half the CTAs per SM; 32-block tiles x 2 stages 0.176)
#endif
constexpr int kBtTile = NTBC_PACK_BT_TILE, kBtStages = NTBC_PACK_BT_STAGES;
// min blocks per SM = 1,280 threads' worth: <= 51 registers (four 320-thread CTAs for C3)
template <int NT>
__global__ void __launch_bounds__(kBtTile * NT, (NTBC_PACK_BT_THREADS / (kBtTile * NT)) > 32 ? 32
                                                 : (NTBC_PACK_BT_THREADS / (kBtTile * NT)) > 2 ? (NTBC_PACK_BT_THREADS / (kBtTile * NT)) : 2)
    pack_kernel_bt(const __grid_constant__ PackParams p) {
  extern __shared__ __align__(16) float psm[];
  float* s_unorm = psm;                                   // 352 UNORM quotients + 32 BC4 weights
  const int rs = 4 * kBtTile * p.n_c;                     // texel-row stride of a staged tile (floats)
  const int ep_floats = (kBtTile * p.n_e + 3) & ~3;
  const int stage_floats = 4 * rs + ep_floats;            // one stage: [4][4 tile N_c] colours, [tile][N_e] endpoints
  uint64_t* bar = reinterpret_cast<uint64_t*>(psm + 384 + kBtStages * stage_floats);   // one per stage
  const int tid = threadIdx.x, lane = tid & 31;
  const int k = tid / kBtTile, b = tid - k * kBtTile;     // texture, block of the tile
  for (int i = tid; i < 352; i += blockDim.x)
    s_unorm[i] = i < 32 ? __fdiv_rn((float)i, 31.0f) : i < 96 ? __fdiv_rn((float)(i - 32), 63.0f)
                                                            : __fdiv_rn((float)(i - 96), 255.0f);
  if (tid < 32) s_unorm[352 + tid] = bc4_weight(tid);
  if (tid == 0) {
    for (int q = 0; q < kBtStages; q++) mbar_init(bar + q, 1);
    fence_mbar_init();
  }
#if NTBC_CHECKS
  NTBC_CHECK((uint32_t)(reinterpret_cast<uint8_t*>(bar + kBtStages) - reinterpret_cast<uint8_t*>(psm)) <= dyn_smem_bytes());
  for (int i = 384 + tid; i < 384 + kBtStages * stage_floats; i += blockDim.x)
    reinterpret_cast<uint32_t*>(psm)[i] = 0x7FC17FC1u;   // poison the staging buffers
  fence_async_smem();
#endif
  __syncthreads();
  // per-texture parameters of this thread (k is warp-uniform: kBtTile threads per texture)
  const int fmt = p.fmt[k], eo = p.ep_off[k], co = p.col_off[k];
  uint64_t* const out = p.out[k];
  const int tpr = (p.BW + kBtTile - 1) / kBtTile, n_tiles = tpr * p.rows;
  // the tile's fp32 MLP outputs: 4 texel-row segments (16-B aligned, 16 nb N_c bytes each) and the endpoints,
  // by bulk asynchronous copies (TMA engine) issued by one thread into stage q; the endpoints by plain loads
  // of all threads when their segment is not 16-B aligned (N_e x the block index odd)
  auto issue = [&](int t, int q) {   // thread 0 only
    const int row = t / tpr, bx0 = (t - row * tpr) * kBtTile, nb = min(kBtTile, p.BW - bx0);
    float* s_col = psm + 384 + q * stage_floats;
    const float* ep_src = p.ep + ((size_t)row * p.BW + bx0) * p.n_e;
    const uint32_t ep_bytes = (uint32_t)(nb * p.n_e * 4), row_bytes = (uint32_t)(16 * nb * p.n_c);
    const bool ep_bulk = ((((uintptr_t)ep_src) | ep_bytes) & 15) == 0;
    mbar_arrive_expect_tx(bar + q, 4 * row_bytes + (ep_bulk ? ep_bytes : 0));
    for (int yi = 0; yi < 4; yi++)
      bulk_g2s(s_col + yi * rs, p.col + ((size_t)(4 * row + yi) * p.W + 4 * bx0) * p.n_c, row_bytes, bar + q);
    if (ep_bulk) bulk_g2s(s_col + 4 * rs, ep_src, ep_bytes, bar + q);
  };
  uint32_t phase[kBtStages];
  for (int q = 0; q < kBtStages; q++) phase[q] = 0;
  if (tid == 0 && (int)blockIdx.x < n_tiles) issue(blockIdx.x, 0);
  int it = 0;
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, it++) {
    const int q = kBtStages > 1 ? (it & 1) : 0;
    const int row = t / tpr, bx0 = (t - row * tpr) * kBtTile;
    const int nb = min(kBtTile, p.BW - bx0);
    float* s_col = psm + 384 + q * stage_floats;           // [4][4 tile N_c]
    float* s_ep = s_col + 4 * rs;                          // [tile][N_e]
    const float* ep_src = p.ep + ((size_t)row * p.BW + bx0) * p.n_e;
    const bool ep_bulk = ((((uintptr_t)ep_src) | (uint32_t)(nb * p.n_e * 4)) & 15) == 0;
    if (kBtStages > 1) {
      __syncthreads();   // every thread is done with the other stage (the previous tile)
      if (tid == 0 && t + (int)gridDim.x < n_tiles) issue(t + gridDim.x, q ^ 1);
    } else if (it > 0) {
      __syncthreads();   // every thread is done with the stage
      if (tid == 0) issue(t, 0);
    }
    if (!ep_bulk) {
      if (kBtStages == 1) __syncthreads();
      for (int i = tid; i < nb * p.n_e; i += blockDim.x) s_ep[i] = ep_src[i];
      __syncthreads();
    }
    mbar_wait(bar + q, phase[q]);
    phase[q] ^= 1u;
    const int bb = min(b, nb - 1);
    const float* e = s_ep + bb * p.n_e + eo;
    const float* c = s_col + 4 * bb * p.n_c + co;        // texel (x, y) of the block at c + y rs + x n_c
    uint64_t word;
    if (fmt == kFmtBC1) {
      float ep6[6];
#pragma unroll
      for (int j = 0; j < 6; j++) ep6[j] = e[j];
      bool swapped;
      const uint32_t hdr = quant_bc1_hdr(ep6, swapped);
      const uint32_t c0 = hdr & 0xFFFFu, c1 = hdr >> 16;
      const float e0[3] = {s_unorm[c0 >> 11], s_unorm[32 + ((c0 >> 5) & 63)], s_unorm[c0 & 31]};
      const float e1[3] = {s_unorm[c1 >> 11], s_unorm[32 + ((c1 >> 5) & 63)], s_unorm[c1 & 31]};
      float pal[12];
      bc1_palette_pairs(e0, e1, pal);
      const bool degenerate = c0 == c1;
      uint32_t bits = 0;
#pragma unroll
      for (int i = 0; i < 16; i++) {
        const float* ci = c + (i >> 2) * rs + (i & 3) * p.n_c;
        const float cc[3] = {ci[0], ci[1], ci[2]};
        bits |= bc1_code_pairs(cc, reinterpret_cast<const float2*>(pal), degenerate) << (2 * i);
      }
      word = (uint64_t)hdr | ((uint64_t)bits << 32);
    } else {
      const float ep2[2] = {e[0], e[1]};
      const uint32_t hdr = quant_bc4_hdr(ep2);
      const uint32_t E0 = hdr & 0xFFu, E1 = (hdr >> 8) & 0xFFu;
      float pl[8];
      bc4_palette_tab(s_unorm[96 + E0], s_unorm[96 + E1], E0 > E1, s_unorm + 352, pl);
      uint64_t bits = 0;
      if (E0 != E1) {   // strictly monotone palette: the one-select argmin (bc4_code_mono)
#pragma unroll
        for (int i = 0; i < 16; i++)
          bits |= (uint64_t)bc4_code_mono(c[(i >> 2) * rs + (i & 3) * p.n_c], pl, E0 > E1) << (3 * i);
      } else {
#pragma unroll 1
        for (int i = 0; i < 16; i++)
          bits |= (uint64_t)bc4_code(c[(i >> 2) * rs + (i & 3) * p.n_c], pl, false) << (3 * i);
      }
      word = (uint64_t)hdr | (bits << 16);
    }
    const size_t oidx = (size_t)row * p.BW + bx0 + b;
    if (p.vec16) {   // b even: this lane and the next hold two adjacent words -> one 16-byte store
      const uint64_t next = __shfl_down_sync(0xFFFFFFFFu, word, 1);
      NTBC_CHECK(!((lane & 1) == 0 && b < nb) || (bx0 + b < p.BW && row < p.rows));
      if ((lane & 1) == 0 && b + 1 < nb) st_words2(out + oidx, word, next);
      else if ((lane & 1) == 0 && b < nb) out[oidx] = word;
    } else if (b < nb) {
      out[oidx] = word;
    }
  }
}

// ---------------------------------------------------------------- kernel (3): BC decode (a9)
__global__ void __launch_bounds__(256) decode_bc_kernel(const uint64_t* __restrict__ blocks, int fmt, int W, int H,
                                                         float* __restrict__ out) {
  const long long n = (long long)W * H;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(t % W), y = (int)(t / W);
    const int BW = W / 4;
    const uint64_t blk = __ldg(blocks + (size_t)(y >> 2) * BW + (x >> 2));
    const int i = (y & 3) * 4 + (x & 3);
    if (fmt == kFmtBC1) {
      const uint32_t c0 = (uint32_t)(blk & 0xFFFF), c1 = (uint32_t)((blk >> 16) & 0xFFFF);
      const uint32_t code = (uint32_t)(blk >> (32 + 2 * i)) & 3u;
      float e0[3], e1[3];
      e0[0] = __fdiv_rn((float)(c0 >> 11), 31.0f); e0[1] = __fdiv_rn((float)((c0 >> 5) & 63), 63.0f);
      e0[2] = __fdiv_rn((float)(c0 & 31), 31.0f);
      e1[0] = __fdiv_rn((float)(c1 >> 11), 31.0f); e1[1] = __fdiv_rn((float)((c1 >> 5) & 63), 63.0f);
      e1[2] = __fdiv_rn((float)(c1 & 31), 31.0f);
      // 4-colour mode: code -> linear n = [0,3,1,2] -> weights n/3 (R18)
      const int n_lin = (0x2130 >> (4 * code)) & 3;
      const float w = n_lin == 0 ? 0.0f : n_lin == 1 ? NTBC_W3_1 : n_lin == 2 ? NTBC_W3_2 : 1.0f;
      const float wb = n_lin == 0 ? 1.0f : n_lin == 1 ? NTBC_WB3_1 : n_lin == 2 ? NTBC_WB3_2 : 0.0f;
      float v[3];
#pragma unroll
      for (int ch = 0; ch < 3; ch++) {
        if (c0 > c1) v[ch] = interp_c(w, wb, e0[ch], e1[ch]);
        else  // DirectX 3-colour mode (never emitted by the encoder, R12)
          v[ch] = code == 0 ? e0[ch] : code == 1 ? e1[ch] : code == 2 ? __fmaf_rn(0.5f, e1[ch], __fmul_rn(0.5f, e0[ch])) : 0.0f;
      }
      float* o = out + (size_t)t * 3;
      o[0] = v[0]; o[1] = v[1]; o[2] = v[2];
    } else {
      const uint32_t E0 = (uint32_t)(blk & 0xFF), E1 = (uint32_t)((blk >> 8) & 0xFF);
      const uint32_t code = (uint32_t)(blk >> (16 + 3 * i)) & 7u;
      float pl[8];
      bc4_palette(E0 | (E1 << 8), pl);
      // code -> linear n: mode8 0->0, 1->7, c->c-1; mode6 0->1, 1->6, 2..5->same, 6->0, 7->7
      const int n_lin = E0 > E1 ? (code == 0 ? 0 : code == 1 ? 7 : (int)code - 1)
                                : (code == 0 ? 1 : code == 1 ? 6 : code == 6 ? 0 : (int)code);
      float v = pl[0];
#pragma unroll
      for (int n = 1; n < 8; n++) v = n_lin == n ? pl[n] : v;
      out[t] = v;
    }
  }
}

// ---------------------------------------------------------------- tensor-core summation probe (R10)
__global__ void __launch_bounds__(128, 1) mma_probe_kernel(const __half* __restrict__ A, const __half* __restrict__ B,
                                                           const float* __restrict__ C, float* __restrict__ D, int K,
                                                           int N) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + 128 * K * 2;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sB + 64 * K * 2);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int r = threadIdx.x, warp = r >> 5;
  for (int k = 0; k < K; k++) {
    *reinterpret_cast<__half*>(sA + kmajor_offset(r, k, K)) = A[(size_t)r * K + k];
    if (r < N) *reinterpret_cast<__half*>(sB + kmajor_offset(r, k, K)) = B[(size_t)r * K + k];
  }
  fence_async_smem();
  if (r == 0) { mbar_init(bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(slot, 64);
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *slot, trow = tbase + ((uint32_t)(32 * warp) << 16);
  if (C) {
    for (int c = 0; c < N; c += 16) {
      uint32_t v[16];
#pragma unroll
      for (int j = 0; j < 16; j++) v[j] = __float_as_uint(C[(size_t)r * N + c + j]);
      tmem_st16(trow + c, v);
    }
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  if (r == 0) {
    tc_fence_after();
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB), idesc = idesc_f16_f32(128, N);
    for (int c = 0; c < K / 16; c++)
      mma_f16(tbase, smem_desc(a0 + c * 256, 128, K * 16), smem_desc(b0 + c * 256, 128, K * 16), idesc,
              (C != nullptr || c > 0) ? 1u : 0u);
    mma_commit(bar);
  }
  mbar_wait(bar, 0);
  tc_fence_after();
  for (int c = 0; c < N; c += 16) {
    uint32_t v[16];
    tmem_ld16p(trow + c, v);
    tmem_wait_ld16(v);
#pragma unroll
    for (int j = 0; j < 16; j++) D[(size_t)r * N + c + j] = __uint_as_float(v[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 64);
}

}  // namespace ntbc
