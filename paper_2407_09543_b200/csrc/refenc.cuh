// refenc.cuh -- reference BC1/BC4 encoder on sm_100a (SPEC encode_block_reference
// S:153-161, the documented stand-in for the paper's Compressonator "two refine steps").
//
// One thread per 4x4 block, fp32 texels [H][W][C] (C = 3 -> BC1, C = 1 -> BC4) read row by row (a warp
// covers 32 horizontally adjacent blocks: 512 B / 1.5 KB contiguous per texel row), the whole block
// in registers, one 8-byte store.  The arithmetic is the pinned reading of DESIGN.md R24-R29 in its
// stated op order (explicit __fmaf_rn, IEEE division, --fmad=false), so the words are bit-identical
// to the oracle's independent implementation.
#pragma once
#include <cstdint>

#include "bc_device.cuh"

namespace ntbc {

__device__ __forceinline__ float clamp01f(float x) { return fminf(fmaxf(x, 0.0f), 1.0f); }

__device__ __forceinline__ uint32_t enc565(const float* e) {
  return (qbits(e[0], 31.0f) << 11) | (qbits(e[1], 63.0f) << 5) | qbits(e[2], 31.0f);
}
__device__ __forceinline__ void dec565(uint32_t c, float* o) {
  o[0] = __fdiv_rn((float)(c >> 11), 31.0f);
  o[1] = __fdiv_rn((float)((c >> 5) & 63u), 63.0f);
  o[2] = __fdiv_rn((float)(c & 31u), 31.0f);
}

// BC1 palette entry n of (q0, q1) and the linear argmin (squared distance, strict <: ties -> lower n)
__device__ __forceinline__ int bc1_nearest(const float* x, const float (*pal)[3]) {
  int best = 0;
  float bd = 0.0f;
#pragma unroll
  for (int n = 0; n < 4; n++) {
    const float dr = x[0] - pal[n][0], dg = x[1] - pal[n][1], db = x[2] - pal[n][2];
    const float d = __fmaf_rn(db, db, __fmaf_rn(dg, dg, dr * dr));
    if (n == 0 || d < bd) { bd = d; best = n; }
  }
  return best;
}
__device__ __forceinline__ void bc1_pal(const float* q0, const float* q1, float (*pal)[3]) {
  const float w[4] = {0.0f, NTBC_W3_1, NTBC_W3_2, 1.0f}, wb[4] = {1.0f, NTBC_WB3_1, NTBC_WB3_2, 0.0f};
#pragma unroll
  for (int n = 0; n < 4; n++)
#pragma unroll
    for (int c = 0; c < 3; c++) pal[n][c] = interp_c(w[n], wb[n], q0[c], q1[c]);
}

// least squares for (e0, e1) of nc channels given per-texel weights (R26); false: keep the old ones
template <int NC>
__device__ __forceinline__ bool ls_fit(const float* w, const float* x, const bool* use, float* e0, float* e1) {
  float A = 0.0f, B = 0.0f, D = 0.0f, P[NC], Q[NC];
#pragma unroll
  for (int c = 0; c < NC; c++) { P[c] = 0.0f; Q[c] = 0.0f; }
#pragma unroll
  for (int i = 0; i < 16; i++) {
    if (use && !use[i]) continue;
    const float wi = w[i], wb = 1.0f - wi;
    A = __fmaf_rn(wb, wb, A);
    B = __fmaf_rn(wi, wb, B);
    D = __fmaf_rn(wi, wi, D);
#pragma unroll
    for (int c = 0; c < NC; c++) {
      P[c] = __fmaf_rn(wb, x[i * NC + c], P[c]);
      Q[c] = __fmaf_rn(wi, x[i * NC + c], Q[c]);
    }
  }
  const float det = __fmaf_rn(A, D, -(B * B));
  if (!(det > 0.0f)) return false;
#pragma unroll
  for (int c = 0; c < NC; c++) {
    e0[c] = clamp01f(__fdiv_rn(__fmaf_rn(D, P[c], -(B * Q[c])), det));
    e1[c] = clamp01f(__fdiv_rn(__fmaf_rn(A, Q[c], -(B * P[c])), det));
  }
  return true;
}

__device__ __forceinline__ uint64_t ref_encode_bc1(const float* x, int n_refine) {
  // ---- R24/R25: mean, covariance, power iteration from the largest-variance covariance column
  float mu[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
  for (int i = 0; i < 16; i++)
#pragma unroll
    for (int c = 0; c < 3; c++) mu[c] = mu[c] + x[3 * i + c];
#pragma unroll
  for (int c = 0; c < 3; c++) mu[c] = mu[c] * 0.0625f;
  float c00 = 0.0f, c01 = 0.0f, c02 = 0.0f, c11 = 0.0f, c12 = 0.0f, c22 = 0.0f;
#pragma unroll
  for (int i = 0; i < 16; i++) {
    const float d0 = x[3 * i] - mu[0], d1 = x[3 * i + 1] - mu[1], d2 = x[3 * i + 2] - mu[2];
    c00 = __fmaf_rn(d0, d0, c00); c01 = __fmaf_rn(d0, d1, c01); c02 = __fmaf_rn(d0, d2, c02);
    c11 = __fmaf_rn(d1, d1, c11); c12 = __fmaf_rn(d1, d2, c12); c22 = __fmaf_rn(d2, d2, c22);
  }
  const float C[3][3] = {{c00, c01, c02}, {c01, c11, c12}, {c02, c12, c22}};
  int k = 0;
  if (C[1][1] > C[k][k]) k = 1;
  if (C[2][2] > C[k][k]) k = 2;
  float v[3] = {C[0][k], C[1][k], C[2][k]};
  bool ok = C[k][k] > 0.0f;
  for (int it = 0; it < 8 && ok; it++) {
    float u[3];
#pragma unroll
    for (int a = 0; a < 3; a++) u[a] = __fmaf_rn(C[a][2], v[2], __fmaf_rn(C[a][1], v[1], C[a][0] * v[0]));
    const float m = fmaxf(fabsf(u[0]), fmaxf(fabsf(u[1]), fabsf(u[2])));
    if (!(m > 0.0f)) { ok = false; break; }
#pragma unroll
    for (int a = 0; a < 3; a++) v[a] = __fdiv_rn(u[a], m);
  }
  float e0[3], e1[3];
  if (!ok) {   // zero covariance: per-channel max / min
#pragma unroll
    for (int c = 0; c < 3; c++) { e0[c] = x[c]; e1[c] = x[c]; }
#pragma unroll
    for (int i = 1; i < 16; i++)
#pragma unroll
      for (int c = 0; c < 3; c++) { e0[c] = fmaxf(e0[c], x[3 * i + c]); e1[c] = fminf(e1[c], x[3 * i + c]); }
  } else {
    float tmin = 0.0f, tmax = 0.0f;
#pragma unroll
    for (int i = 0; i < 16; i++) {
      const float t = __fmaf_rn(x[3 * i + 2] - mu[2], v[2], __fmaf_rn(x[3 * i + 1] - mu[1], v[1], (x[3 * i] - mu[0]) * v[0]));
      if (i == 0 || t < tmin) tmin = t;
      if (i == 0 || t > tmax) tmax = t;
    }
    const float vv = __fmaf_rn(v[2], v[2], __fmaf_rn(v[1], v[1], v[0] * v[0]));
    const float smax = __fdiv_rn(tmax, vv), smin = __fdiv_rn(tmin, vv);
#pragma unroll
    for (int c = 0; c < 3; c++) { e0[c] = clamp01f(__fmaf_rn(smax, v[c], mu[c])); e1[c] = clamp01f(__fmaf_rn(smin, v[c], mu[c])); }
  }
  uint32_t q0c = enc565(e0), q1c = enc565(e1);
  // ---- R26: n_refine least-squares refinements on the current assignment
  for (int rr = 0; rr < n_refine && q0c != q1c; rr++) {
    float q0[3], q1[3], pal[4][3], w[16];
    dec565(q0c, q0);
    dec565(q1c, q1);
    bc1_pal(q0, q1, pal);
#pragma unroll
    for (int i = 0; i < 16; i++) w[i] = __fdiv_rn((float)bc1_nearest(x + 3 * i, pal), 3.0f);
    float n0[3], n1[3];
    if (!ls_fit<3>(w, x, nullptr, n0, n1)) break;
    q0c = enc565(n0);
    q1c = enc565(n1);
  }
  // ---- final word: 4-colour order, per-texel argmin on the final palette (R12, R16)
  if (q0c < q1c) { const uint32_t t = q0c; q0c = q1c; q1c = t; }
  uint64_t word = (uint64_t)q0c | ((uint64_t)q1c << 16);
  if (q0c == q1c) return word;
  float q0[3], q1[3], pal[4][3];
  dec565(q0c, q0);
  dec565(q1c, q1);
  bc1_pal(q0, q1, pal);
#pragma unroll
  for (int i = 0; i < 16; i++) word |= (uint64_t)((0x1320u >> (4 * bc1_nearest(x + 3 * i, pal))) & 3u) << (32 + 2 * i);
  return word;
}

// BC4: one mode's candidate (R27-R29)
__device__ __forceinline__ int bc4_nearest(float x, const float* pal, float* dist = nullptr) {
  int best = 0;
  float bd = 0.0f;
#pragma unroll
  for (int n = 0; n < 8; n++) {
    const float d = fabsf(x - pal[n]);
    if (n == 0 || d < bd) { bd = d; best = n; }
  }
  if (dist) *dist = bd;   // |x - pal[best]|: its square is the oracle's (x - pal[n])^2 exactly
  return best;
}
__device__ __forceinline__ void bc4_order_mode(bool mode8, uint32_t& E0, uint32_t& E1) {
  if (mode8) {
    if (E0 < E1) { const uint32_t t = E0; E0 = E1; E1 = t; }
    if (E0 == E1) { if (E0 < 255u) E0++; else E1--; }
  } else if (E0 > E1) {
    const uint32_t t = E0; E0 = E1; E1 = t;
  }
}
__device__ __forceinline__ float bc4_cand_err(uint32_t E0, uint32_t E1, const float* x) {
  float pal[8], err = 0.0f;
  bc4_palette(E0 | (E1 << 8), pal);
#pragma unroll
  for (int i = 0; i < 16; i++) {
    float d;
    bc4_nearest(x[i], pal, &d);
    err = __fmaf_rn(d, d, err);
  }
  return err;
}
__device__ __forceinline__ float bc4_candidate(bool mode8, const float* x, int n_refine, uint32_t& oE0, uint32_t& oE1) {
  float lo = 2.0f, hi = -1.0f;
#pragma unroll
  for (int i = 0; i < 16; i++) {
    if (!mode8 && (x[i] == 0.0f || x[i] == 1.0f)) continue;
    lo = fminf(lo, x[i]);
    hi = fmaxf(hi, x[i]);
  }
  if (hi < lo) { lo = 0.0f; hi = 1.0f; }
  uint32_t E0 = (uint32_t)qbits(mode8 ? hi : lo, 255.0f), E1 = (uint32_t)qbits(mode8 ? lo : hi, 255.0f);
  bc4_order_mode(mode8, E0, E1);
  for (int rr = 0; rr < n_refine; rr++) {
    float pal[8], w[16];
    bool use[16];
    bc4_palette(E0 | (E1 << 8), pal);
#pragma unroll
    for (int i = 0; i < 16; i++) {
      const int n = bc4_nearest(x[i], pal);
      use[i] = mode8 || (n >= 1 && n <= 6);
      w[i] = mode8 ? __fdiv_rn((float)n, 7.0f) : __fdiv_rn((float)(n - 1), 5.0f);
    }
    float e0, e1;
    if (!ls_fit<1>(w, x, use, &e0, &e1)) break;
    E0 = (uint32_t)qbits(e0, 255.0f);
    E1 = (uint32_t)qbits(e1, 255.0f);
    bc4_order_mode(mode8, E0, E1);
  }
  oE0 = E0;
  oE1 = E1;
  return bc4_cand_err(E0, E1, x);
}
__device__ __forceinline__ uint64_t ref_encode_bc4(const float* x, int n_refine) {
  uint32_t a0, a1, b0, b1;
  const float ea = bc4_candidate(true, x, n_refine, a0, a1), eb = bc4_candidate(false, x, n_refine, b0, b1);
  if (eb < ea) { a0 = b0; a1 = b1; }   // lower error; ties -> the 8-value mode
  float pal[8];
  bc4_palette(a0 | (a1 << 8), pal);
  const uint32_t map = a0 > a1 ? 0x17654320u : 0x71543206u;
  uint64_t word = (uint64_t)a0 | ((uint64_t)a1 << 8);
#pragma unroll
  for (int i = 0; i < 16; i++) word |= (uint64_t)((map >> (4 * bc4_nearest(x[i], pal))) & 7u) << (16 + 3 * i);
  return word;
}

template <int C>
__global__ void __launch_bounds__(128) refenc_kernel(const float* __restrict__ tex, int W, int H, int n_refine,
                                                     uint64_t* __restrict__ out) {
  const int BW = W / 4, BH = H / 4;
  const long long nb = (long long)BW * BH;
  for (long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (long long)gridDim.x * blockDim.x) {
    const int by = (int)(b / BW), bx = (int)(b % BW);
    float x[16 * C];
#pragma unroll
    for (int yy = 0; yy < 4; yy++) {
      const float* row = tex + ((size_t)(4 * by + yy) * W + 4 * bx) * C;
#pragma unroll
      for (int j = 0; j < 4 * C; j++) x[yy * 4 * C + j] = __ldg(row + j);
    }
    out[b] = C == 3 ? ref_encode_bc1(x, n_refine) : ref_encode_bc4(x, n_refine);
  }
}

}  // namespace ntbc
