// train.cuh -- one training step of the NTBC colour network on sm_100a.
//
// PAPER.md: loss L_color = L_c + L_cd (Eq. 14-15) with the colour-network index rule
// (P:274-285), STE through the argmax as the softmax expectation (App. A, T = 0.01), Adam
// with separate grid / MLP learning rates.  DESIGN.md R30-R32 fix the parameter layout,
// the batch-mean loss and this implementation's precision (fp32 throughout, CUDA cores).
//
// Kernel (1) train_step_kernel: one CTA = 128 samples, four threads per sample (each owns a quarter of
// every layer's outputs and inputs).  The MLP
// weights live in shared memory; the layer inputs of the tile (features, three hidden activations)
// are kept in shared memory for the backward pass (selu' is recovered from the activation:
// lambda for a > 0, a + lambda*alpha otherwise).  Weight gradients are reduced over the tile in
// shared memory and added to the global gradient with one atomic per weight per CTA; the grid
// gradient is scattered with atomics (4 vertices x 2 features per level per sample).
// Kernel (2) adam_kernel: bias-corrected Adam over the flat parameter vector.
// The library is compiled with --fmad=false (bit-exact inference); the training loops use explicit
// __fmaf_rn so their dot products still run as FFMA.
#pragma once
#include <cstdint>

namespace ntbc {

constexpr int kTrainTile = 128;
constexpr int kTrainQ = 4;     // threads per sample
constexpr float kSeluL = 1.0507009873554804934f, kSeluLA = 1.0507009873554804934f * 1.6732632423543772848f;

struct TrainParams {
  int n_tex, fmt[kMaxTex], hidden, levels, coarsest, n_c, n_e;
  long long lvl_off[kMaxLevels];      // offsets (floats) of the grid levels in the parameter vector
  long long w_off[4], b_off[4];       // offsets of W_l [in][out] and b_l [out]
  int kin[4], kout[4];
  const float* params;
  float* grads;
  const int* xy;                      // [B][2] texel coordinates
  const float* cref;                  // colour net: [B][n_c] reference colours; endpoint net: [B][16][n_c]
  const float* eref;                  // [B][n_e] reference endpoints (BC1: e0 rgb, e1 rgb; BC4: e0, e1)
  int B, W, H;
  float T;
  float* loss;                        // += batch-mean loss
  const float* qsz;                   // QAT: per level (s, z) of the 8-bit fake quantizer, or nullptr
};

// Eq. 1/3 rounding, read as half away from zero (R33): roundf
// QAT fake quantizer (Eq. 3) of one grid value in binary32; `pass` = 1 where not clamped (STE)
__device__ __forceinline__ float fake_quant(float w, const float* qsz, int l, float& pass) {
  pass = 1.0f;
  if (!qsz) return w;
  const float s = qsz[2 * l], z = qsz[2 * l + 1];
  if (!(s > 0.0f)) return w;
  const float r = roundf(__fdiv_rn(w, s)) + z;
  const float q = fminf(fmaxf(r, 0.0f), 255.0f);
  pass = r == q ? 1.0f : 0.0f;
  return s * (q - z);
}

// per-level min / max of the grid (QAT ranges, Eq. 4): ordered-int atomics on [2*levels] slots
__device__ __forceinline__ int f2ord(float f) { const int i = __float_as_int(f); return i >= 0 ? i : i ^ 0x7FFFFFFF; }
__device__ __forceinline__ float ord2f(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7FFFFFFF); }
struct LevelList { long long off[kMaxLevels], cnt[kMaxLevels]; };
__global__ void __launch_bounds__(256) level_minmax_kernel(const float* __restrict__ params, const LevelList L,
                                                           int levels, int* __restrict__ mm) {
  const int l = blockIdx.y;
  if (l >= levels) return;
  int lo = 0x7FFFFFFF, hi = (int)0x80000000;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < L.cnt[l]; i += (long long)gridDim.x * blockDim.x) {
    const int o = f2ord(params[L.off[l] + i]);
    lo = min(lo, o);
    hi = max(hi, o);
  }
  for (int d = 16; d > 0; d >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xFFFFFFFFu, lo, d));
    hi = max(hi, __shfl_xor_sync(0xFFFFFFFFu, hi, d));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(mm + 2 * l, lo);
    atomicMax(mm + 2 * l + 1, hi);
  }
}
// s = (beta - alpha) / 255, z = round(-alpha / s) (Eq. 4-5, R4, R33), in binary32
__global__ void qat_params_kernel(const int* __restrict__ mm, int levels, float* __restrict__ qsz) {
  const int l = threadIdx.x;
  if (l >= levels) return;
  const float alpha = ord2f(mm[2 * l]), beta = ord2f(mm[2 * l + 1]);
  const float s = __fdiv_rn(beta - alpha, 255.0f);
  qsz[2 * l] = s;
  qsz[2 * l + 1] = s > 0.0f ? roundf(__fdiv_rn(-alpha, s)) : 0.0f;
}

__device__ __forceinline__ float selu_f(float z) { return z > 0.0f ? kSeluL * z : kSeluLA * (expf(z) - 1.0f); }

// reference palette of one texture (Eq. 7 / Eq. 8), linear order: BC1 4 x 3, BC4 8 x 1
__device__ __forceinline__ int train_palette(int fmt, const float* e, float* pal) {
  if (fmt == kFmtBC1) {
    for (int n = 0; n < 4; n++) {
      const float w = (float)n / 3.0f;
      for (int c = 0; c < 3; c++) pal[3 * n + c] = (1.0f - w) * e[c] + w * e[3 + c];
    }
    return 4;
  }
  if (e[0] > e[1]) {
    for (int n = 0; n < 8; n++) { const float w = (float)n / 7.0f; pal[n] = (1.0f - w) * e[0] + w * e[1]; }
  } else {
    pal[0] = 0.0f;
    for (int n = 1; n <= 6; n++) { const float w = (float)(n - 1) / 5.0f; pal[n] = (1.0f - w) * e[0] + w * e[1]; }
    pal[7] = 1.0f;
  }
  return 8;
}

// palette interpolation weight of linear entry n and whether the entry is a constant (BC4 6-value 0/1)
__device__ __forceinline__ float train_weight(int fmt, bool mode8, int n, bool& constant) {
  constant = false;
  if (fmt == kFmtBC1) return (float)n / 3.0f;
  if (mode8) return (float)n / 7.0f;
  constant = n == 0 || n == 7;
  return constant ? 0.0f : (float)(n - 1) / 5.0f;
}

// NET = 1: colour network (samples are texels); NET = 0: endpoint network (samples are blocks)
template <int HID, int NET>
__global__ void __launch_bounds__(kTrainTile * kTrainQ, 1) train_step_kernel(const __grid_constant__ TrainParams p) {
  extern __shared__ float sm[];
  // kTrainQ threads per sample: thread (tid, h) owns sample tid of the tile and the h-th quarter of each
  // layer's outputs / inputs (more warps per SM at the same shared memory)
  const int t = threadIdx.x, tid = t % kTrainTile, h = t / kTrainTile, NT = kTrainTile * kTrainQ;
  const int n_c = NET ? p.n_c : p.n_e, F = 2 * p.levels;   // n_c here = MLP outputs
  // padded row stride: 16-B aligned rows for float4 access, rows 4 banks apart (conflict-free LDS.128)
  constexpr int LD = HID + 4;
  // ---- shared memory: weights, biases, tile activations A0 (features), A1..A3, delta buffer
  auto al4 = [](int n) { return (n + 3) & ~3; };
  float* sW[4];
  float* sb[4];
  float* q = sm;
  for (int l = 0; l < 4; l++) { sW[l] = q; q += al4(p.kin[l] * p.kout[l]); sb[l] = q; q += al4(p.kout[l]); }
  float* A[4];
  A[0] = q; q += al4(kTrainTile * (F + 1));
  for (int l = 1; l < 4; l++) { A[l] = q; q += kTrainTile * LD; }
  float* Dl = q; q += kTrainTile * LD;                          // delta of the current layer output
  float* red = q;                                               // [kTrainTile] loss reduction
  const int ldA[4] = {F + 1, LD, LD, LD};
  for (int l = 0; l < 4; l++) {
    const int nw = p.kin[l] * p.kout[l];
    for (int e = t; e < nw; e += NT) sW[l][e] = p.params[p.w_off[l] + e];
    for (int e = t; e < p.kout[l]; e += NT) sb[l][e] = p.params[p.b_off[l] + e];
  }
  __syncthreads();

  const int s = blockIdx.x * kTrainTile + tid;
  const bool valid = s < p.B;
  const int sc = valid ? s : p.B - 1;
  const float u = ((float)p.xy[2 * sc] + 0.5f) / (float)p.W, v = ((float)p.xy[2 * sc + 1] + 0.5f) / (float)p.H;

  // ---- forward: grid features (R1-R3), hidden layers, sigmoid outputs
  for (int l = h; l < p.levels; l += kTrainQ) {
    const int res = p.coarsest << l;
    const float X = u * (float)(res - 1), Y = v * (float)(res - 1);
    const int i0 = min((int)floorf(X), res - 2), j0 = min((int)floorf(Y), res - 2);
    const float fx = X - (float)i0, fy = Y - (float)j0;
    const float* g = p.params + p.lvl_off[l];
    for (int f = 0; f < 2; f++) {
      float pass;
      const float v00 = fake_quant(g[((size_t)j0 * res + i0) * 2 + f], p.qsz, l, pass);
      const float v10 = fake_quant(g[((size_t)j0 * res + i0 + 1) * 2 + f], p.qsz, l, pass);
      const float v01 = fake_quant(g[((size_t)(j0 + 1) * res + i0) * 2 + f], p.qsz, l, pass);
      const float v11 = fake_quant(g[((size_t)(j0 + 1) * res + i0 + 1) * 2 + f], p.qsz, l, pass);
      const float top = v00 + fx * (v10 - v00), bot = v01 + fx * (v11 - v01);
      A[0][tid * ldA[0] + 2 * l + f] = top + fy * (bot - top);
    }
  }
  __syncthreads();
  constexpr int HQ = HID / kTrainQ;   // this thread's HQ consecutive outputs, register-blocked
  static_assert(HQ % 4 == 0, "quarter width must be a multiple of 4");
  for (int l = 0; l < 3; l++) {
    const float* a = A[l] + tid * ldA[l];
    float* o = A[l + 1] + tid * LD;
    uint64_t z2[HQ / 2];   // output pairs, packed FFMA2 (each lane the same RN fma as the scalar form)
#pragma unroll
    for (int jj = 0; jj < HQ / 2; jj++) z2[jj] = f2pack(sb[l][h * HQ + 2 * jj], sb[l][h * HQ + 2 * jj + 1]);
    for (int k = 0; k < p.kin[l]; k++) {
      const float ak = a[k];
      const uint64_t a2 = f2pack(ak, ak);
      const float4* w4 = reinterpret_cast<const float4*>(sW[l] + k * HID + h * HQ);
#pragma unroll
      for (int q4 = 0; q4 < HQ / 4; q4++) {
        const float4 w = w4[q4];
        z2[2 * q4] = fma2(a2, f2pack(w.x, w.y), z2[2 * q4]);
        z2[2 * q4 + 1] = fma2(a2, f2pack(w.z, w.w), z2[2 * q4 + 1]);
      }
    }
#pragma unroll
    for (int jj = 0; jj < HQ / 2; jj++) {
      float z0, z1;
      f2unpack(z2[jj], z0, z1);
      o[h * HQ + 2 * jj] = selu_f(z0);
      o[h * HQ + 2 * jj + 1] = selu_f(z1);
    }
    __syncthreads();
  }
  float* D = Dl;
  {   // output layer: column j by quarter j % kTrainQ, staged through D
    const float* a = A[3] + tid * LD;
    for (int j = h; j < n_c; j += kTrainQ) {
      float z = sb[3][j];
      for (int k = 0; k < HID; k++) z = __fmaf_rn(a[k], sW[3][k * n_c + j], z);
      D[tid * LD + j] = 1.0f / (1.0f + expf(-z));
    }
  }
  __syncthreads();
  float chat[6 * kMaxTex], g_out[6 * kMaxTex];
  for (int j = 0; j < n_c; j++) chat[j] = D[tid * LD + j];

  if (h == 0) {
  if constexpr (NET == 1) {
      // ---- loss and dL/dc_hat per texture: L_c + L_cd with the STE expectation (App. A)
      float loss = 0.0f;
      {
        int co = 0, eo = 0;
        const float invB = 1.0f / (float)p.B, invT = 1.0f / p.T;
        for (int k = 0; k < p.n_tex; k++) {
          const int w = p.fmt[k] == kFmtBC1 ? 3 : 1;
          float pal[24], e[6], c[3], ch[3];
          for (int t = 0; t < 2 * w; t++) e[t] = p.eref[(size_t)sc * p.n_e + eo + t];
          for (int t = 0; t < w; t++) { c[t] = p.cref[(size_t)sc * n_c + co + t]; ch[t] = chat[co + t]; }
          const int nn = train_palette(p.fmt[k], e, pal);
          float dist[8], dmax = -1e30f;
          int best = 0;
          for (int n = 0; n < nn; n++) {
            float s2 = 0.0f;
            for (int t = 0; t < w; t++) { const float d = ch[t] - pal[n * w + t]; s2 += d * d; }
            dist[n] = sqrtf(fmaxf(s2, 1e-30f));
            if (-dist[n] > dmax) { dmax = -dist[n]; best = n; }        // argmax of d_n = -dist, ties -> lower n
          }
          float sig[8], ssum = 0.0f;
          for (int n = 0; n < nn; n++) { sig[n] = expf((-dist[n] - dmax) * invT); ssum += sig[n]; }
          for (int n = 0; n < nn; n++) sig[n] /= ssum;
          // forward values: L_c = |c_hat - c|^2, L_cd = |c_n(best) - c|^2
          float G[8], gd[3];
          for (int t = 0; t < w; t++) {
            const float dc = ch[t] - c[t], dd = pal[best * w + t] - c[t];
            loss += dc * dc + dd * dd;
            gd[t] = 2.0f * dd;                                         // dL/dc_dec (forward value)
          }
          float sG = 0.0f;
          for (int n = 0; n < nn; n++) {                               // G_n = dL/dc_dec . c_n
            G[n] = 0.0f;
            for (int t = 0; t < w; t++) G[n] += gd[t] * pal[n * w + t];
            sG += sig[n] * G[n];
          }
          for (int x = 0; x < w; x++) {
            // d soft / d c_hat_x = (1/T) sum_n sigma_n (G_n - sum_m sigma_m G_m) dd_n/dc_hat_x,
            // dd_n / dc_hat_x = -(c_hat_x - c_n,x) / dist_n
            float acc = 0.0f;
            for (int n = 0; n < nn; n++) acc += sig[n] * (G[n] - sG) * (-(ch[x] - pal[n * w + x]) / dist[n]);
            const float gx = 2.0f * (ch[x] - c[x]) + invT * acc;
            g_out[co + x] = valid ? gx * invB * ch[x] * (1.0f - ch[x]) : 0.0f;   // through the sigmoid
          }
          co += w;
          eo += 2 * w;
        }
      }
    red[tid] = valid ? loss : 0.0f;
    } else {
    // ---- endpoint network: L_e + L_cd (Eq. 14); indices from the PREDICTED palette and the reference
      //      colours, decoded colour from the REFERENCE palette, STE as for the colour net
      float loss = 0.0f;
      {
        const float invB = 1.0f / (float)p.B, invT = 1.0f / p.T;
        for (int j = 0; j < n_c; j++) {
          const float d = chat[j] - p.eref[(size_t)sc * n_c + j];
          loss += d * d;
          g_out[j] = 2.0f * d;
        }
        int co = 0, eo = 0;
        for (int k = 0; k < p.n_tex; k++) {
          const int w = p.fmt[k] == kFmtBC1 ? 3 : 1;
          float pp[24], pr[24], ep[6], er[6];
          for (int t = 0; t < 2 * w; t++) { ep[t] = chat[eo + t]; er[t] = p.eref[(size_t)sc * n_c + eo + t]; }
          const int nn = train_palette(p.fmt[k], ep, pp);
          train_palette(p.fmt[k], er, pr);
          const bool mode8 = p.fmt[k] == kFmtBC1 || ep[0] > ep[1];
          for (int i = 0; i < 16; i++) {
            float c[3];
            for (int t = 0; t < w; t++) c[t] = p.cref[((size_t)sc * 16 + i) * p.n_c + co + t];
            float dist[8], dmax = -1e30f;
            int best = 0;
            for (int n = 0; n < nn; n++) {
              float s2 = 0.0f;
              for (int t = 0; t < w; t++) { const float d = c[t] - pp[n * w + t]; s2 += d * d; }
              dist[n] = sqrtf(fmaxf(s2, 1e-30f));
              if (-dist[n] > dmax) { dmax = -dist[n]; best = n; }
            }
            float sig[8], ssum = 0.0f;
            for (int n = 0; n < nn; n++) { sig[n] = expf((-dist[n] - dmax) * invT); ssum += sig[n]; }
            for (int n = 0; n < nn; n++) sig[n] /= ssum;
            float gd[3], G[8], sG = 0.0f;
            for (int t = 0; t < w; t++) {
              const float dd = pr[best * w + t] - c[t];
              loss += dd * dd;
              gd[t] = 2.0f * dd;
            }
            for (int n = 0; n < nn; n++) {
              G[n] = 0.0f;
              for (int t = 0; t < w; t++) G[n] += gd[t] * pr[n * w + t];
              sG += sig[n] * G[n];
            }
            for (int n = 0; n < nn; n++) {
              bool constant;
              const float wn = train_weight(p.fmt[k], mode8, n, constant);
              if (constant) continue;
              const float coef = invT * sig[n] * (G[n] - sG);        // dL/dd_n
              for (int x = 0; x < w; x++) {
                const float dpal = coef * (-(pp[n * w + x] - c[x]) / dist[n]);   // dL/d pal_pred[n][x]
                g_out[eo + x] += dpal * (1.0f - wn);
                g_out[eo + w + x] += dpal * wn;
              }
            }
          }
          co += w;
          eo += 2 * w;
        }
        for (int j = 0; j < n_c; j++) g_out[j] = valid ? g_out[j] * invB * chat[j] * (1.0f - chat[j]) : 0.0f;
      }
    red[tid] = valid ? loss : 0.0f;
    }
  }
  // ---- backward: output layer delta -> D, then layers 3..0
  __syncthreads();                                                 // every quarter has read c_hat
  if (h == 0)
    for (int j = 0; j < n_c; j++) D[tid * LD + j] = g_out[j];
  __syncthreads();
  for (int l = 3; l >= 0; l--) {
    const int K = p.kin[l], N = p.kout[l];
    // weight and bias gradients of layer l over the tile: dW[k][j] = sum_i A_l[i][k] D[i][j]
    if (K % 2 == 0 && N % 4 == 0) {
      // 2 x 4 blocks (k pair, j quad): per sample 2 scalar + 1 float4 shared-memory loads for 8 FMAs
      const int nblk = (K / 2) * (N / 4);
      for (int e = t; e < nblk; e += NT) {
        const int kp = e / (N / 4), jq = e - kp * (N / 4), k = 2 * kp, j = 4 * jq;
        uint64_t acc[2][2] = {{0ull, 0ull}, {0ull, 0ull}};   // (j, j+1), (j+2, j+3) pairs, packed FFMA2
        for (int i = 0; i < kTrainTile; i++) {
          const float as0 = A[l][i * ldA[l] + k], as1 = A[l][i * ldA[l] + k + 1];   // ldA[0] is odd
          const float4 d = *reinterpret_cast<const float4*>(D + i * LD + j);
          const uint64_t dxy = f2pack(d.x, d.y), dzw = f2pack(d.z, d.w);
          const uint64_t a0 = f2pack(as0, as0), a1 = f2pack(as1, as1);
          acc[0][0] = fma2(a0, dxy, acc[0][0]); acc[0][1] = fma2(a0, dzw, acc[0][1]);
          acc[1][0] = fma2(a1, dxy, acc[1][0]); acc[1][1] = fma2(a1, dzw, acc[1][1]);
        }
#pragma unroll
        for (int r = 0; r < 2; r++) {   // one 16-byte vector atomic per 4 consecutive weights (sm_90+)
          float4 g4;
          f2unpack(acc[r][0], g4.x, g4.y);
          f2unpack(acc[r][1], g4.z, g4.w);
          atomicAdd(reinterpret_cast<float4*>(p.grads + p.w_off[l] + (size_t)(k + r) * N + j), g4);
        }
      }
    } else {
      for (int e = t; e < K * N; e += NT) {
        const int k = e / N, j = e - k * N;
        float acc = 0.0f;
        for (int i = 0; i < kTrainTile; i++) acc = __fmaf_rn(A[l][i * ldA[l] + k], D[i * LD + j], acc);
        atomicAdd(p.grads + p.w_off[l] + e, acc);
      }
    }
    for (int j = t; j < N; j += NT) {   // bias gradient
      float acc = 0.0f;
      for (int i = 0; i < kTrainTile; i++) acc += D[i * LD + j];
      atomicAdd(p.grads + p.b_off[l] + j, acc);
    }
    // delta of this layer's input: dA[k] = sum_j W[k][j] D[j]; through selu' for hidden inputs;
    // this thread's quarter of the inputs k
    const int KQ = (K + kTrainQ - 1) / kTrainQ, k0 = h * KQ, k1 = min(K, k0 + KQ);
    float dA[HID / kTrainQ];
#pragma unroll
    for (int kk = 0; kk < HID / kTrainQ; kk++) dA[kk] = 0.0f;
    if (N % 4 == 0) {   // per j quad: one float4 of this sample's delta row, one float4 per W row (broadcast)
      const float4* d4 = reinterpret_cast<const float4*>(D + tid * LD);
      uint64_t dA2[HID / kTrainQ / 2];   // input pairs (kk, kk+1), packed FFMA2, same per-lane fma chain
#pragma unroll
      for (int kp = 0; kp < HID / kTrainQ / 2; kp++) dA2[kp] = 0ull;
      for (int jq = 0; jq < N / 4; jq++) {
        const float4 d = d4[jq];
        const uint64_t dx = f2pack(d.x, d.x), dy = f2pack(d.y, d.y), dz = f2pack(d.z, d.z), dw = f2pack(d.w, d.w);
#pragma unroll
        for (int kp = 0; kp < HID / kTrainQ / 2; kp++) {
          if (k0 + 2 * kp >= k1) break;
          const float4 wa = *reinterpret_cast<const float4*>(sW[l] + (k0 + 2 * kp) * N + 4 * jq);
          const float4 wb = *reinterpret_cast<const float4*>(sW[l] + min(k0 + 2 * kp + 1, k1 - 1) * N + 4 * jq);
          dA2[kp] = fma2(f2pack(wa.w, wb.w), dw, fma2(f2pack(wa.z, wb.z), dz,
                    fma2(f2pack(wa.y, wb.y), dy, fma2(f2pack(wa.x, wb.x), dx, dA2[kp]))));
        }
      }
#pragma unroll
      for (int kp = 0; kp < HID / kTrainQ / 2; kp++) f2unpack(dA2[kp], dA[2 * kp], dA[2 * kp + 1]);
    } else {
      for (int k = k0; k < k1; k++)
        for (int j = 0; j < N; j++) dA[k - k0] = __fmaf_rn(sW[l][k * N + j], D[tid * LD + j], dA[k - k0]);
    }
    for (int k = k0; k < k1; k++)
      if (l > 0) {
        const float a = A[l][tid * ldA[l] + k];
        dA[k - k0] *= a > 0.0f ? kSeluL : a + kSeluLA;              // selu'(z) from a = selu(z)
      }
    __syncthreads();                                               // all readers of D are done
    for (int k = k0; k < k1; k++) D[tid * LD + k] = dA[k - k0];
    __syncthreads();
  }
  // ---- grid gradient: scatter d features through the bilinear weights of each level
  if (valid) {
    for (int l = h; l < p.levels; l += kTrainQ) {
      const int res = p.coarsest << l;
      const float X = u * (float)(res - 1), Y = v * (float)(res - 1);
      const int i0 = min((int)floorf(X), res - 2), j0 = min((int)floorf(Y), res - 2);
      const float fx = X - (float)i0, fy = Y - (float)j0;
      float* g = p.grads + p.lvl_off[l];
      const float* gv = p.params + p.lvl_off[l];
      const size_t c00 = ((size_t)j0 * res + i0) * 2, c10 = c00 + 2, c01 = c00 + (size_t)res * 2, c11 = c01 + 2;
      float v00[2], v10[2], v01[2], v11[2];
      for (int f = 0; f < 2; f++) {
        const float d = D[tid * LD + 2 * l + f];
        float m00, m10, m01, m11;   // QAT STE: no gradient through clamped values
        fake_quant(gv[c00 + f], p.qsz, l, m00);
        fake_quant(gv[c10 + f], p.qsz, l, m10);
        fake_quant(gv[c01 + f], p.qsz, l, m01);
        fake_quant(gv[c11 + f], p.qsz, l, m11);
        v00[f] = m00 * d * (1.0f - fx) * (1.0f - fy);
        v10[f] = m10 * d * fx * (1.0f - fy);
        v01[f] = m01 * d * (1.0f - fx) * fy;
        v11[f] = m11 * d * fx * fy;
      }
      // both features of a vertex with one 8-byte vector atomic (sm_90+): half the atomics of the scatter
      atomicAdd(reinterpret_cast<float2*>(g + c00), make_float2(v00[0], v00[1]));
      atomicAdd(reinterpret_cast<float2*>(g + c10), make_float2(v10[0], v10[1]));
      atomicAdd(reinterpret_cast<float2*>(g + c01), make_float2(v01[0], v01[1]));
      atomicAdd(reinterpret_cast<float2*>(g + c11), make_float2(v11[0], v11[1]));
    }
  }
  // ---- batch-mean loss
  __syncthreads();
  for (int st = kTrainTile / 2; st > 0; st >>= 1) {
    if (t < st) red[t] += red[t + st];
    __syncthreads();
  }
  if (t == 0) atomicAdd(p.loss, red[0] / (float)p.B);
}

// bias-corrected Adam: lr_grid for the first n_grid parameters, lr_mlp for the rest
__global__ void __launch_bounds__(256) adam_kernel(float* __restrict__ params, const float* __restrict__ grads,
                                                   float* __restrict__ m, float* __restrict__ v, long long n,
                                                   long long n_grid, float lr_grid, float lr_mlp, float beta1,
                                                   float beta2, float eps, float bc1, float bc2) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float g = grads[i];
    const float mi = beta1 * m[i] + (1.0f - beta1) * g, vi = beta2 * v[i] + (1.0f - beta2) * g * g;
    m[i] = mi;
    v[i] = vi;
    const float lr = i < n_grid ? lr_grid : lr_mlp;
    params[i] -= lr * (mi / bc1) / (sqrtf(vi / bc2) + eps);
  }
}

}  // namespace ntbc
