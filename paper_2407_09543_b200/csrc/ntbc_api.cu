// ntbc_api.cu -- host side of libntbc.so: the C ABI declared in include/ntbc.h.
// Model parsing/validation, device residency, operand re-layout, kernel launches, error reporting.
#include <cuda.h>  // driver types only (entry points resolved at run time, no -lcuda)
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <map>
#include <set>
#include <unordered_map>
#include <string>
#include <vector>

#include "../../include/ntbc.h"
#include "ntbc_kernels.cuh"
#include "refenc.cuh"
#include "train.cuh"

using namespace ntbc;

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};
// ntbc_debug_time_fused: events recorded on the launch stream right before / after each fused-kernel
// launch of this host thread (bench.py's roofline timing of the dominant kernel)
thread_local cudaEvent_t g_time_fused[2] = {nullptr, nullptr};

ntbc_status fail(ntbc_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}
#define CUDA_TRY(x)                                                                              \
  do {                                                                                           \
    cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess) return fail(NTBC_ECUDA, "%s: %s (%s:%d)", #x, cudaGetErrorString(e_), \
                                       __FILE__, __LINE__);                                      \
  } while (0)

size_t al16(size_t n) { return (n + 15) & ~size_t(15); }

// cudaFuncAttributeMaxDynamicSharedMemorySize is per device context: set it once per (device, kernel),
// under a lock (several host threads, several devices per process)
cudaError_t allow_smem(const void* kern, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({dev, kern})) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.insert({dev, kern});
  return e;
}
uint32_t rd32(const uint8_t* p) { uint32_t v; memcpy(&v, p, 4); return v; }

// Parsed architecture of a .ntbc blob.  Offsets index the blob.
struct Arch {
  int n_tex, fmt[kMaxTex], hidden, n_hidden, F;
  int naive;                      // header variant: 0 NTBC colour network, 1 naive weight network
  int levels[2], coarsest[2];
  int dims[2][5];                 // [net][layer boundary]
  size_t level_off[2][kMaxLevels];
  size_t fg_off[2][kMaxLevels];   // dequantized fp32 grid: level offsets inside that region
  size_t fg_zero_off, fg_bytes;   // zero block read by the unused levels; region size
  float s[2][kMaxLevels];
  int z[2][kMaxLevels];
  size_t w_off[2][4], b_off[2][4];
  size_t total;
};

ntbc_status parse(const void* blob, size_t n, Arch& a) {
  if (!blob) return fail(NTBC_EINVAL, "blob is NULL");
  const uint8_t* b = (const uint8_t*)blob;
  if (n < 96) return fail(NTBC_EFORMAT, "blob truncated (%zu bytes < 96-byte header)", n);
  if (memcmp(b, "NTBC", 4) != 0) return fail(NTBC_EFORMAT, "bad magic");
  if (rd32(b + 4) != 1) return fail(NTBC_EFORMAT, "unsupported version %u", rd32(b + 4));
  a.n_tex = (int)rd32(b + 8);
  if (a.n_tex < 1 || a.n_tex > kMaxTex) return fail(NTBC_EFORMAT, "n_textures %d not in [1,8]", a.n_tex);
  for (int i = 0; i < a.n_tex; i++) {
    a.fmt[i] = (int)rd32(b + 12 + 4 * i);
    if (a.fmt[i] != NTBC_BC1 && a.fmt[i] != NTBC_BC4) return fail(NTBC_EFORMAT, "texture %d: bad format %d", i, a.fmt[i]);
  }
  a.hidden = (int)rd32(b + 44);
  a.n_hidden = (int)rd32(b + 48);
  a.F = (int)rd32(b + 52);
  a.levels[0] = (int)rd32(b + 56); a.coarsest[0] = (int)rd32(b + 60);
  a.levels[1] = (int)rd32(b + 64); a.coarsest[1] = (int)rd32(b + 68);
  const int ep_in = (int)rd32(b + 72), n_e = (int)rd32(b + 76), col_in = (int)rd32(b + 80), n_c = (int)rd32(b + 84);
  a.naive = (int)rd32(b + 88);
  if (a.naive != 0 && a.naive != 1) return fail(NTBC_EFORMAT, "unknown model variant %d", a.naive);
  if (a.hidden != 16 && a.hidden != 32 && a.hidden != 64) return fail(NTBC_EFORMAT, "hidden %d not in {16,32,64}", a.hidden);
  if (a.n_hidden != 3) return fail(NTBC_EFORMAT, "n_hidden %d != 3 (PAPER.md:331)", a.n_hidden);
  if (a.F != 2) return fail(NTBC_EFORMAT, "features per level %d != 2 (PAPER.md:336)", a.F);
  int want_e = 0, want_c = 0;
  for (int i = 0; i < a.n_tex; i++) { want_e += a.fmt[i] == NTBC_BC1 ? 6 : 2; want_c += a.fmt[i] == NTBC_BC1 ? 3 : 1; }
  if (a.naive) want_c = a.n_tex;   // one weight per texel per texture
  if (n_e != want_e || n_c != want_c) return fail(NTBC_EFORMAT, "head widths %d/%d inconsistent with formats", n_e, n_c);
  if (n_e > 48) return fail(NTBC_EFORMAT, "N_e = %d > 48 not supported", n_e);
  for (int g = 0; g < 2; g++) {
    if (a.levels[g] < 1 || a.levels[g] > kMaxLevels) return fail(NTBC_EFORMAT, "grid %d: %d levels not in [1,8]", g, a.levels[g]);
    if (a.coarsest[g] < 2 || ((size_t)a.coarsest[g] << (a.levels[g] - 1)) > 8192)
      return fail(NTBC_EFORMAT, "grid %d: bad resolution", g);
  }
  if (ep_in != 2 * a.levels[0] || col_in != 2 * a.levels[1]) return fail(NTBC_EFORMAT, "MLP input widths inconsistent");
  size_t off = 96;
  const size_t qp = off;
  off += al16((size_t)(a.levels[0] + a.levels[1]) * 8);
  int li = 0;
  for (int g = 0; g < 2; g++)
    for (int l = 0; l < a.levels[g]; l++, li++) {
      if (qp + 8 * li + 8 > n) return fail(NTBC_EFORMAT, "blob truncated in quantization params");
      memcpy(&a.s[g][l], b + qp + 8 * li, 4);
      memcpy(&a.z[g][l], b + qp + 8 * li + 4, 4);
    }
  size_t fo = 0, zmax = 0;
  for (int g = 0; g < 2; g++) {
    for (int l = 0; l < a.levels[g]; l++) {
      const size_t res = (size_t)a.coarsest[g] << l, sz = res * res * 2;
      a.level_off[g][l] = off;
      off += al16(sz);
      if (off > n + 15) return fail(NTBC_EFORMAT, "blob truncated in grid %d level %d", g, l);
      a.fg_off[g][l] = fo;
      fo += al16(sz * sizeof(float));
    }
    zmax = std::max(zmax, (size_t)a.coarsest[g] * a.coarsest[g] * 2 * sizeof(float));
  }
  a.fg_zero_off = fo;
  a.fg_bytes = fo + al16(zmax);
  const int ins[2] = {ep_in, col_in}, outs[2] = {n_e, n_c};
  for (int k = 0; k < 2; k++) {
    a.dims[k][0] = ins[k];
    a.dims[k][1] = a.dims[k][2] = a.dims[k][3] = a.hidden;
    a.dims[k][4] = outs[k];
    for (int l = 0; l < 4; l++) {
      a.w_off[k][l] = off;
      off += al16((size_t)a.dims[k][l] * a.dims[k][l + 1] * 2);
      a.b_off[k][l] = off;
      off += al16((size_t)a.dims[k][l + 1] * 2);
    }
  }
  if (off > n + 15 || a.b_off[1][3] + (size_t)n_c * 2 > n) return fail(NTBC_EFORMAT, "blob truncated in MLP weights");
  a.total = n;
  return NTBC_OK;
}

bool same_arch(const Arch& x, const Arch& y) {
  if (x.n_tex != y.n_tex || x.hidden != y.hidden || x.total != y.total || x.naive != y.naive) return false;
  for (int i = 0; i < x.n_tex; i++) if (x.fmt[i] != y.fmt[i]) return false;
  for (int g = 0; g < 2; g++) if (x.levels[g] != y.levels[g] || x.coarsest[g] != y.coarsest[g]) return false;
  return true;
}

int round16(int v) { return (v + 15) & ~15; }

}  // namespace

constexpr int kMaxChunks = 64;
constexpr int kSchedRing = 64;
thread_local long long g_train_total = 0;   // parameter count of the last train_layout
// chunk c is copied on copy stream c % kCopyStreams: each stream-wait operation has a fixed latency,
// so consecutive chunks' waits must not queue behind each other on one stream
constexpr int kCopyStreams = 4;

struct ntbc_model_s {
  int device;
  Arch arch;
  // thread safety (include/ntbc.h): every call that launches work on the model or changes it holds `mu`;
  // decodes of one model on different streams are ordered on the device by `last_done`, recorded after
  // each launch (they share the model's fp32 grid region, rewritten by every decode's dequant launch)
  std::recursive_mutex mu;
  int contract = 0;            // arithmetic contract: 0 = H (binary16 activations), 1 = F,
                               // 2 = P (binary16 selu arithmetic)
  cudaEvent_t last_done = nullptr;
  cudaStream_t last_stream = nullptr;
  uint8_t* d_blob = nullptr;   // weight slot: the blob, then at fg_base its grids dequantized to fp32
  size_t blob_cap = 0;         // slot bytes
  size_t fg_base = 0;          // offset of the fp32 grids in a slot
  size_t img_off = 0;          // offset of the fused kernel's shared-memory prefix image in a slot
  // dynamic-scheduling unit counters: a ring of kSchedRing ints, one per launch (zeroed on the
  // launch's stream), so up to kSchedRing launches of this model may be in flight concurrently
  int* d_sched = nullptr;
  std::atomic<unsigned> sched_next{0};
  NetLayout net[2];
  // lazily sized scratch for ntbc_decode_material_host
  uint8_t* d_scratch = nullptr;
  size_t scratch_bytes = 0;
  // pipelined device->host copies of ntbc_decode_material_host: the fused kernel counts finished
  // units per row chunk in d_progress (monotonic across calls); a copy stream waits on each counter
  // (stream memory operation) and copies that chunk while the kernel works on later rows.
  unsigned long long* d_progress = nullptr;
  unsigned long long progress_target[kMaxChunks] = {};
  cudaStream_t copy_stream[kCopyStreams] = {};
  cudaEvent_t copy_start = nullptr, copy_done[kCopyStreams] = {};
  // double-buffered weights for ntbc_decode_material_host: the next call uploads into the other slot
  // on upload_stream while the previous call's kernel still reads the current one.
  uint8_t* slot_blob[2] = {nullptr, nullptr};
  int cur = 0;
  cudaStream_t upload_stream = nullptr;
  cudaEvent_t uploaded = nullptr, slot_free[2] = {nullptr, nullptr};
  // optional timeline of the last host-path call (NTBC_TIMELINE=1): call start, upload done, kernel
  // start, kernel end, copies done (per copy stream) -- ntbc_debug_host_timeline
  cudaEvent_t tlset[2][4 + kCopyStreams] = {};
  cudaEvent_t* tl = tlset[0];
  int tl_cur = 0;
  bool tl_on = false;
};

namespace {

// Shared-memory B-operand images of both nets (K-major, bias folded as an extra K chunk), built by
// the fused kernel's prologue from the blob's row-major weights (layer offsets and widths here).
void layout_nets(ntbc_model_s* m) {
  const Arch& a = m->arch;
  for (int k = 0; k < 2; k++) {
    NetLayout& L = m->net[k];
    uint32_t o = 0;
    for (int l = 0; l < 4; l++) {
      const int kin16 = l == 0 ? 16 : a.hidden;
      const int npad = l < 3 ? a.hidden : round16(a.dims[k][4]);
      L.layer_off[l] = o;
      L.w_off[l] = (uint32_t)a.w_off[k][l];
      L.b_off[l] = (uint32_t)a.b_off[k][l];
      L.kin[l] = a.dims[k][l];
      L.nout[l] = a.dims[k][l + 1];
      o += (uint32_t)(npad * (kin16 + 16) * 2);
    }
    L.img_bytes = o;
    L.n_out = a.dims[k][4];
    L.n_out16 = round16(a.dims[k][4]);
  }
}

// the model is the blob: one host->device copy into the current weight slot
ntbc_status upload(ntbc_model_s* m, const void* blob, size_t n, cudaStream_t st) {
  CUDA_TRY(cudaMemcpyAsync(m->d_blob, blob, n, cudaMemcpyHostToDevice, st));
  return NTBC_OK;
}

// row a2, first half, at the start of every decode: one kernel dequantizes every grid level of the current
// weight slot (Eq.2, R6) into the slot's fp32 grid region (and zeroes its zero block); the fused kernel
// that follows on the same stream only interpolates
ntbc_status dequant_grids(ntbc_model_s* m, cudaStream_t st) {
  const Arch& a = m->arch;
  DequantParams d{};
  d.slot = m->d_blob;
  for (int g = 0; g < 2; g++)
    for (int l = 0; l < a.levels[g]; l++, d.n_levels++) {
      const long long res = (long long)a.coarsest[g] << l;
      d.src_off[d.n_levels] = a.level_off[g][l];
      d.dst_off[d.n_levels] = m->fg_base + a.fg_off[g][l];
      d.end[d.n_levels] = (d.n_levels ? d.end[d.n_levels - 1] : 0) + (res * res * 2 + 3) / 4;   // 4-code groups
      d.s[d.n_levels] = a.s[g][l];
      d.z[d.n_levels] = a.z[g][l];
    }
  d.zero_off = m->fg_base + a.fg_zero_off;
  d.zero_n = (int)((a.fg_bytes - a.fg_zero_off) / sizeof(float));
  d.net[0] = m->net[0];
  d.net[1] = m->net[1];
  d.H = a.hidden;
  d.img_off = m->img_off;
  const long long total4 = d.end[d.n_levels - 1];
  const int grid = (int)std::min<long long>((total4 + 255) / 256, 148 * 8);
  dequant_grids_kernel<<<grid, 256, 0, st>>>(d);
  g_launches++;
  CUDA_TRY(cudaGetLastError());
  return NTBC_OK;
}

struct DevGuard {
  int prev = -1;
  explicit DevGuard(int d) { cudaGetDevice(&prev); if (prev != d) cudaSetDevice(d); }
  ~DevGuard() { int cur; cudaGetDevice(&cur); if (prev >= 0 && cur != prev) cudaSetDevice(prev); }
};

template <int H, int NWG, bool DUMP, bool SPLIT = false>
ntbc_status launch_fused_t(const FusedLaunch& L, size_t smem, int grid, cudaStream_t st) {
  auto kern = SPLIT          ? fused_decode_kernel<H, NWG, DUMP, false, true>
              : L.m[0].naive ? fused_decode_kernel<H, NWG, DUMP, true>
              : L.m[0].half  ? fused_decode_kernel<H, NWG, DUMP, false, false, true>   // contract P
                             : fused_decode_kernel<H, NWG, DUMP, false>;
  CUDA_TRY(allow_smem((const void*)kern, 227 * 1024));
  if (!DUMP && g_time_fused[0]) CUDA_TRY(cudaEventRecord(g_time_fused[0], st));
  kern<<<grid, NWG * 128, smem, st>>>(L);
  g_launches++;
  CUDA_TRY(cudaGetLastError());
  if (!DUMP && g_time_fused[1]) CUDA_TRY(cudaEventRecord(g_time_fused[1], st));
  return NTBC_OK;
}

// slots per work group of the fused kernel: 2 when the ping-pong variant runs (NTBC_PINGPONG, H = 64, 4 groups)
int fused_slots(int hidden, int nwg, bool dump) { return (NTBC_PINGPONG && hidden == 64 && nwg == 4 && !dump) ? 2 : 1; }
// per work group: SL A operands / staging buffers, the unit's BC word headers (+ naive swap flags), the
// palettes of the SL tiles in flight (8 blocks each)
uint32_t pal_bytes_of(const FusedParams& p, int sl) { return p.tpal_off + (uint32_t)(8 * sl * p.pal_stride * sizeof(float)); }
size_t fused_smem(const FusedParams& p, int nwg, int sl = 1) {
  return (size_t)p.net[0].img_bytes + p.net[1].img_bytes + kOnesBytes + kUnormBytes +
         (size_t)nwg * (sl * p.a_bytes + pal_bytes_of(p, sl)) + 8 * (sl * nwg + 1) + 16 + 4 * 8;
}

ntbc_status launch_fused_locked(ntbc_model_s* m, FusedParams& p, bool dump, cudaStream_t st);

// order this launch after the model's previous one when that ran on another stream
ntbc_status order_after_last(ntbc_model_s* m, cudaStream_t st) {
  if (m->last_done && m->last_stream != st) CUDA_TRY(cudaStreamWaitEvent(st, m->last_done, 0));
  return NTBC_OK;
}
ntbc_status record_last(ntbc_model_s* m, cudaStream_t st) {
  if (!m->last_done) CUDA_TRY(cudaEventCreateWithFlags(&m->last_done, cudaEventDisableTiming));
  CUDA_TRY(cudaEventRecord(m->last_done, st));
  m->last_stream = st;
  return NTBC_OK;
}

ntbc_status launch_fused(ntbc_model_s* m, FusedParams& p, bool dump, cudaStream_t st) {
  std::lock_guard<std::recursive_mutex> lk(m->mu);
  ntbc_status s0 = order_after_last(m, st);
  if (s0) return s0;
  s0 = launch_fused_locked(m, p, dump, st);
  if (s0) return s0;
  return record_last(m, st);
}

// the grid dequantization + prefix build launch of model m, then every kernel parameter of its half of a
// fused launch
ntbc_status prepare_fused(ntbc_model_s* m, FusedParams& p, bool dump, cudaStream_t st) {
  const Arch& a = m->arch;
  ntbc_status dst = dequant_grids(m, st);
  if (dst) return dst;
  if (!dump && m->d_sched && !(getenv("NTBC_STATIC_SCHED") && atoi(getenv("NTBC_STATIC_SCHED")))) {
    p.next_unit = m->d_sched + (m->sched_next++ % kSchedRing);
    CUDA_TRY(cudaMemsetAsync(p.next_unit, 0, sizeof(int), st));
  }
  p.blob = m->d_blob;
  p.prefix = m->d_blob + m->img_off;
  for (int g = 0; g < 2; g++) {
    p.levels[g] = a.levels[g];
    for (int l = 0; l < a.levels[g]; l++) {
      p.lv[g][l].offset = (uint32_t)(m->fg_base + a.fg_off[g][l]);
      p.lv[g][l].res = a.coarsest[g] << l;
      p.lv[g][l].rm1 = (float)((a.coarsest[g] << l) - 1);
      p.lv[g][l].s = a.s[g][l];
      p.lv[g][l].z = a.z[g][l];
    }
    // levels past the grid's count read the slot's zero block at the coarsest resolution: the lookup
    // then yields exactly +0 (every lerp of +0 is +0), the zero feature the architecture defines, so
    // the kernel samples all kMaxLevels levels without branches and can batch their loads.
    for (int l = a.levels[g]; l < kMaxLevels; l++) {
      p.lv[g][l].offset = (uint32_t)(m->fg_base + a.fg_zero_off);
      p.lv[g][l].res = a.coarsest[g];
      p.lv[g][l].rm1 = (float)(a.coarsest[g] - 1);
      p.lv[g][l].s = 0.0f;
      p.lv[g][l].z = 0;
    }
  }
  p.net[0] = m->net[0];
  p.net[1] = m->net[1];
  p.n_tex = a.n_tex;
  int eo = 0, co = 0;
  for (int k = 0; k < a.n_tex; k++) {
    p.fmt[k] = a.fmt[k];
    p.ep_off[k] = eo;
    p.col_off[k] = a.naive ? k : co;
    eo += a.fmt[k] == NTBC_BC1 ? 6 : 2;
    co += a.fmt[k] == NTBC_BC1 ? 3 : 1;
  }
  p.BW = p.W / 4;
  p.BH = p.H / 4;
  p.units_per_row = (p.BW + kUnitBlocks - 1) / kUnitBlocks;
  p.n_units = p.units_per_row * (p.row_end - p.row_begin);
  const int maxo = a.dims[0][4] > a.dims[1][4] ? a.dims[0][4] : a.dims[1][4];
  p.split = m->contract == 1;
  p.half = m->contract == 2;
  const uint32_t a_kmajor = 128u * a.hidden * 2u * (p.split ? 2u : 1u);   // F: hi and lo chunks
  const uint32_t a_stage = 128u * 4u * (uint32_t)((maxo + 1) & ~1);      // fp32 staging [ch][128], pairs
  p.a_bytes = (uint32_t)((std::max(a_kmajor, a_stage) + 127) & ~127u);
  // per work group: BC word headers (+ BC1 swap flags, naive models) of the unit's 128 blocks, then the palettes of the
  // current colour tile's 8 blocks (BC1 12 floats, BC4 8 floats per texture; 16-B aligned records)
  p.pal_stride = 0;
  for (int k = 0; k < a.n_tex; k++) {
    p.pal_off[k] = p.pal_stride;
    p.pal_stride += a.fmt[k] == NTBC_BC1 ? 12 : 8;
  }
  p.pal_stride = (p.pal_stride + 3) & ~3;
  p.tpal_off = (uint32_t)((a.n_tex * 128 * (a.naive ? 5 : 4) + 15) & ~15u);   // BC1 swap flags: naive only
  p.pal_bytes = p.tpal_off + (uint32_t)(8 * p.pal_stride * sizeof(float));
  p.naive = a.naive;
  p.vec16 = (p.BW % 2) == 0;
  for (int k = 0; k < a.n_tex; k++)
    if ((uintptr_t)p.out[k] & 15) p.vec16 = 0;
  p.n_bc1 = p.n_bc4 = 0;
  for (int k = 0; k < a.n_tex; k++) {
    if (a.fmt[k] == NTBC_BC1) p.tex_bc1[p.n_bc1++] = k;
    else p.tex_bc4[p.n_bc4++] = k;
  }
  return NTBC_OK;
}

// work groups per CTA: more independent groups per SM hide more latency (C3: NWG 4 -> 2.70 ms, 6 -> 2.65
// with 8% wave-quantisation loss, 8 -> 2.46) but each group's unit takes ~1.8x longer, so 8 groups pay only
// with at least two full waves of units (C2, 512 units: NWG 4 = 0.19 ms on 128 SMs in one wave, NWG 8 =
// 0.34 ms on 64 SMs); 5 and 6 quantise badly on power-of-two unit counts.  One launch runs one model, or
// the two models of a conservative pair on disjoint CTA ranges (each CTA holds one model's operand images).
ntbc_status launch_prepared(FusedParams* ps, int n, int hidden, bool dump, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t cap = 227 * 1024;
  int units = 0;
  for (int i = 0; i < n; i++) units += ps[i].n_units;
  auto smem_of = [&](int w) {
    size_t m = 0;
    for (int i = 0; i < n; i++) m = std::max(m, fused_smem(ps[i], w, fused_slots(hidden, w, dump)));
    return m;
  };
  int nwg = 2;
  for (int w : {8, 4, 3})
    if ((w != 8 || units >= 2 * 8 * sms) && (w != 8 || !NTBC_PINGPONG || hidden != 64 || dump) && (w != 8 || !ps[0].split) &&
        smem_of(w) <= cap) {
      nwg = w;
      break;
    }
  if (const char* e = getenv("NTBC_NWG")) {  // measurement override (bench sweeps); clamped to what fits
    const int want = atoi(e);
    if ((want >= 2 && want <= 4 || (want == 8 && !ps[0].split)) && smem_of(want) <= cap) nwg = want;
  }
  const size_t smem = smem_of(nwg);
  if (smem > cap) return fail(NTBC_EINVAL, "model needs %zu B of shared memory (> %zu)", smem, cap);
  for (int i = 0; i < n; i++) ps[i].pal_bytes = pal_bytes_of(ps[i], fused_slots(hidden, nwg, dump));
  FusedLaunch L{};
  L.m[0] = ps[0];
  L.m[1] = n > 1 ? ps[1] : ps[0];
  int grid;
  if (n == 1) {
    grid = std::max(1, std::min(sms, (ps[0].n_units + nwg - 1) / nwg));
    L.split = grid;
  } else {
    // CTAs in proportion to each model's work: units x (per-texel MLP + per-texture index/pack cost),
    // measured ~90 SASS instructions per texel per texture against ~2,700 for the MLPs
    double w[2];
    for (int i = 0; i < 2; i++) w[i] = ps[i].n_units * (2700.0 + 90.0 * ps[i].n_tex);
    grid = sms;
    int split = (int)std::lround(grid * w[0] / (w[0] + w[1]));
    if (const char* e = getenv("NTBC_PAIR_SPLIT")) split = atoi(e);   // measurement override
    L.split = std::max(1, std::min(grid - 1, split));
  }
#define NTBC_DISPATCH_SPLIT(HH)                                                                  \
  if (hidden == HH && ps[0].split) {                                                             \
    if (nwg == 4) return dump ? launch_fused_t<HH, 4, true, true>(L, smem, grid, st)             \
                              : launch_fused_t<HH, 4, false, true>(L, smem, grid, st);           \
    if (nwg == 3) return dump ? launch_fused_t<HH, 3, true, true>(L, smem, grid, st)             \
                              : launch_fused_t<HH, 3, false, true>(L, smem, grid, st);           \
    return dump ? launch_fused_t<HH, 2, true, true>(L, smem, grid, st) : launch_fused_t<HH, 2, false, true>(L, smem, grid, st); \
  }
  NTBC_DISPATCH_SPLIT(16)
  NTBC_DISPATCH_SPLIT(32)
  NTBC_DISPATCH_SPLIT(64)
#undef NTBC_DISPATCH_SPLIT
#define NTBC_DISPATCH(HH)                                                                        \
  if (hidden == HH) {                                                                            \
    if (nwg == 8) return dump ? launch_fused_t<HH, 8, true>(L, smem, grid, st)                   \
                              : launch_fused_t<HH, 8, false>(L, smem, grid, st);                 \
    if (nwg == 4) return dump ? launch_fused_t<HH, 4, true>(L, smem, grid, st)                   \
                              : launch_fused_t<HH, 4, false>(L, smem, grid, st);                 \
    if (nwg == 3) return dump ? launch_fused_t<HH, 3, true>(L, smem, grid, st)                   \
                              : launch_fused_t<HH, 3, false>(L, smem, grid, st);                 \
    return dump ? launch_fused_t<HH, 2, true>(L, smem, grid, st) : launch_fused_t<HH, 2, false>(L, smem, grid, st); \
  }
  NTBC_DISPATCH(16)
  NTBC_DISPATCH(32)
  NTBC_DISPATCH(64)
#undef NTBC_DISPATCH
  return fail(NTBC_EINVAL, "unsupported hidden width");
}

ntbc_status launch_fused_locked(ntbc_model_s* m, FusedParams& p, bool dump, cudaStream_t st) {
  ntbc_status s0 = prepare_fused(m, p, dump, st);
  if (s0) return s0;
  return launch_prepared(&p, 1, m->arch.hidden, dump, st);
}

// cuStreamWaitValue64 through the runtime's driver entry-point query (no link-time libcuda dependency)
typedef CUresult (*wait64_fn)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
typedef CUresult (*dev_attr_fn)(int*, CUdevice_attribute, CUdevice);
typedef CUresult (*dev_get_fn)(CUdevice*, int);
wait64_fn g_wait64 = nullptr;

bool stream_waits_supported(int device) {
  static std::atomic<int> cached[64];  // 0 unknown, 1 yes, 2 no (several host threads may probe at once)
  static std::mutex probe_mu;
  if (device < 0 || device >= 64) return false;
  if (cached[device].load()) return cached[device].load() == 1;
  std::lock_guard<std::mutex> lk(probe_mu);
  if (cached[device].load()) return cached[device].load() == 1;
  if (const char* e = getenv("NTBC_NO_PIPELINED_COPY")) if (atoi(e)) { cached[device] = 2; return false; }
  void *w = nullptr, *ga = nullptr, *gd = nullptr;
  cudaDriverEntryPointQueryResult q1, q2, q3;
  bool ok = cudaGetDriverEntryPoint("cuStreamWaitValue64", &w, cudaEnableDefault, &q1) == cudaSuccess &&
            q1 == cudaDriverEntryPointSuccess &&
            cudaGetDriverEntryPoint("cuDeviceGetAttribute", &ga, cudaEnableDefault, &q2) == cudaSuccess &&
            q2 == cudaDriverEntryPointSuccess &&
            cudaGetDriverEntryPoint("cuDeviceGet", &gd, cudaEnableDefault, &q3) == cudaSuccess &&
            q3 == cudaDriverEntryPointSuccess;
  if (ok) {
    CUdevice d;
    int v = 0;
    ok = ((dev_get_fn)gd)(&d, device) == CUDA_SUCCESS &&
         ((dev_attr_fn)ga)(&v, CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS, d) == CUDA_SUCCESS && v;
  }
  cudaGetLastError();
  if (ok) g_wait64 = (wait64_fn)w;
  cached[device] = ok ? 1 : 2;
  return ok;
}

bool create_copy_streams(ntbc_model_s* m) {
  for (int i = 0; i < kCopyStreams; i++)
    if (cudaStreamCreateWithFlags(&m->copy_stream[i], cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&m->copy_done[i], cudaEventDisableTiming) != cudaSuccess)
      return false;
  return true;
}

// streams, events, progress counters and the second weight slot of the pipelined host path
// (allocated once per model; on failure the host path falls back to serial copies on `stream`)
bool ensure_copy_state(ntbc_model_s* m) {
  if (m->d_progress) return true;
  const unsigned f = cudaEventDisableTiming;
  bool ok = cudaMalloc(&m->slot_blob[1], m->blob_cap) == cudaSuccess &&
            create_copy_streams(m) &&
            cudaStreamCreateWithFlags(&m->upload_stream, cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&m->copy_start, f) == cudaSuccess &&
            cudaEventCreateWithFlags(&m->uploaded, f) == cudaSuccess &&
            cudaEventCreateWithFlags(&m->slot_free[0], f) == cudaSuccess &&
            cudaEventCreateWithFlags(&m->slot_free[1], f) == cudaSuccess &&
            cudaMalloc(&m->d_progress, kMaxChunks * sizeof(unsigned long long)) == cudaSuccess &&
            cudaMemset(m->d_progress, 0, kMaxChunks * sizeof(unsigned long long)) == cudaSuccess &&
            cudaDeviceSynchronize() == cudaSuccess;
  if (!ok) {   // release what was created, so a later call starts from scratch (no leaks on retry)
    cudaGetLastError();
    cudaFree(m->d_progress);
    m->d_progress = nullptr;
    cudaFree(m->slot_blob[1]);
    m->slot_blob[1] = nullptr;
    for (int i = 0; i < kCopyStreams; i++) {
      if (m->copy_stream[i]) cudaStreamDestroy(m->copy_stream[i]);
      if (m->copy_done[i]) cudaEventDestroy(m->copy_done[i]);
      m->copy_stream[i] = nullptr;
      m->copy_done[i] = nullptr;
    }
    for (cudaEvent_t* e : {&m->copy_start, &m->uploaded, &m->slot_free[0], &m->slot_free[1]}) {
      if (*e) cudaEventDestroy(*e);
      *e = nullptr;
    }
    if (m->upload_stream) cudaStreamDestroy(m->upload_stream);
    m->upload_stream = nullptr;
    cudaGetLastError();
    return false;
  }
  m->slot_blob[0] = m->d_blob;
  m->cur = 0;
  return true;
}

ntbc_status check_dims(int W, int H, int r0, int r1) {
  if (W <= 0 || H <= 0 || W % 4 || H % 4) return fail(NTBC_EINVAL, "width/height %dx%d must be positive multiples of 4", W, H);
  if (r0 < 0 || r0 >= r1 || r1 > H / 4) return fail(NTBC_EINVAL, "block rows [%d,%d) not within [0,%d)", r0, r1, H / 4);
  if ((long long)W * H > (1ll << 30)) return fail(NTBC_EINVAL, "texture too large");
  return NTBC_OK;
}

}  // namespace

// ---------------------------------------------------------------- peer-memory gather plumbing (CUDA IPC)
typedef CUresult (*addr_range_fn)(CUdeviceptr*, size_t*, CUdeviceptr);
static addr_range_fn get_addr_range() {
  static addr_range_fn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<addr_range_fn>(f);
  }();
  return fn;
}
// [p, p + bytes) lies inside one CUDA allocation (device memory, or pinned host memory through its UVA address)
static bool one_allocation(const void* p, size_t bytes) {
  addr_range_fn fn = get_addr_range();
  CUdeviceptr base = 0;
  size_t size = 0;
  if (!fn || fn(&base, &size, (CUdeviceptr)p) != CUDA_SUCCESS) { cudaGetLastError(); return false; }
  return (CUdeviceptr)p >= base && (CUdeviceptr)p + bytes <= base + size;
}
static std::mutex g_peer_mu;
static std::unordered_map<void*, void*> g_peer_base;   // pointer returned by ntbc_peer_open -> mapped base

extern "C" {

ntbc_status ntbc_load_model(const void* blob, size_t nbytes, int cuda_device, ntbc_model* out) {
  if (!out) return fail(NTBC_EINVAL, "out is NULL");
  *out = nullptr;
  Arch a;
  ntbc_status st = parse(blob, nbytes, a);
  if (st) return st;
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (cuda_device < 0 || cuda_device >= ndev) return fail(NTBC_EINVAL, "cuda_device %d out of range", cuda_device);
  DevGuard dg(cuda_device);
  auto* m = new ntbc_model_s();
  m->device = cuda_device;
  m->arch = a;
  layout_nets(m);
  m->fg_base = (al16(nbytes) + 255) & ~size_t(255);
  m->img_off = (m->fg_base + a.fg_bytes + 255) & ~size_t(255);
  m->blob_cap = m->img_off + m->net[0].img_bytes + m->net[1].img_bytes + kOnesBytes + kUnormBytes;
  if (cudaMalloc(&m->d_blob, m->blob_cap) != cudaSuccess) {
    cudaGetLastError();
    ntbc_free_model(m);
    return fail(NTBC_ENOMEM, "device allocation of %zu bytes failed", m->blob_cap);
  }
  if (cudaMalloc(&m->d_sched, kSchedRing * sizeof(int)) != cudaSuccess) { cudaGetLastError(); m->d_sched = nullptr; }
  st = upload(m, blob, nbytes, 0);
  if (st == NTBC_OK && cudaDeviceSynchronize() != cudaSuccess) st = fail(NTBC_ECUDA, "model upload: %s", cudaGetErrorString(cudaGetLastError()));
  if (st) { ntbc_free_model(m); return st; }
  *out = m;
  return NTBC_OK;
}

ntbc_status ntbc_model_upload_async(ntbc_model m, const void* blob, size_t nbytes, void* stream) {
  if (!m || !blob) return fail(NTBC_EINVAL, "NULL argument");
  Arch a;
  ntbc_status st = parse(blob, nbytes, a);
  if (st) return st;
  if (!same_arch(a, m->arch)) return fail(NTBC_EMISMATCH, "blob architecture differs from the loaded model");
  DevGuard dg(m->device);
  std::lock_guard<std::recursive_mutex> lk(m->mu);
  st = order_after_last(m, (cudaStream_t)stream);   // the previous decode (any stream) still reads the weights
  if (st) return st;
  m->arch = a;  // same layout; refresh the per-level (s, z)
  st = upload(m, blob, nbytes, (cudaStream_t)stream);
  if (st) return st;
  return record_last(m, (cudaStream_t)stream);
}

ntbc_status ntbc_model_get_info(ntbc_model m, ntbc_model_info* out) {
  if (!m || !out) return fail(NTBC_EINVAL, "NULL argument");
  std::lock_guard<std::recursive_mutex> lk(m->mu);   // slot and scratch sizes change under host-path calls
  const Arch& a = m->arch;
  memset(out, 0, sizeof *out);
  out->n_textures = a.n_tex;
  for (int i = 0; i < a.n_tex; i++) out->fmt[i] = a.fmt[i];
  out->hidden = a.hidden;
  out->n_hidden = a.n_hidden;
  out->n_endpoint_out = a.dims[0][4];
  out->n_color_out = a.dims[1][4];
  out->block_levels = a.levels[0];
  out->block_coarsest = a.coarsest[0];
  out->texel_levels = a.levels[1];
  out->texel_coarsest = a.coarsest[1];
  out->features = a.F;
  out->variant = a.naive;
  out->device_bytes = m->blob_cap * (m->slot_blob[1] ? 2 : 1) + m->scratch_bytes;
  return NTBC_OK;
}

void ntbc_free_model(ntbc_model m) {
  if (!m) return;
  DevGuard dg(m->device);
  cudaFree(m->slot_blob[0] ? m->slot_blob[0] : m->d_blob);
  cudaFree(m->d_scratch);
  cudaFree(m->d_sched);
  cudaFree(m->d_progress);
  if (m->copy_start) cudaEventDestroy(m->copy_start);
  for (int i = 0; i < kCopyStreams; i++) {
    if (m->copy_stream[i]) cudaStreamDestroy(m->copy_stream[i]);
    if (m->copy_done[i]) cudaEventDestroy(m->copy_done[i]);
  }
  for (int i = 0; i < 2; i++) if (m->slot_free[i]) cudaEventDestroy(m->slot_free[i]);
  for (auto& row : m->tlset)
    for (auto e : row) if (e) cudaEventDestroy(e);
  if (m->uploaded) cudaEventDestroy(m->uploaded);
  if (m->last_done) cudaEventDestroy(m->last_done);
  if (m->upload_stream) cudaStreamDestroy(m->upload_stream);
  cudaFree(m->slot_blob[1]);
  delete m;
}

ntbc_status ntbc_decode_material(const ntbc_model* models, int n_models, int width, int height, int r0, int r1,
                                 void* const* out_blocks, void* stream) {
  if (!models || !out_blocks) return fail(NTBC_EINVAL, "NULL argument");
  if (n_models < 1 || n_models > 2) return fail(NTBC_EINVAL, "n_models %d not in {1,2}", n_models);
  ntbc_status st = check_dims(width, height, r0, r1);
  if (st) return st;
  for (int i = 0; i < n_models; i++) if (!models[i]) return fail(NTBC_EINVAL, "model %d is NULL", i);
  if (n_models == 2) {  // conservative pair: one all-BC1 model and one all-BC4 model
    auto all = [](const Arch& a, int f) { for (int k = 0; k < a.n_tex; k++) if (a.fmt[k] != f) return false; return true; };
    const Arch &x = models[0]->arch, &y = models[1]->arch;
    if (!((all(x, NTBC_BC1) && all(y, NTBC_BC4)) || (all(x, NTBC_BC4) && all(y, NTBC_BC1))))
      return fail(NTBC_EMISMATCH, "conservative pair must be one all-BC1 and one all-BC4 model");
    if (models[0]->device != models[1]->device) return fail(NTBC_EMISMATCH, "models on different devices");
  }
  FusedParams ps[2] = {};
  int t = 0;
  for (int i = 0; i < n_models; i++) {
    FusedParams& p = ps[i];
    p.W = width; p.H = height; p.row_begin = r0; p.row_end = r1;
    for (int k = 0; k < models[i]->arch.n_tex; k++, t++) {
      if (!out_blocks[t] || ((uintptr_t)out_blocks[t] & 7)) return fail(NTBC_EINVAL, "out_blocks[%d] NULL or not 8-B aligned", t);
      p.out[k] = (uint64_t*)out_blocks[t];
    }
  }
  cudaStream_t cs = (cudaStream_t)stream;
  if (n_models == 1 || models[0]->arch.hidden != models[1]->arch.hidden || models[0]->arch.naive != models[1]->arch.naive ||
      models[0]->contract != models[1]->contract ||
      (getenv("NTBC_PAIR_LAUNCHES") && atoi(getenv("NTBC_PAIR_LAUNCHES")))) {
    for (int i = 0; i < n_models; i++) {   // one fused launch per model
      DevGuard dg(models[i]->device);
      st = launch_fused(models[i], ps[i], false, cs);
      if (st) return st;
    }
    return NTBC_OK;
  }
  // conservative pair in ONE persistent launch: both models' prep launches, then one fused kernel whose
  // CTAs are partitioned by model (f1)
  DevGuard dg(models[0]->device);
  ntbc_model_s* lk0 = models[0] < models[1] ? models[0] : models[1];   // fixed lock order
  ntbc_model_s* lk1 = models[0] < models[1] ? models[1] : models[0];
  std::lock_guard<std::recursive_mutex> g0(lk0->mu);
  std::unique_lock<std::recursive_mutex> g1(lk1->mu, std::defer_lock);
  if (lk1 != lk0) g1.lock();
  for (int i = 0; i < 2; i++) {
    st = order_after_last(models[i], cs);
    if (st) return st;
  }
  for (int i = 0; i < 2; i++) {
    st = prepare_fused(models[i], ps[i], false, cs);
    if (st) return st;
  }
  st = launch_prepared(ps, 2, models[0]->arch.hidden, false, cs);
  if (st) return st;
  for (int i = 0; i < 2; i++) {
    st = record_last(models[i], cs);
    if (st) return st;
  }
  return NTBC_OK;
}

ntbc_status ntbc_decode_material_host(const ntbc_model* models, int n_models, const void* const* blobs,
                                      const size_t* blob_sizes, int width, int height, void* const* host_out,
                                      void* stream) {
  if (!models || !blobs || !blob_sizes || !host_out) return fail(NTBC_EINVAL, "NULL argument");
  if (n_models < 1 || n_models > 2) return fail(NTBC_EINVAL, "n_models %d not in {1,2}", n_models);
  ntbc_status st = check_dims(width, height, 0, height / 4);
  if (st) return st;
  if (n_models == 2) {  // reuse the pair validation of ntbc_decode_material without launching anything
    for (int i = 0; i < 2; i++) if (!models[i]) return fail(NTBC_EINVAL, "model %d is NULL", i);
    auto all = [](const Arch& a, int f) { for (int k = 0; k < a.n_tex; k++) if (a.fmt[k] != f) return false; return true; };
    const Arch &x = models[0]->arch, &y = models[1]->arch;
    if (!((all(x, NTBC_BC1) && all(y, NTBC_BC4)) || (all(x, NTBC_BC4) && all(y, NTBC_BC1))))
      return fail(NTBC_EMISMATCH, "conservative pair must be one all-BC1 and one all-BC4 model");
  }
  const int BW = width / 4, BH = height / 4;
  const size_t plane = (size_t)BW * BH * 8, row_bytes = (size_t)BW * 8;
  cudaStream_t cs = (cudaStream_t)stream;
  int t = 0;
  for (int i = 0; i < n_models; i++) {
    ntbc_model_s* m = models[i];
    if (!m) return fail(NTBC_EINVAL, "model %d is NULL", i);
    DevGuard dg(m->device);
    std::lock_guard<std::recursive_mutex> lk(m->mu);   // the call swaps the model's weight slot
    const int n_tex = m->arch.n_tex;
    for (int k = 0; k < n_tex; k++)
      if (!host_out[t + k]) return fail(NTBC_EINVAL, "host_out[%d] is NULL", t + k);
    const size_t need = plane * n_tex;
    if (m->scratch_bytes < need) {
      cudaFree(m->d_scratch);
      m->d_scratch = nullptr;
      m->scratch_bytes = 0;
      if (cudaMalloc(&m->d_scratch, need) != cudaSuccess) { cudaGetLastError(); return fail(NTBC_ENOMEM, "scratch %zu B", need); }
      m->scratch_bytes = need;
    }
    if (m->tlset[1][0] && getenv("NTBC_TIMELINE") && atoi(getenv("NTBC_TIMELINE"))) {
      m->tl_cur ^= 1;
      m->tl = m->tlset[m->tl_cur];
      CUDA_TRY(cudaEventRecord(m->tl[0], cs));
    }
    FusedParams p{};
    p.W = width; p.H = height; p.row_begin = 0; p.row_end = BH;
    for (int k = 0; k < n_tex; k++) p.out[k] = (uint64_t*)(m->d_scratch + k * plane);
    // row chunks for the pipelined copy-back: ~16 chunks of whole block rows
    const int upr = (BW + kUnitBlocks - 1) / kUnitBlocks;
    // 1/16 of the rows per chunk, except the last three such chunks, which are split 4 ways: their
    // rows finish last, and only the final chunk's copy is exposed after the kernel
    // 16 chunks (measured with the upload placed under the kernel: 4/8/16/32 chunks -> 2.67/2.60/2.57/
    // 2.59 ms per C3 call; each stream wait + its copies has a fixed cost, the last chunk is the tail)
    // > 0 when host_out[t..t+n_tex) are planes at one fixed pitch inside ONE pinned allocation (e.g. views of a
    // [tex][BH][BW] tensor): then one 2-D copy per chunk moves every texture (fewer, larger copies: the
    // per-copy cost is what limits fine chunking)
    size_t host_pitch = 0;
    if (n_tex > 1) {
      const ptrdiff_t d = (const uint8_t*)host_out[t + 1] - (const uint8_t*)host_out[t];
      bool uniform = d >= (ptrdiff_t)plane;
      for (int k = 2; k < n_tex && uniform; k++)
        uniform = (const uint8_t*)host_out[t + k] - (const uint8_t*)host_out[t + k - 1] == d;
      if (uniform && one_allocation(host_out[t], (size_t)d * (n_tex - 1) + plane)) host_pitch = (size_t)d;
    }
    // copy-back chunks: 1/16 of the rows each; with 2-D copies the last quarter in 1/64 chunks: the rows of the
    // kernel's last wave of units finish only at its end, and the smaller the chunks they fall into, the less
    // is copied after it (exposed tail 0.12 -> 0.06 ms).  With one copy per texture and chunk, the per-copy
    // cost of the extra chunks outweighs that (measured 0.31 ms tail), so those stay uniform.
    const int big = std::max(1, (BH + 15) / 16);
    const int tail_row0 = host_pitch ? std::min(BH, (3 * BH / 4) / big * big) : BH;
    const int small = std::max(1, big / 4);
    const int n_big = (tail_row0 + big - 1) / big;   // the last one partial when tail_row0 = BH is no multiple
    const int n_chunks = n_big + (BH - tail_row0 + small - 1) / small;
    auto chunk_rows = [&](int c, int& r0, int& r1) {
      if (c < n_big) { r0 = c * big; r1 = std::min(tail_row0, r0 + big); }
      else { r0 = tail_row0 + (c - n_big) * small; r1 = std::min(BH, r0 + small); }
    };
    const bool pipelined = stream_waits_supported(m->device) && n_chunks <= kMaxChunks && ensure_copy_state(m);
    if (!pipelined) {
      st = ntbc_model_upload_async(m, blobs[i], blob_sizes[i], stream);
      if (st) return st;
    } else {
      // upload into the idle weight slot on upload_stream (overlaps the previous call's kernel) once
      // that kernel has STARTED: the slot's last reader (the kernel before it) is done by then, and the
      // upload no longer competes with the copy-back tail of the call before (measured: 2.75 -> 2.6 ms
      // per call when it waited only for the slot); the kernel below waits for the upload.
      Arch a;
      st = parse(blobs[i], blob_sizes[i], a);
      if (st) return st;
      if (!same_arch(a, m->arch)) return fail(NTBC_EMISMATCH, "blob architecture differs from the loaded model");
      const int s = m->cur ^ 1;
      m->arch = a;
      m->cur = s;
      m->d_blob = m->slot_blob[s];
      CUDA_TRY(cudaStreamWaitEvent(m->upload_stream, m->copy_start, 0));   // the previous call's kernel start
      st = upload(m, blobs[i], blob_sizes[i], m->upload_stream);
      if (st) return st;
      CUDA_TRY(cudaEventRecord(m->uploaded, m->upload_stream));
      if (getenv("NTBC_TIMELINE") && atoi(getenv("NTBC_TIMELINE")) && m->tl[1]) CUDA_TRY(cudaEventRecord(m->tl[1], m->upload_stream));
      CUDA_TRY(cudaStreamWaitEvent(cs, m->uploaded, 0));
    }
    if (pipelined) {
      p.progress = m->d_progress;
      p.chunk_rows = big;
      p.tail_row0 = tail_row0;
      p.tail_rows = small;
    }
    const bool tl = pipelined && getenv("NTBC_TIMELINE") && atoi(getenv("NTBC_TIMELINE"));
    if (tl && !m->tlset[1][0])
      for (auto& row : m->tlset)
        for (auto& e : row) CUDA_TRY(cudaEventCreate(&e));
    m->tl_on = tl;
    if (tl) CUDA_TRY(cudaEventRecord(m->tl[2], cs));
    if (pipelined) {  // copy stream: ordered after the upload and whatever precedes it on `stream`
      CUDA_TRY(cudaEventRecord(m->copy_start, cs));
      for (int i = 0; i < kCopyStreams; i++) CUDA_TRY(cudaStreamWaitEvent(m->copy_stream[i], m->copy_start, 0));
    }
    st = launch_fused(m, p, false, cs);
    if (st) return st;
    if (tl) CUDA_TRY(cudaEventRecord(m->tl[3], cs));
    if (pipelined) CUDA_TRY(cudaEventRecord(m->slot_free[m->cur], cs));
    if (!pipelined) {
      for (int k = 0; k < n_tex; k++)
        CUDA_TRY(cudaMemcpyAsync(host_out[t + k], p.out[k], plane, cudaMemcpyDeviceToHost, cs));
    } else {
      // the launched kernel publishes every chunk: advance all targets first, so an error below cannot
      // leave later chunks' targets one call behind the device counters
      for (int c = 0; c < n_chunks; c++) {
        int r0, r1;
        chunk_rows(c, r0, r1);
        m->progress_target[c] += (unsigned long long)(r1 - r0) * upr;
      }
      // chunk c's copies wait until all units of chunk c have been published by the running kernel
      for (int c = 0; c < n_chunks; c++) {
        int r0, r1;
        chunk_rows(c, r0, r1);
        // the last chunk finishes with the kernel: copy it in stream order right behind the kernel
        // (no counter wait, whose latency would add to the exposed tail)
        const bool last = c == n_chunks - 1 && n_chunks > 1;
        cudaStream_t xs = last ? cs : m->copy_stream[c % kCopyStreams];
        if (!last && g_wait64((CUstream)xs, (CUdeviceptr)(m->d_progress + c), m->progress_target[c],
                              CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
          return fail(NTBC_ECUDA, "stream wait on progress counter failed");
        if (host_pitch)   // the caller's planes are equally spaced: one 2-D copy moves the chunk of every texture
          CUDA_TRY(cudaMemcpy2DAsync((uint8_t*)host_out[t] + r0 * row_bytes, host_pitch,
                                     (const uint8_t*)p.out[0] + r0 * row_bytes, plane, (size_t)(r1 - r0) * row_bytes,
                                     n_tex, cudaMemcpyDeviceToHost, xs));
        else
          for (int k = 0; k < n_tex; k++)
            CUDA_TRY(cudaMemcpyAsync((uint8_t*)host_out[t + k] + r0 * row_bytes, (const uint8_t*)p.out[k] + r0 * row_bytes,
                                     (size_t)(r1 - r0) * row_bytes, cudaMemcpyDeviceToHost, xs));
      }
      for (int i = 0; i < kCopyStreams; i++) {   // the caller's stream sees every finished copy
        if (tl) CUDA_TRY(cudaEventRecord(m->tl[4 + i], m->copy_stream[i]));
        CUDA_TRY(cudaEventRecord(m->copy_done[i], m->copy_stream[i]));
        CUDA_TRY(cudaStreamWaitEvent(cs, m->copy_done[i], 0));
      }
    }
    t += n_tex;
  }
  return NTBC_OK;
}

ntbc_status ntbc_debug_host_timeline(ntbc_model m, float* ms_out, int n) {
  if (!m || !ms_out || n < 5 + 2 * kCopyStreams) return fail(NTBC_EINVAL, "need %d outputs", 5 + 2 * kCopyStreams);
  if (!m->tl_on || !m->tlset[1][0]) return fail(NTBC_EINVAL, "no timeline recorded (set NTBC_TIMELINE=1)");
  DevGuard dg(m->device);
  cudaEvent_t* prev = m->tlset[m->tl_cur ^ 1];
  for (int i = 0; i < 4 + kCopyStreams; i++) {
    CUDA_TRY(cudaEventSynchronize(m->tl[i]));
    CUDA_TRY(cudaEventElapsedTime(ms_out + i, m->tl[0], m->tl[i]));
  }
  // the previous call's start and copy completions relative to this call's start
  CUDA_TRY(cudaEventElapsedTime(ms_out + 4 + kCopyStreams, m->tl[0], prev[0]));
  for (int i = 0; i < kCopyStreams; i++)
    CUDA_TRY(cudaEventElapsedTime(ms_out + 5 + kCopyStreams + i, m->tl[0], prev[4 + i]));
  return NTBC_OK;
}

ntbc_status ntbc_encode_bc(const float* texels, ntbc_format fmt, int width, int height, int n_refine,
                           void* out_blocks, void* stream) {
  if (!texels || !out_blocks) return fail(NTBC_EINVAL, "NULL argument");
  if (fmt != NTBC_BC1 && fmt != NTBC_BC4) return fail(NTBC_EINVAL, "bad format %d", (int)fmt);
  if (n_refine < 0 || n_refine > 8) return fail(NTBC_EINVAL, "n_refine %d not in [0,8]", n_refine);
  if ((uintptr_t)out_blocks & 7) return fail(NTBC_EINVAL, "out_blocks not 8-B aligned");
  ntbc_status st = check_dims(width, height, 0, height / 4);
  if (st) return st;
  const long long nb = (long long)(width / 4) * (height / 4);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<long long>((nb + 127) / 128, (long long)sms * 16);
  if (fmt == NTBC_BC1)
    refenc_kernel<3><<<grid, 128, 0, (cudaStream_t)stream>>>(texels, width, height, n_refine, (uint64_t*)out_blocks);
  else
    refenc_kernel<1><<<grid, 128, 0, (cudaStream_t)stream>>>(texels, width, height, n_refine, (uint64_t*)out_blocks);
  g_launches++;
  CUDA_TRY(cudaGetLastError());
  return NTBC_OK;
}

namespace {
bool train_layout(const ntbc_train_arch* a, TrainParams& p, int net) {
  if (!a || a->n_textures < 1 || a->n_textures > kMaxTex || a->hidden != 64 || a->levels < 1 ||
      a->levels > kMaxLevels || a->coarsest < 2 || ((long long)a->coarsest << (a->levels - 1)) > 8192)
    return false;
  p.n_tex = a->n_textures;
  p.n_c = p.n_e = 0;
  for (int k = 0; k < p.n_tex; k++) {
    if (a->fmt[k] != NTBC_BC1 && a->fmt[k] != NTBC_BC4) return false;
    p.fmt[k] = a->fmt[k];
    p.n_c += a->fmt[k] == NTBC_BC1 ? 3 : 1;
    p.n_e += a->fmt[k] == NTBC_BC1 ? 6 : 2;
  }
  p.hidden = a->hidden;
  p.levels = a->levels;
  p.coarsest = a->coarsest;
  long long off = 0;
  for (int l = 0; l < p.levels; l++) {
    p.lvl_off[l] = off;
    const long long res = (long long)p.coarsest << l;
    off += res * res * 2;
  }
  const int dims[5] = {2 * p.levels, p.hidden, p.hidden, p.hidden, net == 1 ? p.n_c : p.n_e};
  for (int l = 0; l < 4; l++) {
    p.kin[l] = dims[l];
    p.kout[l] = dims[l + 1];
    p.w_off[l] = off;
    off += (long long)dims[l] * dims[l + 1];
    p.b_off[l] = off;
    off += dims[l + 1];
  }
  g_train_total = off;
  return true;
}
}  // namespace

long long ntbc_train_param_count(const ntbc_train_arch* arch) {
  TrainParams p{};
  if (!train_layout(arch, p, 1)) return -1;
  return g_train_total;
}

long long ntbc_train_endpoint_param_count(const ntbc_train_arch* arch) {
  TrainParams p{};
  if (!train_layout(arch, p, 0)) return -1;
  return g_train_total;
}

namespace {
ntbc_status train_step(int net, const ntbc_train_arch* arch, float* params, float* grads, float* adam_m,
                       float* adam_v, int step, const int* xy, const float* cref, const float* eref, int batch,
                       int width, int height, float temperature, float lr_grid, float lr_mlp, float* loss,
                       void* stream) {
  TrainParams p{};
  if (!train_layout(arch, p, net)) return fail(NTBC_EINVAL, "unsupported training architecture (hidden must be 64)");
  const long long n = g_train_total, n_grid = p.w_off[0];
  if (!params || !grads || !adam_m || !adam_v || !xy || !cref || !eref || !loss) return fail(NTBC_EINVAL, "NULL argument");
  if (batch < 1 || width < 1 || height < 1 || step < 1 || !(temperature > 0.0f)) return fail(NTBC_EINVAL, "bad batch/size/step/T");
  if ((uintptr_t)grads & 15) return fail(NTBC_EINVAL, "grads not 16-B aligned (vector atomics)");
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaMemsetAsync(grads, 0, (size_t)n * sizeof(float), st));
  CUDA_TRY(cudaMemsetAsync(loss, 0, sizeof(float), st));
  p.qsz = nullptr;
  if (arch->qat) {   // QAT: per-level min/max -> (s, z) of the 8-bit fake quantizer, on the GPU
    // [2*kMaxLevels] ordered-int min/max, then [2*kMaxLevels] (s, z): one scratch per (device, stream), so
    // steps on other devices or concurrent streams never share it
    static std::mutex q_mu;
    static std::map<std::pair<int, cudaStream_t>, int*> q_scratch;
    int q_dev = 0;
    cudaGetDevice(&q_dev);
    int* d_q = nullptr;
    {
      std::lock_guard<std::mutex> lk(q_mu);
      int*& slot = q_scratch[{q_dev, st}];
      if (!slot && cudaMalloc(&slot, 4 * kMaxLevels * sizeof(int)) != cudaSuccess) { cudaGetLastError(); slot = nullptr; return fail(NTBC_ENOMEM, "QAT scratch"); }
      d_q = slot;
    }
    int init[2 * kMaxLevels];
    for (int l = 0; l < kMaxLevels; l++) { init[2 * l] = 0x7FFFFFFF; init[2 * l + 1] = (int)0x80000000; }
    CUDA_TRY(cudaMemcpyAsync(d_q, init, sizeof(init), cudaMemcpyHostToDevice, st));
    LevelList L{};
    for (int l = 0; l < p.levels; l++) {
      const long long res = (long long)p.coarsest << l;
      L.off[l] = p.lvl_off[l];
      L.cnt[l] = res * res * 2;
    }
    level_minmax_kernel<<<dim3(148, p.levels), 256, 0, st>>>(params, L, p.levels, d_q);
    qat_params_kernel<<<1, 32, 0, st>>>(d_q, p.levels, reinterpret_cast<float*>(d_q + 2 * kMaxLevels));
    g_launches += 2;
    p.qsz = reinterpret_cast<const float*>(d_q + 2 * kMaxLevels);
  }
  p.params = params; p.grads = grads; p.xy = xy; p.cref = cref; p.eref = eref;
  p.B = batch; p.W = width; p.H = height; p.T = temperature; p.loss = loss;
  auto al4 = [](size_t n) { return (n + 3) & ~(size_t)3; };
  size_t smem = 0;
  for (int l = 0; l < 4; l++) smem += al4((size_t)p.kin[l] * p.kout[l]) + al4((size_t)p.kout[l]);
  smem += al4((size_t)kTrainTile * (2 * p.levels + 1)) + 4 * (size_t)kTrainTile * (64 + 4) + kTrainTile;
  smem *= sizeof(float);
  auto kern = net == 1 ? train_step_kernel<64, 1> : train_step_kernel<64, 0>;
  CUDA_TRY(allow_smem((const void*)kern, 227 * 1024));
  kern<<<(batch + kTrainTile - 1) / kTrainTile, kTrainTile * kTrainQ, smem, st>>>(p);
  g_launches++;
  const double bc1 = 1.0 - std::pow(0.9, step), bc2 = 1.0 - std::pow(0.999, step);
  const int grid = (int)std::min<long long>((n + 255) / 256, 148 * 32);
  adam_kernel<<<grid, 256, 0, st>>>(params, grads, adam_m, adam_v, n, n_grid, lr_grid, lr_mlp, 0.9f, 0.999f, 1e-15f,
                                    (float)bc1, (float)bc2);
  g_launches++;
  CUDA_TRY(cudaGetLastError());
  return NTBC_OK;
}
}  // namespace

ntbc_status ntbc_train_colour_step(const ntbc_train_arch* arch, float* params, float* grads, float* adam_m,
                                   float* adam_v, int step, const int* xy, const float* cref, const float* eref,
                                   int batch, int width, int height, float temperature, float lr_grid,
                                   float lr_mlp, float* loss, void* stream) {
  return train_step(1, arch, params, grads, adam_m, adam_v, step, xy, cref, eref, batch, width, height, temperature,
                    lr_grid, lr_mlp, loss, stream);
}

ntbc_status ntbc_train_endpoint_step(const ntbc_train_arch* arch, float* params, float* grads, float* adam_m,
                                     float* adam_v, int step, const int* bxy, const float* cref16, const float* eref,
                                     int batch, int blocks_w, int blocks_h, float temperature, float lr_grid,
                                     float lr_mlp, float* loss, void* stream) {
  return train_step(0, arch, params, grads, adam_m, adam_v, step, bxy, cref16, eref, batch, blocks_w, blocks_h,
                    temperature, lr_grid, lr_mlp, loss, stream);
}

ntbc_status ntbc_decode_bc(const void* blocks, ntbc_format fmt, int width, int height, float* out, void* stream) {
  if (!blocks || !out) return fail(NTBC_EINVAL, "NULL argument");
  if (fmt != NTBC_BC1 && fmt != NTBC_BC4) return fail(NTBC_EINVAL, "bad format %d", (int)fmt);
  ntbc_status st = check_dims(width, height, 0, height / 4);
  if (st) return st;
  const long long n = (long long)width * height;
  const int grid = (int)std::min<long long>((n + 255) / 256, 148 * 16);
  decode_bc_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>((const uint64_t*)blocks, (int)fmt, width, height, out);
  g_launches++;
  CUDA_TRY(cudaGetLastError());
  return NTBC_OK;
}

ntbc_status ntbc_debug_mlp(ntbc_model m, int width, int height, int r0, int r1, float* endpoints, float* colors,
                           void* stream) {
  if (!m || !endpoints || !colors) return fail(NTBC_EINVAL, "NULL argument");
  ntbc_status st = check_dims(width, height, r0, r1);
  if (st) return st;
  DevGuard dg(m->device);
  FusedParams p{};
  p.W = width; p.H = height; p.row_begin = r0; p.row_end = r1;
  p.dump_ep = endpoints;
  p.dump_col = colors;
  return launch_fused(m, p, true, (cudaStream_t)stream);
}

ntbc_status ntbc_debug_features(ntbc_model m, int width, int height, int r0, int r1, float* block_features,
                                float* texel_features, void* stream) {
  if (!m || !block_features || !texel_features) return fail(NTBC_EINVAL, "NULL argument");
  ntbc_status st = check_dims(width, height, r0, r1);
  if (st) return st;
  DevGuard dg(m->device);
  FusedParams p{};
  p.W = width; p.H = height; p.row_begin = r0; p.row_end = r1;
  p.dump_ep = block_features;
  p.dump_col = texel_features;
  p.debug_flags = 2;
  return launch_fused(m, p, true, (cudaStream_t)stream);
}

ntbc_status ntbc_pack(int n_tex, const int* fmts, const float* endpoints, const float* colors, int width, int height,
                      int r0, int r1, void* const* out_blocks, void* stream) {
  if (!fmts || !endpoints || !colors || !out_blocks) return fail(NTBC_EINVAL, "NULL argument");
  if (n_tex < 1 || n_tex > kMaxTex) return fail(NTBC_EINVAL, "n_textures %d not in [1,8]", n_tex);
  ntbc_status st = check_dims(width, height, r0, r1);
  if (st) return st;
  PackParams p{};
  p.ep = endpoints; p.col = colors; p.W = width; p.BW = width / 4; p.rows = r1 - r0; p.n_tex = n_tex;
  int eo = 0, co = 0;
  for (int k = 0; k < n_tex; k++) {
    if (fmts[k] != NTBC_BC1 && fmts[k] != NTBC_BC4) return fail(NTBC_EINVAL, "bad format %d", fmts[k]);
    if (!out_blocks[k] || ((uintptr_t)out_blocks[k] & 7)) return fail(NTBC_EINVAL, "out_blocks[%d] NULL or misaligned", k);
    p.fmt[k] = fmts[k]; p.ep_off[k] = eo; p.col_off[k] = co; p.out[k] = (uint64_t*)out_blocks[k];
    p.pal_off[k] = p.pal_stride;
    eo += fmts[k] == NTBC_BC1 ? 6 : 2;
    co += fmts[k] == NTBC_BC1 ? 3 : 1;
    p.pal_stride += fmts[k] == NTBC_BC1 ? 12 : 8;
  }
  p.n_e = eo; p.n_c = co;
  p.vec16 = (p.BW % 2) == 0;
  for (int k = 0; k < n_tex; k++)
    if ((uintptr_t)p.out[k] & 15) p.vec16 = 0;
  p.tiles_per_row = (p.BW + kPackTileBlocks - 1) / kPackTileBlocks;
  p.n_tiles = p.tiles_per_row * p.rows;
  const size_t smem = (384 + (size_t)kPackStages * (4 * (4 * kPackTileBlocks * p.n_c + 4) +
                                                    ((kPackTileBlocks * p.n_e + 3) & ~3)) +
                       (NTBC_PACK_PAL == 1 ? (size_t)kPackTileBlocks * p.pal_stride : 0) +
                       (NTBC_PACK_PAL == 2 ? (size_t)(kPackThreads / 32) * 2 * p.pal_stride : 0)) * sizeof(float) +
                      kPackTileBlocks * kMaxTex * sizeof(uint32_t);
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  static void (*const kernels[kMaxTex])(PackParams) = {pack_kernel<1>, pack_kernel<2>, pack_kernel<3>, pack_kernel<4>,
                                                       pack_kernel<5>, pack_kernel<6>, pack_kernel<7>, pack_kernel<8>};
  static void (*const kernels_bt[kMaxTex])(PackParams) = {pack_kernel_bt<1>, pack_kernel_bt<2>, pack_kernel_bt<3>,
                                                          pack_kernel_bt<4>, pack_kernel_bt<5>, pack_kernel_bt<6>,
                                                          pack_kernel_bt<7>, pack_kernel_bt<8>};
  static_assert(kMaxTex == 8, "pack kernel instantiations");
  // default: one thread per (block, texture) (pack_kernel_bt); NTBC_PACK_WARP=1: the warp-per-two-blocks form
  // (the bulk copies of the thread form need 16-B aligned colour rows: a misaligned `colors` takes the warp form)
  const bool warp_form = (getenv("NTBC_PACK_WARP") && atoi(getenv("NTBC_PACK_WARP"))) || ((uintptr_t)colors & 15);
  const auto kern = warp_form ? kernels[n_tex - 1] : kernels_bt[n_tex - 1];
  const int threads = warp_form ? kPackThreads : kBtTile * n_tex;
  const size_t smem_k = warp_form ? smem : (384 + (size_t)kBtStages * (4 * (size_t)(4 * kBtTile * p.n_c) +
                                                                        (size_t)((kBtTile * p.n_e + 3) & ~3))) * sizeof(float) +
                                            8 * kBtStages;
  CUDA_TRY(allow_smem((const void*)kern, 227 * 1024));
  // the whole unified L1 as shared memory: several CTAs of staged tiles per SM
  CUDA_TRY(cudaFuncSetAttribute((const void*)kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                cudaSharedmemCarveoutMaxShared));
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem_k));
  // persistent grid: exactly the resident CTAs (a second partial wave of grid-stride CTAs would double
  // the tail), each striding over 64-block tiles
  const int n_tiles = warp_form ? p.n_tiles : (p.BW + kBtTile - 1) / kBtTile * p.rows;
  const int grid = std::max(1, std::min(n_tiles, sms * std::max(per_sm, 1)));
  if (smem_k > 227 * 1024) return fail(NTBC_EINVAL, "pack tile needs %zu B of shared memory", smem_k);
  kern<<<grid, threads, smem_k, (cudaStream_t)stream>>>(p);
  g_launches++;
  CUDA_TRY(cudaGetLastError());
  return NTBC_OK;
}

ntbc_status ntbc_debug_mma(const void* A, const void* B, const float* C, float* D, int K, int N, void* stream) {
  if (!A || !B || !D) return fail(NTBC_EINVAL, "NULL argument");
  if (K <= 0 || K % 16 || K > 128 || (N != 16 && N != 32 && N != 64)) return fail(NTBC_EINVAL, "bad K=%d N=%d", K, N);
  const size_t smem = 128 * K * 2 + 64 * K * 2 + 64;
  CUDA_TRY(allow_smem((const void*)mma_probe_kernel, 227 * 1024));
  mma_probe_kernel<<<1, 128, smem, (cudaStream_t)stream>>>((const __half*)A, (const __half*)B, C, D, K, N);
  g_launches++;
  CUDA_TRY(cudaGetLastError());
  return NTBC_OK;
}

uint64_t ntbc_launch_count(void) { return g_launches.load(); }

ntbc_status ntbc_set_contract(ntbc_model m, int contract) {
  if (!m) return fail(NTBC_EINVAL, "model is NULL");
  if (contract < 0 || contract > 2) return fail(NTBC_EINVAL, "contract %d not in {0 (H), 1 (F), 2 (P)}", contract);
  if (contract != 0 && m->arch.naive) return fail(NTBC_EINVAL, "contracts F and P are not provided for the naive variant");
  std::lock_guard<std::recursive_mutex> lk(m->mu);
  m->contract = contract;
  return NTBC_OK;
}

ntbc_status ntbc_debug_time_fused(void* start_event, void* end_event) {
  if ((start_event == nullptr) != (end_event == nullptr)) return fail(NTBC_EINVAL, "pass both events or neither");
  g_time_fused[0] = (cudaEvent_t)start_event;
  g_time_fused[1] = (cudaEvent_t)end_event;
  return NTBC_OK;
}

ntbc_status ntbc_peer_export(const void* device_ptr, void* handle_out) {
  if (!device_ptr || !handle_out) return fail(NTBC_EINVAL, "NULL argument");
  cudaPointerAttributes at{};
  CUDA_TRY(cudaPointerGetAttributes(&at, device_ptr));
  if (at.type != cudaMemoryTypeDevice) return fail(NTBC_EINVAL, "not a device allocation");
  DevGuard dg(at.device);
  addr_range_fn fn = get_addr_range();
  if (!fn) return fail(NTBC_ECUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (fn(&base, &size, (CUdeviceptr)device_ptr) != CUDA_SUCCESS)
    return fail(NTBC_ECUDA, "cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, (void*)base));
  const uint64_t off = (uint64_t)((CUdeviceptr)device_ptr - base);
  std::memcpy(handle_out, &h, sizeof(h));
  std::memcpy((uint8_t*)handle_out + 64, &off, sizeof(off));
  return NTBC_OK;
}

ntbc_status ntbc_peer_open(const void* handle, int cuda_device, void** device_ptr_out) {
  if (!handle || !device_ptr_out) return fail(NTBC_EINVAL, "NULL argument");
  *device_ptr_out = nullptr;
  DevGuard dg(cuda_device);
  cudaIpcMemHandle_t h;
  uint64_t off = 0;
  std::memcpy(&h, handle, sizeof(h));
  std::memcpy(&off, (const uint8_t*)handle + 64, sizeof(off));
  void* base = nullptr;
  CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  void* p = (uint8_t*)base + off;
  {
    std::lock_guard<std::mutex> lk(g_peer_mu);
    g_peer_base[p] = base;
  }
  *device_ptr_out = p;
  return NTBC_OK;
}

ntbc_status ntbc_peer_close(void* device_ptr) {
  void* base = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_peer_mu);
    auto it = g_peer_base.find(device_ptr);
    if (it == g_peer_base.end()) return fail(NTBC_EINVAL, "pointer was not returned by ntbc_peer_open");
    base = it->second;
    g_peer_base.erase(it);
  }
  CUDA_TRY(cudaIpcCloseMemHandle(base));
  return NTBC_OK;
}

const char* ntbc_last_error(void) { return g_err.c_str(); }

}  // extern "C"
