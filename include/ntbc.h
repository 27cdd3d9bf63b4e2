/* ntbc.h -- C ABI of libntbc.so, the B200 (sm_100a) NTBC inference hot path.
 *
 * Neural Texture Block Compression (arXiv 2407.09543).  "Network weights are stored in the disk
 * which are loaded into the memory.  Then inference is executed to reconstruct block-compressed
 * texture data which are copied to VRAM"; "NTBC predicts block-compressed data
 * instead of loading block-compressed textures from the disk, and then texel values are decoded
 * from the compressed data using the existing BC decompression method".
 *
 * Conventions (all entry points):
 *   - return ntbc_status (0 = OK, < 0 = error) and never throw; on error a thread-local message is
 *     available from ntbc_last_error();
 *   - "device" pointers are CUDA device memory of the model's device, allocated and owned by the
 *     caller (typically torch tensors); "host" pointers are host memory owned by the caller;
 *   - stream = a cudaStream_t passed as void* (NULL = legacy default stream); calls taking a
 *     stream are asynchronous: launch errors are returned, device faults surface at the caller's
 *     next synchronisation of that stream;
 *   - no entry point allocates device memory on the hot path (ntbc_decode_material,
 *     ntbc_decode_bc, ntbc_pack); scratch is owned by the model and sized at load time;
 *   - thread safety: any call may be made from any host thread.  Calls that use or change a model
 *     (decode, upload, debug dumps) are serialised per model on the host, and decodes of one model
 *     issued on different streams are ordered on the device (each waits for the model's previous
 *     launch: they share the model's fp32 grid region), so concurrent use of ONE model on several
 *     streams is correct but not concurrent on the GPU; use one model per stream for overlap.
 * Readings of silent passages are numbered R1..R20 in DESIGN.md §2.
 */
#ifndef NTBC_H
#define NTBC_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ntbc_model_s* ntbc_model;               /* opaque, library-owned */

typedef enum { NTBC_BC1 = 1, NTBC_BC4 = 4 } ntbc_format;

typedef enum {
  NTBC_OK = 0,
  NTBC_EINVAL = -1,    /* bad argument: NULL, size/alignment/range (W,H % 4, rows, pointer alignment) */
  NTBC_EFORMAT = -2,   /* bad .ntbc blob: magic, version, truncation, dims inconsistent with header */
  NTBC_EMISMATCH = -3, /* models vs request (e.g. conservative pair not one all-BC1 + one all-BC4) */
  NTBC_ENOMEM = -4,    /* device allocation failed */
  NTBC_ECUDA = -5      /* CUDA runtime error (message has the CUDA error string) */
} ntbc_status;

typedef struct {
  int n_textures;          /* textures in head order (<= 8) */
  int fmt[8];              /* NTBC_BC1 / NTBC_BC4 per texture */
  int hidden, n_hidden;    /* MLP width (16/32/64) and depth (3) */
  int n_endpoint_out;      /* N_e = 6 N_RGB + 2 N_SC */
  int n_color_out;         /* N_c = 3 N_RGB + N_SC */
  int block_levels, block_coarsest, texel_levels, texel_coarsest, features;
  int variant;             /* 0: NTBC colour network; 1: naive weight network with
                              n_color_out = n_textures weights per texel (DESIGN R21-R23) */
  size_t device_bytes;     /* device memory held by the model */
} ntbc_model_info;

/* Parse and validate a host .ntbc blob (int8 grids + per-level (s, z) + fp16 MLPs,
 * PAPER.md:321-322, 342) and upload it to `cuda_device` as-is (one copy into a device weight slot that
 * also holds the fp32 grid region every decode dequantizes into; the fused kernel builds the tcgen05
 * shared-memory operand images of the MLPs, bias folded in as an extra K chunk, in its prologue).
 * The blob is not retained (caller may free it after return).  Synchronous.
 * Errors: NTBC_EINVAL (NULL args), NTBC_EFORMAT, NTBC_ENOMEM, NTBC_ECUDA. */
ntbc_status ntbc_load_model(const void* blob, size_t nbytes, int cuda_device, ntbc_model* out);

/* Re-upload the parameters of an already loaded model from a (preferably pinned) host blob of the
 * same architecture, asynchronously on `stream` (host->device copies only; the blob must stay
 * valid until the stream reaches this point).  Errors: NTBC_EINVAL, NTBC_EFORMAT,
 * NTBC_EMISMATCH (architecture differs), NTBC_ECUDA. */
ntbc_status ntbc_model_upload_async(ntbc_model m, const void* blob, size_t nbytes, void* stream);

ntbc_status ntbc_model_get_info(ntbc_model m, ntbc_model_info* out);
void ntbc_free_model(ntbc_model m);                     /* NULL ok; caller guarantees no in-flight use */

/* Rows a1-a8 of SURVEY §8: per model a prep launch -- the grid dequantization (Eq.2; every level's
 * codes -> fp32 in the model's weight slot) and the fused kernel's shared-memory prefix image (tcgen05
 * operand images of both MLPs, copied into every CTA by the TMA engine) -- then ONE fused sm_100a kernel
 * (shared by the two models of a conservative pair, CTAs partitioned by model): bilinear sampling
 * (P:334-337), endpoint MLP per block and colour MLP per texel on tcgen05 tensor cores
 * (P:257-272), endpoint quantization (R11-R13), palettes (Eq.7/8), per-texel
 * argmax of negative distance (Eq.9-10) and BC1/BC4 bit packing.
 *   models / n_models: 1 = aggressive (one model), 2 = conservative (an all-BC1 model and
 *     an all-BC4 model);
 *   width, height: texels, multiples of 4, identical for every texture of the material;
 *   [block_row_begin, block_row_end): shard of the H/4 block rows to decode (0 <= begin < end <= H/4);
 *   out_blocks: one device pointer per texture, models[0]'s textures then models[1]'s, each
 *     (end-begin) * (width/4) * 8 bytes, 8-B aligned (16-B aligned pointers and an even width/4 let
 *     the kernel write two adjacent blocks' words as one 16-byte store); row-major little-endian
 *     64-bit BC words:
 *     BC1 = c0 | c1<<16 | sum code_i << (32+2i), BC4 = e0 | e1<<8 | sum code_i << (16+3i), texel i = 4y+x.
 * Errors: NTBC_EINVAL, NTBC_EMISMATCH, NTBC_ECUDA. */
ntbc_status ntbc_decode_material(const ntbc_model* models, int n_models, int width, int height,
                                 int block_row_begin, int block_row_end, void* const* out_blocks,
                                 void* stream);

/* End-to-end variant of ntbc_decode_material for host buffers: per model, copies its host blob
 * (pinned recommended; same architecture as the loaded model) host->device, decodes all block rows,
 * and copies every texture's BC words device->host into host_out[t] (height/4 * width/4 * 8 bytes).
 * Uses model-owned device scratch (allocated on first use for a given size, outside any timed loop).
 * Asynchronous on `stream`; call cudaStreamSynchronize before reading host_out.
 * Pipelining (when the device supports 64-bit stream memory operations; NTBC_NO_PIPELINED_COPY=1
 * disables it): the blob is uploaded into the model's idle second weight slot on an internal stream
 * that does NOT wait for earlier work on `stream` -- the blob must hold its final contents when this
 * function is called and stay unchanged until `stream` reaches this call -- so the upload overlaps the
 * previous call's kernel; the kernel publishes finished row chunks (1/16 of the rows each) through
 * device counters and an internal copy stream copies each chunk back while later rows are decoded.
 * `stream` waits for all of it, so host_out is complete once `stream` reaches this call.
 * When host_out[t..] of a model are equally spaced planes inside one pinned allocation (e.g. views of a
 * [tex][H/4][W/4] buffer), each chunk is one 2-D copy for all textures and the last quarter of the rows
 * is copied in smaller chunks (a shorter exposed tail); otherwise one copy per texture and chunk.
 * Not re-entrant per model: calls on the same model must not run concurrently on different streams.
 * Errors: as ntbc_decode_material, plus NTBC_ENOMEM. */
ntbc_status ntbc_decode_material_host(const ntbc_model* models, int n_models, const void* const* blobs,
                                      const size_t* blob_sizes, int width, int height,
                                      void* const* host_out, void* stream);

/* Debug: with NTBC_TIMELINE=1 in the environment, ntbc_decode_material_host records CUDA events;
 * this returns, for the model's last call, the times (ms) relative to the call's start on `stream` of:
 * [0] call start, [1] its upload done (negative when it overlapped the previous call), [2] kernel
 * start, [3] kernel end, [4..7] copy-back done per internal copy stream, [8] the previous call's start,
 * [9..12] the previous call's copy-back done per stream (negative).  n >= 13.  Synchronizes. */
ntbc_status ntbc_debug_host_timeline(ntbc_model m, float* ms_out, int n);

/* reference BC1/BC4 encoder -- the documented stand-in for the paper's Compressonator
 * "two refine steps" (SPEC encode_block_reference S:153-161; R24-R29):
 * PCA (BC1) or min/max (BC4, both modes) endpoints, n_refine least-squares refinements of the
 * endpoints on the current index assignment, BC1 4-colour order, BC4 lower-error mode, per-texel
 * optimal indices on the final palette.  One thread per block.
 *   texels: device, height*width*(3 for BC1 | 1 for BC4) fp32 in [0,1], row-major, RGB interleaved;
 *   out_blocks: device, (height/4)*(width/4) u64 words, row-major, 8-B aligned; n_refine in [0, 8].
 * Errors: NTBC_EINVAL, NTBC_ECUDA. */
ntbc_status ntbc_encode_bc(const float* texels, ntbc_format fmt, int width, int height, int n_refine,
                           void* out_blocks, void* stream);

/* one training step of the colour network (Eq. 14-15 / P:285-304 / App. A,
 * Adam P:340-341; R30-R32).  fp32 parameters in one flat device vector, layout: the texel
 * grid levels coarse -> fine, each [res][res][2] (res = coarsest << l), then per layer l = 0..3
 * W_l [in][out] and b_l [out] of the 2*levels -> hidden x3 -> N_c colour MLP.  The step zeroes `grads`,
 * computes loss = mean over the batch of sum over textures (|c_hat - c|^2 + |c_dec - c|^2) with the
 * STE expectation at temperature T for the argmax, accumulates its gradient, and applies one
 * bias-corrected Adam update (beta1 0.9, beta2 0.999, eps 1e-15; lr_grid for the grid entries, lr_mlp
 * for the MLP) with step number `step` (>= 1).
 *   xy: device int32 [B][2] texel coordinates (< W, H); cref: device fp32 [B][N_c] reference colours
 *   (head order); eref: device fp32 [B][N_e] reference endpoints of each texel's block (BC1: e0 rgb,
 *   e1 rgb; BC4: e0, e1); loss: device fp32 scalar (overwritten).  grads must be 16-B aligned (gradients
 *   are accumulated with 8- and 16-byte vector atomics).  Not deterministic in the last bits (atomic
 *   accumulation order).  Errors: NTBC_EINVAL, NTBC_ECUDA. */
typedef struct {
  int n_textures, fmt[8], hidden, levels, coarsest;
  int qat;   /* 1: the grid passes the per-level 8-bit fake quantizer (Eq. 1-5; DESIGN R33) */
} ntbc_train_arch;
long long ntbc_train_param_count(const ntbc_train_arch* arch);   /* floats in the parameter vector; <0: invalid */
ntbc_status ntbc_train_colour_step(const ntbc_train_arch* arch, float* params, float* grads, float* adam_m,
                                   float* adam_v, int step, const int* xy, const float* cref, const float* eref,
                                   int batch, int width, int height, float temperature, float lr_grid,
                                   float lr_mlp, float* loss, void* stream);
/* The endpoint network's step (Eq. 14: L_e + L_cd): parameters = the BLOCK grid levels and
 * the 2*levels -> hidden x3 -> N_e MLP (same layout rules); samples are blocks: bxy [B][2] block
 * coordinates (< blocks_w, blocks_h), eref [B][N_e] reference endpoints, cref16 [B][16][N_c] the
 * reference colours of the block's texels (texel i = 4y + x).  Each texel's index comes from the
 * PREDICTED endpoints' palette and its reference colour; the decoded colour is the REFERENCE
 * endpoints' palette entry at that index; STE and Adam as above. */
long long ntbc_train_endpoint_param_count(const ntbc_train_arch* arch);
ntbc_status ntbc_train_endpoint_step(const ntbc_train_arch* arch, float* params, float* grads, float* adam_m,
                                     float* adam_v, int step, const int* bxy, const float* cref16, const float* eref,
                                     int batch, int blocks_w, int blocks_h, float temperature, float lr_grid,
                                     float lr_mlp, float* loss, void* stream);

/* Row a9 (verification): decode a BC1/BC4 surface with the DirectX palettes (decode uses
 * the same float palette arithmetic as the encoder, R18) into fp32 texels.
 *   blocks: device, (height/4)*(width/4) words; out_texels: device, height*width*(3|1) fp32,
 *   row-major, RGB interleaved.  Errors: NTBC_EINVAL, NTBC_ECUDA. */
ntbc_status ntbc_decode_bc(const void* blocks, ntbc_format fmt, int width, int height, float* out_texels,
                           void* stream);

/* Verification only (not timed): rows a1-a4, the fp32 MLP outputs of block rows [row_begin,row_end):
 *   endpoints: device [rows][width/4][N_e] fp32;  colors: device [rows*4][width][N_c] fp32. */
ntbc_status ntbc_debug_mlp(ntbc_model m, int width, int height, int row_begin, int row_end,
                           float* endpoints, float* colors, void* stream);

/* Verification only (not timed): rows a1-a2, the fp32 grid features (after Eq.2 dequantization and
 * bilinear interpolation, before the fp16 rounding of the first MMA operand) of block rows
 * [row_begin,row_end): block_features: device [rows][width/4][16]; texel_features: device
 * [rows*4][width][16] (levels coarse->fine x 2 features; unused levels 0).  Written by the same
 * fused kernel as ntbc_decode_material (dump mode) from the values it feeds the first MMA. */
ntbc_status ntbc_debug_features(ntbc_model m, int width, int height, int row_begin, int row_end,
                                float* block_features, float* texel_features, void* stream);

/* Rows a5-a8 as a standalone kernel (quantize + palette + index + pack) fed fp32 MLP outputs in the
 * ntbc_debug_mlp layouts; same output convention as ntbc_decode_material.  fmts: host array of
 * n_textures formats (head order, R17).  One thread per (block, texture), tiles staged by bulk copies when
 * `colors` is 16-B aligned (any alignment accepted; out_blocks 8-B aligned).  Errors: NTBC_EINVAL,
 * NTBC_ECUDA. */
ntbc_status ntbc_pack(int n_textures, const int* fmts, const float* endpoints, const float* colors,
                      int width, int height, int row_begin, int row_end, void* const* out_blocks,
                      void* stream);

/* Measurement support: tcgen05.mma kind::f16 probe used to pin the tensor-core summation reading
 * (R10).  D[128][N] = C[128][N] (if C != NULL) + sum over K/16 MMAs of A[128][K] B[N][K]^T.
 * A, B fp16 row-major device; C, D fp32 device; N in {16,32,64}, K % 16 == 0, K <= 128. */
ntbc_status ntbc_debug_mma(const void* A, const void* B, const float* C, float* D, int K, int N, void* stream);

/* Peer-memory gather (BASELINE north star: "only a final gather of packed bytes, counted in
 * the timing").  The gather is fused into the decode: a rank passes pointers into rank 0's output
 * buffer as the out_blocks of ntbc_decode_material, so the fused kernel's BC-word stores travel over
 * NVLink straight into rank 0's HBM, unit by unit, while later units are still being computed; no
 * separate collective moves the bytes.  These three calls are the CUDA-IPC plumbing.
 *   ntbc_peer_export: device_ptr = any address inside a cudaMalloc allocation of this process;
 *     writes NTBC_PEER_HANDLE_BYTES opaque bytes (IPC handle of the allocation + the offset of
 *     device_ptr in it) to handle_out (host memory), to be sent to the other ranks.
 *   ntbc_peer_open: maps an exported handle of ANOTHER process into `cuda_device`'s address space
 *     (peer access enabled lazily) and returns the pointer equivalent to the exporter's device_ptr;
 *     valid until ntbc_peer_close.  The exporter must keep the allocation alive until every opener
 *     has closed it.  Writes through the pointer are visible to the exporter's device once the
 *     writing kernel has completed and the processes have synchronised (e.g. a process-group barrier).
 *   ntbc_peer_close: unmaps a pointer returned by ntbc_peer_open.
 * Errors: NTBC_EINVAL (NULL, not device memory, unknown pointer), NTBC_ECUDA. */
#define NTBC_PEER_HANDLE_BYTES 72
ntbc_status ntbc_peer_export(const void* device_ptr, void* handle_out);
ntbc_status ntbc_peer_open(const void* handle, int cuda_device, void** device_ptr_out);
ntbc_status ntbc_peer_close(void* device_ptr);

/* Number of kernel launches the library issued since load (all entry points), for bench accounting. */
uint64_t ntbc_launch_count(void);

/* The arithmetic contract of the model's MLP operands.  0 = H (default):
 * every layer input rounded to binary16, the paper's half-precision inference.
 * 1 = F: activations stay binary32 and each tcgen05 operand is the split hi = RN16(a), lo = RN16(a - hi),
 * multiplied by the same weights (2x the MMAs, half the work groups per SM) -- the contract under which the
 * decode meets north_star's agreement rule against the plain definitions literally.  2 = P: as H, but the
 * hidden selu is evaluated in binary16 ARITHMETIC on packed f16x2 lanes (DESIGN.md
 * §8.f2: the most literal reading of P:322; faster, and ~21% of the activations one or more binary16 ulps
 * from the correctly rounded selu).  All three are bit-exact against the oracle's matching mode.  Applies
 * to later decodes of the model (serialised with them).  A conservative pair runs in one launch only when
 * both models have the same contract.
 * Errors: NTBC_EINVAL (NULL, contract not in {0, 1, 2}, F or P for a naive model). */
ntbc_status ntbc_set_contract(ntbc_model m, int contract);

/* Measurement hook (bench.py's roofline of the dominant kernel): while set, every fused-kernel launch
 * made by THIS host thread through ntbc_decode_material / ntbc_decode_material_host records
 * `start_event` right before and `end_event` right after it on the launch stream (cudaEvent_t as
 * void*, created by the caller with timing enabled).  Pass NULL, NULL to clear.  Not for concurrent
 * use of the same events.  Errors: NTBC_EINVAL (exactly one of the two is NULL). */
ntbc_status ntbc_debug_time_fused(void* start_event, void* end_event);

const char* ntbc_last_error(void);                     /* thread-local message of the last failure */

#ifdef __cplusplus
}
#endif
#endif
