/* ntbc_oracle.h -- CPU ORACLE for NTBC inference.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this library.  The product path (paper_2407_09543_b200/) never
 * includes, links or executes anything under oracle/, and this file shares no
 * code, header, table or constant generator with it.
 *
 * Plain, slow, obviously-correct C99 following PAPER.md (arXiv 2407.09543).
 * Every function cites the passage it implements ("P:n" = PAPER.md line n,
 * "S:n" = SPEC.md line n).  Readings of silent/garbled passages are numbered
 * R1..Rn and listed in DESIGN.md §2.
 *
 * Build: gcc -O2 -fno-fast-math -ffp-contract=off -fopenmp -shared -fPIC
 * (no contraction: every fused multiply-add below is an explicit fmaf()).
 */
#ifndef NTBC_ORACLE_H
#define NTBC_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct o_model o_model;

/* ---- model container (.ntbc v1) ---- */
int  o_model_parse(const void* blob, size_t nbytes, o_model** out);   /* 0 ok, <0 error */
void o_model_free(o_model* m);
/* out[0]=n_tex out[1..8]=fmt out[9]=hidden out[10]=n_e out[11]=n_c
   out[12]=block_levels out[13]=block_coarsest out[14]=texel_levels out[15]=texel_coarsest
   out[16]=variant (0 NTBC colour network, 1 naive weight network) */
void o_model_info(const o_model* m, int* out17);

/* ---- scalar building blocks ---- */
float    o_f16_to_f32(uint16_t h);
uint16_t o_f32_to_f16(float f);                               /* IEEE RN-even */
void     o_f32_to_f16_n(const float* x, uint16_t* out, size_t n);
float    o_dequant(uint8_t q, float s, int32_t z);             /* Eq.2 */
float    o_exp(float x);                                       /* pinned E, R9 */
float    o_expm1(float x);                                     /* selu_neg(x)/(lambda alpha), accuracy pin only */
float    o_selu(float z);                                      /* P:333, R8 */
float    o_sigmoid(float z);                                   /* P:332, R8 */
/* activation model: 0 = pinned op sequences (R9, default), 1 = plain float64/libm definitions,
   2 = binary32 libm (sensitivity variant), 3 = contract P: selu in binary16 arithmetic (R9-P) */
void     o_set_act_model(int plain);
int      o_get_act_model(void);
/* IEEE binary16 arithmetic (contract P): each op is the exact result rounded once to
   binary16, nearest-even */
uint16_t o_f64_to_f16(double x);                               /* RN-even, directly from binary64 */
uint16_t o_h16_fma(uint16_t a, uint16_t b, uint16_t c);
uint16_t o_h16_mul(uint16_t a, uint16_t b);
uint16_t o_h16_sub(uint16_t a, uint16_t b);
uint16_t o_selu_half(float z);                                 /* R9-P, the contract-P hidden activation */

/* Summation model of one layer's dot product (R10).
   mode 0 = CR  : b + sum_k w_k a_k exactly, one RN to fp32.
   mode 1 = CHUNK (default, R10): acc = b; per chunk of `chunk` products acc = F(acc, chunk)
                   where R = max over the chunk's non-zero terms of the exponent SUM
                   e_w + e_a of each fp16 product (and the fp32 acc's exponent); every
                   term is truncated toward zero to a multiple of 2^(R-p), the terms are
                   added exactly and the sum is rounded once (rmode 0 = RN-even, 1 = RZ).
                   Default chunk=16, p=25, RZ. */
void  o_set_dot_model(int mode, int chunk, int p_bits, int rmode);
void  o_get_dot_model(int* out4);
float o_dot(float bias, const uint16_t* w, int w_stride, const uint16_t* a, int k);
float o_fused_sum(const float* acc_in, const uint16_t* a, const uint16_t* b, int n,
                  int p_bits, int rmode);       /* exposed for the pins */

/* ---- grid encoding (Eq.2) ----
   which: 0 = block grid (endpoint network), 1 = texel grid (colour network) */
void o_grid_encode(const o_model* m, int which, float p, float q, float* out);
/* ---- MLP: which 0 = endpoint net, 1 = colour net ---- */
void o_mlp_forward(const o_model* m, int which, const float* in, float* out);
/* operand contract: 0 = H (binary16 layer inputs, the paper's and the kernels'), 1 = F (fp32 activations,
   hi/lo split operands; sensitivity study of DESIGN.md §5.1 only) */
void o_set_operand_model(int split);
/* raw MLP on caller-given fp16 params (for the torch pins) */
void o_mlp_raw(int n_layers, const int* dims, const uint16_t* const* W, const uint16_t* const* b,
               const float* in, float* out);

/* ---- BC formats (Eq.7/8 P:187-205) ---- */
uint16_t o_rgb565(const float e[3]);                           /* R11 */
uint8_t  o_unorm8(float e);                                    /* R11 */
void     o_expand565(uint16_t c, float out[3]);
void     o_palette_bc1(const float e0[3], const float e1[3], float pal[4][3]);   /* Eq.7 */
void     o_palette_bc4(uint8_t E0, uint8_t E1, float pal[8]);                    /* Eq.7+8 */
int      o_argmin_bc1(const float c[3], float pal[4][3]);      /* Eq.9-10 */
int      o_argmin_bc4(float c, const float pal[8]);            /* Eq.9-10 */
uint64_t o_encode_bc1(const float ep[6], const float* texels /* 16 x 3 */);
uint64_t o_encode_bc4(const float ep[2], const float* texels /* 16 */);
/* reference encoder (SPEC encode_block_reference, DESIGN R24-R29): PCA / min-max endpoints,
   n_refine least-squares refinements (2 = the paper's Compressonator setting) */
uint64_t o_encode_ref_bc1(const float* texels /* 16 x 3 */, int n_refine);
uint64_t o_encode_ref_bc4(const float* texels /* 16 */, int n_refine);
void     o_encode_ref_texture(const float* tex /* [H][W][C] */, int W, int H, int C, int n_refine,
                              uint64_t* out /* [H/4][W/4] */, int nthreads);
/* naive approach: nearest palette weight (ties -> lower n), linear index */
int      o_quantize_weight(float w, int fmt, int mode8);
uint64_t o_encode_bc1_naive(const float ep[6], const float* weights /* 16 */);
uint64_t o_encode_bc4_naive(const float ep[2], const float* weights /* 16 */);
void     o_decode_block(uint64_t blk, int fmt, float* out /* 16 x (3|1) */);

/* ---- whole-material paths ---- */
/* out: n_tex planes of (row_end-row_begin) x (W/4) uint64 words, plane-major */
void o_decode_material(const o_model* m, int W, int H, int row_begin, int row_end,
                       uint64_t* out, int nthreads);
/* fp32 MLP outputs: ep [rows][BW][n_e], col [rows*4][W][n_c] */
void o_mlp_outputs(const o_model* m, int W, int H, int row_begin, int row_end,
                   float* ep, float* col, int nthreads);
/* quantize + palette + index + pack from given fp32 MLP outputs (same layouts) */
void o_pack(int n_tex, const int* fmts, const float* ep, const float* col, int W, int H,
            int row_begin, int row_end, uint64_t* out, int nthreads);
/* BC decode of a whole surface: out [H][W][3|1] */
void o_decode_bc(const uint64_t* blocks, int fmt, int W, int H, float* out);
double o_psnr(const float* a, const float* b, size_t n);

/* ---- brute force (tiny inputs) ---- */
uint64_t o_bruteforce_bc4(const float* texels16, double* best_err);
double   o_block_sq_error(uint64_t blk, int fmt, const float* texels);

/* ---- storage arithmetic ---- */
uint64_t o_storage_bytes(int block_levels, int block_coarsest, int texel_levels, int texel_coarsest,
                         int features, int hidden, int n_hidden, int n_e, int n_c, int with_bias);

/* accuracy sweep vs libm over [lo,hi], every `step`-th float: which 0 = E vs exp, 1 = selu's negative branch vs lambda*alpha*expm1 */
double o_exp_max_relerr(float lo, float hi, int step, int which);

#ifdef __cplusplus
}
#endif
#endif
