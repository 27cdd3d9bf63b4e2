/* ntbc_oracle.c -- CPU ORACLE for NTBC inference (arXiv 2407.09543).
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / reference arm.  Never used by the product path.
 * Shares no code with paper_2407_09543_b200/ (see ntbc_oracle.h).
 *
 * Plain, slow, IEEE-exact C99.  Compiled with -ffp-contract=off so that the
 * only fused multiply-adds are the explicit fmaf() calls written below; every
 * other operation is one IEEE-754 binary32 operation rounded to nearest-even.
 *
 * Two arithmetic modes.  PINNED (default): the op sequences the CUDA kernels execute bit for bit
 * -- R9's exponential, R10's tensor-core summation order.  PLAIN (o_set_dot_model(0, ...) +
 * o_set_act_model(1)): the definitions themselves -- every dot product exact and rounded once,
 * selu / sigmoid in float64 with libm and rounded once -- the reference the faithfulness tests
 * (tests/test_faithfulness.py) measure both the pinned oracle and the CUDA path against under
 * north_star's tolerance rule.  The binary16 operand rounding at every layer input
 * is part of the method and is the same in both modes.  Two more arithmetic contracts of the kernels
 * have their own pinned modes: F (o_set_operand_model(1): binary32 activations, hi/lo split operands)
 * and P (o_set_act_model(3): the selu in binary16 arithmetic, R9-P).
 *
 * Parity status per function: every function below is pinned by -m "not gpu"
 * tests.  o_dot's summation ORDER (R10: chunks of 16, window p = 25, round toward zero) is a
 * reading of a passage the paper leaves silent ("half-precision floating points"); the
 * mathematics pins it through its error bound and its exactness on representable sums.
 */
#include "ntbc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define BC1 1
#define BC4 4
#define MAXTEX 8
#define MAXLV 8

/* ------------------------------------------------------------------------- */
/* model container                                                            */
/* ------------------------------------------------------------------------- */
typedef struct { float s; int32_t z; int res; const uint8_t* q; } o_level;
typedef struct { int levels, coarsest; o_level lv[MAXLV]; } o_grid;
typedef struct { int n_layers; int dims[8]; const uint16_t* W[7]; const uint16_t* b[7]; } o_mlp;
struct o_model {
    int n_tex, fmt[MAXTEX], hidden, n_hidden, F;
    int naive;             /* header variant: 0 NTBC colour network, 1 naive weight network */
    o_grid grid[2];        /* 0 = block grid, 1 = texel grid */
    o_mlp mlp[2];          /* 0 = endpoint net, 1 = colour net */
    uint8_t* blob;         /* private copy; all pointers above point into it */
};

static uint32_t rd32(const uint8_t* p) { uint32_t v; memcpy(&v, p, 4); return v; }
static size_t al16(size_t n) { return (n + 15) & ~(size_t)15; }

int o_model_parse(const void* blob, size_t n, o_model** out) {
    const uint8_t* b = (const uint8_t*)blob;
    if (n < 96 || memcmp(b, "NTBC", 4) != 0 || rd32(b + 4) != 1) return -2;
    o_model* m = (o_model*)calloc(1, sizeof(o_model));
    m->blob = (uint8_t*)malloc(n);
    memcpy(m->blob, b, n);
    b = m->blob;
    m->n_tex = (int)rd32(b + 8);
    if (m->n_tex < 1 || m->n_tex > MAXTEX) { o_model_free(m); return -2; }
    for (int i = 0; i < m->n_tex; i++) {
        m->fmt[i] = (int)rd32(b + 12 + 4 * i);
        if (m->fmt[i] != BC1 && m->fmt[i] != BC4) { o_model_free(m); return -2; }
    }
    m->hidden = (int)rd32(b + 44); m->n_hidden = (int)rd32(b + 48); m->F = (int)rd32(b + 52);
    m->grid[0].levels = (int)rd32(b + 56); m->grid[0].coarsest = (int)rd32(b + 60);
    m->grid[1].levels = (int)rd32(b + 64); m->grid[1].coarsest = (int)rd32(b + 68);
    int ep_in = (int)rd32(b + 72), n_e = (int)rd32(b + 76), col_in = (int)rd32(b + 80), n_c = (int)rd32(b + 84);
    m->naive = (int)rd32(b + 88);
    if (m->naive != 0 && m->naive != 1) { o_model_free(m); return -2; }
    if (m->n_hidden < 1 || m->n_hidden > 5 || m->F < 1 || m->grid[0].levels < 1 ||
        m->grid[0].levels > MAXLV || m->grid[1].levels < 1 || m->grid[1].levels > MAXLV) { o_model_free(m); return -2; }
    size_t off = 96;
    const uint8_t* qp = b + off;
    int nl = m->grid[0].levels + m->grid[1].levels;
    off += al16((size_t)nl * 8);
    int li = 0;
    for (int g = 0; g < 2; g++)
        for (int l = 0; l < m->grid[g].levels; l++, li++) {
            o_level* L = &m->grid[g].lv[l];
            memcpy(&L->s, qp + 8 * li, 4);
            memcpy(&L->z, qp + 8 * li + 4, 4);
            L->res = m->grid[g].coarsest << l;
        }
    for (int g = 0; g < 2; g++)
        for (int l = 0; l < m->grid[g].levels; l++) {
            o_level* L = &m->grid[g].lv[l];
            size_t sz = (size_t)L->res * L->res * m->F;
            if (off + sz > n) { o_model_free(m); return -2; }
            L->q = b + off;
            off += al16(sz);
        }
    int ins[2] = {ep_in, col_in}, outs[2] = {n_e, n_c};
    for (int k = 0; k < 2; k++) {
        o_mlp* M = &m->mlp[k];
        M->n_layers = m->n_hidden + 1;
        M->dims[0] = ins[k];
        for (int l = 1; l <= m->n_hidden; l++) M->dims[l] = m->hidden;
        M->dims[M->n_layers] = outs[k];
        for (int l = 0; l < M->n_layers; l++) {
            size_t wsz = (size_t)M->dims[l] * M->dims[l + 1] * 2, bsz = (size_t)M->dims[l + 1] * 2;
            if (off + al16(wsz) + bsz > n) { o_model_free(m); return -2; }
            M->W[l] = (const uint16_t*)(b + off); off += al16(wsz);
            M->b[l] = (const uint16_t*)(b + off); off += al16(bsz);
        }
    }
    int want_e = 0, want_c = 0;
    for (int i = 0; i < m->n_tex; i++) { want_e += m->fmt[i] == BC1 ? 6 : 2; want_c += m->fmt[i] == BC1 ? 3 : 1; }
    if (m->naive) want_c = m->n_tex;                          /* one weight per texel per texture */
    if (want_e != n_e || want_c != n_c || ep_in != m->grid[0].levels * m->F ||
        col_in != m->grid[1].levels * m->F) { o_model_free(m); return -2; }
    *out = m;
    return 0;
}

void o_model_free(o_model* m) { if (m) { free(m->blob); free(m); } }

void o_model_info(const o_model* m, int* o) {
    memset(o, 0, 17 * sizeof(int));
    o[16] = m->naive;
    o[0] = m->n_tex;
    for (int i = 0; i < m->n_tex; i++) o[1 + i] = m->fmt[i];
    o[9] = m->hidden;
    o[10] = m->mlp[0].dims[m->mlp[0].n_layers];
    o[11] = m->mlp[1].dims[m->mlp[1].n_layers];
    o[12] = m->grid[0].levels; o[13] = m->grid[0].coarsest;
    o[14] = m->grid[1].levels; o[15] = m->grid[1].coarsest;
}

/* ------------------------------------------------------------------------- */
/* IEEE binary16 <-> binary32 ("half-precision floating points")       */
/* ------------------------------------------------------------------------- */
float o_f16_to_f32(uint16_t h) {
    int sign = h >> 15, e = (h >> 10) & 31, f = h & 1023;
    float v;
    if (e == 0) v = ldexpf((float)f, -24);                 /* subnormal (and zero) */
    else if (e == 31) v = f ? NAN : INFINITY;
    else v = ldexpf((float)(1024 + f), e - 25);
    return sign ? -v : v;
}

uint16_t o_f32_to_f16(float x) {
    uint32_t u; memcpy(&u, &x, 4);
    uint16_t sign = (uint16_t)((u >> 16) & 0x8000);
    float a = fabsf(x);
    if (a != a) return (uint16_t)(sign | 0x7e00);
    if (a >= 65520.0f) return (uint16_t)(sign | 0x7c00);     /* rounds to inf */
    /* exact value a = M * 2^E with integer M < 2^24 */
    int E; (void)frexpf(a, &E);                              /* a = fr * 2^E, fr in [0.5,1) */
    if (a == 0.0f) return sign;
    /* binary16 quantum for this binade: normal if a >= 2^-14 -> 2^(E-1-10), else 2^-24 */
    int qexp = (E - 1 >= -14) ? (E - 1 - 10) : -24;
    double scaled = ldexp((double)a, -qexp);                 /* exact in double */
    double fl = floor(scaled), rem = scaled - fl;
    uint32_t mant = (uint32_t)fl;
    if (rem > 0.5 || (rem == 0.5 && (mant & 1))) mant++;    /* round half to even */
    /* value = mant * 2^qexp; re-encode */
    if (qexp == -24)            /* subnormals and the first normal binade share the quantum 2^-24: */
        return (uint16_t)(sign | mant);   /* bits == mant (mant <= 2048 = 2^-13 after rounding up) */
    int bexp = qexp + 25;                                    /* biased exponent for mant in [1024,2048) */
    if (mant == 2048) { mant = 1024; bexp++; }
    if (bexp >= 31) return (uint16_t)(sign | 0x7c00);
    return (uint16_t)(sign | (bexp << 10) | (mant - 1024));
}

void o_f32_to_f16_n(const float* x, uint16_t* out, size_t n) {
    for (size_t i = 0; i < n; i++) out[i] = o_f32_to_f16(x[i]);
}

/* Eq.2: r = s * (q - z) -- one fp32 multiply of an exact integer (R6) */
float o_dequant(uint8_t q, float s, int32_t z) { return s * (float)((int32_t)q - z); }

/* ------------------------------------------------------------------------- */
/* pinned exponential (R9): 2^n * (1 + f*Q(f)), Q a degree-3 polynomial       */
/* ------------------------------------------------------------------------- */
static const float LOG2E = 0x1.715476p+0f;
static const float MAGIC = 12582912.0f;                      /* 1.5 * 2^23 */
/* Q(f) ~ (2^f - 1)/f on |f| <= 1/2, minimax in relative error of Q (so that both e^x and the selu
   branch's e^z - 1 = 2^n (1 + f Q) - 1 keep it, including f -> 0).  Degree 4 (R9 v4): the degree-3
   polynomial of v3 (|rel| 1.5e-5 = 1/30 of a binary16 ulp) flips the binary16 rounding of ~3% of the
   hidden activations against the plain definition, and the fp16 re-rounding of every layer input
    amplifies each flip (tests/test_faithfulness.py: 163 vs 10 mismatched words on 8,192 C2
   blocks).  Degrees 3 and 5 are kept for that sensitivity study (-DNTBC_QDEG). */
#ifndef NTBC_QDEG
#define NTBC_QDEG 4
#endif
#if NTBC_QDEG == 3   /* |rel| <= 1.5e-5 */
static const float QC[4] = {0x1.62e2d6p-1f, 0x1.ebff08p-3f, 0x1.c96b34p-5f, 0x1.3b2a76p-7f};
#elif NTBC_QDEG == 4 /* |rel| <= 4.7e-7 */
static const float QC[5] = {0x1.62e42ep-1f, 0x1.ebfa4ep-3f, 0x1.c6b26ep-5f, 0x1.3cbe58p-7f, 0x1.5d87dep-10f};
#else                /* degree 5, |rel| <= 2.1e-8 */
static const float QC[6] = {0x1.62e430p-1f, 0x1.ebfbdep-3f, 0x1.c6af6ep-5f, 0x1.3b2ba0p-7f, 0x1.5f07b4p-10f, 0x1.4308fap-13f};
#endif
static const float SELU_L = 0x1.0cfabep+0f;                  /* RN32(1.0507009873554804934) */
static const float SELU_LA = 0x1.c212ccp+0f;                 /* RN32(lambda * alpha)        */

/* e^x = 2^n (1 + f Q(f)): n = rint(x log2e) (magic-number rounding of the exactly-computed product),
   f = RN(x log2e - n) (exact product, one rounding), q = Q(f) by Horner.  Returns n, f and q. */
static int exp_reduce(float x, float* f_out, float* q_out) {
    float r = fmaf(x, LOG2E, MAGIC);              /* rint(x log2e) + 1.5*2^23, one rounding */
    float negnf = MAGIC - r;                      /* -n, exact */
    float f = fmaf(x, LOG2E, negnf);              /* x log2e - n, one rounding */
    *f_out = f;
    float q = QC[NTBC_QDEG];                      /* Horner, highest coefficient first */
    for (int i = NTBC_QDEG - 1; i >= 0; i--) q = fmaf(q, f, QC[i]);
    *q_out = q;
    int32_t ri, mi; memcpy(&ri, &r, 4); float mg = MAGIC; memcpy(&mi, &mg, 4);
    return ri - mi;
}
static float pow2i(int n, float scale) {          /* scale * 2^n by exponent insertion (exact) */
    uint32_t b; memcpy(&b, &scale, 4);
    b += (uint32_t)n << 23;
    float v; memcpy(&v, &b, 4);
    return v;
}
/* E(x) = 2^n + 2^n RN(f q), x clamped to [-80, 80] */
float o_exp(float x) {
    float xc = fminf(fmaxf(x, -80.0f), 80.0f), f, q;
    int n = exp_reduce(xc, &f, &q);
    float s = pow2i(n, 1.0f);
    return fmaf(s, f * q, s);
}
/* selu negative branch (R8/R9): lambda*alpha*(e^z - 1) = fma(S, RN(f q), S - lambda*alpha),
   S = lambda*alpha*2^n exact.  For n = 0 the addend S - lambda*alpha is exactly 0, so there is no
   cancellation as z -> 0^- (the result keeps the polynomial's relative accuracy down to the
   smallest z; pinned by test_selu_branch_relative_error_near_zero). */
static float selu_neg_pinned(float z) {
    float x = fmaxf(z, -80.0f), f, q;
    int n = exp_reduce(x, &f, &q);
    float S = pow2i(n, SELU_LA);
    return fmaf(S, f * q, S - SELU_LA);
}

/* ------------------------------------------------------------------------- */
/* activation model: 0 = the pinned op sequences above (R9, what the kernel computes);          */
/* 3 = contract P (below: the selu in binary16 arithmetic, R9-P; the sigmoid stays pinned R9);   */
/* 2 = the same in binary32 libm (expm1f / expf; a sensitivity variant, not a reference); */
/* 1 = the PLAIN definitions (P:332-333 with the standard selu constants): evaluated in  */
/* float64 with libm exp/expm1 and rounded once to binary32 -- the faithfulness reference.      */
/* ------------------------------------------------------------------------- */
static int g_act_plain = 0;
void o_set_act_model(int plain) { g_act_plain = plain; }
int  o_get_act_model(void) { return g_act_plain; }
static const double SELU_LAMBDA_D = 1.0507009873554804934, SELU_ALPHA_D = 1.6732632423543772848;

static float selu_neg(float z) {
    if (g_act_plain == 2) return SELU_LA * expm1f(z);        /* a binary32 libm variant (sensitivity study) */
    if (g_act_plain == 1) return (float)(SELU_LAMBDA_D * SELU_ALPHA_D * expm1((double)z));
    return selu_neg_pinned(z);
}
float o_expm1(float x) { return selu_neg_pinned(x) / SELU_LA; }   /* for the accuracy pin only (x <= 0) */

/* ------------------------------------------------------------------------- */
/* contract P (R9-P): the selu evaluated in IEEE binary16 arithmetic,    */
/* the most literal reading of "inference is executed in the half-precision floating points". */
/* Every step is ONE binary16 operation: the exact result (computed exactly in binary64 -- a product   */
/* of two binary16 values has 22 bits, and a binary16 fma's exact result is either representable in   */
/* binary64 or, when it is not, lies farther than 2^-53 |x| from every binary16 rounding midpoint, so  */
/* the binary64 fma followed by one binary16 rounding equals the single rounding; pinned against      */
/* exact rational arithmetic by test_h16_ops_are_single_roundings) rounded once to nearest-even.      */
/* ------------------------------------------------------------------------- */
uint16_t o_f64_to_f16(double x) {
    uint64_t u; memcpy(&u, &x, 8);
    uint16_t sign = (uint16_t)((u >> 48) & 0x8000);
    double a = fabs(x);
    if (a != a) return (uint16_t)(sign | 0x7e00);
    if (a >= 65520.0) return (uint16_t)(sign | 0x7c00);       /* rounds to inf */
    if (a == 0.0) return sign;
    int E; (void)frexp(a, &E);                                /* a = fr * 2^E, fr in [0.5,1) */
    int qexp = (E - 1 >= -14) ? (E - 1 - 10) : -24;           /* the binary16 quantum of a's binade */
    double scaled = ldexp(a, -qexp);                          /* exact (a power-of-two scaling) */
    double fl = floor(scaled), rem = scaled - fl;             /* rem exact: fl and scaled share the binade */
    uint32_t mant = (uint32_t)fl;
    if (rem > 0.5 || (rem == 0.5 && (mant & 1))) mant++;      /* round half to even */
    if (qexp == -24) return (uint16_t)(sign | mant);
    int bexp = qexp + 25;
    if (mant == 2048) { mant = 1024; bexp++; }
    if (bexp >= 31) return (uint16_t)(sign | 0x7c00);
    return (uint16_t)(sign | (bexp << 10) | (mant - 1024));
}
static double h2d(uint16_t h) { return (double)o_f16_to_f32(h); }
uint16_t o_h16_fma(uint16_t a, uint16_t b, uint16_t c) { return o_f64_to_f16(fma(h2d(a), h2d(b), h2d(c))); }
uint16_t o_h16_mul(uint16_t a, uint16_t b) { return o_f64_to_f16(h2d(a) * h2d(b)); }
uint16_t o_h16_sub(uint16_t a, uint16_t b) { return o_f64_to_f16(h2d(a) - h2d(b)); }

/* R9-P, step by step (the constants are binary16 bit patterns):
   h = RN16(z); z's sign decides (h = -0 takes the negative branch, which gives +0 there);
   positive: RN16(lambda16 h), lambda16 = RN16(1.0507...) = 0x3C34;
   negative: x = max(h, -10) (below -10, lambda alpha e^x is under a quarter ulp of lambda alpha16);
     t = RN16(x log2e16 + 1039), an integer in [1025, 1039] (the binary16 quantum is 1 there), n = t - 1039;
     g = RN16(x - n ln2hi), ln2hi = 0.693359375 (exact: Cody-Waite); g = RN16(g - n ln2lo16);
     P = RN16(RN16(C2 g + C1) g + C0), u = RN16(g RN16(g P) + g)  -- u ~ e^g - 1 on |g| <= 0.37;
     S = lambda alpha16 2^n (exact: the binary16 exponent field of 0x3F08 lowered by -n, n >= -14);
     neg = RN16(S u + RN16(S - lambda alpha16)). */
uint16_t o_selu_half(float z) {
    const uint16_t h = o_f32_to_f16(z);
    if (!(h & 0x8000)) return o_h16_mul(h, 0x3C34);
    const uint16_t x = h2d(h) > -10.0 ? h : 0xC900;           /* max(h, -10); h = -0 stays -0 */
    const uint16_t t = o_h16_fma(x, 0x3DC5, 0x640F);
    const uint16_t nf = o_h16_sub(t, 0x640F);
    uint16_t g = o_h16_fma(nf, 0xB98C, x);
    g = o_h16_fma(nf, 0x0AF4, g);
    uint16_t P = o_h16_fma(0x295B, g, 0x315B);
    P = o_h16_fma(P, g, 0x3800);
    const uint16_t u = o_h16_fma(g, o_h16_mul(g, P), g);
    const int n = (int)h2d(nf);                                /* exact integer in [-14, 0] */
    const uint16_t S = (uint16_t)(0x3F08 + n * 1024);          /* lambda alpha16 * 2^n, a normal binary16 */
    return o_h16_fma(S, u, o_h16_sub(S, 0x3F08));
}

/* selu ([selu] Klambauer et al.): lambda z (z > 0) else lambda alpha (e^z - 1) */
float o_selu(float z) {
    if (g_act_plain == 3) return o_f16_to_f32(o_selu_half(z));
    if (g_act_plain == 2) return z > 0.0f ? SELU_L * z : selu_neg(z);
    if (g_act_plain == 1) return z > 0.0f ? (float)(SELU_LAMBDA_D * (double)z) : selu_neg(z);
    return z > 0.0f ? SELU_L * z : selu_neg(z);
}
/* sigmoid: 1 / (1 + e^-z), IEEE division */
float o_sigmoid(float z) {
    if (g_act_plain == 2) return 1.0f / (1.0f + expf(-z));
    if (g_act_plain == 1) return (float)(1.0 / (1.0 + exp(-(double)z)));
    float d = 1.0f + o_exp(-z); return 1.0f / d;
}

double o_exp_max_relerr(float lo, float hi, int step, int which) {
    double worst = 0.0;
    float x = lo;
    while (x <= hi) {
        double ref = which == 0 ? exp((double)x) : (double)SELU_LA * expm1((double)x);
        double got = which == 0 ? (double)o_exp(x) : (double)selu_neg_pinned(x);
        double den = fabs(ref);
        if (den > 0) { double e = fabs(got - ref) / den; if (e > worst) worst = e; }
        for (int k = 0; k < step; k++) x = nextafterf(x, INFINITY);
    }
    return worst;
}

/* ------------------------------------------------------------------------- */
/* exact fused summation of fp16 products (R10)                               */
/* ------------------------------------------------------------------------- */
/* A term of a fused sum: value = (-1)^neg * m * 2^e.  `ref` is the exponent the R10 alignment
   rule uses: for an fp16 x fp16 product the SUM of the two operands' unbiased exponents (subnormal
   operands count as -14), for the fp32 accumulator its unbiased exponent (subnormal: -126). */
typedef struct { int neg; uint64_t m; int e; int ref; } term;

static term t_f16(uint16_t h) {
    term t; int e = (h >> 10) & 31, f = h & 1023;
    t.neg = h >> 15;
    if (e == 0) { t.m = (uint64_t)f; t.e = -24; t.ref = -14; }
    else { t.m = (uint64_t)(1024 + f); t.e = e - 25; t.ref = e - 15; }
    return t;
}
static term t_mul(term a, term b) {
    term t; t.neg = a.neg ^ b.neg; t.m = a.m * b.m; t.e = a.e + b.e; t.ref = a.ref + b.ref; return t;
}
static term t_f32(float x) {
    term t; uint32_t u; memcpy(&u, &x, 4);
    int e = (u >> 23) & 255; uint32_t f = u & 0x7fffff;
    t.neg = (int)(u >> 31);
    if (e == 0) { t.m = f; t.e = -149; t.ref = -126; } else { t.m = (uint64_t)(0x800000 | f); t.e = e - 150; t.ref = e - 127; }
    return t;
}
static int bitlen128(unsigned __int128 v) { int n = 0; while (v) { n++; v >>= 1; } return n; }

/* value = S * 2^q rounded to binary32 (rmode 0: nearest-even, 1: toward zero) */
static float round_f32(__int128 S, int q, int rmode) {
    if (S == 0) return 0.0f;
    int neg = S < 0;
    unsigned __int128 M = neg ? (unsigned __int128)(-S) : (unsigned __int128)S;
    int L = q + bitlen128(M) - 1;                             /* exponent of the leading bit */
    if (L > 127) return neg ? -INFINITY : INFINITY;
    int lsb = (L >= -126) ? L - 23 : -149;                    /* exponent of the result's ulp */
    unsigned __int128 mant;
    if (lsb <= q) mant = M << (q - lsb);
    else {
        int sh = lsb - q;
        mant = M >> sh;
        unsigned __int128 rem = M - (mant << sh), half = (unsigned __int128)1 << (sh - 1);
        if (rmode == 0 && (rem > half || (rem == half && (mant & 1)))) mant++;
    }
    float r = ldexpf((float)(uint64_t)mant, lsb);             /* mant <= 2^24: exact */
    return neg ? -r : r;
}

/* R10 fused sum: R = max ref over the non-zero terms; every term is truncated toward zero to a
   multiple of 2^(R - p); the truncated terms are added exactly; the sum is rounded once (rmode 0 =
   nearest-even, 1 = toward zero).  With p >= 100 nothing is truncated for fp16 products, so the
   result is the exact sum rounded once. */
static float fused(const term* t, int n, int p, int rmode) {
    int R = -100000;
    for (int i = 0; i < n; i++) if (t[i].m && t[i].ref > R) R = t[i].ref;
    if (R == -100000) return 0.0f;
    if (p > 100) p = 100;
    int q = R - p;
    __int128 S = 0;
    for (int i = 0; i < n; i++) {
        if (!t[i].m) continue;
        int sh = t[i].e - q;
        __int128 v;
        if (sh >= 0) v = (__int128)t[i].m << sh;
        else v = -sh > 63 ? 0 : (__int128)(t[i].m >> (-sh));          /* magnitude truncation */
        S += t[i].neg ? -v : v;
    }
    return round_f32(S, q, rmode);
}

/* R10: fp32 accumulation in chunks of 16 products, each chunk fused with the running
   accumulator under window p = 25 and a final round-toward-zero. */
static int g_mode = 1, g_chunk = 16, g_p = 25, g_rmode = 1;
void o_set_dot_model(int mode, int chunk, int p_bits, int rmode) { g_mode = mode; g_chunk = chunk; g_p = p_bits; g_rmode = rmode; }
void o_get_dot_model(int* o) { o[0] = g_mode; o[1] = g_chunk; o[2] = g_p; o[3] = g_rmode; }

float o_fused_sum(const float* acc_in, const uint16_t* a, const uint16_t* b, int n, int p_bits, int rmode) {
    term* t = (term*)malloc(sizeof(term) * (size_t)(n + 1));
    int k = 0;
    if (acc_in) t[k++] = t_f32(*acc_in);
    for (int i = 0; i < n; i++) t[k++] = t_mul(t_f16(a[i]), t_f16(b[i]));
    float r = fused(t, k, p_bits, rmode);
    free(t);
    return r;
}

/* z_j = b_j + sum_k W[k][j] * a_k under the pinned summation model (R10). */
float o_dot(float bias, const uint16_t* w, int ws, const uint16_t* a, int K) {
    term t[257];
    if (g_mode == 0 || K + 1 > 256) {                         /* CR: one exact sum, one RN */
        int k = 0; t[k++] = t_f32(bias);
        for (int i = 0; i < K; i++) t[k++] = t_mul(t_f16(w[(size_t)i * ws]), t_f16(a[i]));
        return fused(t, k, 100, 0);
    }
    float acc = bias;                                         /* bias enters first, exactly */
    for (int k0 = 0; k0 < K; k0 += g_chunk) {
        int k1 = k0 + g_chunk < K ? k0 + g_chunk : K, n = 0;
        t[n++] = t_f32(acc);
        for (int i = k0; i < k1; i++) t[n++] = t_mul(t_f16(w[(size_t)i * ws]), t_f16(a[i]));
        acc = fused(t, n, g_p, g_rmode);
    }
    return acc;
}

/* ------------------------------------------------------------------------- */
/* grid encoding: vertex-centred dense grids (R1), centres (R2), concat (R3)  */
/* ------------------------------------------------------------------------- */
static float lerp(float a, float b, float t) { return fmaf(t, b - a, a); }

void o_grid_encode(const o_model* m, int which, float p, float q, float* out) {
    const o_grid* g = &m->grid[which];
    for (int l = 0; l < g->levels; l++) {
        const o_level* L = &g->lv[l];
        float X = p * (float)(L->res - 1), Y = q * (float)(L->res - 1);
        int i0 = (int)floorf(X), j0 = (int)floorf(Y);
        if (i0 > L->res - 2) i0 = L->res - 2;
        if (j0 > L->res - 2) j0 = L->res - 2;
        if (i0 < 0) i0 = 0;
        if (j0 < 0) j0 = 0;
        float fx = X - (float)i0, fy = Y - (float)j0;
        for (int f = 0; f < m->F; f++) {
#define QV(j, i) o_dequant(L->q[((size_t)(j) * L->res + (i)) * m->F + f], L->s, L->z)
            float v00 = QV(j0, i0), v10 = QV(j0, i0 + 1), v01 = QV(j0 + 1, i0), v11 = QV(j0 + 1, i0 + 1);
#undef QV
            out[l * m->F + f] = lerp(lerp(v00, v10, fx), lerp(v01, v11, fx), fy);
        }
    }
}

/* ------------------------------------------------------------------------- */
/* MLP: fp16 operands at every layer input, selu hidden,       */
/* sigmoid output                                                 */
/* ------------------------------------------------------------------------- */
/* Operand contract of every layer input.  0 = H, the paper's half precision (P:322,
   P:331): a -> RN16(a), what the kernels compute.  1 = F ("fp32-faithful", a sensitivity study only, not
   implemented on the GPU): activations stay binary32 and each MMA operand is the split hi = RN16(a),
   lo = RN16(a - hi), the dot product running over [hi 0:16, lo 0:16, hi 16:32, lo 16:32, ...] with the
   weights repeated. */
static int g_operand_split = 0;
void o_set_operand_model(int split) { g_operand_split = split; }

void o_mlp_raw(int n_layers, const int* dims, const uint16_t* const* W, const uint16_t* const* b,
               const float* in, float* out) {
    float act[256];
    uint16_t a16[512], w2[512];
    for (int i = 0; i < dims[0]; i++) act[i] = in[i];
    for (int l = 0; l < n_layers; l++) {
        int K = dims[l], N = dims[l + 1];
        if (!g_operand_split) {
            for (int i = 0; i < K; i++) a16[i] = o_f32_to_f16(act[i]);
            for (int j = 0; j < N; j++) {
                float z = o_dot(o_f16_to_f32(b[l][j]), W[l] + j, N, a16, K);
                act[j] = (l + 1 < n_layers) ? o_selu(z) : o_sigmoid(z);
            }
        } else {
            /* interleaved hi / lo chunks of 16 entries (a partial chunk padded with zero operands, which
               add no term to any sum), so that R10's chunks of 16 are exactly the tensor core's K = 16 MMAs */
            int K2 = 0;
            for (int k0 = 0; k0 < K; k0 += 16) {
                for (int i = k0; i < k0 + 16; i++) a16[K2++] = i < K ? o_f32_to_f16(act[i]) : 0;
                for (int i = k0; i < k0 + 16; i++) {
                    if (i >= K) { a16[K2++] = 0; continue; }
                    float hi = o_f16_to_f32(o_f32_to_f16(act[i]));
                    a16[K2++] = o_f32_to_f16(act[i] - hi);
                }
            }
            for (int j = 0; j < N; j++) {
                int n2 = 0;
                for (int k0 = 0; k0 < K; k0 += 16)
                    for (int rep = 0; rep < 2; rep++)
                        for (int i = k0; i < k0 + 16; i++) w2[n2++] = i < K ? W[l][(size_t)i * N + j] : 0;
                float z = o_dot(o_f16_to_f32(b[l][j]), w2, 1, a16, K2);
                act[j] = (l + 1 < n_layers) ? o_selu(z) : o_sigmoid(z);
            }
        }
    }
    for (int j = 0; j < dims[n_layers]; j++) out[j] = act[j];
}

void o_mlp_forward(const o_model* m, int which, const float* in, float* out) {
    const o_mlp* M = &m->mlp[which];
    o_mlp_raw(M->n_layers, M->dims, M->W, M->b, in, out);
}

/* ------------------------------------------------------------------------- */
/* BC1 / BC4 (Eq.7, Eq.8)                      */
/* ------------------------------------------------------------------------- */
static int qbits(float e, float maxv) {                       /* R11: floor(e*(2^b-1) + 1/2) */
    float v = floorf(fmaf(e, maxv, 0.5f));
    if (v < 0.0f) v = 0.0f;
    if (v > maxv) v = maxv;
    return (int)v;
}
uint16_t o_rgb565(const float e[3]) {
    return (uint16_t)((qbits(e[0], 31.0f) << 11) | (qbits(e[1], 63.0f) << 5) | qbits(e[2], 31.0f));
}
uint8_t o_unorm8(float e) { return (uint8_t)qbits(e, 255.0f); }
void o_expand565(uint16_t c, float o[3]) {
    o[0] = (float)(c >> 11) / 31.0f; o[1] = (float)((c >> 5) & 63) / 63.0f; o[2] = (float)(c & 31) / 31.0f;
}

/* Eq.7: c_n = (1 - w_n) e0 + w_n e1, evaluated as fmaf(w_n, e1, RN((1 - w_n) * e0)) */
static float interp(float w, float e0, float e1) { float wb = 1.0f - w; return fmaf(w, e1, wb * e0); }

void o_palette_bc1(const float e0[3], const float e1[3], float pal[4][3]) {
    for (int n = 0; n < 4; n++) {
        float w = (float)n / 3.0f;                            /* w_n = n/3 */
        for (int c = 0; c < 3; c++) pal[n][c] = interp(w, e0[c], e1[c]);
    }
}

void o_palette_bc4(uint8_t E0, uint8_t E1, float pal[8]) {
    float e0 = (float)E0 / 255.0f, e1 = (float)E1 / 255.0f;
    if (E0 > E1) {                                            /* w_n = n/7 */
        for (int n = 0; n < 8; n++) pal[n] = interp((float)n / 7.0f, e0, e1);
    } else {                                                  /* Eq.8: c_0 = 0, c_7 = 1 */
        pal[0] = 0.0f;
        for (int n = 1; n <= 6; n++) pal[n] = interp((float)(n - 1) / 5.0f, e0, e1);
        pal[7] = 1.0f;
    }
}

/* Eq.9-10: n = argmax(-||c - c_n||) = argmin of the squared distance (R14); ties -> lowest n (R15) */
int o_argmin_bc1(const float c[3], float pal[4][3]) {
    int best = 0; float bd = 0.0f;
    for (int n = 0; n < 4; n++) {
        float dr = c[0] - pal[n][0], dg = c[1] - pal[n][1], db = c[2] - pal[n][2];
        float d = fmaf(db, db, fmaf(dg, dg, dr * dr));
        if (n == 0 || d < bd) { bd = d; best = n; }
    }
    return best;
}
int o_argmin_bc4(float c, const float pal[8]) {
    int best = 0; float bd = 0.0f;
    for (int n = 0; n < 8; n++) {
        float d = fabsf(c - pal[n]);
        if (n == 0 || d < bd) { bd = d; best = n; }
    }
    return best;
}

/* linear palette index -> DirectX stored code (R16) */
static const int MAP1[4] = {0, 2, 3, 1};
static const int MAP4_8[8] = {0, 2, 3, 4, 5, 6, 7, 1};
static const int MAP4_6[8] = {6, 0, 2, 3, 4, 5, 1, 7};

uint64_t o_encode_bc1(const float ep[6], const float* tx) {
    uint16_t c0 = o_rgb565(ep), c1 = o_rgb565(ep + 3);
    if (c0 < c1) { uint16_t t = c0; c0 = c1; c1 = t; }        /* 4-colour mode order (R12) */
    uint64_t w = (uint64_t)c0 | ((uint64_t)c1 << 16);
    if (c0 == c1) return w;                                   /* all codes 0 (R12) */
    float e0[3], e1[3], pal[4][3];
    o_expand565(c0, e0); o_expand565(c1, e1);
    o_palette_bc1(e0, e1, pal);
    for (int i = 0; i < 16; i++) w |= (uint64_t)MAP1[o_argmin_bc1(tx + 3 * i, pal)] << (32 + 2 * i);
    return w;
}

uint64_t o_encode_bc4(const float ep[2], const float* tx) {
    uint8_t E0 = o_unorm8(ep[0]), E1 = o_unorm8(ep[1]);       /* mode from stored order, no swap (R13) */
    float pal[8];
    o_palette_bc4(E0, E1, pal);
    const int* map = E0 > E1 ? MAP4_8 : MAP4_6;
    uint64_t w = (uint64_t)E0 | ((uint64_t)E1 << 8);
    for (int i = 0; i < 16; i++) w |= (uint64_t)map[o_argmin_bc4(tx[i], pal)] << (16 + 3 * i);
    return w;
}

/* Naive approach: the weight network's floating-point weight w_f is quantized to the
   nearest palette weight w_n of the block's format and mode ("quantizes w_f to w_n"; SPEC
   quantize_weight: minimize |w_f - w_n|, ties -> lower n).  Weights are the fp32 values the palette
   uses: n/3 (BC1), n/7 (BC4, E0 > E1), (n-1)/5 for linear n = 1..6 (BC4, E0 <= E1: entries 0 and 7
   are the constants 0 and 1, which carry no weight).  Returns the linear palette index n. */
int o_quantize_weight(float w, int fmt, int mode8) {
    int lo = 0, hi = 3;
    if (fmt == BC4) { lo = mode8 ? 0 : 1; hi = mode8 ? 7 : 6; }
    int best = lo; float bd = 0.0f;
    for (int n = lo; n <= hi; n++) {
        float wn = fmt == BC1 ? (float)n / 3.0f : mode8 ? (float)n / 7.0f : (float)(n - 1) / 5.0f;
        float d = fabsf(w - wn);
        if (n == lo || d < bd) { bd = d; best = n; }
    }
    return best;
}

/* BC1: the weights are relative to the predicted endpoint order; when the 4-colour-mode rule swaps
   the stored endpoints, index n maps to 3 - n (SPEC infer_surfaces "swap + index remap"). */
uint64_t o_encode_bc1_naive(const float ep[6], const float* w) {
    uint16_t c0 = o_rgb565(ep), c1 = o_rgb565(ep + 3);
    int swapped = c0 < c1;
    if (swapped) { uint16_t t = c0; c0 = c1; c1 = t; }
    uint64_t blk = (uint64_t)c0 | ((uint64_t)c1 << 16);
    if (c0 == c1) return blk;                                 /* all codes 0 (R12) */
    for (int i = 0; i < 16; i++) {
        int n = o_quantize_weight(w[i], BC1, 0);
        if (swapped) n = 3 - n;
        blk |= (uint64_t)MAP1[n] << (32 + 2 * i);
    }
    return blk;
}

uint64_t o_encode_bc4_naive(const float ep[2], const float* w) {
    uint8_t E0 = o_unorm8(ep[0]), E1 = o_unorm8(ep[1]);       /* mode from stored order, no swap (R13) */
    const int* map = E0 > E1 ? MAP4_8 : MAP4_6;
    uint64_t blk = (uint64_t)E0 | ((uint64_t)E1 << 8);
    for (int i = 0; i < 16; i++) blk |= (uint64_t)map[o_quantize_weight(w[i], BC4, E0 > E1)] << (16 + 3 * i);
    return blk;
}

/* ------------------------------------------------------------------------- */
/* Reference BC1/BC4 encoder: the stand-in for Compressonator's "two refine steps"  */
/* specified by SPEC encode_block_reference, in the op order of       */
/* DESIGN.md R24-R29.  Texel values in [0,1]; fp32 with explicit fmaf, IEEE division.               */
/* ------------------------------------------------------------------------- */
static float clamp01(float x) { return fminf(fmaxf(x, 0.0f), 1.0f); }

/* R26: 2x2 least squares for the endpoints of one channel set given per-texel weights w_i
   (e0 has weight 0, e1 weight 1): A = sum (1-w)^2, B = sum w(1-w), D = sum w^2, P = sum (1-w)x,
   Q = sum w x; e0 = (D P - B Q)/det, e1 = (A Q - B P)/det, det = A D - B^2.  Returns 0 (keep the
   previous endpoints) when det is not positive. */
static int ls_endpoints(int n, const float* w, const float* x, int nc, const int* use, float* e0, float* e1) {
    float A = 0.0f, B = 0.0f, D = 0.0f, P[3] = {0, 0, 0}, Q[3] = {0, 0, 0};
    for (int i = 0; i < n; i++) {
        if (use && !use[i]) continue;
        float wi = w[i], wb = 1.0f - wi;
        A = fmaf(wb, wb, A); B = fmaf(wi, wb, B); D = fmaf(wi, wi, D);
        for (int c = 0; c < nc; c++) { P[c] = fmaf(wb, x[i * nc + c], P[c]); Q[c] = fmaf(wi, x[i * nc + c], Q[c]); }
    }
    float det = fmaf(A, D, -(B * B));
    if (!(det > 0.0f)) return 0;
    for (int c = 0; c < nc; c++) {
        e0[c] = clamp01(fmaf(D, P[c], -(B * Q[c])) / det);
        e1[c] = clamp01(fmaf(A, Q[c], -(B * P[c])) / det);
    }
    return 1;
}

/* R24/R25: BC1 initial endpoints = extremes of the texels projected on the principal axis */
static void bc1_pca_endpoints(const float* tx, float e0[3], float e1[3]) {
    float mu[3] = {0, 0, 0};
    for (int i = 0; i < 16; i++) for (int c = 0; c < 3; c++) mu[c] += tx[3 * i + c];
    for (int c = 0; c < 3; c++) mu[c] *= 0.0625f;
    float C[3][3] = {{0}};
    for (int i = 0; i < 16; i++) {
        float d[3] = {tx[3 * i] - mu[0], tx[3 * i + 1] - mu[1], tx[3 * i + 2] - mu[2]};
        for (int a = 0; a < 3; a++) for (int b = a; b < 3; b++) C[a][b] = fmaf(d[a], d[b], C[a][b]);
    }
    C[1][0] = C[0][1]; C[2][0] = C[0][2]; C[2][1] = C[1][2];
    /* start vector: the covariance column of the channel with the largest variance (first maximum);
       never orthogonal to the principal axis of a line of texels (a fixed start like (1,1,1) is, e.g.
       for a red-blue line) */
    int k = 0;
    for (int a = 1; a < 3; a++) if (C[a][a] > C[k][k]) k = a;
    float v[3] = {C[0][k], C[1][k], C[2][k]};
    int ok = C[k][k] > 0.0f;
    for (int it = 0; it < 8 && ok; it++) {                     /* power iteration, max-abs normalised */
        float u[3];
        for (int a = 0; a < 3; a++) u[a] = fmaf(C[a][2], v[2], fmaf(C[a][1], v[1], C[a][0] * v[0]));
        float m = fmaxf(fabsf(u[0]), fmaxf(fabsf(u[1]), fabsf(u[2])));
        if (!(m > 0.0f)) { ok = 0; break; }
        for (int a = 0; a < 3; a++) v[a] = u[a] / m;
    }
    if (!ok) {                                                 /* zero covariance: per-channel max / min */
        for (int c = 0; c < 3; c++) { e0[c] = tx[c]; e1[c] = tx[c]; }
        for (int i = 1; i < 16; i++) for (int c = 0; c < 3; c++) {
            e0[c] = fmaxf(e0[c], tx[3 * i + c]); e1[c] = fminf(e1[c], tx[3 * i + c]);
        }
        return;
    }
    float tmin = 0.0f, tmax = 0.0f;
    for (int i = 0; i < 16; i++) {
        float t = fmaf(tx[3 * i + 2] - mu[2], v[2], fmaf(tx[3 * i + 1] - mu[1], v[1], (tx[3 * i] - mu[0]) * v[0]));
        if (i == 0 || t < tmin) tmin = t;
        if (i == 0 || t > tmax) tmax = t;
    }
    /* extremes along the axis: mu + (t / |v|^2) v (v is max-abs normalised, not unit length) */
    float vv = fmaf(v[2], v[2], fmaf(v[1], v[1], v[0] * v[0]));
    float smax = tmax / vv, smin = tmin / vv;
    for (int c = 0; c < 3; c++) { e0[c] = clamp01(fmaf(smax, v[c], mu[c])); e1[c] = clamp01(fmaf(smin, v[c], mu[c])); }
}

/* final BC1 word for quantized endpoints (c0, c1) in either order: 4-colour order, per-texel argmin */
static uint64_t bc1_word(uint16_t c0, uint16_t c1, const float* tx) {
    if (c0 < c1) { uint16_t t = c0; c0 = c1; c1 = t; }
    uint64_t w = (uint64_t)c0 | ((uint64_t)c1 << 16);
    if (c0 == c1) return w;
    float e0[3], e1[3], pal[4][3];
    o_expand565(c0, e0); o_expand565(c1, e1);
    o_palette_bc1(e0, e1, pal);
    for (int i = 0; i < 16; i++) w |= (uint64_t)MAP1[o_argmin_bc1(tx + 3 * i, pal)] << (32 + 2 * i);
    return w;
}

uint64_t o_encode_ref_bc1(const float* tx, int n_refine) {
    float e0[3], e1[3];
    bc1_pca_endpoints(tx, e0, e1);
    uint16_t c0 = o_rgb565(e0), c1 = o_rgb565(e1);
    for (int r = 0; r < n_refine && c0 != c1; r++) {           /* R26: least squares on the assignment */
        float q0[3], q1[3], pal[4][3], w[16];
        o_expand565(c0, q0); o_expand565(c1, q1);
        o_palette_bc1(q0, q1, pal);
        for (int i = 0; i < 16; i++) w[i] = (float)o_argmin_bc1(tx + 3 * i, pal) / 3.0f;
        float n0[3], n1[3];
        if (!ls_endpoints(16, w, tx, 3, NULL, n0, n1)) break;
        c0 = o_rgb565(n0); c1 = o_rgb565(n1);
    }
    return bc1_word(c0, c1, tx);
}

/* BC4 candidate of one mode: squared error of the final assignment, word via o_encode_bc4's rules */
static float bc4_err(uint8_t E0, uint8_t E1, const float* tx, int* n_out) {
    float pal[8], err = 0.0f;
    o_palette_bc4(E0, E1, pal);
    for (int i = 0; i < 16; i++) {
        int n = o_argmin_bc4(tx[i], pal);
        if (n_out) n_out[i] = n;
        float d = tx[i] - pal[n];
        err = fmaf(d, d, err);
    }
    return err;
}
/* R27: enforce the candidate's mode on quantized endpoints (mode 8: E0 > E1, mode 6: E0 <= E1) */
static void bc4_order(int mode8, uint8_t* E0, uint8_t* E1) {
    if (mode8) {
        if (*E0 < *E1) { uint8_t t = *E0; *E0 = *E1; *E1 = t; }
        if (*E0 == *E1) { if (*E0 < 255) (*E0)++; else (*E1)--; }
    } else if (*E0 > *E1) { uint8_t t = *E0; *E0 = *E1; *E1 = t; }
}

static float bc4_candidate(int mode8, const float* tx, int n_refine, uint8_t* oE0, uint8_t* oE1) {
    float lo = 2.0f, hi = -1.0f;                              /* R28: min/max (mode 6: without exact 0 and 1) */
    for (int i = 0; i < 16; i++) {
        if (!mode8 && (tx[i] == 0.0f || tx[i] == 1.0f)) continue;
        lo = fminf(lo, tx[i]); hi = fmaxf(hi, tx[i]);
    }
    if (hi < lo) { lo = 0.0f; hi = 1.0f; }                    /* mode 6 with only 0/1 texels */
    uint8_t E0 = mode8 ? o_unorm8(hi) : o_unorm8(lo), E1 = mode8 ? o_unorm8(lo) : o_unorm8(hi);
    bc4_order(mode8, &E0, &E1);
    for (int r = 0; r < n_refine; r++) {
        int n[16], use[16];
        float w[16];
        bc4_err(E0, E1, tx, n);
        for (int i = 0; i < 16; i++) {
            use[i] = mode8 || (n[i] >= 1 && n[i] <= 6);         /* the constants 0 and 1 carry no weight */
            w[i] = mode8 ? (float)n[i] / 7.0f : (float)(n[i] - 1) / 5.0f;
        }
        float e0, e1;
        if (!ls_endpoints(16, w, tx, 1, use, &e0, &e1)) break;
        E0 = o_unorm8(e0); E1 = o_unorm8(e1);
        bc4_order(mode8, &E0, &E1);
    }
    *oE0 = E0; *oE1 = E1;
    return bc4_err(E0, E1, tx, NULL);
}

uint64_t o_encode_ref_bc4(const float* tx, int n_refine) {
    uint8_t a0, a1, b0, b1;
    float ea = bc4_candidate(1, tx, n_refine, &a0, &a1), eb = bc4_candidate(0, tx, n_refine, &b0, &b1);
    float ep[2];
    if (eb < ea) { a0 = b0; a1 = b1; }                        /* R29: lower error, ties -> 8-value mode */
    ep[0] = (float)a0 / 255.0f; ep[1] = (float)a1 / 255.0f;   /* re-quantizes to exactly (a0, a1) */
    return o_encode_bc4(ep, tx);
}

/* whole texture: row-major blocks; tex = fp32 [H][W][C] (C = 3 -> BC1, 1 -> BC4) */
void o_encode_ref_texture(const float* tex, int W, int H, int C, int n_refine, uint64_t* out, int nthreads) {
    int BW = W / 4, BH = H / 4;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 4)
    for (int by = 0; by < BH; by++)
        for (int bx = 0; bx < BW; bx++) {
            float tx[48];
            for (int i = 0; i < 16; i++)
                for (int c = 0; c < C; c++) tx[i * C + c] = tex[((size_t)(4 * by + (i >> 2)) * W + 4 * bx + (i & 3)) * C + c];
            out[(size_t)by * BW + bx] = C == 3 ? o_encode_ref_bc1(tx, n_refine) : o_encode_ref_bc4(tx, n_refine);
        }
}

void o_decode_block(uint64_t blk, int fmt, float* out) {
    if (fmt == BC1) {
        uint16_t c0 = (uint16_t)blk, c1 = (uint16_t)(blk >> 16);
        float e0[3], e1[3], pal[4][3], byc[4][3];
        o_expand565(c0, e0); o_expand565(c1, e1);
        if (c0 > c1) {
            o_palette_bc1(e0, e1, pal);
            for (int n = 0; n < 4; n++) for (int c = 0; c < 3; c++) byc[MAP1[n]][c] = pal[n][c];
        } else {                                              /* DirectX 3-colour mode (never emitted, R12) */
            for (int c = 0; c < 3; c++) {
                byc[0][c] = e0[c]; byc[1][c] = e1[c];
                byc[2][c] = fmaf(0.5f, e1[c], 0.5f * e0[c]); byc[3][c] = 0.0f;
            }
        }
        for (int i = 0; i < 16; i++) {
            int code = (int)((blk >> (32 + 2 * i)) & 3);
            for (int c = 0; c < 3; c++) out[3 * i + c] = byc[code][c];
        }
    } else {
        uint8_t E0 = (uint8_t)blk, E1 = (uint8_t)(blk >> 8);
        float pal[8], byc[8];
        o_palette_bc4(E0, E1, pal);
        const int* map = E0 > E1 ? MAP4_8 : MAP4_6;
        for (int n = 0; n < 8; n++) byc[map[n]] = pal[n];
        for (int i = 0; i < 16; i++) out[i] = byc[(blk >> (16 + 3 * i)) & 7];
    }
}

/* ------------------------------------------------------------------------- */
/* whole material (Fig. 3a)                                 */
/* ------------------------------------------------------------------------- */
static int set_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
    return omp_get_max_threads();
#else
    (void)nthreads; return 1;
#endif
}

/* endpoint MLP of block (bx,by) and colour MLP of its 16 texels (texel i = 4y+x) */
static void block_mlp(const o_model* m, int W, int H, int bx, int by, float* ep, float* col) {
    int BW = W / 4, BH = H / 4, n_c = m->mlp[1].dims[m->mlp[1].n_layers];
    float fe[16], fc[16];
    float s = ((float)bx + 0.5f) / (float)BW, t = ((float)by + 0.5f) / (float)BH;      /* R2 */
    o_grid_encode(m, 0, s, t, fe);
    o_mlp_forward(m, 0, fe, ep);
    for (int i = 0; i < 16; i++) {
        int x = 4 * bx + (i & 3), y = 4 * by + (i >> 2);
        float u = ((float)x + 0.5f) / (float)W, v = ((float)y + 0.5f) / (float)H;     /* R2 */
        o_grid_encode(m, 1, u, v, fc);
        o_mlp_forward(m, 1, fc, col + i * n_c);
    }
}

/* quantize + palette + index + pack one block position for every texture.
   ep: N_e endpoint outputs; col: 16 texels x N_c colour outputs; head layout R17. */
static void encode_all(int n_tex, const int* fmts, const float* ep, const float* col, int n_c,
                       uint64_t* out, size_t plane_stride, int naive) {
    int eo = 0, co = 0;
    for (int k = 0; k < n_tex; k++) {
        int w = fmts[k] == BC1 ? 3 : 1;
        float tx[48];
        if (naive) {                                          /* weight of texture k = output channel k */
            for (int i = 0; i < 16; i++) tx[i] = col[i * n_c + k];
            out[(size_t)k * plane_stride] = fmts[k] == BC1 ? o_encode_bc1_naive(ep + eo, tx) : o_encode_bc4_naive(ep + eo, tx);
        } else {
            for (int i = 0; i < 16; i++) for (int c = 0; c < w; c++) tx[i * w + c] = col[i * n_c + co + c];
            out[(size_t)k * plane_stride] = fmts[k] == BC1 ? o_encode_bc1(ep + eo, tx) : o_encode_bc4(ep + eo, tx);
        }
        eo += 2 * w; co += w;
    }
}

void o_mlp_outputs(const o_model* m, int W, int H, int r0, int r1, float* ep, float* col, int nthreads) {
    int BW = W / 4, n_e = m->mlp[0].dims[m->mlp[0].n_layers], n_c = m->mlp[1].dims[m->mlp[1].n_layers];
    set_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
    for (int by = r0; by < r1; by++)
        for (int bx = 0; bx < BW; bx++) {
            float c16[16 * 32];
            size_t r = (size_t)(by - r0);
            block_mlp(m, W, H, bx, by, ep + (r * BW + bx) * n_e, c16);
            for (int i = 0; i < 16; i++) {
                size_t y = r * 4 + (i >> 2), x = 4 * (size_t)bx + (i & 3);
                memcpy(col + (y * W + x) * n_c, c16 + i * n_c, sizeof(float) * n_c);
            }
        }
}

void o_pack(int n_tex, const int* fmts, const float* ep, const float* col, int W, int H,
            int r0, int r1, uint64_t* out, int nthreads) {
    int BW = W / 4, rows = r1 - r0, n_e = 0, n_c = 0;
    (void)H;
    for (int k = 0; k < n_tex; k++) { n_e += fmts[k] == BC1 ? 6 : 2; n_c += fmts[k] == BC1 ? 3 : 1; }
    set_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
    for (int r = 0; r < rows; r++)
        for (int bx = 0; bx < BW; bx++) {
            float c16[16 * 32];
            for (int i = 0; i < 16; i++) {
                size_t y = (size_t)r * 4 + (i >> 2), x = 4 * (size_t)bx + (i & 3);
                memcpy(c16 + i * n_c, col + (y * W + x) * n_c, sizeof(float) * n_c);
            }
            encode_all(n_tex, fmts, ep + ((size_t)r * BW + bx) * n_e, c16, n_c,
                       out + (size_t)r * BW + bx, (size_t)rows * BW, 0);
        }
}

void o_decode_material(const o_model* m, int W, int H, int r0, int r1, uint64_t* out, int nthreads) {
    int BW = W / 4, rows = r1 - r0, n_c = m->mlp[1].dims[m->mlp[1].n_layers];
    set_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
    for (int r = 0; r < rows; r++)
        for (int bx = 0; bx < BW; bx++) {
            float ep[64], c16[16 * 32];
            block_mlp(m, W, H, bx, r0 + r, ep, c16);
            encode_all(m->n_tex, m->fmt, ep, c16, n_c, out + (size_t)r * BW + bx, (size_t)rows * BW, m->naive);
        }
}

void o_decode_bc(const uint64_t* blocks, int fmt, int W, int H, float* out) {
    int BW = W / 4, BH = H / 4, ch = fmt == BC1 ? 3 : 1;
    for (int by = 0; by < BH; by++)
        for (int bx = 0; bx < BW; bx++) {
            float tx[48];
            o_decode_block(blocks[(size_t)by * BW + bx], fmt, tx);
            for (int i = 0; i < 16; i++) {
                size_t y = 4 * (size_t)by + (i >> 2), x = 4 * (size_t)bx + (i & 3);
                for (int c = 0; c < ch; c++) out[(y * W + x) * ch + c] = tx[i * ch + c];
            }
        }
}

/* PSNR: 10 log10(1 / MSE) for values in [0,1] */
double o_psnr(const float* a, const float* b, size_t n) {
    double se = 0.0;
    for (size_t i = 0; i < n; i++) { double d = (double)a[i] - (double)b[i]; se += d * d; }
    if (se == 0.0) return INFINITY;
    return 10.0 * log10((double)n / se);
}

/* ------------------------------------------------------------------------- */
/* brute force                                                                */
/* ------------------------------------------------------------------------- */
double o_block_sq_error(uint64_t blk, int fmt, const float* tx) {
    float dec[48]; int ch = fmt == BC1 ? 3 : 1;
    o_decode_block(blk, fmt, dec);
    double se = 0.0;
    for (int i = 0; i < 16 * ch; i++) { double d = (double)dec[i] - (double)tx[i]; se += d * d; }
    return se;
}

/* exhaustive BC4 encoder: all 65,536 endpoint pairs, per-texel nearest entry */
uint64_t o_bruteforce_bc4(const float* tx, double* best_err) {
    double best = INFINITY; uint64_t bb = 0;
    for (int E0 = 0; E0 < 256; E0++)
        for (int E1 = 0; E1 < 256; E1++) {
            float pal[8]; o_palette_bc4((uint8_t)E0, (uint8_t)E1, pal);
            const int* map = E0 > E1 ? MAP4_8 : MAP4_6;
            double se = 0.0; uint64_t w = (uint64_t)E0 | ((uint64_t)E1 << 8);
            for (int i = 0; i < 16; i++) {
                int bn = 0; double bd = INFINITY;
                for (int n = 0; n < 8; n++) { double d = (double)tx[i] - (double)pal[n]; d *= d; if (d < bd) { bd = d; bn = n; } }
                se += bd; w |= (uint64_t)map[bn] << (16 + 3 * i);
            }
            if (se < best) { best = se; bb = w; }
        }
    if (best_err) *best_err = best;
    return bb;
}

/* ------------------------------------------------------------------------- */
/* storage arithmetic (13.37 / 26.74 MB; P:321 int8 grids, P:342 fp16 MLPs) */
/* ------------------------------------------------------------------------- */
uint64_t o_storage_bytes(int bl, int bc, int tl, int tc, int F, int hidden, int n_hidden,
                         int n_e, int n_c, int with_bias) {
    uint64_t bytes = 0;
    for (int l = 0; l < bl; l++) bytes += (uint64_t)(bc << l) * (uint64_t)(bc << l) * F;
    for (int l = 0; l < tl; l++) bytes += (uint64_t)(tc << l) * (uint64_t)(tc << l) * F;
    int ins[2] = {bl * F, tl * F}, outs[2] = {n_e, n_c};
    for (int k = 0; k < 2; k++) {
        int prev = ins[k];
        for (int l = 0; l <= n_hidden; l++) {
            int o = l < n_hidden ? hidden : outs[k];
            bytes += 2ull * ((uint64_t)prev * o + (with_bias ? o : 0));
            prev = o;
        }
    }
    return bytes;
}
