/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the residual-compensated
 * 16-bit optimizer step of arXiv 2309.12381 ("16-bit-only mixed precision").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2309_12381_b200/) never imports, links or executes it, and this file shares no
 * code, header, table or constant with the CUDA path.
 *
 * Build: gcc -std=c99 -O2 -ffp-contract=off -fno-fast-math -fPIC -shared (x86-64 SSE2
 * scalar binary32/binary64 arithmetic, FLT_EVAL_METHOD == 0, no contraction, no FTZ/DAZ).
 *
 * Citation keys: "P:n" = PAPER.md line n (section named alongside), "S:n" = SPEC.md line n,
 * "R<k>" = a reading of a paper-silent point, listed in DESIGN.md section 3.
 *
 * Every function processes one element at a time in the order the paper (or the reading
 * it cites) states; nothing is blocked, fused or reordered.
 *
 * Parity pins: see tests/test_oracle_*.py.  Every function here is pinned (no function is
 * "parity unpinned"): formats by exhaustive sweeps against numpy/torch casts and closed-form
 * counts; SGD/Adam by closed forms and by torch.optim (library routine) within tolerance;
 * the norm by exact-sum constructions and by math.fsum; the byte model by the paper's
 * printed inventory.
 */
#include <stdint.h>
#include <string.h>
#include <math.h>
#if defined(__x86_64__) || defined(__i386__)
#include <xmmintrin.h>
#endif

/* Element loops are independent (the method is elementwise), so the all-core baseline build
 * (gcc -fopenmp: liboracle_omp.so, bench.py's cpu_baseline "threads_all") splits them across
 * threads with no other change; the plain build ignores the annotation.  Both builds are
 * bit-identical (tests/test_oracle_omp.py). */
#ifdef _OPENMP
#include <omp.h>
#define OR_PARALLEL_FOR _Pragma("omp parallel for schedule(static)")
#else
#define OR_PARALLEL_FOR
#endif

/* Threads of the parallel build (1 in the plain build). */
int or_threads(int set) {
#ifdef _OPENMP
    if (set > 0) omp_set_num_threads(set);
    return omp_get_max_threads();
#else
    (void)set;
    return 1;
#endif
}

/* Format codes of THIS oracle (independent of the CUDA library's enum). */
#define OR_FP16 0
#define OR_BF16 1
#define OR_FP32 2

/* ------------------------------------------------------------------------------------- */
/* Host floating-point environment: subnormals must not be flushed.  */
/* ------------------------------------------------------------------------------------- */

/* Clears FTZ (bit 15) and DAZ (bit 6) of MXCSR; returns the MXCSR value found on entry. */
unsigned or_fpenv_clear(void) {
#if defined(__x86_64__) || defined(__i386__)
    unsigned old = _mm_getcsr();
    _mm_setcsr(old & ~((1u << 15) | (1u << 6)));
    return old;
#else
    return 0;
#endif
}

/* 1 if FTZ and DAZ are both clear. */
int or_fpenv_ok(void) {
#if defined(__x86_64__) || defined(__i386__)
    unsigned c = _mm_getcsr();
    return (c & ((1u << 15) | (1u << 6))) == 0;
#else
    return 1;
#endif
}

static uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

/* ------------------------------------------------------------------------------------- */
/* L0 numeric formats (Table 1; sec. 1.1 "Floating Point Format Basics")  */
/* ------------------------------------------------------------------------------------- */

/*
 * IEEE-754 round-to-nearest-even of a binary32 pattern to binary16 (fp16, 1/5/10) or
 * bfloat16 (1/8/7), by explicit integer arithmetic (guard/round/sticky on the dropped bits).
 * Reading R2 (BASELINE north_star "explicit IEEE round-to-nearest-even"; P:84 calls
 * round-to-nearest "the standard" rounding).  Subnormals are produced (R5: P:50's claim that
 * bf16 has none is not followed).  Overflow rounds to +-Inf (IEEE).  NaN -> 0x7FFF (R4).
 */
uint16_t or_rne16(int fmt, uint32_t u) {
    uint32_t sign = u & 0x80000000u;
    uint32_t a = u & 0x7FFFFFFFu;
    if (a > 0x7F800000u) return 0x7FFF;                  /* NaN (R4) */
    if (fmt == OR_BF16) {
        /* bf16 keeps the binary32 exponent: drop the low 16 significand bits. */
        uint32_t h = a >> 16;
        uint32_t rem = a & 0xFFFFu;
        if (rem > 0x8000u || (rem == 0x8000u && (h & 1u))) h += 1u;   /* carry may reach Inf */
        return (uint16_t)((sign >> 16) | h);
    }
    /* fp16 */
    if (a == 0x7F800000u) return (uint16_t)((sign >> 16) | 0x7C00u);
    {
        uint32_t e = a >> 23, mant = a & 0x7FFFFFu;
        uint32_t sig;        /* significand with explicit leading bit, value = sig * 2^(ee-23) */
        int ee;              /* unbiased exponent of bit 23 of sig */
        uint32_t h, rem, half;
        int s;
        if (e == 0) { sig = mant; ee = -126; } else { sig = mant | 0x800000u; ee = (int)e - 127; }
        if (ee >= -14) {
            /* normal fp16 candidate: keep 11 significand bits, drop 13 */
            if (ee > 15) return (uint16_t)((sign >> 16) | 0x7C00u);   /* >= 2^16: overflow */
            h = ((uint32_t)(ee + 15) << 10) + ((sig >> 13) - 0x400u);
            rem = sig & 0x1FFFu; half = 0x1000u;
            if (rem > half || (rem == half && (h & 1u))) h += 1u;      /* carry into exponent */
            if (h >= 0x7C00u) h = 0x7C00u;                            /* rounded to Inf */
            return (uint16_t)((sign >> 16) | h);
        }
        /* fp16 subnormal: value / 2^-24 = sig * 2^(ee+1); drop s = -1-ee bits (s >= 14) */
        s = -1 - ee;
        if (s >= 25) return (uint16_t)(sign >> 16);                  /* < half of 2^-24 */
        h = sig >> s;
        rem = sig & ((1u << s) - 1u);
        half = 1u << (s - 1);
        if (rem > half || (rem == half && (h & 1u))) h += 1u;          /* may become 0x400 */
        return (uint16_t)((sign >> 16) | h);
    }
}

/* Exact widening of a 16-bit pattern to a binary32 pattern (P:21-32, P:44 implicit bit;
 * subnormals normalised).  NaN -> 0x7FFFFFFF (R4). */
uint32_t or_widen16(int fmt, uint16_t h) {
    uint32_t sign = ((uint32_t)h & 0x8000u) << 16;
    if (fmt == OR_BF16) {
        uint32_t u = (uint32_t)h << 16;
        if ((u & 0x7FFFFFFFu) > 0x7F800000u) return 0x7FFFFFFFu;
        return u;
    } else {
        uint32_t E = ((uint32_t)h >> 10) & 0x1Fu, m = (uint32_t)h & 0x3FFu;
        if (E == 31u) return m ? 0x7FFFFFFFu : (sign | 0x7F800000u);
        if (E == 0u) {
            int p;
            if (m == 0u) return sign;
            p = 9;                                   /* position of the leading one of m */
            while (!(m & (1u << p))) p--;
            /* value = m * 2^-24 = 2^(p-24) * (m / 2^p) */
            return sign | ((uint32_t)(p - 24 + 127) << 23) | ((m << (23 - p)) & 0x7FFFFFu);
        }
        return sign | ((E - 15u + 127u) << 23) | (m << 13);
    }
}

/* 16-bit value of the paper's storage scheme ("storing only the difference between the
 * two formats"; P:68 13/16 extra bits; "the 16bits value used in the computations").
 * Reading R1: the residual is the signed difference of the two binary32 patterns, saturated
 * to int16 (R3: the RNE upper tie gives +32768 and saturates to +32767). */
static void split1(int fmt, uint32_t u, uint16_t* h_out, int16_t* r_out) {
    uint16_t h;
    uint32_t wu;
    int64_t d;
    if ((u & 0x7FFFFFFFu) > 0x7F800000u) { *h_out = 0x7FFF; *r_out = 0; return; }   /* R4 */
    h = or_rne16(fmt, u);
    wu = or_widen16(fmt, h);
    if ((wu & 0x7FFFFFFFu) == 0x7F800000u) { *h_out = h; *r_out = 0; return; }      /* Inf */
    d = (int64_t)u - (int64_t)wu;          /* same sign: RNE never changes the sign */
    if (d > 32767) d = 32767;
    if (d < -32768) d = -32768;
    *h_out = h;
    *r_out = (int16_t)d;
}

/* Reconstruct the full-precision value from the 16-bit value and its extra bits (P:70
 * "performs the operation in full precision using the extra bits saved separately"). */
static uint32_t reconstruct1(int fmt, uint16_t h, int16_t r) {
    uint32_t wu = or_widen16(fmt, h);
    if ((wu & 0x7FFFFFFFu) > 0x7F800000u) return 0x7FFFFFFFu;
    if ((wu & 0x7FFFFFFFu) == 0x7F800000u) return wu;
    return (uint32_t)((int64_t)wu + (int64_t)r);   /* two's-complement 32-bit wrap */
}

void or_split(int fmt, const float* w, uint16_t* value, int16_t* resid, int64_t n) {
    int64_t i;
    OR_PARALLEL_FOR
    for (i = 0; i < n; i++) split1(fmt, f2u(w[i]), &value[i], &resid[i]);
}

void or_reconstruct(int fmt, const uint16_t* value, const int16_t* resid, float* w, int64_t n) {
    int64_t i;
    OR_PARALLEL_FOR
    for (i = 0; i < n; i++) w[i] = u2f(reconstruct1(fmt, value[i], resid[i]));
}

/* Plain 16-bit cast used for the "16-bit only" baseline ("fp16" row) and for grads. */
void or_cast16(int fmt, const float* w, uint16_t* out, int64_t n) {
    int64_t i;
    for (i = 0; i < n; i++) out[i] = or_rne16(fmt, f2u(w[i]));
}

void or_widen(int fmt, const uint16_t* h, float* out, int64_t n) {
    int64_t i;
    for (i = 0; i < n; i++) out[i] = u2f(or_widen16(fmt, h[i]));
}

static float load_grad(int gfmt, const void* grad, int64_t i) {
    if (gfmt == OR_FP32) return ((const float*)grad)[i];
    return u2f(or_widen16(gfmt, ((const uint16_t*)grad)[i]));
}

/* ------------------------------------------------------------------------------------- */
/* L2 optimizers ("classic optimizers (Adam and SGD)"; P:86 fused stream)            */
/* Hyper-parameters arrive as doubles; each derived kernel scalar is rounded ONCE to float */
/* (reading R7).  Update formulas and operation order: reading R6 (torch.optim single-    */
/* tensor semantics, "does not necessitate any alterations to the hyperparameters or */
/* the training framework", P:210 PyTorch 2.0.1).                                         */
/* ------------------------------------------------------------------------------------- */

typedef struct {
    double lr, momentum, dampening, weight_decay, grad_scale;
    int32_t nesterov, first_step;
    double clip_value;     /* > 0: clamp the scaled gradient to [-c, c]; 0: off */
} or_sgd_hp;

typedef struct {
    double lr, beta1, beta2, eps, weight_decay, grad_scale;
    int32_t adamw;
    int64_t step;          /* 1-based */
    double clip_value;     /* > 0: clamp the scaled gradient to [-c, c]; 0: off */
} or_adam_hp;

/* Clip-by-value of the (scaled) gradient: the paper's hook "torch.clamp(grad, -clip_value,
 * clip_value)", applied as the optimizer's gradient ingest.  NaN stays NaN
 * (torch.clamp semantics), +-Inf clamps to +-c. */
static float clamp_grad(float g, double clip_value) {
    float c;
    if (!(clip_value > 0.0)) return g;
    c = (float)clip_value;
    if (g > c) return c;
    if (g < -c) return -c;
    return g;
}

/* SGD(-momentum) element update on the fp32 value w (torch.optim.SGD). */
static float sgd_update(float w, float g, float* buf, const or_sgd_hp* hp) {
    float lr = (float)hp->lr, mom = (float)hp->momentum;
    float damp1 = (float)(1.0 - hp->dampening), wd = (float)hp->weight_decay;
    float t;
    if (hp->weight_decay != 0.0) { t = wd * w; g = g + t; }
    if (hp->momentum != 0.0) {
        float b;
        if (hp->first_step) {
            b = g;                                    /* buffer = clone(grad) */
        } else {
            b = *buf * mom; t = damp1 * g; b = b + t;
        }
        *buf = b;
        if (hp->nesterov) { t = mom * b; g = g + t; } else { g = b; }
    }
    t = lr * g;
    w = w - t;
    return w;
}

/* Adam / AdamW element update on the fp32 value w (Kingma & Ba; torch.optim). */
typedef struct { float b1c, b2, b2c, bc2s, ss, eps, dec, wd; int adamw, l2; } adam_scalars;

static adam_scalars adam_derive(const or_adam_hp* hp) {
    adam_scalars c;
    double t = (double)hp->step;
    c.b1c = (float)(1.0 - hp->beta1);                      /* lerp weight 1-beta1 */
    c.b2 = (float)hp->beta2;
    c.b2c = (float)(1.0 - hp->beta2);
    c.bc2s = (float)sqrt(1.0 - pow(hp->beta2, t));         /* sqrt(bias_correction2) */
    c.ss = (float)(hp->lr / (1.0 - pow(hp->beta1, t)));    /* step size lr/bias_correction1 */
    c.eps = (float)hp->eps;
    c.dec = (float)(1.0 - hp->lr * hp->weight_decay);      /* AdamW decoupled decay */
    c.wd = (float)hp->weight_decay;
    c.adamw = hp->adamw != 0;
    c.l2 = (!hp->adamw) && hp->weight_decay != 0.0;
    return c;
}

static float adam_update(float w, float g, float* m, float* v, const adam_scalars* c) {
    float d, t, s, mm, vv;
    if (c->adamw) { w = w * c->dec; }
    else if (c->l2) { t = c->wd * w; g = g + t; }
    /* m = lerp(m, g, 1-beta1); the lerp formula switches at weight 0.5 (R6) */
    if (c->b1c < 0.5f) { d = g - *m; t = c->b1c * d; mm = *m + t; }
    else { d = g - *m; t = (1.0f - c->b1c); t = t * d; mm = g - t; }
    /* v = v*beta2 + (1-beta2)*g*g */
    vv = *v * c->b2; t = c->b2c * g; t = t * g; vv = vv + t;
    *m = mm; *v = vv;
    /* w = w - (ss*m) / (sqrt(v)/bc2s + eps) */
    s = sqrtf(vv); s = s / c->bc2s; s = s + c->eps;
    t = c->ss * mm; t = t / s;
    w = w - t;
    return w;
}

/* Residual-compensated SGD step, one tensor: reconstruct -> update at fp32 -> re-split
 * ("outputs both the updated 16 bits float and its extra bits"). */
void or_sgd_step(int vfmt, int gfmt, uint16_t* value, int16_t* resid, const void* grad,
                 float* buf, int64_t n, const or_sgd_hp* hp) {
    int64_t i;
    float gs = (float)hp->grad_scale;
    OR_PARALLEL_FOR
    for (i = 0; i < n; i++) {
        float g = clamp_grad(load_grad(gfmt, grad, i) * gs, hp->clip_value);
        float w = u2f(reconstruct1(vfmt, value[i], resid[i]));
        w = sgd_update(w, g, buf ? &buf[i] : 0, hp);
        split1(vfmt, f2u(w), &value[i], &resid[i]);
    }
}

/* Residual-compensated Adam/AdamW step, one tensor.  clip_coef multiplies the scaled grad
 * when global-norm clipping is active ("every operations on the gradient (eg. clipping
 * or scaling) has to be done through the optimizer"); pass a negative value for no clip. */
void or_adam_step(int vfmt, int gfmt, uint16_t* value, int16_t* resid, const void* grad,
                  float* m, float* v, int64_t n, const or_adam_hp* hp, float clip_coef) {
    int64_t i;
    float gs = (float)hp->grad_scale;
    adam_scalars c = adam_derive(hp);
    OR_PARALLEL_FOR
    for (i = 0; i < n; i++) {
        float g = clamp_grad(load_grad(gfmt, grad, i) * gs, hp->clip_value);
        float w;
        if (clip_coef >= 0.0f || clip_coef != clip_coef) g = g * clip_coef;
        w = u2f(reconstruct1(vfmt, value[i], resid[i]));
        w = adam_update(w, g, &m[i], &v[i], &c);
        split1(vfmt, f2u(w), &value[i], &resid[i]);
    }
}

/* fp32-master comparators ("full precision copy for each parameter"): the same
 * updates applied to an fp32 weight that is never split.  Used by pin P6. */
void or_sgd_step_master(int gfmt, float* w, const void* grad, float* buf, int64_t n,
                        const or_sgd_hp* hp) {
    int64_t i;
    float gs = (float)hp->grad_scale;
    OR_PARALLEL_FOR
    for (i = 0; i < n; i++) {
        float g = clamp_grad(load_grad(gfmt, grad, i) * gs, hp->clip_value);
        w[i] = sgd_update(w[i], g, buf ? &buf[i] : 0, hp);
    }
}

void or_adam_step_master(int gfmt, float* w, const void* grad, float* m, float* v, int64_t n,
                         const or_adam_hp* hp, float clip_coef) {
    int64_t i;
    float gs = (float)hp->grad_scale;
    adam_scalars c = adam_derive(hp);
    OR_PARALLEL_FOR
    for (i = 0; i < n; i++) {
        float g = clamp_grad(load_grad(gfmt, grad, i) * gs, hp->clip_value);
        if (clip_coef >= 0.0f || clip_coef != clip_coef) g = g * clip_coef;
        w[i] = adam_update(w[i], g, &m[i], &v[i], &c);
    }
}

/* ------------------------------------------------------------------------------------- */
/* Paper variants of the storage scheme                               */
/*   OR_S_RNE  round-to-nearest-even value + int16 signed difference (R1-R5, the default)  */
/*   OR_S_RTZ  round-to-zero value + uint16 extra bits: "saving only the first part   */
/*             of the 32bit significand is equivalent to applying a round-to-zero          */
/*             operation on the full precision value"                                      */
/*   OR_S_SR   stochastic rounding + the signed difference, whose sign is the paper's one  */
/*             extra "un-round" bit ("we store one additional extra-bit to keep in     */
/*             memory whether or not the value was changed when rounded-up"); fp16 only,    */
/*             as in the paper's "fp16 + 13 stochastic" run -- 13 + 1 bits fit 16   */
/*   OR_S_X8   RNE value + only 8 extra bits (int8): "We also explore the performance  */
/*             when keeping only part of those bits"; "fp16 + 8"; reading R14         */
/*   OR_S_X8Z  the paper's own fp16+8 / bf16+8: round-to-zero value + the NEXT 8 bits of the  */
/*             fp32 significand, truncated (uint8) -- P:84 "saving only the first part of   */
/*             the 32bit significand is equivalent to applying a round-to-zero"; R20        */
/* ------------------------------------------------------------------------------------- */
#define OR_S_RNE 0
#define OR_S_RTZ 1
#define OR_S_SR 2
#define OR_S_X8 3
#define OR_S_X8Z 4

/* IEEE round-toward-zero of a binary32 pattern to fp16 / bf16 by integer truncation of the
 * dropped significand bits (no rounding increment).  Finite values never overflow to Inf: they
 * saturate at the largest finite 16-bit value (IEEE RTZ).  NaN -> 0x7FFF (R4). */
uint16_t or_rtz16(int fmt, uint32_t u) {
    uint32_t sign = u & 0x80000000u;
    uint32_t a = u & 0x7FFFFFFFu;
    if (a > 0x7F800000u) return 0x7FFF;
    if (fmt == OR_BF16) return (uint16_t)((sign >> 16) | (a >> 16));
    if (a == 0x7F800000u) return (uint16_t)((sign >> 16) | 0x7C00u);
    {
        uint32_t e = a >> 23, mant = a & 0x7FFFFFu, sig;
        int ee, s;
        if (e == 0) { sig = mant; ee = -126; } else { sig = mant | 0x800000u; ee = (int)e - 127; }
        if (ee > 15) return (uint16_t)((sign >> 16) | 0x7BFFu);                 /* >= 2^16 */
        if (ee >= -14) return (uint16_t)((sign >> 16) | (((uint32_t)(ee + 15) << 10) + ((sig >> 13) - 0x400u)));
        s = -1 - ee;                                                           /* subnormal */
        if (s >= 24) return (uint16_t)(sign >> 16);
        return (uint16_t)((sign >> 16) | (sig >> s));
    }
}

/* The counter-based generator both sides implement (the draws of stochastic rounding are an
 * input of the method, not its arithmetic): splitmix64's finaliser over a key mixed from
 * (seed, stream, index) with two odd 64-bit constants. */
uint64_t or_mix64(uint64_t seed, uint64_t stream, uint64_t index) {
    uint64_t x = seed ^ (stream * 0x9E3779B97F4A7C15ull) ^ (index * 0xD1B54A32D192ED03ull);
    x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27; x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}

/* Stochastic rounding to fp16 with a 32-bit draw `rnd`: t = RTZ(x); with D = bits(x) -
 * bits(widen(t)) and U = bits(widen(t + 1 ulp)) - bits(widen(t)) (binary32 patterns), round
 * up in magnitude iff rnd < floor(D * 2^32 / U), i.e. with probability D/U.  |x| >= 2^16
 * -> Inf (as RNE overflow).  NaN -> 0x7FFF, Inf -> Inf. */
uint16_t or_sr16(uint32_t u, uint32_t rnd) {
    uint32_t a = u & 0x7FFFFFFFu;
    uint16_t t, up;
    uint64_t d, uu;
    if (a > 0x7F800000u) return 0x7FFF;
    if (a >= 0x47800000u) return (uint16_t)(((u & 0x80000000u) >> 16) | 0x7C00u);   /* >= 2^16 or Inf */
    t = or_rtz16(OR_FP16, u);
    up = (uint16_t)(t + 1u);                           /* next magnitude (may become Inf) */
    d = (uint64_t)(a - (or_widen16(OR_FP16, t) & 0x7FFFFFFFu));
    uu = (uint64_t)((or_widen16(OR_FP16, up) & 0x7FFFFFFFu) - (or_widen16(OR_FP16, t) & 0x7FFFFFFFu));
    if ((uint64_t)rnd < ((d << 32) / uu)) return up;
    return t;
}

static int64_t floordiv_pow2(int64_t x, int sh) {
    int64_t q = (int64_t)1 << sh;
    return x >= 0 ? x / q : -((-x + q - 1) / q);
}

/* Split under a scheme.  resid receives the stored residual as an integer: int16 range (RNE,
 * SR), 0..65535 (RTZ, stored as the uint16 bit pattern), int8 range (X8). */
static void split_s(int scheme, int fmt, uint32_t u, uint32_t rnd, uint16_t* h_out, int32_t* r_out) {
    uint16_t h;
    uint32_t wu;
    int64_t d;
    if ((u & 0x7FFFFFFFu) > 0x7F800000u) { *h_out = 0x7FFF; *r_out = 0; return; }   /* R4 */
    if (scheme == OR_S_RTZ || scheme == OR_S_X8Z) h = or_rtz16(fmt, u);
    else if (scheme == OR_S_SR) h = or_sr16(u, rnd);
    else h = or_rne16(fmt, u);
    wu = or_widen16(fmt, h);
    *h_out = h;
    if ((wu & 0x7FFFFFFFu) >= 0x7F800000u) { *r_out = 0; return; }                    /* Inf */
    d = (int64_t)u - (int64_t)wu;          /* same sign: none of the roundings changes it */
    if (scheme == OR_S_RTZ) {              /* |x| >= |t|: d >= 0 */
        *r_out = (int32_t)(d > 65535 ? 65535 : d);
    } else if (scheme == OR_S_X8Z) {       /* |x| >= |t|: the next 8 bits, truncated (R20) */
        int64_t q = d >> (fmt == OR_BF16 ? 8 : 5);
        *r_out = (int32_t)(q > 255 ? 255 : q);
    } else if (scheme == OR_S_X8) {        /* keep the top 8 of the extra bits, nearest (R14) */
        int sh = fmt == OR_BF16 ? 8 : 5;
        int64_t q = floordiv_pow2(d + ((int64_t)1 << (sh - 1)), sh);
        *r_out = (int32_t)(q > 127 ? 127 : (q < -128 ? -128 : q));
    } else {
        *r_out = (int32_t)(d > 32767 ? 32767 : (d < -32768 ? -32768 : d));
    }
}

static uint32_t reconstruct_s(int scheme, int fmt, uint16_t h, int32_t r) {
    uint32_t wu = or_widen16(fmt, h);
    int64_t add;
    if ((wu & 0x7FFFFFFFu) > 0x7F800000u) return 0x7FFFFFFFu;
    if ((wu & 0x7FFFFFFFu) == 0x7F800000u) return wu;
    if (scheme == OR_S_X8 || scheme == OR_S_X8Z) add = (int64_t)r * (fmt == OR_BF16 ? 256 : 32);
    else add = r;
    return (uint32_t)((int64_t)wu + add);
}

static int32_t load_resid(int scheme, const void* resid, int64_t i) {
    if (scheme == OR_S_X8) return ((const int8_t*)resid)[i];
    if (scheme == OR_S_X8Z) return ((const uint8_t*)resid)[i];
    if (scheme == OR_S_RTZ) return ((const uint16_t*)resid)[i];
    return ((const int16_t*)resid)[i];
}

static void store_resid(int scheme, void* resid, int64_t i, int32_t r) {
    if (scheme == OR_S_X8) ((int8_t*)resid)[i] = (int8_t)r;
    else if (scheme == OR_S_X8Z) ((uint8_t*)resid)[i] = (uint8_t)r;
    else if (scheme == OR_S_RTZ) ((uint16_t*)resid)[i] = (uint16_t)r;
    else ((int16_t*)resid)[i] = (int16_t)r;
}

/* Draw of element i: one 64-bit output serves an element pair -- the upper half for even i,
 * the lower half for odd i (reading R14). */
static uint32_t draw(int scheme, uint64_t seed, uint64_t stream, int64_t i) {
    uint64_t x;
    if (scheme != OR_S_SR) return 0u;
    x = or_mix64(seed, stream, (uint64_t)i >> 1);
    return (i & 1) ? (uint32_t)x : (uint32_t)(x >> 32);
}

void or_split_s(int scheme, int fmt, const float* w, uint16_t* value, void* resid, int64_t n, uint64_t seed,
                uint64_t stream) {
    int64_t i;
    OR_PARALLEL_FOR
    for (i = 0; i < n; i++) {
        uint16_t h; int32_t r;
        split_s(scheme, fmt, f2u(w[i]), draw(scheme, seed, stream, i), &h, &r);
        value[i] = h;
        store_resid(scheme, resid, i, r);
    }
}

void or_reconstruct_s(int scheme, int fmt, const uint16_t* value, const void* resid, float* w, int64_t n) {
    int64_t i;
    OR_PARALLEL_FOR
    for (i = 0; i < n; i++) w[i] = u2f(reconstruct_s(scheme, fmt, value[i], load_resid(scheme, resid, i)));
}

/* The steps under a scheme: reconstruct -> the same fp32 update -> split (SR draws keyed by
 * (seed, stream, element index)). */
void or_sgd_step_s(int scheme, int vfmt, int gfmt, uint16_t* value, void* resid, const void* grad, float* buf,
                   int64_t n, const or_sgd_hp* hp, uint64_t seed, uint64_t stream) {
    int64_t i;
    float gs = (float)hp->grad_scale;
    OR_PARALLEL_FOR
    for (i = 0; i < n; i++) {
        float g = clamp_grad(load_grad(gfmt, grad, i) * gs, hp->clip_value);
        float w = u2f(reconstruct_s(scheme, vfmt, value[i], load_resid(scheme, resid, i)));
        uint16_t h; int32_t r;
        w = sgd_update(w, g, buf ? &buf[i] : 0, hp);
        split_s(scheme, vfmt, f2u(w), draw(scheme, seed, stream, i), &h, &r);
        value[i] = h;
        store_resid(scheme, resid, i, r);
    }
}

void or_adam_step_s(int scheme, int vfmt, int gfmt, uint16_t* value, void* resid, const void* grad, float* m,
                    float* v, int64_t n, const or_adam_hp* hp, float clip_coef, uint64_t seed, uint64_t stream) {
    int64_t i;
    float gs = (float)hp->grad_scale;
    adam_scalars c = adam_derive(hp);
    OR_PARALLEL_FOR
    for (i = 0; i < n; i++) {
        float g = clamp_grad(load_grad(gfmt, grad, i) * gs, hp->clip_value);
        float w;
        uint16_t h; int32_t r;
        if (clip_coef >= 0.0f || clip_coef != clip_coef) g = g * clip_coef;
        w = u2f(reconstruct_s(scheme, vfmt, value[i], load_resid(scheme, resid, i)));
        w = adam_update(w, g, &m[i], &v[i], &c);
        split_s(scheme, vfmt, f2u(w), draw(scheme, seed, stream, i), &h, &r);
        value[i] = h;
        store_resid(scheme, resid, i, r);
    }
}

/* ------------------------------------------------------------------------------------- */
/* Global-norm clipping ("Gradient Clipping"; reading R9: torch clip_grad_norm_     */
/* formula, fp64 accumulation; only in multi-tensor / sharded modes)                */
/* ------------------------------------------------------------------------------------- */

static double sumsq_pairwise(int gfmt, const void* grad, int64_t lo, int64_t hi, float gs) {
    if (hi - lo <= 8) {
        double s = 0.0;
        int64_t i;
        for (i = lo; i < hi; i++) {
            double g = (double)(load_grad(gfmt, grad, i) * gs);
            s += g * g;                       /* exact: a float squared fits in a double */
        }
        return s;
    } else {
        int64_t mid = lo + (hi - lo) / 2;
        return sumsq_pairwise(gfmt, grad, lo, mid, gs) + sumsq_pairwise(gfmt, grad, mid, hi, gs);
    }
}

/* Sum over i of (double)(f32(grad_i)*gs)^2, pairwise summation. */
double or_sumsq(int gfmt, const void* grad, int64_t n, double grad_scale) {
    if (n <= 0) return 0.0;
    return sumsq_pairwise(gfmt, grad, 0, n, (float)grad_scale);
}

/* coef = min(1, max_norm / (sqrt(S) + 1e-6)); a NaN quotient propagates (R9). */
float or_clip_coef(double sumsq, double max_norm) {
    double q = max_norm / (sqrt(sumsq) + 1e-6);
    return (float)(q > 1.0 ? 1.0 : q);
}

/* ------------------------------------------------------------------------------------- */
/* Data-parallel gradient reduction of the P2P fused sharded step (BJ north_star (c);     */
/* reading R15: the sum over ranks of the 16-bit gradients, each widened exactly to        */
/* binary32 and accumulated in binary32 in rank order, g = ((g_0 + g_1) + g_2) + ...)       */
/* ------------------------------------------------------------------------------------- */

/* grads: `world` pointers to n 16-bit gradient patterns of format fmt (rank order). */
void or_reduce_sum16(int fmt, int world, const uint16_t* const* grads, float* out, int64_t n) {
    int64_t i;
    int k;
    for (i = 0; i < n; i++) {
        float s = u2f(or_widen16(fmt, grads[0][i]));
        for (k = 1; k < world; k++) s = s + u2f(or_widen16(fmt, grads[k][i]));
        out[i] = s;
    }
}

/* ------------------------------------------------------------------------------------- */
/* Per-parameter byte accounting (reading R11)                                   */
/* ------------------------------------------------------------------------------------- */

/* scheme: 0 = paper's AMP inventory (fp32 master 4 + 16-bit copy 2 + grad 4 + state),
 *         1 = ours, fused backward (16-bit value 2 + residual 2 + no persistent grad + state),
 *         2 = ours, multi-tensor with 16-bit grads (2 + 2 + 2 + state).
 * optim: 0 = SGD-momentum (state 4 B), 1 = Adam (state 8 B). */
int or_bytes_per_param(int scheme, int optim) {
    int state = optim == 1 ? 8 : 4;
    if (scheme == 0) return 4 + 2 + 4 + state;
    if (scheme == 1) return 2 + 2 + 0 + state;
    if (scheme == 2) return 2 + 2 + 2 + state;
    return -1;
}
