/*
 * lora_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU reference for the multi-LoRA delta
 * (InfiniLoRA, arxiv 2604.07173).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.  It
 * shares no code, header or constant with the CUDA path
 * (paper_2604_07173_b200/csrc) and must never be reached from the product.
 *
 * What it computes (the plain per-row definition; segmentation is only an
 * execution strategy of the GPU path, so it does not appear here):
 *
 *   P:165 (Sec. 2.2)  W' = W + AB,  A in R^{h x r},  B in R^{r x d},
 *                     y' = xW' = xW + xAB          (row-vector x)
 *   P:167 (Sec. 2.2)  each request computes its own xAB, "added to the base
 *                     output"
 *   P:185 (Sec. 2.3)  expert-specific A/B: the unit is (adapter a, expert e)
 *   P:233 (Fig. 4b)   "followed by a final addition of the two outputs"
 *   north_star        y += s * (x A_{a,e}) B_{a,e}; a = -1 means "no LoRA"
 *
 * For every row i whose unit u_i >= 0:
 *     v[k]   = sum_{j ascending} x[i,j] * A_u[j,k]            (fp64)
 *     d[c]   = s_i * sum_{k ascending} v[k] * B_u[k,c]        (fp64)
 *     y[i,c] = round_to_y_dtype( y[i,c] + d[c] )              (one rounding, RNE)
 * Rows with u_i < 0 are not touched (bit-identical).  Arithmetic is fp64
 * (the paper fixes no precision; reading R3), inputs are bf16 bit
 * patterns.  Each row's summation order is fixed, so the result is identical
 * for any thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static double bf16_to_double(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, sizeof f);
    return (double)f;
}

/* Round a double to the nearest bf16 (ties to even), single rounding. */
static uint16_t double_to_bf16_rne(double d) {
    if (isnan(d)) return 0x7FC0;
    uint16_t sign = signbit(d) ? 0x8000 : 0;
    double a = fabs(d);
    if (a == 0.0) return sign;
    int ex;
    (void)frexp(a, &ex);                 /* a = m * 2^ex, m in [0.5, 1) */
    int q = ex - 8;                      /* 8 significant bits: ulp = 2^(ex-8) */
    if (q < -133) q = -133;              /* bf16 subnormal quantum 2^-133 */
    double m = nearbyint(ldexp(a, -q));  /* default rounding mode: to nearest even */
    double r = ldexp(m, q);
    if (r > 3.3895313892515355e38) return (uint16_t)(sign | 0x7F80);   /* overflow -> inf */
    float f = (float)r;                  /* exact: r has <= 8 significant bits */
    uint32_t u;
    memcpy(&u, &f, sizeof u);
    return (uint16_t)(sign | ((u >> 16) & 0x7FFF));
}

/* Exposed for the tests' rounding pins. */
uint16_t oracle_round_bf16(double d) { return double_to_bf16_rne(d); }

/*
 * oracle_lora_apply
 *   T            rows
 *   x            bf16 bits [T][h_in]
 *   unit_of_row  [T]; index into A/B, or -1 for "no LoRA"
 *   scale_of_row [T]; s_a of the row's adapter
 *   A            bf16 bits [U][h_in][r]   (paper orientation)
 *   B            bf16 bits [U][r][h_out]
 *   y            [T][h_out]; bf16 bits (y_is_fp32 = 0) or fp32 (1); updated in place
 *   n_threads    OpenMP threads (<= 0: library default)
 * Returns 0, or -1 on a bad argument.
 */
int oracle_lora_apply(int64_t T, int32_t h_in, int32_t h_out, int32_t r,
                      const uint16_t *x, const int32_t *unit_of_row, const double *scale_of_row,
                      const uint16_t *A, const uint16_t *B, int64_t U,
                      void *y, int32_t y_is_fp32, int32_t n_threads) {
    if (T < 0 || h_in <= 0 || h_out <= 0 || r <= 0 || !x || !unit_of_row || !scale_of_row || !y)
        return -1;
    for (int64_t i = 0; i < T; ++i)
        if (unit_of_row[i] >= U) return -1;
#ifdef _OPENMP
    /* per-call thread count (a num_threads clause, so the library default is
       not changed for later calls) */
    const int nt = n_threads > 0 ? n_threads : omp_get_max_threads();
#else
    (void)n_threads;
#endif
    int bad = 0;
#pragma omp parallel num_threads(nt)
    {
        double *v = (double *)malloc(sizeof(double) * (size_t)r);
        double *d = (double *)malloc(sizeof(double) * (size_t)h_out);
        if (!v || !d) {
#pragma omp atomic write
            bad = 1;
        }
#pragma omp for schedule(dynamic, 1)
        for (int64_t i = 0; i < T; ++i) {
            if (!v || !d) continue;
            const int64_t u = unit_of_row[i];
            if (u < 0) continue;                               /* a = -1: untouched */
            const uint16_t *xi = x + i * (int64_t)h_in;
            const uint16_t *Au = A + u * (int64_t)h_in * r;
            const uint16_t *Bu = B + u * (int64_t)r * h_out;
            /* shrink: v = x_i A_u  (j outer, k inner: each v[k] sums j ascending) */
            for (int k = 0; k < r; ++k) v[k] = 0.0;
            for (int j = 0; j < h_in; ++j) {
                const double xj = bf16_to_double(xi[j]);
                const uint16_t *Aj = Au + (int64_t)j * r;
                for (int k = 0; k < r; ++k) v[k] += xj * bf16_to_double(Aj[k]);
            }
            /* expand: d = v B_u  (k outer, c inner) */
            for (int c = 0; c < h_out; ++c) d[c] = 0.0;
            for (int k = 0; k < r; ++k) {
                const double vk = v[k];
                const uint16_t *Bk = Bu + (int64_t)k * h_out;
                for (int c = 0; c < h_out; ++c) d[c] += vk * bf16_to_double(Bk[c]);
            }
            /* scale, then the final addition into the base output, one rounding */
            const double s = scale_of_row[i];
            if (y_is_fp32) {
                float *yi = (float *)y + i * (int64_t)h_out;
                for (int c = 0; c < h_out; ++c) yi[c] = (float)((double)yi[c] + s * d[c]);
            } else {
                uint16_t *yi = (uint16_t *)y + i * (int64_t)h_out;
                for (int c = 0; c < h_out; ++c)
                    yi[c] = double_to_bf16_rne(bf16_to_double(yi[c]) + s * d[c]);
            }
        }
        free(v);
        free(d);
    }
    return bad ? -1 : 0;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
