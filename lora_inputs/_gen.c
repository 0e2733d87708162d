/*
 * _gen.c -- C implementation of lora_inputs' counter-based generator (inputs
 * only; no arithmetic of the method).  Same recipe as lora_inputs/__init__.py:
 *     base  = mix64(seed*G ^ tag*T ^ major*M)
 *     h     = mix64(base + minor*G)
 *     value = ((h >> 56) - 128) * 2^-shift     -> bf16 bits
 * Used to regenerate large touched-unit weight sets quickly for the oracle;
 * tests pin it bit-for-bit against the numpy implementation.
 */
#include <stdint.h>
#include <string.h>

static uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static uint16_t bits_of(uint64_t base, uint64_t minor, float scale) {
    uint64_t h = mix64(base + minor * 0x9E3779B97F4A7C15ull);
    int q = (int)(h >> 56) - 128;
    float f = (float)q * scale;
    uint32_t u;
    memcpy(&u, &f, 4);
    return (uint16_t)(u >> 16);
}

/* out[i][m] for majors[i] (i < n_major), minor m in [0, n_minor) */
void gen_bf16_rows(uint64_t seed, uint32_t tag, const uint64_t *majors, int64_t n_major, int64_t n_minor,
                   int32_t shift, uint16_t *out) {
    float scale = 1.0f;
    for (int i = 0; i < shift; ++i) scale *= 0.5f;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n_major; ++i) {
        uint64_t base = mix64(seed * 0x9E3779B97F4A7C15ull ^ (uint64_t)tag * 0xD1B54A32D192ED03ull ^
                              majors[i] * 0xC2B2AE3D27D4EB4Full);
        uint16_t *o = out + i * n_minor;
        for (int64_t m = 0; m < n_minor; ++m) o[m] = bits_of(base, (uint64_t)m, scale);
    }
}
