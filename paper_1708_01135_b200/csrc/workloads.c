/*
 * Synthetic-input generator for the BASELINE.json "random charged gas"
 * workload (config 4): N positions uniform in a cubic periodic box with a
 * hard-core minimum pair distance under the minimum-image convention,
 * placed by random sequential adsorption on a hash grid.
 *
 * This is harness code (input generation), not part of the Ewald hot path.
 * Deterministic for a given seed: xoshiro256** seeded through splitmix64.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static uint64_t splitmix64(uint64_t *x) {
    uint64_t z = (*x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

typedef struct { uint64_t s[4]; } rng_t;

static uint64_t rng_next(rng_t *r) {
    uint64_t *s = r->s;
    uint64_t result = rotl(s[1] * 5, 7) * 9;
    uint64_t t = s[1] << 17;
    s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3];
    s[2] ^= t; s[3] = rotl(s[3], 45);
    return result;
}

static double rng_uniform(rng_t *r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }

static double min_image(double d, double L) { return d - L * floor(d / L + 0.5); }

/* Returns 0 on success, 1 on bad arguments, 2 if max_attempts was exceeded. */
int ewb_gen_hardcore_gas(int64_t n, double L, double min_sep, uint64_t seed,
                         int64_t max_attempts, double *pos_out,
                         int64_t *attempts_out) {
    if (n < 1 || !(L > 0.0) || !(min_sep >= 0.0)) return 1;
    rng_t rng;
    uint64_t sm = seed;
    for (int i = 0; i < 4; ++i) rng.s[i] = splitmix64(&sm);

    int ng = (min_sep > 0.0) ? (int)floor(L / min_sep) : 1;
    if (ng < 1) ng = 1;
    if (ng > 1024) ng = 1024;
    const int brute = ng < 3;
    const double edge = L / ng;
    const int cap = 16;
    int64_t ncell = (int64_t)ng * ng * ng;
    int32_t *cnt = brute ? NULL : (int32_t *)calloc((size_t)ncell, sizeof(int32_t));
    int64_t *mem = brute ? NULL : (int64_t *)malloc((size_t)ncell * cap * sizeof(int64_t));
    if (!brute && (!cnt || !mem)) { free(cnt); free(mem); return 1; }

    const double s2 = min_sep * min_sep;
    int64_t placed = 0, attempts = 0;
    while (placed < n) {
        if (attempts >= max_attempts) { free(cnt); free(mem); if (attempts_out) *attempts_out = attempts; return 2; }
        ++attempts;
        double c[3];
        for (int a = 0; a < 3; ++a) {
            c[a] = rng_uniform(&rng) * L;
            if (c[a] >= L) c[a] = 0.0;
        }
        int ok = 1;
        if (brute) {
            for (int64_t j = 0; j < placed && ok; ++j) {
                double dx = min_image(pos_out[3 * j] - c[0], L);
                double dy = min_image(pos_out[3 * j + 1] - c[1], L);
                double dz = min_image(pos_out[3 * j + 2] - c[2], L);
                if (dx * dx + dy * dy + dz * dz < s2) ok = 0;
            }
        } else {
            int ci[3];
            for (int a = 0; a < 3; ++a) {
                ci[a] = (int)floor(c[a] / edge);
                if (ci[a] < 0) ci[a] = 0;
                if (ci[a] >= ng) ci[a] = ng - 1;
            }
            for (int oz = -1; oz <= 1 && ok; ++oz)
                for (int oy = -1; oy <= 1 && ok; ++oy)
                    for (int ox = -1; ox <= 1 && ok; ++ox) {
                        int nx = (ci[0] + ox + ng) % ng, ny = (ci[1] + oy + ng) % ng,
                            nz = (ci[2] + oz + ng) % ng;
                        int64_t cell = nx + (int64_t)ng * (ny + (int64_t)ng * nz);
                        for (int k = 0; k < cnt[cell]; ++k) {
                            int64_t j = mem[cell * cap + k];
                            double dx = min_image(pos_out[3 * j] - c[0], L);
                            double dy = min_image(pos_out[3 * j + 1] - c[1], L);
                            double dz = min_image(pos_out[3 * j + 2] - c[2], L);
                            if (dx * dx + dy * dy + dz * dz < s2) { ok = 0; break; }
                        }
                    }
            if (ok) {
                int64_t cell = ci[0] + (int64_t)ng * (ci[1] + (int64_t)ng * ci[2]);
                if (cnt[cell] >= cap) ok = 0; /* cannot happen with edge >= min_sep */
                else mem[cell * cap + cnt[cell]++] = placed;
            }
        }
        if (ok) {
            memcpy(pos_out + 3 * placed, c, sizeof c);
            ++placed;
        }
    }
    free(cnt);
    free(mem);
    if (attempts_out) *attempts_out = attempts;
    return 0;
}
