/*
 * tmgen.c -- seeded, counter-based synthetic input generator (host side).
 *
 * This module holds NONE of the method's arithmetic: it only draws the
 * paper's synthetic workload (section 3.5):
 *   x in {+1,-1}^N i.i.d. equiprobable (or x ~ N(0,1) in fp32),
 *   k0 uniform in [0, N)               (reading C18),
 *   t = [x_{k0}, ..., x_{k0+K-1}] (mod N) with independent bit flips
 *       (int8) or additive N(0, sigma^2) noise (fp32).
 * It is shared by tests (host inputs for the oracle and the GPU) and is
 * re-implemented, bit-for-bit for the integer outputs, by the device
 * generator tm_generate() in paper_1509_04863_b200/csrc (DESIGN.md
 * "Input recipe").  Neither side calls the other.
 *
 * Definition (both sides):
 *   mix64(z)        SplitMix64 finaliser
 *   key(seed, b)    = mix64(mix64(seed) + (b + 1) * 0x9E3779B97F4A7C15)
 *   H(seed, b, c)   = mix64(key(seed, b) ^ (c * 0xD1B54A32D192ED03))
 *   x_i   (int8)    = 1 - 2 * bit (i mod 64) of H(seed, b, i / 64)
 *   x_i   (fp32)    = gauss(H(seed, b, i))
 *   k0              = floor(H(seed, b, TAG_K0) * N / 2^64)
 *   flip_j          = (H(seed, b, TAG_FLIP + j) mod 2^32) < round(p * 2^32)
 *   tnoise_j        = gauss(H(seed, b, TAG_TNOISE + j))
 *   gauss(h)        = sqrt(-2 ln u1) cos(2 pi u2),
 *                     u1 = ((h >> 40) + 1) / 2^24,  u2 = (h mod 2^24) / 2^24
 */
#include <math.h>
#include <stdint.h>

#define TG_TAG_K0     0x4000000000000000ULL
#define TG_TAG_FLIP   0x5000000000000000ULL
#define TG_TAG_TNOISE 0x6000000000000000ULL
#define TG_TAG_XNOISE 0x7000000000000000ULL

static uint64_t mix64(uint64_t z) {
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27; z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}

uint64_t tg_key(uint64_t seed, uint64_t pair) {
    return mix64(mix64(seed) + (pair + 1ULL) * 0x9E3779B97F4A7C15ULL);
}

uint64_t tg_hash(uint64_t seed, uint64_t pair, uint64_t ctr) {
    return mix64(tg_key(seed, pair) ^ (ctr * 0xD1B54A32D192ED03ULL));
}

static uint64_t hk(uint64_t key, uint64_t ctr) { return mix64(key ^ (ctr * 0xD1B54A32D192ED03ULL)); }

double tg_gauss(uint64_t h) {
    double u1 = (double)((h >> 40) + 1ULL) * (1.0 / 16777216.0);
    double u2 = (double)(h & 0xFFFFFFULL) * (1.0 / 16777216.0);
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
}

int64_t tg_k0(uint64_t seed, uint64_t pair, int64_t N) {
    uint64_t h = tg_hash(seed, pair, TG_TAG_K0);
    return (int64_t)(((unsigned __int128)h * (unsigned __int128)(uint64_t)N) >> 64);
}

static int8_t x_i8_at(uint64_t key, int64_t i) {
    uint64_t h = hk(key, (uint64_t)i >> 6);
    return (int8_t)(1 - 2 * (int)((h >> (i & 63)) & 1ULL));
}

/* x[lo .. lo+len) of pair `pair` */
void tg_x_i8(uint64_t seed, uint64_t pair, int64_t lo, int64_t len, int8_t *out) {
    uint64_t key = tg_key(seed, pair);
    int64_t i = lo, end = lo + len;
    while (i < end) {
        uint64_t h = hk(key, (uint64_t)i >> 6);
        int64_t stop = ((i >> 6) + 1) << 6;
        if (stop > end) stop = end;
        for (; i < stop; ++i) out[i - lo] = (int8_t)(1 - 2 * (int)((h >> (i & 63)) & 1ULL));
    }
}

void tg_x_f32(uint64_t seed, uint64_t pair, int64_t lo, int64_t len, float *out) {
    uint64_t key = tg_key(seed, pair);
    for (int64_t i = 0; i < len; ++i) out[i] = (float)tg_gauss(hk(key, (uint64_t)(lo + i)));
}

static uint64_t flip_threshold(double p) {
    if (p <= 0.0) return 0ULL;
    if (p >= 1.0) return 1ULL << 32;
    return (uint64_t)llround(p * 4294967296.0);
}

/* t[j] = x[(k0 + j) mod N] * (flip_j ? -1 : +1),  j < K */
void tg_t_i8(uint64_t seed, uint64_t pair, int64_t N, int64_t K, double flip_p, int8_t *t) {
    uint64_t key = tg_key(seed, pair);
    int64_t k0 = tg_k0(seed, pair, N);
    uint64_t thr = flip_threshold(flip_p);
    for (int64_t j = 0; j < K; ++j) {
        int64_t pos = (k0 + j) % N;
        int8_t v = x_i8_at(key, pos);
        uint64_t f = hk(key, TG_TAG_FLIP + (uint64_t)j) & 0xFFFFFFFFULL;
        t[j] = (f < thr) ? (int8_t)(-v) : v;
    }
}

/* t[j] = x[(k0 + j) mod N] + sigma * tnoise_j  (fp32 data) */
void tg_t_f32(uint64_t seed, uint64_t pair, int64_t N, int64_t K, double sigma, float *t) {
    uint64_t key = tg_key(seed, pair);
    int64_t k0 = tg_k0(seed, pair, N);
    for (int64_t j = 0; j < K; ++j) {
        int64_t pos = (k0 + j) % N;
        double xv = (double)(float)tg_gauss(hk(key, (uint64_t)pos));
        double v = xv + sigma * tg_gauss(hk(key, TG_TAG_TNOISE + (uint64_t)j));
        t[j] = (float)v;
    }
}

/* batch helpers: pairs [pair0, pair0 + B), x rows of stride ldx */
void tg_batch_i8(uint64_t seed, uint64_t pair0, int64_t B, int64_t N, int64_t K, double flip_p,
                 int8_t *x, int64_t ldx, int8_t *t, int64_t *k0) {
    for (int64_t b = 0; b < B; ++b) {
        if (x) tg_x_i8(seed, pair0 + b, 0, N, x + b * ldx);
        if (t) tg_t_i8(seed, pair0 + b, N, K, flip_p, t + b * K);
        if (k0) k0[b] = tg_k0(seed, pair0 + b, N);
    }
}

void tg_batch_f32(uint64_t seed, uint64_t pair0, int64_t B, int64_t N, int64_t K, double sigma,
                  float *x, int64_t ldx, float *t, int64_t *k0) {
    for (int64_t b = 0; b < B; ++b) {
        if (x) tg_x_f32(seed, pair0 + b, 0, N, x + b * ldx);
        if (t) tg_t_f32(seed, pair0 + b, N, K, sigma, t + b * K);
        if (k0) k0[b] = tg_k0(seed, pair0 + b, N);
    }
}
