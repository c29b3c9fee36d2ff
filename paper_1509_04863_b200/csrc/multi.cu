// multi.cu -- Theorem 4 with alpha moduli (SURVEY 8(f)
// f4(ii)): alpha pairwise co-prime moduli M_j >= K with prod M_j > N; each
// modulus is folded / correlated / argmax-ed as in Algorithm 1 (steps 3-7) by
// two-modulus sub-plans (M, M + 1) that reuse the whole single-plan path
// (packed fold, tensor-core or NTT correlation), and steps 8-9 become Garner's
// mixed-radix CRT over the alpha residues (one thread per pair).
#include <cstdlib>
#include <cstring>

#include "tm_internal.cuh"

namespace {

constexpr int AMAX = 8;

struct Garner {
    int alpha;
    int64_t N;
    int64_t M[AMAX];
    int64_t C[AMAX];   // C_j = (M_0 ... M_{j-1})^{-1} mod M_j (j >= 1)
    // gather: residue j of pair b is src[j][b * 2 + col[j]]
    const int32_t *src[AMAX];
    int col[AMAX];
};

int64_t inv_mod64(int64_t a, int64_t m) {  // a^{-1} mod m (gcd 1), extended Euclid
    int64_t r0 = m, r1 = a % m, s0 = 0, s1 = 1;
    while (r1 != 0) {
        const int64_t qq = r0 / r1;
        int64_t t = r0 - qq * r1; r0 = r1; r1 = t;
        t = s0 - qq * s1; s0 = s1; s1 = t;
    }
    int64_t v = s0 % m;
    return v < 0 ? v + m : v;
}

int64_t gcd64(int64_t a, int64_t b) {
    while (b) { const int64_t r = a % b; a = b; b = r; }
    return a;
}

// Garner: z = t_0 + t_1 M_0 + t_2 M_0 M_1 + ..., t_j = (m_j - (t_0 + ... )) C_j mod M_j
// (the partial sum reduced mod M_j by Horner); k = z if z < N, evaluated from
// the top digit with an overflow-free comparison, else -1.
__global__ void garner_kernel(Garner g, int64_t batch, int32_t *residues_out, int64_t *k) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= batch) return;
    int64_t m[AMAX], t[AMAX];
#pragma unroll
    for (int j = 0; j < AMAX; ++j) {
        if (j >= g.alpha) break;
        m[j] = g.src[j][g.col[j] >= 0 ? b * 2 + g.col[j] : b * g.alpha + j];
        if (residues_out) residues_out[b * g.alpha + j] = (int32_t)m[j];
    }
    t[0] = m[0];
#pragma unroll
    for (int j = 1; j < AMAX; ++j) {
        if (j >= g.alpha) break;
        const int64_t Mj = g.M[j];
        int64_t s = t[j - 1] % Mj;
        for (int i = j - 2; i >= 0; --i) s = (s * (g.M[i] % Mj) + t[i]) % Mj;
        int64_t d = (m[j] - s) % Mj;
        if (d < 0) d += Mj;
        t[j] = (d * g.C[j]) % Mj;
    }
    // z = (((t_{a-1}) M_{a-2} + t_{a-2}) M_{a-3} + ...) M_0 + t_0, stop once >= N
    int64_t z = t[g.alpha - 1];
    bool big = false;
    for (int i = g.alpha - 2; i >= 0; --i) {
        if (z > (g.N - t[i]) / g.M[i]) { big = true; break; }   // z M_i + t_i >= N
        z = z * g.M[i] + t[i];
    }
    k[b] = (big || z >= g.N) ? -1 : z;
}

int check_moduli(int64_t N, int64_t K, const int64_t *M, int alpha, const char *who) {
    if (!M || alpha < 2 || alpha > AMAX) { tm_set_error("%s: need 2 <= alpha <= %d moduli", who, AMAX); return TM_EINVAL; }
    __int128 P = 1;
    for (int j = 0; j < alpha; ++j) {
        if (M[j] < K || M[j] < 2 || M[j] >= (int64_t(1) << 31)) {
            tm_set_error("%s: modulus %lld outside [max(K, 2), 2^31)", who, (long long)M[j]);
            return TM_EINVAL;
        }
        for (int i = 0; i < j; ++i)
            if (gcd64(M[i], M[j]) != 1) {
                tm_set_error("%s: moduli %lld and %lld are not co-prime (Theorem 4)", who, (long long)M[i],
                             (long long)M[j]);
                return TM_EINVAL;
            }
        P *= M[j];
        if (P > ((__int128)1 << 100)) P = (__int128)1 << 100;
    }
    if (P <= (__int128)N) { tm_set_error("%s: prod M_j <= N (Theorem 4 needs prod M_j > N)", who); return TM_EINVAL; }
    return TM_OK;
}

void fill_garner(Garner &g, int64_t N, const int64_t *M, int alpha) {
    g.alpha = alpha; g.N = N;
    for (int j = 0; j < alpha; ++j) {
        g.M[j] = M[j];
        int64_t P = 1;  // prod_{i<j} M_i mod M_j
        for (int i = 0; i < j; ++i) P = (P * (M[i] % M[j])) % M[j];
        g.C[j] = j ? inv_mod64(P, M[j]) : 0;
    }
}

}  // namespace

struct tm_mplan_s {
    int64_t N, K;
    int alpha, nsub;
    int64_t M[AMAX];
    tm_plan sub[AMAX];
    int sub_of[AMAX], col_of[AMAX];  // modulus j -> (sub-plan, residue column)
};

extern "C" __attribute__((visibility("default"))) int tm_mplan_create(tm_mplan *out, int64_t N, int64_t K,
                                                                      const int64_t *moduli, int alpha,
                                                                      uint64_t seed, int dtype, uint32_t flags) {
    if (!out) { tm_set_error("tm_mplan_create: out is NULL"); return TM_EINVAL; }
    *out = nullptr;
    if (N < 1 || K < 1) { tm_set_error("tm_mplan_create: N, K must be >= 1"); return TM_EINVAL; }
    if (flags & TM_ALIAS_REPAIR) { tm_set_error("tm_mplan_create: TM_ALIAS_REPAIR needs alpha = 2"); return TM_EINVAL; }
    int rc = check_moduli(N, K, moduli, alpha, "tm_mplan_create");
    if (rc) return rc;
    tm_mplan_s *p = (tm_mplan_s *)calloc(1, sizeof(tm_mplan_s));
    if (!p) { tm_set_error("tm_mplan_create: out of host memory"); return TM_EINVAL; }
    p->N = N; p->K = K; p->alpha = alpha;
    for (int j = 0; j < alpha; ++j) { p->M[j] = moduli[j]; p->sub_of[j] = -1; }
    for (int j = 0; j < alpha; ++j) {
        if (p->sub_of[j] >= 0) continue;
        // sub-plan (M_j, M_j + 1); if M_j + 1 is also a modulus it is served too
        const int s = p->nsub++;
        rc = tm_plan_create_impl(&p->sub[s], N, K, moduli[j], seed, dtype, flags, 0);
        if (rc) { tm_mplan_destroy(p); return rc; }
        p->sub_of[j] = s; p->col_of[j] = 0;
        for (int i = 0; i < alpha; ++i)
            if (p->sub_of[i] < 0 && moduli[i] == moduli[j] + 1) { p->sub_of[i] = s; p->col_of[i] = 1; }
    }
    *out = p;
    return TM_OK;
}

// workspace: [the largest sub-plan run workspace][nsub x batch x 2 int32 residues][batch int64 k]
extern "C" __attribute__((visibility("default"))) size_t tm_mplan_workspace_bytes(tm_mplan p, int64_t batch) {
    if (!p || batch < 0) return 0;
    size_t w = 0;
    for (int s = 0; s < p->nsub; ++s) {
        const size_t v = tm_workspace_bytes(p->sub[s], batch);
        if (v > w) w = v;
    }
    w = (w + 255) & ~size_t(255);
    return w + (size_t)p->nsub * batch * 8 + 256 + (size_t)batch * 8 + 256;
}

extern "C" __attribute__((visibility("default"))) int tm_mplan_run(tm_mplan p, const void *x, int64_t ldx,
                                                                   const void *t, int64_t batch, int32_t *residues,
                                                                   int64_t *k, void *ws, void *stream) {
    if (!p) { tm_set_error("tm_mplan_run: NULL plan"); return TM_EINVAL; }
    if (batch < 0) { tm_set_error("tm_mplan_run: batch < 0"); return TM_EINVAL; }
    if (batch == 0) return TM_OK;
    if (!x || !t || !k || !ws) { tm_set_error("tm_mplan_run: NULL pointer"); return TM_EINVAL; }
    size_t w = 0;
    for (int s = 0; s < p->nsub; ++s) {
        const size_t v = tm_workspace_bytes(p->sub[s], batch);
        if (v > w) w = v;
    }
    w = (w + 255) & ~size_t(255);
    int32_t *res_sub = (int32_t *)((char *)ws + w);
    int64_t *k_sub = (int64_t *)((char *)ws + w + (((size_t)p->nsub * batch * 8 + 255) & ~size_t(255)));
    for (int s = 0; s < p->nsub; ++s) {  // steps 3-7 for each pair of moduli (its own k is discarded)
        const int rc = tm_run(p->sub[s], x, ldx, t, batch, res_sub + (size_t)s * batch * 2, k_sub, ws, stream);
        if (rc) return rc;
    }
    Garner g{};
    fill_garner(g, p->N, p->M, p->alpha);
    for (int j = 0; j < p->alpha; ++j) {
        g.src[j] = res_sub + (size_t)p->sub_of[j] * batch * 2;
        g.col[j] = p->col_of[j];
    }
    garner_kernel<<<(unsigned)((batch + 127) / 128), 128, 0, (cudaStream_t)stream>>>(g, batch, residues, k);
    TM_CHECK_LAUNCH("tm_mplan_run: garner_kernel");
    return TM_OK;
}

extern "C" __attribute__((visibility("default"))) int tm_crt_multi(const int32_t *residues, int64_t batch, int alpha,
                                                                   const int64_t *moduli, int64_t N, int64_t *k,
                                                                   void *stream) {
    if (batch < 0 || N < 1) { tm_set_error("tm_crt_multi: bad batch or N"); return TM_EINVAL; }
    int rc = check_moduli(N, 1, moduli, alpha, "tm_crt_multi");
    if (rc) return rc;
    if (batch == 0) return TM_OK;
    if (!residues || !k) { tm_set_error("tm_crt_multi: NULL pointer"); return TM_EINVAL; }
    Garner g{};
    fill_garner(g, N, moduli, alpha);
    for (int j = 0; j < alpha; ++j) { g.src[j] = residues; g.col[j] = -1; }
    garner_kernel<<<(unsigned)((batch + 127) / 128), 128, 0, (cudaStream_t)stream>>>(g, batch, nullptr, k);
    TM_CHECK_LAUNCH("tm_crt_multi: garner_kernel");
    return TM_OK;
}

extern "C" __attribute__((visibility("default"))) void tm_mplan_destroy(tm_mplan p) {
    if (!p) return;
    for (int s = 0; s < p->nsub; ++s) tm_plan_destroy(p->sub[s]);
    free(p);
}
