/* A plain-C consumer of the C ABI (include/epk/epk.h): no C++, no torch --
 * what an FFI binding (cgo, JNI, ctypes) sees.  One bf16 block step of a
 * 2-layer, 4-head cache through epk_evict_step (tensor-core scorer, fused
 * selection, compaction into a second cache), then the invariants the
 * reference guarantees: every layer keeps exactly min(live, H * budget)
 * entries, each head's kept positions stay sorted, and every kept position
 * existed in the input.  Prints "abi_c_step ok" on success.
 *
 * Build: tests/cpp/Makefile (gcc, -lepk -lcudart); run by
 * tests/test_gpu_cpp_dropin.py. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "epk/epk.h"

#define CHECK(x)                                                                           \
    do {                                                                                   \
        int rc_ = (x);                                                                     \
        if (rc_ != 0) {                                                                    \
            fprintf(stderr, "%s:%d: %s -> %d (%s)\n", __FILE__, __LINE__, #x, rc_, epk_last_error()); \
            return 1;                                                                      \
        }                                                                                  \
    } while (0)
#define CUCHECK(x)                                                                          \
    do {                                                                                    \
        cudaError_t e_ = (x);                                                               \
        if (e_ != cudaSuccess) {                                                            \
            fprintf(stderr, "%s:%d: %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            return 1;                                                                       \
        }                                                                                   \
    } while (0)

enum { L = 2, H = 4, HQ = 12, D = 128, P = 16, N = 300, BUDGET = 200, SLACK = 8 };

static uint16_t bf16(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    return (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}

static uint32_t rng_state = 12345u;
static float frand(void) {
    rng_state = rng_state * 1664525u + 1013904223u;
    return ((float)(rng_state >> 8) / 16777216.0f) * 2.0f - 1.0f;
}

int main(void) {
    const int64_t cap = (int64_t)H * (N + SLACK);
    const int64_t rows = (int64_t)L * cap;
    int64_t base[L + 1];
    for (int l = 0; l <= L; ++l) base[l] = l * cap;

    /* host data: every head holds N entries at positions 0..N-1 */
    uint16_t* hk = malloc(sizeof(uint16_t) * rows * D);
    int32_t* hpos = malloc(sizeof(int32_t) * rows);
    int32_t hoff[L][H + 1], hlen[L][H];
    for (int64_t i = 0; i < rows * D; ++i) hk[i] = bf16(frand());
    for (int l = 0; l < L; ++l)
        for (int h = 0; h <= H; ++h) {
            hoff[l][h] = h * (N + SLACK);
            if (h < H) hlen[l][h] = N;
        }
    for (int64_t r = 0; r < rows; ++r) hpos[r] = (int32_t)((r % cap) % (N + SLACK));
    uint16_t* hq = malloc(sizeof(uint16_t) * L * HQ * P * D);
    uint16_t* hkp = malloc(sizeof(uint16_t) * L * H * P * D);
    for (int i = 0; i < L * HQ * P * D; ++i) hq[i] = bf16(frand());
    for (int i = 0; i < L * H * P * D; ++i) hkp[i] = bf16(frand());

    void *k_in, *v_in, *k_out, *v_out, *q, *kp;
    int32_t *pos_in, *pos_out, *off_in, *off_out, *len_in, *len_out, *kept;
    CUCHECK(cudaMalloc(&k_in, rows * D * 2));
    CUCHECK(cudaMalloc(&v_in, rows * D * 2));
    CUCHECK(cudaMalloc(&k_out, rows * D * 2));
    CUCHECK(cudaMalloc(&v_out, rows * D * 2));
    CUCHECK(cudaMalloc(&q, (size_t)L * HQ * P * D * 2));
    CUCHECK(cudaMalloc(&kp, (size_t)L * H * P * D * 2));
    CUCHECK(cudaMalloc((void**)&pos_in, rows * 4));
    CUCHECK(cudaMalloc((void**)&pos_out, rows * 4));
    CUCHECK(cudaMalloc((void**)&off_in, sizeof hoff));
    CUCHECK(cudaMalloc((void**)&off_out, sizeof hoff));
    CUCHECK(cudaMalloc((void**)&len_in, sizeof hlen));
    CUCHECK(cudaMalloc((void**)&len_out, sizeof hlen));
    CUCHECK(cudaMalloc((void**)&kept, L * 4));
    CUCHECK(cudaMemcpy(k_in, hk, rows * D * 2, cudaMemcpyHostToDevice));
    CUCHECK(cudaMemcpy(v_in, hk, rows * D * 2, cudaMemcpyHostToDevice));
    CUCHECK(cudaMemcpy(q, hq, (size_t)L * HQ * P * D * 2, cudaMemcpyHostToDevice));
    CUCHECK(cudaMemcpy(kp, hkp, (size_t)L * H * P * D * 2, cudaMemcpyHostToDevice));
    CUCHECK(cudaMemcpy(pos_in, hpos, rows * 4, cudaMemcpyHostToDevice));
    CUCHECK(cudaMemcpy(off_in, hoff, sizeof hoff, cudaMemcpyHostToDevice));
    CUCHECK(cudaMemcpy(len_in, hlen, sizeof hlen, cudaMemcpyHostToDevice));

    epk_cache_desc in = {L, H, D, EPK_BF16, k_in, v_in, pos_in, off_in, len_in, base};
    epk_cache_desc out = {L, H, D, EPK_BF16, k_out, v_out, pos_out, off_out, len_out, base};
    const int64_t budgets[L] = {BUDGET, BUDGET / 2};

    epk_ctx* ctx = NULL;
    CHECK(epk_ctx_create(0, NULL, &ctx));
    CHECK(epk_evict_step(ctx, &in, &out, q, kp, HQ, P, budgets, NULL, 0, EPK_AGG_MAX, EPK_SCORE_TC_BF16, N, SLACK,
                         NULL, kept));
    CHECK(epk_ctx_synchronize(ctx));
    CHECK(epk_ctx_poll_error(ctx));

    int32_t hkept[L], ooff[L][H + 1], olen[L][H];
    int32_t* opos = malloc(sizeof(int32_t) * rows);
    CUCHECK(cudaMemcpy(hkept, kept, sizeof hkept, cudaMemcpyDeviceToHost));
    CUCHECK(cudaMemcpy(ooff, off_out, sizeof ooff, cudaMemcpyDeviceToHost));
    CUCHECK(cudaMemcpy(olen, len_out, sizeof olen, cudaMemcpyDeviceToHost));
    CUCHECK(cudaMemcpy(opos, pos_out, rows * 4, cudaMemcpyDeviceToHost));
    for (int l = 0; l < L; ++l) {
        const int want = (H * N < H * (int)budgets[l]) ? H * N : H * (int)budgets[l];
        int total = 0;
        for (int h = 0; h < H; ++h) {
            total += olen[l][h];
            for (int i = 0; i < olen[l][h]; ++i) {
                const int32_t p = opos[base[l] + ooff[l][h] + i];
                if (p < 0 || p >= N || (i > 0 && p <= opos[base[l] + ooff[l][h] + i - 1])) {
                    fprintf(stderr, "layer %d head %d: bad kept position order\n", l, h);
                    return 1;
                }
            }
        }
        if (total != want || hkept[l] != want) {
            fprintf(stderr, "layer %d: kept %d / %d, want %d\n", l, total, hkept[l], want);
            return 1;
        }
    }
    CHECK(epk_ctx_destroy(ctx));
    printf("abi_c_step ok\n");
    return 0;
}
