// Bring-up self-test for the tcgen05 PPMM kernel (not the parity suite):
// random centred digit planes, GPU result vs a host loop on sampled rows,
// plus a timed full-size launch. Prints mismatch structure for debugging.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "../../paper_2601_17561_b200/csrc/ppmm.h"

using namespace irl;

#define CK(x)                                                                        \
    do {                                                                             \
        cudaError_t e_ = (x);                                                        \
        if (e_ != cudaSuccess) {                                                     \
            std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, \
                        __LINE__);                                                   \
            std::exit(2);                                                            \
        }                                                                            \
    } while (0)

static const uint32_t kPrimes[24] = {127, 131, 137, 139, 149, 151, 157, 163, 167, 173, 179, 181,
                                     191, 193, 197, 199, 211, 223, 227, 229, 233, 239, 241, 251};

static int run_case(uint32_t parts, uint32_t nprimes, uint32_t M, uint32_t N, uint32_t K,
                    int sample_rows, int timed_iters) {
    const uint32_t ldk = (K + 15) / 16 * 16;
    const size_t a_elems = (size_t)parts * nprimes * 2 * M * ldk;
    const size_t b_elems = (size_t)nprimes * 2 * N * ldk;
    const size_t o_elems = (size_t)parts * nprimes * N * M;
    std::vector<int8_t> ha(a_elems), hb(b_elems);
    std::mt19937_64 rng(1234 + M + N + K);
    for (uint32_t g = 0; g < parts; ++g)
        for (uint32_t i = 0; i < nprimes; ++i) {
            const int half = (kPrimes[i] - 1) / 2;
            for (int d = 0; d < 2; ++d)
                for (uint32_t r = 0; r < M; ++r) {
                    int8_t* row = &ha[((((size_t)g * nprimes + i) * 2 + d) * M + r) * ldk];
                    for (uint32_t k = 0; k < ldk; ++k)
                        row[k] = k < K ? (int8_t)((int)(rng() % (2 * half + 1)) - half) : 0;
                }
        }
    for (uint32_t i = 0; i < nprimes; ++i) {
        const int half = (kPrimes[i] - 1) / 2;
        for (int d = 0; d < 2; ++d)
            for (uint32_t r = 0; r < N; ++r) {
                int8_t* row = &hb[(((size_t)i * 2 + d) * N + r) * ldk];
                for (uint32_t k = 0; k < ldk; ++k)
                    row[k] = k < K ? (int8_t)((int)(rng() % (2 * half + 1)) - half) : 0;
            }
    }
    int8_t *da, *db;
    uint16_t* dout;
    CK(cudaMalloc(&da, a_elems));
    CK(cudaMalloc(&db, b_elems));
    CK(cudaMalloc(&dout, o_elems * 2));
    CK(cudaMemcpy(da, ha.data(), a_elems, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(db, hb.data(), b_elems, cudaMemcpyHostToDevice));
    CK(cudaMemset(dout, 0xFF, o_elems * 2));

    PpmmLaunch L;
    L.a_planes = da;
    L.b_planes = db;
    L.out = dout;
    L.M = M;
    L.N = N;
    L.K = K;
    L.ldk = ldk;
    L.parts = parts;
    L.nprimes = nprimes;
    uint32_t* prog = nullptr;
    CK(cudaMalloc(&prog, kScheduleScratchBytes));
    L.progress = prog;
    for (uint32_t i = 0; i < nprimes; ++i) L.mc[i] = make_modconst(kPrimes[i], 2);
    CK(launch_ppmm_planes(L, 0));
    CK(cudaDeviceSynchronize());
    std::vector<uint16_t> hout(o_elems);
    CK(cudaMemcpy(hout.data(), dout, o_elems * 2, cudaMemcpyDeviceToHost));

    // Host check on sampled rows (all rows if sample_rows <= 0).
    long bad = 0, checked = 0;
    int printed = 0;
    std::vector<uint32_t> rows;
    if (sample_rows <= 0 || (uint32_t)sample_rows >= M) {
        for (uint32_t r = 0; r < M; ++r) rows.push_back(r);
    } else {
        for (int s = 0; s < sample_rows; ++s) rows.push_back((uint32_t)(rng() % M));
        rows.push_back(0);
        rows.push_back(M - 1);
    }
    for (uint32_t g = 0; g < parts; ++g)
        for (uint32_t i = 0; i < nprimes; ++i) {
            const int64_t p = kPrimes[i], p2 = p * p;
            for (uint32_t r : rows) {
                const int8_t* x0 = &ha[((((size_t)g * nprimes + i) * 2 + 0) * M + r) * ldk];
                const int8_t* x1 = &ha[((((size_t)g * nprimes + i) * 2 + 1) * M + r) * ldk];
                for (uint32_t n = 0; n < N; ++n) {
                    const int8_t* y0 = &hb[(((size_t)i * 2 + 0) * N + n) * ldk];
                    const int8_t* y1 = &hb[(((size_t)i * 2 + 1) * N + n) * ldk];
                    int64_t t00 = 0, t01 = 0, t10 = 0;
                    for (uint32_t k = 0; k < K; ++k) {
                        t00 += x0[k] * y0[k];
                        t01 += x0[k] * y1[k];
                        t10 += x1[k] * y0[k];
                    }
                    int64_t v = (t00 + p * (t01 + t10)) % p2;
                    if (v < 0) v += p2;
                    const uint16_t got = hout[(((size_t)g * nprimes + i) * N + n) * M + r];
                    ++checked;
                    if (got != v) {
                        ++bad;
                        if (printed < 12) {
                            std::printf("  mismatch part %u prime %u row %u col %u: got %u want %lld"
                                        " (t00 %lld t01 %lld t10 %lld)\n",
                                        g, i, r, n, got, (long long)v, (long long)t00,
                                        (long long)t01, (long long)t10);
                            ++printed;
                        }
                    }
                }
            }
        }
    std::printf("case parts=%u primes=%u M=%u N=%u K=%u: %ld / %ld mismatches\n", parts, nprimes, M,
                N, K, bad, checked);

    if (timed_iters > 0) {
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        for (int w = 0; w < 2; ++w) CK(launch_ppmm_planes(L, 0));
        CK(cudaEventRecord(e0));
        for (int it = 0; it < timed_iters; ++it) CK(launch_ppmm_planes(L, 0));
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        ms /= timed_iters;
        const double ops = 6.0 * parts * nprimes * (double)M * N * K;
        std::printf("  timed: %.3f ms/launch, %.1f TOPS (int8-op equiv, 6PMNK)\n", ms,
                    ops / (ms * 1e-3) / 1e12);
    }
    CK(cudaFree(da));
    CK(cudaFree(db));
    CK(cudaFree(dout));
    CK(cudaFree(prog));
    return bad == 0 ? 0 : 1;
}

int main(int argc, char** argv) {
    int fails = 0;
    fails += run_case(1, 1, 256, 256, 128, 0, 0);
    fails += run_case(1, 2, 256, 256, 1024, 0, 0);
    fails += run_case(2, 3, 512, 992, 2048, 0, 0);
    fails += run_case(1, 2, 300, 200, 1000, 0, 0);   // ragged M, N, K
    fails += run_case(1, 1, 16384, 992, 24576, 16, 5);
    if (argc > 1 && std::strcmp(argv[1], "big") == 0)
        fails += run_case(1, 24, 16384, 992, 24576, 2, 3);
    std::printf(fails ? "SELFTEST FAIL\n" : "SELFTEST PASS\n");
    return fails ? 1 : 0;
}
