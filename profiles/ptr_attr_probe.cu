#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
int main() {
    cudaFree(0);
    size_t n = 64 << 20;
    char* pg = (char*)malloc(n); memset(pg, 1, n);
    char* pin; cudaMallocHost(&pin, n);
    char* dev; cudaMalloc(&dev, n);
    const char* names[3] = {"pageable", "pinned", "device"};
    char* ptrs[3] = {pg + 12345, pin + 12345, dev + 12345};
    for (int k = 0; k < 3; ++k) {
        auto t0 = std::chrono::steady_clock::now();
        int type = -1;
        for (int i = 0; i < 1000; ++i) { cudaPointerAttributes a; cudaPointerGetAttributes(&a, ptrs[k]); type = a.type; }
        auto t1 = std::chrono::steady_clock::now();
        printf("%s: %.2f us per call (type %d)\n", names[k], std::chrono::duration<double, std::micro>(t1 - t0).count() / 1000, type);
    }
    // pageable D2H memcpyAsync of 7.3 MB vs pinned
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    for (size_t b : {size_t(4) << 20, size_t(7300000), size_t(29) << 20}) {
        for (int k = 0; k < 2; ++k) {
            char* dst = k ? pin : pg;
            cudaMemcpyAsync(dst, dev, b, cudaMemcpyDeviceToHost, s); cudaStreamSynchronize(s);
            auto t0 = std::chrono::steady_clock::now();
            for (int i = 0; i < 10; ++i) { cudaMemcpyAsync(dst, dev, b, cudaMemcpyDeviceToHost, s); cudaStreamSynchronize(s); }
            auto t1 = std::chrono::steady_clock::now();
            printf("D2H %zu B to %s: %.3f ms\n", b, k ? "pinned" : "pageable", std::chrono::duration<double, std::milli>(t1 - t0).count() / 10);
        }
    }
    return 0;
}
