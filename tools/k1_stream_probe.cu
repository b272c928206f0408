// Microbenchmark (not product code): how fast can one warp per request stream
// each request's first `m` tokens (K1's access pattern, no trie side)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o k1probe tools/k1_stream_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

template <int U, int MODE>
__global__ void __launch_bounds__(256) k_stream(const int32_t *__restrict__ arena, const int64_t *__restrict__ off,
                                                const int32_t *__restrict__ m, int32_t n, int32_t *out) {
    const int lane = threadIdx.x & 31;
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i >= n) return;
    const int32_t *rq = arena + off[i];
    const int32_t len = m[i];
    int32_t acc = 0;
    if (MODE == 1) {
        const int32_t nb = (len * 4 + 4095) >> 12;
        if (lane < nb) {
            const int32_t b0 = lane << 10;
            const uint32_t bytes = (uint32_t)(((min(len, b0 + 1024) - b0) * 4 + 15) & ~15);
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(rq + b0), "r"(bytes) : "memory");
        }
    }
    if (MODE == 2) {
        // int4 loads: 4 tokens per lane per load
        for (int32_t k = 0; k < len; k += 128 * U) {
            bool bad = false;
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int32_t p = k + u * 128 + lane * 4;
                if (p + 3 < len) {
                    const int4 v = __ldg(reinterpret_cast<const int4 *>(rq + p));
                    bad |= (v.x == -7) | (v.y == -7) | (v.z == -7) | (v.w == -7);
                }
            }
            if (__ballot_sync(0xffffffffu, bad)) { acc = 1; break; }
        }
    } else {
        for (int32_t k = 0; k < len; k += 32 * U) {
            bool bad[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int32_t p = k + u * 32 + lane;
                bad[u] = p < len && __ldg(rq + p) == -7;
            }
#pragma unroll
            for (int u = 0; u < U; u++)
                if (__ballot_sync(0xffffffffu, bad[u])) { acc = 1; break; }
        }
    }
    if (lane == 0 && acc) out[i] = acc;
}

template <int U, int MODE>
float run(const int32_t *arena, const int64_t *off, const int32_t *m, int n, int32_t *out) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    const int blocks = (n * 32 + 255) / 256;
    k_stream<U, MODE><<<blocks, 256>>>(arena, off, m, n, out);
    cudaEventRecord(a);
    for (int r = 0; r < 3; r++) k_stream<U, MODE><<<blocks, 256>>>(arena, off, m, n, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 3;
}

int main() {
    const int n = 1 << 20;
    const int64_t L = 8192;
    int32_t *arena; int64_t *off; int32_t *m, *out;
    cudaMalloc(&arena, sizeof(int32_t) * n * L);
    cudaMemset(arena, 1, sizeof(int32_t) * n * L);
    cudaMalloc(&off, sizeof(int64_t) * n); cudaMalloc(&m, sizeof(int32_t) * n); cudaMalloc(&out, sizeof(int32_t) * n);
    std::vector<int64_t> ho(n); std::vector<int32_t> hm(n);
    uint64_t x = 88172645463325252ull;
    double bytes = 0;
    for (int i = 0; i < n; i++) {
        ho[i] = (int64_t)i * L;
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        hm[i] = 1024 + (int32_t)(x % 4096);  // ~2.6k tokens read per request, like config 5
        bytes += 4.0 * hm[i];
    }
    cudaMemcpy(off, ho.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice);
    cudaMemcpy(m, hm.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice);
    auto rep = [&](const char *name, float ms) { printf("%-28s %.3f ms  %.0f GB/s\n", name, ms, bytes / ms / 1e6); };
    rep("scalar U=4", run<4, 0>(arena, off, m, n, out));
    rep("scalar U=8", run<8, 0>(arena, off, m, n, out));
    rep("scalar U=16", run<16, 0>(arena, off, m, n, out));
    rep("scalar U=8 + bulk prefetch", run<8, 1>(arena, off, m, n, out));
    rep("int4 U=1", run<1, 2>(arena, off, m, n, out));
    rep("int4 U=2", run<2, 2>(arena, off, m, n, out));
    rep("int4 U=4", run<4, 2>(arena, off, m, n, out));
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
