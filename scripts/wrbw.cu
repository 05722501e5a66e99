// Write-pattern microbenchmark (development aid): every warp owns S streams
// (contiguous regions) and writes C bytes to each in turn (round robin),
// 32-bit coalesced stores (128 B per instruction), like k_write_pairs' target
// column.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/wrbw.cu -o /tmp/wrbw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_wr(uint32_t *out, uint64_t words_per_warp, int S, uint32_t C_words, int vec) {
    const int lane = threadIdx.x & 31;
    const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    uint32_t *base = out + wid * words_per_warp;
    const uint64_t per_stream = words_per_warp / S;
    for (uint64_t off = 0; off < per_stream; off += C_words) {
        for (int s = 0; s < S; ++s) {
            uint32_t *p = base + s * per_stream + off;
            const uint32_t n = (uint32_t)(per_stream - off < C_words ? per_stream - off : C_words);
            if (vec) {
                for (uint32_t k = lane * 4; k + 3 < n; k += 128)
                    *reinterpret_cast<uint4 *>(p + k) = make_uint4(k, s, 1, 2);
            } else {
                for (uint32_t k = lane; k < n; k += 32) p[k] = k + s;
            }
        }
    }
}
int main() {
    const uint64_t total = 32ull << 30;   // bytes
    uint32_t *out;
    cudaMalloc(&out, total);
    const int blocks = 148 * 8, threads = 128;
    const uint64_t warps = (uint64_t)blocks * threads / 32;
    const uint64_t wpw = total / 4 / warps;
    int Ss[] = {1, 8, 64};
    uint32_t Cs[] = {128, 512, 1728, 4096, 16384, 65536};
    for (int vec = 0; vec < 2; ++vec)
        for (int S : Ss)
            for (uint32_t C : Cs) {
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0);
                cudaEventCreate(&e1);
                float best = 1e9;
                for (int it = 0; it < 3; ++it) {
                    cudaEventRecord(e0);
                    k_wr<<<blocks, threads>>>(out, wpw - wpw % (S * 4), S, C / 4, vec);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    best = ms < best ? ms : best;
                }
                printf("vec=%d streams/warp=%2d chunk=%6u B: %.2f ms %.0f GB/s\n", vec, S, C, best, total / best / 1e6);
            }
    return 0;
}
