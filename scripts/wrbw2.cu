// Write-pattern microbenchmark 2 (development aid): the PAIRS output pattern.
// Two columns (arrays); source s owns the run [s*L, (s+1)*L) of both; warp w
// writes the runs of sources 64w..64w+63 chunk by chunk (round robin over its
// 64 sources), C bytes per chunk and column, STG.128.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/wrbw2.cu -o scripts/wrbw2.bin
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_wr2(uint32_t *A, uint32_t *B, uint64_t L, uint32_t C, uint64_t nsrc, int twocol, int order) {
    const int lane = threadIdx.x & 31;
    const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t)gridDim.x * blockDim.x >> 5;
    for (uint64_t g = wid; g * 64 < nsrc; g += nwarps) {
        for (uint64_t off = 0; off < L; off += C) {
            for (int b = 0; b < 64; ++b) {
                const uint64_t s = order ? g + (uint64_t)b * (nsrc / 64) : g * 64 + b;   // order 1: strided sources
                if (s >= nsrc) break;
                const uint32_t n = (uint32_t)(L - off < C ? L - off : C);
                uint4 *pa = reinterpret_cast<uint4 *>(A + s * L + off);
                uint4 *pb = reinterpret_cast<uint4 *>(B + s * L + off);
                for (uint32_t k = lane; k < n / 4; k += 32) {
                    pa[k] = make_uint4(k, b, 1, 2);
                    if (twocol) pb[k] = make_uint4(b, b, b, b);
                }
            }
        }
    }
}
int main() {
    const uint64_t cols = 32ull << 30;   // bytes per column
    uint32_t *A, *B;
    cudaMalloc(&A, cols);
    cudaMalloc(&B, cols);
    const uint64_t L = 83200;                 // elements per source run
    const uint64_t nsrc = cols / 4 / L / 64 * 64;
    for (int order = 0; order < 2; ++order)
    for (int twocol = 0; twocol < 2; ++twocol)
        for (int blocks : {148 * 4, 148 * 6, 148 * 12})
            for (uint32_t C : {512u, 1728u, 6912u}) {
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0);
                cudaEventCreate(&e1);
                float best = 1e9;
                for (int it = 0; it < 3; ++it) {
                    cudaEventRecord(e0);
                    k_wr2<<<blocks, 128>>>(A, B, L, C / 4, nsrc, twocol, order);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    best = ms < best ? ms : best;
                }
                const double bytes = (double)nsrc * L * 4 * (twocol ? 2 : 1);
                printf("order=%d cols=%d blocks=%5d chunk=%5u B: %.2f ms %.0f GB/s\n", order, twocol + 1, blocks, C, best,
                       bytes / best / 1e6);
            }
    return 0;
}
