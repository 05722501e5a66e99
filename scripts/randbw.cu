// Random-access bandwidth microbenchmark (development aid, not product code):
// what HBM delivers for the k_level access pattern -- warp-coalesced 256-byte
// segments at random 256-B-aligned offsets of a multi-GB array -- as plain
// loads, as red.or, and as load-then-red.or of the same segment.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/randbw scripts/randbw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t hash64(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
    return x;
}

// SEGW = 256-byte blocks per contiguous segment (a warp reads SEGW x 256 B)
template <int MODE, int ILP, int SEGW = 1>
__global__ void __launch_bounds__(256) k_rand(uint64_t *a, uint64_t nseg, uint64_t iters, unsigned long long *sink) {
    const int lane = threadIdx.x & 31;
    const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    uint64_t acc = 0;
    for (uint64_t it = 0; it < iters; ++it) {
        uint64_t seg[ILP], v[ILP];
#pragma unroll
        for (int k = 0; k < ILP; ++k)
            seg[k] = (hash64(wid * 1000003ull + (it * ILP + k) / SEGW) % (nseg / SEGW)) * SEGW + (it * ILP + k) % SEGW;
        if (MODE != 1) {
#pragma unroll
            for (int k = 0; k < ILP; ++k) v[k] = __ldcg((const unsigned long long *)(a + seg[k] * 32 + lane));
        }
#pragma unroll
        for (int k = 0; k < ILP; ++k) {
            if (MODE == 0) acc += v[k];
            else {
                uint64_t m = (MODE == 2) ? (~v[k] & (1ull << ((it + k) & 63))) : (1ull << ((it + k) & 63));
                if (m) asm volatile("red.relaxed.gpu.global.or.b64 [%0], %1;" ::"l"(a + seg[k] * 32 + lane), "l"(m) : "memory");
            }
        }
    }
    if (acc == 0x1234567) atomicAdd(sink, acc);
}

template <int MODE, int ILP, int SEGW = 1>
void run(const char *name, uint64_t *a, uint64_t nseg, unsigned long long *sink, int blocks_per_sm) {
    const int blocks = 148 * blocks_per_sm;
    const uint64_t warps = blocks * 8ull;
    const uint64_t iters = 2000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    k_rand<MODE, ILP, SEGW><<<blocks, 256>>>(a, nseg, 10, sink);
    cudaEventRecord(e0);
    k_rand<MODE, ILP, SEGW><<<blocks, 256>>>(a, nseg, iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double segs = (double)warps * iters * ILP;
    const double bytes = segs * 256.0 * (MODE == 0 ? 1 : MODE == 1 ? 2 : 2);   // red = read+write of the line
    printf("%-28s seg=%5dB ILP=%d CTAs/SM=%d: %.3f ms, %.1f G256B/s, %.0f GB/s (x%s)\n", name, 256 * SEGW, ILP,
           blocks_per_sm, ms,
           segs / ms / 1e6, bytes / ms / 1e6, MODE == 0 ? "1 read" : "read+write");
}

int main() {
    const uint64_t bytes = 4ull << 30;   // 4 GiB >> L2
    uint64_t *a;
    unsigned long long *sink;
    cudaMalloc(&a, bytes);
    cudaMalloc(&sink, 8);
    cudaMemset(a, 0, bytes);
    const uint64_t nseg = bytes / 256;
    for (int occ : {3, 8}) {
        run<0, 8, 1>("random load", a, nseg, sink, occ);
        run<0, 8, 2>("random load", a, nseg, sink, occ);
        run<0, 8, 4>("random load", a, nseg, sink, occ);
        run<0, 8, 8>("random load", a, nseg, sink, occ);
        run<0, 16, 16>("random load", a, nseg, sink, occ);
        run<1, 8, 1>("random red.or", a, nseg, sink, occ);
        run<2, 8, 1>("random load+red.or", a, nseg, sink, occ);
        run<2, 8, 8>("random load+red.or", a, nseg, sink, occ);
    }
    // streaming copy reference
    uint64_t *b;
    cudaMalloc(&b, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaMemcpy(b, a, bytes, cudaMemcpyDeviceToDevice);
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) cudaMemcpy(b, a, bytes, cudaMemcpyDeviceToDevice);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-28s %.0f GB/s (read+write)\n", "cudaMemcpy D2D 4 GiB", 5 * 2.0 * bytes / ms / 1e6);
    return 0;
}
