// Micro-benchmark: does SHFL share the LSU data pipe with LDS?  Independent
// conflict-free LDS.32 (lane-distinct banks), SHFL.IDX, and both interleaved.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_bcast micro_bcast.cu
#include <cstdio>
#include <cstdint>

template <int MODE>   // 1 = LDS only, 2 = SHFL only, 3 = both, 4 = LDS.128 broadcast
__global__ void k(uint32_t* out, int iters) {
    __shared__ __align__(16) uint32_t s[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = i * 2654435761u;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    uint32_t a0 = 0, a1 = 1, a2 = 2, a3 = 3, b0 = 5, b1 = 6, b2 = 7, b3 = 8;
    for (int it = 0; it < iters; ++it) {
        const uint32_t base = (it & 63) * 128;
        if (MODE & 1) {
            a0 ^= s[base + lane];
            a1 ^= s[base + 32 + lane];
            a2 ^= s[base + 64 + lane];
            a3 ^= s[base + 96 + lane];
        }
        if (MODE & 2) {
            b0 += __shfl_sync(0xFFFFFFFFu, b0, it & 31);
            b1 += __shfl_sync(0xFFFFFFFFu, b1, (it + 1) & 31);
            b2 += __shfl_sync(0xFFFFFFFFu, b2, (it + 2) & 31);
            b3 += __shfl_sync(0xFFFFFFFFu, b3, (it + 3) & 31);
        }
        if (MODE == 4) {
            const uint4 v = *reinterpret_cast<const uint4*>(s + base);
            const uint4 w = *reinterpret_cast<const uint4*>(s + base + 4);
            a0 ^= v.x; a1 ^= v.y; a2 ^= w.z; a3 ^= w.w;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + b0 + b1 + b2 + b3;
}

int main() {
    uint32_t* d;
    cudaMalloc(&d, 148 * 512 * 4);
    const int iters = 1 << 15;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](auto kern, const char* name, int per_iter) {
        kern<<<148, 512>>>(d, iters);
        cudaEventRecord(e0);
        kern<<<148, 512>>>(d, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = 16.0 * iters * per_iter;   // warp ops per SM
        printf("%-10s %.3f ms  %.3f warp-ops per SM-clock\n", name, ms, ops / (ms * 1e-3 * 1.965e9));
    };
    run(k<1>, "lds", 4);
    run(k<2>, "shfl", 4);
    run(k<3>, "lds+shfl", 8);
    run(k<4>, "lds128bc", 2);
    return 0;
}
