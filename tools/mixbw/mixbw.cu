// Achievable HBM bandwidth for the quantizer's two access mixes, no compute:
//   STATS-like: read A, B (fp32) + codes (u8), write scratch x (fp32)   13 B/element
//   BIN-like:   read scratch x (fp32), write codes (u8)                  5 B/element
//   copy:       read fp32, write fp32                                    8 B/element
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mixbw mixbw.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void stats_like(const float4* __restrict__ a, const float4* __restrict__ b,
                           const unsigned* __restrict__ c, float4* __restrict__ x, size_t n4) {
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n4; q += (size_t)gridDim.x * blockDim.x) {
        float4 va = __ldcs(a + q), vb = __ldcs(b + q);
        unsigned cc = __ldcs(c + q);
        float f = (float)(cc & 0xff);
        x[q] = make_float4(va.x - vb.x + f, va.y - vb.y, va.z - vb.z, va.w - vb.w);
    }
}
__global__ void bin_like(const float4* __restrict__ x, unsigned* __restrict__ c, size_t n4) {
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n4; q += (size_t)gridDim.x * blockDim.x) {
        float4 v = __ldcg(x + q);
        c[q] = (unsigned)(int)v.x ^ (unsigned)(int)v.y ^ (unsigned)(int)v.z ^ (unsigned)(int)v.w;
    }
}
__global__ void copy_like(const float4* __restrict__ a, float4* __restrict__ b, size_t n4) {
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n4; q += (size_t)gridDim.x * blockDim.x)
        b[q] = __ldcs(a + q);
}

int main() {
    const size_t n = 250000000, n4 = n / 4;
    float4 *a, *b, *x;
    unsigned* c;
    cudaMalloc(&a, n * 4); cudaMalloc(&b, n * 4); cudaMalloc(&x, n * 4); cudaMalloc(&c, n);
    cudaMemset(a, 0, n * 4); cudaMemset(b, 0, n * 4); cudaMemset(c, 0, n);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int blocks_per_sm : {4, 8, 16}) {
        const int grid = sms * blocks_per_sm;
        float best[3] = {1e9f, 1e9f, 1e9f};
        for (int rep = 0; rep < 6; ++rep) {
            float ms;
            cudaEventRecord(e0); stats_like<<<grid, 256>>>(a, b, c, x, n4); cudaEventRecord(e1);
            cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best[0]) best[0] = ms;
            cudaEventRecord(e0); bin_like<<<grid, 256>>>(x, c, n4); cudaEventRecord(e1);
            cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best[1]) best[1] = ms;
            cudaEventRecord(e0); copy_like<<<grid, 256>>>(a, x, n4); cudaEventRecord(e1);
            cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best[2]) best[2] = ms;
        }
        printf("grid %d x 256: STATS-like %.3f ms (%.0f GB/s)  BIN-like %.3f ms (%.0f GB/s)  copy %.3f ms (%.0f GB/s)  "
               "STATS+BIN %.3f ms\n", grid, best[0], 13.0 * n / best[0] / 1e6, best[1], 5.0 * n / best[1] / 1e6,
               best[2], 8.0 * n / best[2] / 1e6, best[0] + best[1]);
    }
    return 0;
}
