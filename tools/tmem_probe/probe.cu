// Feasibility probe for the segment-resident quantizer (round 2): can tensor
// memory hold the quantizer's x between its STATS and BIN passes, and what
// does a 1-CTA-per-SM, 16-warp streaming loop reach on the quantizer's access
// mix (read theta_g, theta_l, codes: 9 B/element; write codes: 1 B/element)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe probe.cu
// Modes (250M elements, one warp unit = 1024 elements = 8 float4 per lane):
//   0 stream only: x = a - b + lut[c], fp64 sum, x -> TMEM
//   1 + bin back from TMEM right away (codes out)
//   2 + bin of the PREVIOUS unit (one unit of lag) + L2 bulk prefetch of the next unit
//   3 like 1 but x round-trips through shared memory
//   4 like 1 but x round-trips through global memory (L2)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kWarps = 16, kThreads = kWarps * 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void tm_st32(uint32_t taddr, const float (&x)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
        "f"(x[0]), "f"(x[1]), "f"(x[2]), "f"(x[3]), "f"(x[4]), "f"(x[5]), "f"(x[6]), "f"(x[7]), "f"(x[8]), "f"(x[9]),
        "f"(x[10]), "f"(x[11]), "f"(x[12]), "f"(x[13]), "f"(x[14]), "f"(x[15]), "f"(x[16]), "f"(x[17]), "f"(x[18]),
        "f"(x[19]), "f"(x[20]), "f"(x[21]), "f"(x[22]), "f"(x[23]), "f"(x[24]), "f"(x[25]), "f"(x[26]), "f"(x[27]),
        "f"(x[28]), "f"(x[29]), "f"(x[30]), "f"(x[31])
        : "memory");
}
__device__ __forceinline__ void tm_ld32(uint32_t taddr, float (&x)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3]), "=f"(x[4]), "=f"(x[5]), "=f"(x[6]), "=f"(x[7]), "=f"(x[8]),
          "=f"(x[9]), "=f"(x[10]), "=f"(x[11]), "=f"(x[12]), "=f"(x[13]), "=f"(x[14]), "=f"(x[15]), "=f"(x[16]),
          "=f"(x[17]), "=f"(x[18]), "=f"(x[19]), "=f"(x[20]), "=f"(x[21]), "=f"(x[22]), "=f"(x[23]), "=f"(x[24]),
          "=f"(x[25]), "=f"(x[26]), "=f"(x[27]), "=f"(x[28]), "=f"(x[29]), "=f"(x[30]), "=f"(x[31])
        : "r"(taddr)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

struct f8 { float v[8]; };
// 256-bit streaming loads (LDG.E.256, sm_100): 8 floats / 8 codes per lane
__device__ __forceinline__ f8 ld_stream8(const float* p) {
    f8 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]), "=f"(r.v[6]),
                   "=f"(r.v[7])
                 : "l"(p));
    return r;
}
__device__ __forceinline__ uint2 ld_stream_u64(const uint8_t* p) {
    uint2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1)
probe(const float4* __restrict__ a, const float4* __restrict__ b, const uint32_t* __restrict__ c, uint32_t* codes,
      float4* gx, uint64_t nunits, double* sums, uint32_t* ctr) {
    extern __shared__ __align__(16) unsigned char sm_raw[];
    float* lut = reinterpret_cast<float*>(sm_raw);
    uint32_t* tbase = reinterpret_cast<uint32_t*>(sm_raw + 1024);
    float4* sx = reinterpret_cast<float4*>(sm_raw + 2048);  // [warp][8][32] float4 (mode 3)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x < 256) lut[threadIdx.x] = (float)threadIdx.x * 1e-3f;
    if (MODE != 3 && MODE != 4 && warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tb = *tbase;
    const uint32_t tq = tb + ((uint32_t)(32 * (warp & 3)) << 16) + 128u * (uint32_t)(warp >> 2);
    double s = 0.0;
    uint32_t slot = 0;
    uint64_t prev_u = ~0ull;
    for (uint64_t u = (uint64_t)blockIdx.x * kWarps + warp; u < nunits; u += (uint64_t)gridDim.x * kWarps) {
        if (MODE == 2 && lane == 0) {
            const uint64_t nu = u + (uint64_t)gridDim.x * kWarps;
            if (nu < nunits) {
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], 4096;" ::"l"(a + nu * 256));
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], 4096;" ::"l"(b + nu * 256));
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], 1024;" ::"l"(c + nu * 256));
            }
        }
        f8 va[4], vb[4];
        uint2 vc[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint64_t e = u * 1024 + j * 256 + lane * 8;
            va[j] = ld_stream8(reinterpret_cast<const float*>(a) + e);
            vb[j] = ld_stream8(reinterpret_cast<const float*>(b) + e);
            vc[j] = ld_stream_u64(reinterpret_cast<const uint8_t*>(c) + e);
        }
        if (MODE == 2 && prev_u != ~0ull) {  // bin the previous unit while this unit's loads fly
            float y[32];
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            tm_ld32(tq + 32u * ((slot + 3) & 3), y);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                uint32_t p0 = 0, p1 = 0;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    p0 |= ((uint32_t)(int)__fmaf_rn(y[8 * j + e], 100.f, 128.f) & 0xffu) << (8 * e);
                    p1 |= ((uint32_t)(int)__fmaf_rn(y[8 * j + 4 + e], 100.f, 128.f) & 0xffu) << (8 * e);
                }
                *reinterpret_cast<uint2*>(reinterpret_cast<uint8_t*>(codes) + prev_u * 1024 + j * 256 + lane * 8) = make_uint2(p0, p1);
            }
        }
        float x[32];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const uint32_t cw = e < 4 ? vc[j].x : vc[j].y;
                const float v = __fadd_rn(__fsub_rn(va[j].v[e], vb[j].v[e]), lut[(cw >> (8 * (e & 3))) & 0xff]);
                x[8 * j + e] = v;
                s = __dadd_rn(s, (double)v);
            }
        }
        if (MODE == 3) {
#pragma unroll
            for (int j = 0; j < 8; ++j) sx[(warp * 8 + j) * 32 + lane] = make_float4(x[4 * j], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3]);
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float4 v = sx[(warp * 8 + j) * 32 + lane];
                x[4 * j] = v.x; x[4 * j + 1] = v.y; x[4 * j + 2] = v.z; x[4 * j + 3] = v.w;
            }
        } else if (MODE == 4) {
#pragma unroll
            for (int j = 0; j < 8; ++j) gx[u * 256 + j * 32 + lane] = make_float4(x[4 * j], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3]);
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float4 v = __ldcg(gx + u * 256 + j * 32 + lane);
                x[4 * j] = v.x; x[4 * j + 1] = v.y; x[4 * j + 2] = v.z; x[4 * j + 3] = v.w;
            }
        } else {
            tm_st32(tq + 32u * slot, x);
            if (MODE == 1) {
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                tm_ld32(tq + 32u * slot, x);
            }
        }
        if (MODE == 1 || MODE == 3 || MODE == 4) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                uint32_t p0 = 0, p1 = 0;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    p0 |= ((uint32_t)(int)__fmaf_rn(x[8 * j + e], 100.f, 128.f) & 0xffu) << (8 * e);
                    p1 |= ((uint32_t)(int)__fmaf_rn(x[8 * j + 4 + e], 100.f, 128.f) & 0xffu) << (8 * e);
                }
                *reinterpret_cast<uint2*>(reinterpret_cast<uint8_t*>(codes) + u * 1024 + j * 256 + lane * 8) = make_uint2(p0, p1);
            }
        }
        prev_u = u;
        slot = (slot + 1) & 3;
    }
    if (MODE == 2 && prev_u != ~0ull) {
        float y[32];
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tm_ld32(tq + 32u * ((slot + 3) & 3), y);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint32_t p0 = 0, p1 = 0;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                p0 |= ((uint32_t)(int)__fmaf_rn(y[8 * j + e], 100.f, 128.f) & 0xffu) << (8 * e);
                p1 |= ((uint32_t)(int)__fmaf_rn(y[8 * j + 4 + e], 100.f, 128.f) & 0xffu) << (8 * e);
            }
            *reinterpret_cast<uint2*>(reinterpret_cast<uint8_t*>(codes) + prev_u * 1024 + j * 256 + lane * 8) =
                make_uint2(p0, p1);
        }
    }
    for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
    if (lane == 0) atomicAdd(&sums[0], s);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (MODE != 3 && MODE != 4 && warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

int main() {
    const uint64_t n = 250000000ull / 1024 * 1024, nunits = n / 1024;
    float4 *a, *b, *gx;
    uint32_t *c, *codes, *ctr;
    double* sums;
    cudaMalloc(&a, n * 4); cudaMalloc(&b, n * 4); cudaMalloc(&gx, n * 4);
    cudaMalloc(&c, n); cudaMalloc(&codes, n); cudaMalloc(&sums, 64); cudaMalloc(&ctr, 64);
    // a = small values, b = 0, c = pattern: x = a + lut[c]
    cudaMemset(a, 0, n * 4); cudaMemset(b, 0, n * 4); cudaMemset(c, 0x11, n);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    const size_t smem = 2048 + (size_t)kWarps * 8 * 32 * 16;  // 66 KB (mode 3 uses it)
    void (*fns[5])(const float4*, const float4*, const uint32_t*, uint32_t*, float4*, uint64_t, double*, uint32_t*) = {
        probe<0>, probe<1>, probe<2>, probe<3>, probe<4>};
    const char* names[5] = {"stream->TMEM", "stream->TMEM->bin", "stream + lagged bin + L2 pf", "stream->smem->bin",
                            "stream->gmem->bin"};
    const double bytes[5] = {9.0, 10.0, 10.0, 10.0, 10.0};
    for (int m = 0; m < 5; ++m) {
        cudaFuncSetAttribute(fns[m], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        float best = 1e9f;
        for (int rep = 0; rep < 8; ++rep) {
            cudaMemset(sums, 0, 64);
            cudaEventRecord(e0);
            fns[m]<<<sms, kThreads, smem>>>(a, b, c, codes, gx, nunits, sums, ctr);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        cudaError_t err = cudaGetLastError();
        double hs = 0;
        cudaMemcpy(&hs, sums, 8, cudaMemcpyDeviceToHost);
        uint32_t hc[4] = {0, 0, 0, 0};
        cudaMemcpy(hc, codes + nunits * 256 - 4, 16, cudaMemcpyDeviceToHost);
        printf("mode %d %-28s %.3f ms  %.0f GB/s (%.0f B/elt)  sum %.6g (expect %.6g)  code %08x  %s\n", m, names[m],
               best, bytes[m] * n / best / 1e6, bytes[m], hs, (double)n * 0x11 * 1e-3, hc[3], cudaGetErrorString(err));
        cudaMemset(codes, 0, n);
    }
    return 0;
}
