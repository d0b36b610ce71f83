// tmem_bench.cu -- TMEM -> register load throughput on one SM (tcgen05.ld 32x32b.x64),
// to size a tensor-core distance filter.  One CTA of 4 warps per SM;
// each warp reads its 32-lane quarter of a 512-column allocation repeatedly.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gtime() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }

#define R8(i) "=r"(v[i]), "=r"(v[i + 1]), "=r"(v[i + 2]), "=r"(v[i + 3]), "=r"(v[i + 4]), "=r"(v[i + 5]), "=r"(v[i + 6]), "=r"(v[i + 7])

__global__ void __launch_bounds__(128) tmem_ld(unsigned *out, unsigned long long *clk, int iters)
{
    __shared__ uint32_t taddr_s;
    const int warp = threadIdx.x / 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&taddr_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tbase = taddr_s + ((uint32_t)(warp * 32) << 16);
    unsigned acc = 0;
    unsigned long long c0 = clock64(), t0 = gtime();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < 512; c += 64) {
            unsigned v[64];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,"
                "%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
                : R8(0), R8(8), R8(16), R8(24), R8(32), R8(40), R8(48), R8(56)
                : "r"(tbase + c));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int i = 0; i < 64; i += 2) acc = min(acc ^ v[i], v[i + 1]);
        }
    }
    unsigned long long c1 = clock64(), t1 = gtime();
    if (acc == 0x12345) out[0] = acc;
    if (blockIdx.x == 0 && threadIdx.x == 0) { clk[0] = c1 - c0; clk[1] = t1 - t0; }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s));
}

int main()
{
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned *out; unsigned long long *clk; cudaMalloc(&out, 4); cudaMalloc(&clk, 16);
    const int iters = 4096;
    tmem_ld<<<sms, 128>>>(out, clk, 16);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    tmem_ld<<<sms, 128>>>(out, clk, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaError_t e = cudaGetLastError();
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long h[2]; cudaMemcpy(h, clk, 16, cudaMemcpyDeviceToHost);
    const double mhz = (double)h[0] / (double)h[1] * 1e3;
    const double bytes_per_sm = (double)iters * 512 * 128 * 4;
    printf("{\"err\": \"%s\", \"tmem_ld_bytes_per_clk_sm\": %.1f, \"in_kernel_cycles_per_iter\": %.1f, \"mhz\": %.0f}\n",
           cudaGetErrorString(e), bytes_per_sm / (ms * 1e-3 * mhz * 1e6), (double)h[0] / iters, mhz);
    return 0;
}
