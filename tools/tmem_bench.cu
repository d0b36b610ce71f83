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

#define LD64(dst, addr) asm volatile( \
    "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15," \
    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39," \
    "%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];" \
    : "=r"(dst[0]), "=r"(dst[1]), "=r"(dst[2]), "=r"(dst[3]), "=r"(dst[4]), "=r"(dst[5]), "=r"(dst[6]), "=r"(dst[7]), \
      "=r"(dst[8]), "=r"(dst[9]), "=r"(dst[10]), "=r"(dst[11]), "=r"(dst[12]), "=r"(dst[13]), "=r"(dst[14]), "=r"(dst[15]), \
      "=r"(dst[16]), "=r"(dst[17]), "=r"(dst[18]), "=r"(dst[19]), "=r"(dst[20]), "=r"(dst[21]), "=r"(dst[22]), "=r"(dst[23]), \
      "=r"(dst[24]), "=r"(dst[25]), "=r"(dst[26]), "=r"(dst[27]), "=r"(dst[28]), "=r"(dst[29]), "=r"(dst[30]), "=r"(dst[31]), \
      "=r"(dst[32]), "=r"(dst[33]), "=r"(dst[34]), "=r"(dst[35]), "=r"(dst[36]), "=r"(dst[37]), "=r"(dst[38]), "=r"(dst[39]), \
      "=r"(dst[40]), "=r"(dst[41]), "=r"(dst[42]), "=r"(dst[43]), "=r"(dst[44]), "=r"(dst[45]), "=r"(dst[46]), "=r"(dst[47]), \
      "=r"(dst[48]), "=r"(dst[49]), "=r"(dst[50]), "=r"(dst[51]), "=r"(dst[52]), "=r"(dst[53]), "=r"(dst[54]), "=r"(dst[55]), \
      "=r"(dst[56]), "=r"(dst[57]), "=r"(dst[58]), "=r"(dst[59]), "=r"(dst[60]), "=r"(dst[61]), "=r"(dst[62]), "=r"(dst[63]) \
    : "r"(addr))

// 2 x64 loads in flight per wait, minimal consumer work (one min per value).
__global__ void __launch_bounds__(128) tmem_ld2(unsigned *out, unsigned long long *clk, int iters)
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
    unsigned acc = 0xffffffffu;
    unsigned long long c0 = clock64(), t0 = gtime();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < 512; c += 128) {
            unsigned a[64], b[64];
            LD64(a, tbase + c);
            LD64(b, tbase + c + 64);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int i = 0; i < 64; i += 2) acc = min(acc, min(min(a[i], a[i + 1]), min(b[i], b[i + 1])));
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
    tmem_ld2<<<sms, 128>>>(out, clk, 16);
    cudaEventRecord(a);
    tmem_ld2<<<sms, 128>>>(out, clk, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    e = cudaGetLastError();
    cudaEventElapsedTime(&ms, a, b);
    cudaMemcpy(h, clk, 16, cudaMemcpyDeviceToHost);
    printf("{\"variant\": \"2 loads in flight\", \"err\": \"%s\", \"tmem_ld_bytes_per_clk_sm\": %.1f, \"cycles_per_iter\": %.1f}\n",
           cudaGetErrorString(e), bytes_per_sm / (ms * 1e-3 * mhz * 1e6), (double)h[0] / iters);
    return 0;
}
