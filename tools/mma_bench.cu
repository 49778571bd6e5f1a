// Microbenchmark: sustained tcgen05.mma throughput per SM for the shapes the
// abs-GEMM uses (kind::tf32 M=128, N=64/128/256, SS operands in SWIZZLE_64B/128B
// smem) vs kind::f16 (bf16).  One CTA per SM, a single thread issues MMAs back
// to back into one TMEM accumulator; commit + wait every 16 MMAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_bench tools/mma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, int row_bytes) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)1u << 16;
    d |= (uint64_t)((8u * row_bytes) >> 4) << 32;
    d |= (uint64_t)1u << 46;
    d |= (uint64_t)(row_bytes == 128 ? 2u : 4u) << 61;
    return d;
}

template <int KIND, int N>  // KIND 0 = tf32, 1 = f16(bf16), 2 = f16 with A in TMEM (TS)
__global__ void __launch_bounds__(128, 1) k_mma(int iters, unsigned long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    if (threadIdx.x == 0) {
        const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
        const uint32_t idesc = (1u << 4) | ((KIND == 0 ? 2u : 1u) << 7) | ((KIND == 0 ? 2u : 1u) << 10) |
                               ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint64_t ad = make_desc(a, 128), bd = make_desc(b, 128);
        uint32_t phase = 0;
        long long t0 = clock64();
        for (int it = 0; it < iters; it++) {
            for (int j = 0; j < 16; j++) {
                if (KIND == 0)
                    asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;}"
                                 ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(1));
                else if (KIND == 1)
                    asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
                                 ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(1));
                else  // A operand from TMEM columns 384.. (128 lanes x 8 columns per k16)
                    asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}"
                                 ::"r"(tmem), "r"(tmem + 384u), "l"(bd), "r"(idesc), "r"(1));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
            asm volatile("{.reg .pred P1; W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1; @P1 bra D; bra W; D: }" ::"r"(smem_u32(&bar)), "r"(phase));
            phase ^= 1;
        }
        long long t1 = clock64();
        cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int KIND, int N>
void run(const char* name) {
    const int iters = 2000, sms = 148;
    unsigned long long* d;
    cudaMalloc(&d, sms * 8);
    cudaFuncSetAttribute(k_mma<KIND, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    k_mma<KIND, N><<<sms, 128, 64 * 1024>>>(10, d);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_mma<KIND, N><<<sms, 128, 64 * 1024>>>(iters, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[148];
    cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
    const double mmas = (double)iters * 16;
    const double k = KIND == 0 ? 8 : 16;  // k per instruction
    const double flops = 2.0 * 128 * N * k * mmas * sms;
    printf("{\"mma\": \"%s\", \"N\": %d, \"cycles_per_mma\": %.1f, \"TFLOP/s\": %.1f, \"err\": \"%s\"}\n", name, N,
           (double)h[0] / mmas, flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    run<0, 64>("tf32");
    run<0, 128>("tf32");
    run<0, 256>("tf32");
    run<1, 128>("bf16");
    run<1, 256>("bf16");
    run<2, 128>("bf16_ts");
    run<2, 256>("bf16_ts");
    return 0;
}
