// Probe: how close does a hand-written SIMT FP32 GEMM (the value half of a
// fused value + abs-bound GEMM) get to cuBLAS on the B200?
//   C[M,N] = A[M,K] @ B[K,N], FP32, row-major; 128x128 tile, 256 threads,
//   8x8 outputs per thread (rows ty*4+{0..3}, 64+ty*4+{0..3}; cols likewise),
//   A staged transposed in smem (LDG.128 -> 4 STS.32), B by cp.async 16 B,
//   double-buffered smem, one __syncthreads per k-tile.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/sgemm_probe.cu -lcublas -o tools/sgemm_probe
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <cuda_runtime.h>
#include <cublas_v2.h>

constexpr int BM = 128, BN = 128, BK = 16, NT = 256;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

#ifndef MINB
#define MINB 2
#endif
__global__ void __launch_bounds__(NT, MINB) k_sgemm(const float* __restrict__ A,
                                                 const float* __restrict__ B,
                                                 float* __restrict__ C, int M, int N, int K) {
    __shared__ __align__(16) float As[2][BK][BM];
    __shared__ __align__(16) float Bs[2][BK][BN];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    // A loader: 128 rows x 16 k = 512 float4; thread t loads rows (t>>2) and 64+(t>>2), k-chunk t&3
    const int ar = tid >> 2, ac = (tid & 3) * 4;
    const float* Ag0 = A + (size_t)(m0 + ar) * K + ac;
    const float* Ag1 = A + (size_t)(m0 + 64 + ar) * K + ac;
    // B loader: 16 k x 128 n = 512 float4; thread t loads k-rows (t>>5) and 8+(t>>5), col chunk t&31
    const int br = tid >> 5, bc = (tid & 31) * 4;
    const float* Bg0 = B + (size_t)br * N + n0 + bc;
    const float* Bg1 = B + (size_t)(br + 8) * N + n0 + bc;

    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 8; j++) acc[i][j] = 0.f;

    float4 ra0 = *reinterpret_cast<const float4*>(Ag0);
    float4 ra1 = *reinterpret_cast<const float4*>(Ag1);
    cp_async16(&Bs[0][br][bc], Bg0);
    cp_async16(&Bs[0][br + 8][bc], Bg1);
    cp_commit();
    As[0][ac + 0][ar] = ra0.x; As[0][ac + 1][ar] = ra0.y; As[0][ac + 2][ar] = ra0.z; As[0][ac + 3][ar] = ra0.w;
    As[0][ac + 0][64 + ar] = ra1.x; As[0][ac + 1][64 + ar] = ra1.y;
    As[0][ac + 2][64 + ar] = ra1.z; As[0][ac + 3][64 + ar] = ra1.w;
    cp_wait0();
    __syncthreads();

    const int nkt = K / BK;
    for (int kt = 0; kt < nkt; kt++) {
        const int cur = kt & 1, nxt = cur ^ 1;
        const bool more = kt + 1 < nkt;
        if (more) {
            ra0 = *reinterpret_cast<const float4*>(Ag0 + (kt + 1) * BK);
            ra1 = *reinterpret_cast<const float4*>(Ag1 + (kt + 1) * BK);
            cp_async16(&Bs[nxt][br][bc], Bg0 + (size_t)(kt + 1) * BK * N);
            cp_async16(&Bs[nxt][br + 8][bc], Bg1 + (size_t)(kt + 1) * BK * N);
            cp_commit();
        }
        // fragments double-buffered in registers: loads of k+1 overlap FFMAs of k
        float4 fa0[2], fa1[2], fb0[2], fb1[2];
        fa0[0] = *reinterpret_cast<const float4*>(&As[cur][0][ty * 4]);
        fa1[0] = *reinterpret_cast<const float4*>(&As[cur][0][64 + ty * 4]);
        fb0[0] = *reinterpret_cast<const float4*>(&Bs[cur][0][tx * 4]);
        fb1[0] = *reinterpret_cast<const float4*>(&Bs[cur][0][64 + tx * 4]);
#pragma unroll
        for (int k = 0; k < BK; k++) {
            const int p = k & 1, q = p ^ 1;
            if (k + 1 < BK) {
                fa0[q] = *reinterpret_cast<const float4*>(&As[cur][k + 1][ty * 4]);
                fa1[q] = *reinterpret_cast<const float4*>(&As[cur][k + 1][64 + ty * 4]);
                fb0[q] = *reinterpret_cast<const float4*>(&Bs[cur][k + 1][tx * 4]);
                fb1[q] = *reinterpret_cast<const float4*>(&Bs[cur][k + 1][64 + tx * 4]);
            }
            const float a[8] = {fa0[p].x, fa0[p].y, fa0[p].z, fa0[p].w, fa1[p].x, fa1[p].y, fa1[p].z, fa1[p].w};
            const float b[8] = {fb0[p].x, fb0[p].y, fb0[p].z, fb0[p].w, fb1[p].x, fb1[p].y, fb1[p].z, fb1[p].w};
#pragma unroll
            for (int i = 0; i < 8; i++)
#pragma unroll
                for (int j = 0; j < 8; j++) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        if (more) {
            As[nxt][ac + 0][ar] = ra0.x; As[nxt][ac + 1][ar] = ra0.y;
            As[nxt][ac + 2][ar] = ra0.z; As[nxt][ac + 3][ar] = ra0.w;
            As[nxt][ac + 0][64 + ar] = ra1.x; As[nxt][ac + 1][64 + ar] = ra1.y;
            As[nxt][ac + 2][64 + ar] = ra1.z; As[nxt][ac + 3][64 + ar] = ra1.w;
            cp_wait0();
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 8; i++) {
        const int r = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
        float* c = C + (size_t)r * N + n0;
        *reinterpret_cast<float4*>(c + tx * 4) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        *reinterpret_cast<float4*>(c + 64 + tx * 4) = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
    }
}

int main(int argc, char** argv) {
    const int shapes[3][3] = {{2048, 4096, 4096}, {2048, 4096, 12288}, {2048, 12288, 4096}};
    cublasHandle_t h;
    cublasCreate(&h);
    cublasSetMathMode(h, CUBLAS_PEDANTIC_MATH);
    for (auto& s : shapes) {
        const int M = s[0], K = s[1], N = s[2];
        std::vector<float> ha((size_t)M * K), hb((size_t)K * N);
        for (auto& v : ha) v = (float)((rand() % 2001) - 1000) / 1000.f;
        for (auto& v : hb) v = (float)((rand() % 2001) - 1000) / 1000.f;
        float *a, *b, *c, *cr;
        cudaMalloc(&a, ha.size() * 4); cudaMalloc(&b, hb.size() * 4);
        cudaMalloc(&c, (size_t)M * N * 4); cudaMalloc(&cr, (size_t)M * N * 4);
        cudaMemcpy(a, ha.data(), ha.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(b, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice);
        dim3 grid(N / BN, M / BM);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        float best = 1e9f, bestc = 1e9f;
        const float one = 1.f, zero = 0.f;
        for (int r = 0; r < 6; r++) {
            cudaEventRecord(e0);
            k_sgemm<<<grid, NT>>>(a, b, c, M, N, K);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); if (r) best = fminf(best, ms);
            cudaEventRecord(e0);
            // row-major C = A B  <=>  column-major C^T = B^T A^T
            cublasSgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, N, M, K, &one, b, N, a, K, &zero, cr, N);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1); if (r) bestc = fminf(bestc, ms);
        }
        std::vector<float> hc((size_t)M * N), hr((size_t)M * N);
        cudaMemcpy(hc.data(), c, hc.size() * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(hr.data(), cr, hr.size() * 4, cudaMemcpyDeviceToHost);
        double maxd = 0;
        for (size_t i = 0; i < hc.size(); i++) maxd = fmax(maxd, fabs((double)hc[i] - hr[i]));
        const double fl = 2.0 * M * N * K;
        printf("{\"shape\": [%d, %d, %d], \"ours_ms\": %.4f, \"ours_tflops\": %.1f, \"cublas_ms\": %.4f, "
               "\"cublas_tflops\": %.1f, \"max_abs_diff\": %.3g, \"err\": \"%s\"}\n",
               M, K, N, best, fl / best / 1e9, bestc, fl / bestc / 1e9, maxd,
               cudaGetErrorString(cudaGetLastError()));
        cudaFree(a); cudaFree(b); cudaFree(c); cudaFree(cr);
    }
    return 0;
}
