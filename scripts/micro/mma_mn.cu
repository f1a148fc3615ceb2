// Microbenchmark: tcgen05.mma M128 N64 K16 bf16 with both operands in shared
// memory, K-major (no swizzle) vs MN-major no-swizzle with the compositor's
// padded stride (SBO = 144 B) vs MN-major no-swizzle with SBO = 128 B; one
// CTA per SM, one thread issues back-to-back MMAs into one accumulator.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2605_24290_b200/csrc/tc_util.cuh"
using namespace rxgs_b200;

template <int MODE>  // 0 K-major, 1 MN-major SBO 144, 2 MN-major SBO 128
__global__ void k(int iters, long long* out) {
    __shared__ __align__(1024) uint8_t sA[2 * 16 * 144 * 2];
    __shared__ __align__(1024) uint8_t sB[2 * 8 * 144 * 2];
    __shared__ uint64_t bar;
    __shared__ uint32_t tb;
    const int tid = threadIdx.x;
    for (int i = tid; i < static_cast<int>(sizeof(sA)) / 2; i += blockDim.x) reinterpret_cast<uint16_t*>(sA)[i] = 0x3f80;
    for (int i = tid; i < static_cast<int>(sizeof(sB)) / 2; i += blockDim.x) reinterpret_cast<uint16_t*>(sB)[i] = 0x3f80;
    if (tid < 32) { tc::tmem_alloc(&tb, 64); tc::tmem_relinquish(); }
    if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
    tc::fence_proxy_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    uint32_t idesc = tc::idesc_bf16_f32(128, 64);
    uint64_t ad, bd;
    if (MODE == 0) {
        ad = tc::sdesc_kmajor_noswizzle(tc::smem_u32(sA), 128, 256);
        bd = tc::sdesc_kmajor_noswizzle(tc::smem_u32(sB), 128, 256);
    } else {
        const uint32_t sbo = MODE == 1 ? 144 : 128;
        idesc |= (1u << 15) | (1u << 16);
        ad = tc::sdesc_kmajor_noswizzle(tc::smem_u32(sA), 16 * sbo, sbo);
        bd = tc::sdesc_kmajor_noswizzle(tc::smem_u32(sB), 8 * sbo, sbo);
    }
    long long t0 = clock64();
    if (tid == 0) {
        for (int i = 0; i < iters; ++i) tc::mma_ss(tb, ad, bd, idesc, 1u);
        tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (tid == 0) out[blockIdx.x] = t1 - t0;
    tc::fence_before_sync();
    __syncthreads();
    if (tid < 32) tc::tmem_dealloc(tb, 64);
}

template <int MODE>
void run(const char* name) {
    long long* d; cudaMalloc(&d, 148 * 8);
    const int iters = 4096;
    k<MODE><<<148, 128>>>(iters, d);
    cudaDeviceSynchronize();
    k<MODE><<<148, 128>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
    printf("%-24s %s  %.1f clk/MMA\n", name, cudaGetErrorString(e), avg / iters);
    cudaFree(d);
}

int main() {
    run<0>("K-major ss");
    run<1>("MN-major ss SBO 144");
    run<2>("MN-major ss SBO 128");
    return 0;
}
