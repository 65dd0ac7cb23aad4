// Throughput of back-to-back CTA-pair UMMAs (kind::f16, M = 256, K = 16, A in
// TMEM, B in shared memory) as a function of N: cycles per UMMA vs the ideal N/2
// (4096 bf16 MAC/clk/SM). Decides how finely the MLP's output parts may be cut.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2506_12787_b200/csrc tools/umma_n_bench.cu -o tools/umma_n_bench.bin
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tc_ptx.cuh"
using namespace swr::tc;

template <int N>
__global__ void __cluster_dims__(2, 1, 1) bench(long long *out, int iters)
{
    __shared__ __align__(1024) uint16_t b_s[10][N / 2 * 16];
    __shared__ uint64_t done;
    __shared__ uint32_t tslot;
    const uint32_t rank = cluster_rank();
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 10 * N / 2 * 16; i += blockDim.x)
        (&b_s[0][0])[i] = 0x3c00;
    if (threadIdx.x == 0)
    {
        mbar_init(&done, 1);
        fence_mbar_init();
    }
    if (warp == 0)
        tmem_alloc2<512>(&tslot);
    fence_proxy_async_smem();
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (rank == 0 && warp == 0)
    {
        constexpr uint32_t IDESC = make_idesc(1, 256, N);
        const uint32_t b0 = desc_lo(smem_u32(b_s), N / 2 / 8 * 128);
        long long t0 = clock64();
        if (elect_one())
        {
            for (int it = 0; it < iters; it++)
            {
#pragma unroll
                for (int k = 0; k < 10; k++)
                    mma2_f16_ts(tmem + 256, tmem + 8 * k, desc_of(b0 + (k * N / 2 * 16 * 2 >> 4), desc_hi(128)), IDESC,
                                1u);
            }
            mma2_commit(&done, 3);
        }
        __syncwarp();
        mbar_wait(&done, 0);
        long long t1 = clock64();
        if (threadIdx.x == 0)
            out[0] = t1 - t0;
    }
    else if (warp == 0)
        mbar_wait(&done, 0);
    tc_fence_before();
    cluster_sync();
    if (warp == 0)
    {
        tc_fence_after();
        tmem_dealloc2<512>(tmem);
    }
}

template <int N>
void run()
{
    long long *d, h;
    cudaMalloc(&d, 8);
    const int iters = 300;
    bench<N><<<2, 128>>>(d, iters);
    bench<N><<<2, 128>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("N=%3d: %.1f clk per UMMA (ideal %d) %s\n", N, (double)h / (iters * 10), N / 2, cudaGetErrorString(e));
    cudaFree(d);
}

int main()
{
    run<32>();
    run<64>();
    run<96>();
    run<128>();
    run<160>();
    return 0;
}
