// Tensor-pipe time of one MLP layer issued as output parts, without the epilogue:
// the mlp_tc_kernel issue pattern (M = 256 CTA pair, A from TMEM, bf16x3 = 3 UMMAs
// per K step, 10 K steps, D regions rotating over 3 x 160 columns, two commits per
// part). Compares part splits; ideal = 2400 clk per layer (N/2 clk per UMMA).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2506_12787_b200/csrc tools/umma_parts_bench.cu -o tools/umma_parts_bench.bin
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tc_ptx.cuh"
using namespace swr::tc;

template <int N, int K0, int NK>
__device__ __forceinline__ void issue(uint32_t d, uint32_t bh, uint32_t areg)
{
    constexpr uint32_t KB = N / 2 * 16 * 2, LBO = N / 2 / 8 * 128;
    constexpr uint32_t IDESC = make_idesc(1, 256, N);
    const uint32_t b0 = desc_lo(bh, LBO);
#pragma unroll
    for (int kk = 0; kk < NK; kk++)
    {
        const int k = K0 + kk;
        const uint64_t dbh = desc_of(b0 + (k * 2 * KB >> 4), desc_hi(128));
        const uint32_t ahi = areg + 16 * k;
        mma2_f16_ts(d, ahi, dbh, IDESC, kk > 0 ? 1u : 0u);
        mma2_f16_ts(d, ahi + 8, dbh, IDESC, 1u);
        mma2_f16_ts(d, ahi, desc_of(b0 + ((k * 2 + 1) * KB >> 4), desc_hi(128)), IDESC, 1u);
    }
}

// SPLITS: 0 = (96, 64), 1 = (64, 32, 32, 32), 2 = (160), 3 = (32 x 5)
// NOISE: warps 1.. run independent FFMA chains (the epilogue's issue pressure) until the layers are done
template <int SPLITS, int NOISE = 0, int ISSUER = 0>
__global__ void __cluster_dims__(2, 1, 1) bench(long long *out, int layers)
{
    extern __shared__ __align__(1024) uint8_t smem[]; // B: 10 K x hi/lo x 80 cols x 16 x 2 B = 51 KB
    __shared__ uint64_t done, bar[8];
    __shared__ uint32_t tslot;
    __shared__ volatile int stop;
    const uint32_t rank = cluster_rank();
    const int warp = ((threadIdx.x >> 5) + 26 - ISSUER) % 26; // the issuer runs as hardware warp ISSUER
    for (int i = threadIdx.x; i < 10 * 2 * 80 * 16; i += blockDim.x)
        reinterpret_cast<uint16_t *>(smem)[i] = 0x3c00;
    if (warp == 0 && (threadIdx.x & 31) == 0)
    {
        stop = 0;
        mbar_init(&done, 1);
        for (int k = 0; k < 8; k++)
            mbar_init(&bar[k], 1);
        fence_mbar_init();
    }
    if (warp == 0)
        tmem_alloc2<512>(&tslot);
    fence_proxy_async_smem();
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = tslot;
    const uint32_t b = smem_u32(smem);
    if (rank == 0 && warp == 0)
    {
        long long t0 = clock64();
        for (int l = 0; l < layers; l++)
        {
            const uint32_t dreg = tmem + (l % 3) * 160, areg = tmem + ((l + 2) % 3) * 160;
            if (elect_one())
            {
                if (SPLITS == 0)
                {
                    issue<96, 0, 10>(dreg, b, areg);
                    mma2_commit(&bar[0], 3);
                    mma2_commit(&bar[1], 3);
                    issue<64, 0, 10>(dreg + 96, b, areg);
                    mma2_commit(&bar[2], 3);
                    mma2_commit(&bar[3], 3);
                }
                else if (SPLITS == 1)
                {
                    issue<64, 0, 10>(dreg, b, areg);
                    mma2_commit(&bar[0], 3);
                    mma2_commit(&bar[1], 3);
#pragma unroll
                    for (int p = 1; p < 4; p++)
                    {
                        issue<32, 0, 10>(dreg + 32 + 32 * p, b, areg);
                        mma2_commit(&bar[2 * p], 3);
                        mma2_commit(&bar[2 * p + 1], 3);
                    }
                }
                else if (SPLITS == 2)
                {
                    issue<160, 0, 10>(dreg, b, areg);
                    mma2_commit(&bar[0], 3);
                }
                else
                {
#pragma unroll
                    for (int p = 0; p < 5; p++)
                    {
                        issue<32, 0, 10>(dreg + 32 * p, b, areg);
                        mma2_commit(&bar[p], 3);
                    }
                }
            }
            __syncwarp();
        }
        if (elect_one())
            mma2_commit(&done, 3);
        __syncwarp();
        mbar_wait(&done, 0);
        long long t1 = clock64();
        if ((threadIdx.x & 31) == 0)
        {
            out[SPLITS] = t1 - t0;
            stop = 1;
        }
    }
    else if (warp == 0)
    {
        mbar_wait(&done, 0);
        if ((threadIdx.x & 31) == 0)
            stop = 1;
    }
    else if (NOISE)
    {
        float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
        while (!stop)
            for (int i = 0; i < 64; i++)
            {
                x0 = fmaf(x0, 0.999f, 1e-3f);
                x1 = fmaf(x1, 0.999f, 1e-3f);
                x2 = fmaf(x2, 0.999f, 1e-3f);
                x3 = fmaf(x3, 0.999f, 1e-3f);
            }
        if (x0 + x1 + x2 + x3 == 12345.f)
            out[7] = 1;
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 0)
    {
        tc_fence_after();
        tmem_dealloc2<512>(tmem);
    }
}

template <int S, int NOISE = 0, int ISSUER = 0>
void run(long long *d, const char *name)
{
    const int layers = 200;
    const int threads = NOISE ? 32 * 26 : 128;
    cudaFuncSetAttribute(bench<S, NOISE, ISSUER>, cudaFuncAttributeMaxDynamicSharedMemorySize, 60 * 1024);
    bench<S, NOISE, ISSUER><<<2, threads, 60 * 1024>>>(d, layers);
    bench<S, NOISE, ISSUER><<<2, threads, 60 * 1024>>>(d, layers);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[4];
    cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("%-22s %.0f clk per layer (ideal 2400) %s\n", name, (double)h[S] / layers, cudaGetErrorString(e));
    fflush(stdout);
}

int main()
{
    long long *d;
    cudaMalloc(&d, 64);
    run<2>(d, "one part (160)");
    run<0>(d, "parts 96/64");
    run<1>(d, "parts 64/32/32/32");
    run<3>(d, "parts 32 x 5");
    run<2, 1>(d, "one part + noise");
    run<0, 1>(d, "96/64 + noise");
    run<1, 1>(d, "64/32/32/32 + noise");
    run<3, 1>(d, "32 x 5 + noise");
    run<0, 1, 25>(d, "96/64 + noise, w25");
    run<1, 1, 25>(d, "64/32x3 + noise, w25");
    run<0, 1, 13>(d, "96/64 + noise, w13");
    return 0;
}
