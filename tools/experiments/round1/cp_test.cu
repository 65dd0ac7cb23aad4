// tcgen05.cp.cta_group::2.32x128b.warpx4 check: does a CTA pair copy each CTA's
// own 32-row shared-memory block into all four TMEM lane quarters of its own
// TMEM, and does a following UMMA (issued by the same thread) accumulate on top
// of the copied values? nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2506_12787_b200/csrc
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
#include <vector>
#include <cmath>
#include "tc_ptx.cuh"
using namespace swr::tc;

constexpr int NC = 32; // copied fp32 columns
constexpr int N = 32;  // UMMA N (cta_group::2: each CTA holds N/2 columns of B)

__device__ __forceinline__ void cp2_32x128b_x4(uint32_t taddr, uint64_t desc)
{
    asm volatile("tcgen05.cp.cta_group::2.32x128b.warpx4 [%0], %1;" ::"r"(taddr), "l"(desc) : "memory");
}

// src: [2 ranks][32 rows][NC] f32; A: [256][16] bf16 bits; B: [N][16] bf16 bits; D: [2][128][NC]
__global__ void __cluster_dims__(2, 1, 1) cp_test(const float *src, const uint16_t *A, const uint16_t *B, float *D,
                                                  int mode)
{
    __shared__ __align__(1024) float c_s[NC / 4][32][4]; // per 4-column group: 32 rows x 16 B, row-major
    __shared__ __align__(1024) uint16_t a_s[128 * 16];
    __shared__ __align__(1024) uint16_t b_s[N / 2 * 16];
    __shared__ uint64_t done;
    __shared__ uint32_t tslot;
    const uint32_t rank = cluster_rank();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 32 * NC; i += blockDim.x)
    {
        const int r = i / NC, c = i % NC;
        c_s[c / 4][r][c % 4] = src[(rank * 32 + r) * NC + c];
    }
    for (int i = threadIdx.x; i < 128 * 16; i += blockDim.x)
    {
        const int row = i / 16, k = i % 16;
        a_s[((k / 8) * 16 + row / 8) * 64 + (row % 8) * 8 + k % 8] = A[(rank * 128 + row) * 16 + k];
    }
    const int nb = N / 2, n0 = rank * N / 2;
    for (int i = threadIdx.x; i < nb * 16; i += blockDim.x)
    {
        const int n = i / 16, k = i % 16;
        b_s[((k / 8) * (nb / 8) + n / 8) * 64 + (n % 8) * 8 + k % 8] = B[(n0 + n) * 16 + k];
    }
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
        if (elect_one())
        {
            for (int g = 0; g < NC / 4; g++)
                cp2_32x128b_x4(tmem + 4 * g, desc_of(desc_lo(smem_u32(&c_s[g][0][0]), 16), desc_hi(128)));
            if (mode == 1)
            {
                constexpr uint32_t IDESC = make_idesc(1, 256, N);
                const uint64_t da = desc_of(desc_lo(smem_u32(a_s), 16 * 128), desc_hi(128));
                const uint64_t db = desc_of(desc_lo(smem_u32(b_s), N / 2 / 8 * 128), desc_hi(128));
                mma2_f16(tmem, da, db, IDESC, 1u);
            }
            mma2_commit(&done, 3);
        }
        __syncwarp();
    }
    if (warp < 4)
    {
        mbar_wait(&done, 0);
        tc_fence_after();
        float v[16];
        for (int c0 = 0; c0 < NC; c0 += 16)
        {
            tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
            for (int i = 0; i < 16; i++)
                D[((size_t)rank * 128 + warp * 32 + lane) * NC + c0 + i] = v[i];
        }
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 0)
    {
        tc_fence_after();
        tmem_dealloc2<512>(tmem);
    }
}

static float bf(uint16_t h)
{
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

int main()
{
    std::vector<float> src(2 * 32 * NC);
    for (int i = 0; i < (int)src.size(); i++)
        src[i] = (float)(i + 1) * 0.25f;
    std::vector<uint16_t> A(256 * 16), B(N * 16);
    for (int i = 0; i < (int)A.size(); i++)
        A[i] = 0x3f80 + (uint16_t)((i * 7) % 5) * 0x10; // small exact bf16 values
    for (int i = 0; i < (int)B.size(); i++)
        B[i] = 0x3e00 + (uint16_t)((i * 3) % 7) * 0x8;
    float *dsrc, *dD;
    uint16_t *dA, *dB;
    cudaMalloc(&dsrc, src.size() * 4);
    cudaMalloc(&dA, A.size() * 2);
    cudaMalloc(&dB, B.size() * 2);
    cudaMalloc(&dD, 2 * 128 * NC * 4);
    cudaMemcpy(dsrc, src.data(), src.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
    int fails = 0;
    for (int mode = 0; mode < 2; mode++)
    {
        cudaMemset(dD, 0xff, 2 * 128 * NC * 4);
        cp_test<<<2, 128>>>(dsrc, dA, dB, dD, mode);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess)
        {
            printf("mode %d: %s\n", mode, cudaGetErrorString(e));
            return 1;
        }
        std::vector<float> D(2 * 128 * NC);
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int r = 0; r < 2; r++)
            for (int row = 0; row < 128; row++)
                for (int c = 0; c < NC; c++)
                {
                    double want = src[(r * 32 + row % 32) * NC + c];
                    if (mode == 1)
                        for (int k = 0; k < 16; k++)
                            want += (double)bf(A[(r * 128 + row) * 16 + k]) * bf(B[c * 16 + k]);
                    const float got = D[((size_t)r * 128 + row) * NC + c];
                    if (fabs(got - want) > 1e-3 * fabs(want) + 1e-6)
                    {
                        if (bad < 8)
                            printf("mode %d rank %d row %d col %d: got %g want %g\n", mode, r, row, c, got, want);
                        bad++;
                    }
                }
        printf("mode %d (%s): %d mismatches of %d\n", mode, mode ? "cp + accumulating UMMA" : "cp only", bad,
               2 * 128 * NC);
        fails += bad;
    }
    return fails ? 2 : 0;
}
