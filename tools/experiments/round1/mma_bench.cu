// Microbenchmark: tcgen05.mma kind::f16 throughput per SM for M=128 and a few N,
// A from shared memory (SS) or from TMEM (TS). Build + run on a B200:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2506_12787_b200/csrc tools/mma_bench.cu -o /tmp/mma_bench && /tmp/mma_bench
#include <cstdio>
#include <cstdint>
#include "tc_ptx.cuh"

using namespace swr::tc;

template <int N, bool TS, int CEVERY = 0, int FENCE = 0>
__global__ void bench(long long *out, int iters)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint64_t bar2[8];
    __shared__ uint64_t bar3;
    __shared__ int flag;
    __shared__ uint32_t tslot;
    if (threadIdx.x == 0)
    {
        mbar_init(&bar, 1);
        for (int k = 0; k < 8; k++)
            mbar_init(&bar2[k], 1);
        mbar_init(&bar3, 1);
        flag = 1;
        fence_mbar_init();
    }
    if (threadIdx.x < 32)
        tmem_alloc<512>(&tslot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    const uint32_t idesc = make_idesc(1, 128, N);
    long long t0 = 0, t1 = 0;
    if ((FENCE & 64) && threadIdx.x == 32)
    {
        for (int i = 0; i < iters * 2; i++)
            mbar_wait(&bar3, 1);
    }
    if ((FENCE & 128) && threadIdx.x < 32)
    {
        const uint32_t a = smem_u32(sm), b = a + 128 * 16 * 2 * 8;
        const uint64_t da = make_desc(a, 128 * 16, 128), db = make_desc(b, N * 16, 128);
        t0 = clock64();
        for (int i = 0; i < iters; i++)
        {
            uint32_t pred;
            asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
            if (pred)
                mma_f16_ts(tmem, tmem + 256, db, idesc, i > 0);
            __syncwarp();
            if (CEVERY && (i % CEVERY) == CEVERY - 1)
            {
                if (pred)
                    mma_commit(&bar2[(i / CEVERY) & 7]);
                __syncwarp();
                if (FENCE & 2)
                    mbar_wait(&bar3, 1);
            }
        }
        if (threadIdx.x == 0)
        {
            mma_commit(&bar);
            mbar_wait(&bar, 0);
            t1 = clock64();
            out[blockIdx.x] = t1 - t0;
        }
    }
    else if (!(FENCE & 128) && threadIdx.x == 0)
    {
        const uint32_t a = smem_u32(sm), b = a + 128 * 16 * 2 * 8;
        const uint64_t da = make_desc(a, 128 * 16, 128), db = make_desc(b, N * 16, 128);
        t0 = clock64();
        for (int i = 0; i < iters; i++)
        {
            if (TS)
                mma_f16_ts(tmem, tmem + 256, db, idesc, i > 0);
            else
                mma_f16(tmem, da, db, idesc, i > 0);
            if (CEVERY && (i % CEVERY) == CEVERY - 1)
            {
                if (!(FENCE & 16))
                    mma_commit(&bar2[(i / CEVERY) & 7]);
                if (FENCE & 1)
                    tc_fence_after();
                if (FENCE & 2)
                    mbar_wait(&bar3, 1); // already-complete phase: returns at once
                if (FENCE & 4)
                    while (!mbar_test_wait(&bar3, 1)) {}
                if (FENCE & 8)
                    while (!mbar_try_wait_relaxed(&bar3, 1)) {}
                if (FENCE & 32)
                {
                    int f;
                    asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(f) : "r"(smem_u32(&flag)));
                    if (f != 1)
                        printf("x");
                }
            }
        }
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32)
    {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

template <int N, bool TS, int CEVERY = 0, int FENCE = 0>
void run(int sms)
{
    long long *d, h[256];
    cudaMalloc(&d, sizeof(h));
    const int iters = 4000;
    cudaFuncSetAttribute(bench<N, TS, CEVERY, FENCE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    bench<N, TS, CEVERY, FENCE><<<sms, 128, 200 * 1024>>>(d, iters);
    bench<N, TS, CEVERY, FENCE><<<sms, 128, 200 * 1024>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < sms; i++)
        avg += h[i];
    avg /= sms;
    const double cyc = avg / iters;
    const double macs = 128.0 * N * 16;
    printf("fence%d commit/%d M=128 N=%3d %s: %6.1f cycles/MMA  ideal %5.1f  (%.0f MAC/cycle/SM) %s\n", FENCE, CEVERY, N,
           TS ? "TS" : "SS", cyc, 128.0 * N / 256.0, macs / cyc, cudaGetErrorString(e));
    cudaFree(d);
}


// stage-loop mimic: converged warp, per batch: wait (complete barrier) -> BATCH MMAs -> commit
template <int N, int BATCH, int WAITMODE>
__global__ void stage_bench(long long *out, int batches)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full, empty[4];
    __shared__ uint32_t tslot;
    if (threadIdx.x == 0)
    {
        mbar_init(&full, 1);
        for (int k = 0; k < 4; k++)
            mbar_init(&empty[k], 1);
        fence_mbar_init();
    }
    if (threadIdx.x < 32)
        tmem_alloc<512>(&tslot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (threadIdx.x == 0)
        mbar_arrive(&full); // phase 0 complete
    __syncthreads();
    const uint32_t idesc = make_idesc(1, 128, N);
    if (threadIdx.x < 32)
    {
        const uint32_t b = smem_u32(sm) + 65536;
        const uint64_t db = make_desc(b, N * 16, 128);
        long long t0 = clock64();
        for (int j = 0; j < batches; j++)
        {
            if (WAITMODE == 1)
                mbar_wait(&full, 0);
            if (WAITMODE == 2)
                mbar_poll(&full, 0);
            tc_fence_after();
            if (elect_one())
            {
#pragma unroll
                for (int k = 0; k < BATCH; k++)
                    mma_f16_ts(tmem, tmem + 256 + 8 * (k % 8), db + 16 * (k % 4), idesc, (j | k) > 0);
                mma_commit(&empty[j & 3]);
            }
            __syncwarp();
        }
        if (threadIdx.x == 0)
        {
            mma_commit(&full);
            mbar_wait(&full, 1);
            out[blockIdx.x] = clock64() - t0;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32)
    {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

template <int N, int BATCH, int WAITMODE>
void run_stage(int sms)
{
    long long *d, h[256];
    cudaMalloc(&d, sizeof(h));
    const int batches = 4000 / BATCH;
    cudaFuncSetAttribute(stage_bench<N, BATCH, WAITMODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    stage_bench<N, BATCH, WAITMODE><<<sms, 128, 200 * 1024>>>(d, batches);
    stage_bench<N, BATCH, WAITMODE><<<sms, 128, 200 * 1024>>>(d, batches);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < sms; i++)
        avg += h[i];
    avg /= sms;
    printf("stage N=%3d batch=%2d wait=%d: %6.1f cycles/MMA ideal %5.1f %s\n", N, BATCH, WAITMODE,
           avg / (batches * BATCH), 128.0 * N / 256.0, cudaGetErrorString(e));
    cudaFree(d);
}

// stage loop with SPIN extra warps blocked in mbar_wait, SS: A from shared memory
template <int N, int BATCH, int SPIN, int SS, int NACC = 2>
__global__ void stage_bench2(long long *out, int batches)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full, done, empty[4];
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0)
    {
        mbar_init(&full, 1);
        mbar_init(&done, 1);
        for (int k = 0; k < 4; k++)
            mbar_init(&empty[k], 1);
        fence_mbar_init();
    }
    if (warp == SPIN)
        tmem_alloc<512>(&tslot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (threadIdx.x == 0)
        mbar_arrive(&full);
    __syncthreads();
    const uint32_t idesc = make_idesc(1, 128, N);
    if (warp == SPIN)
    {
        const uint32_t b = smem_u32(sm) + 65536;
        const uint32_t abase = smem_u32(sm);
        const uint64_t db = make_desc(b, N * 16, 128);
        long long t0 = clock64();
        for (int j = 0; j < batches; j++)
        {
            mbar_wait(&full, 0);
            tc_fence_after();
            if (elect_one())
            {
#pragma unroll
                for (int k = 0; k < BATCH; k++)
                {
                    const uint32_t d = tmem + 160 * (j % 3) + (NACC == 1 ? 0 : 80 * (k & 1));
                    if (SS)
                        mma_f16(d, make_desc(abase + 4096 * (k % 3), 2048, 128), db + 16 * (k % 4), idesc, (j | k) > 0);
                    else
                        mma_f16_ts(d, tmem + 160 * ((j + 2) % 3) + 16 * (k % 10) + 8 * (k & 1), db + 16 * (k % 4),
                                   idesc, (j | k) > 0);
                }
                mma_commit(&empty[j & 3]);
            }
            __syncwarp();
        }
        if (threadIdx.x == 32 * SPIN)
        {
            mma_commit(&full);
            mbar_wait(&full, 1);
            out[blockIdx.x] = clock64() - t0;
            mbar_arrive(&done);
        }
    }
    else
        mbar_wait(&done, 0);
    tc_fence_before();
    __syncthreads();
    if (warp == SPIN)
    {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

template <int N, int BATCH, int SPIN, int SS, int NACC = 2>
void run_stage2(int sms)
{
    long long *d, h[256];
    cudaMalloc(&d, sizeof(h));
    const int batches = 4000 / BATCH;
    auto k = stage_bench2<N, BATCH, SPIN, SS, NACC>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    k<<<sms, 32 * (SPIN + 1), 200 * 1024>>>(d, batches);
    k<<<sms, 32 * (SPIN + 1), 200 * 1024>>>(d, batches);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < sms; i++)
        avg += h[i];
    avg /= sms;
    printf("stage2 nacc=%d N=%3d batch=%2d spin=%2d ss=%d: %6.1f cycles/MMA ideal %5.1f %s\n", NACC, N, BATCH, SPIN, SS,
           avg / (batches * BATCH), 128.0 * N / 256.0, cudaGetErrorString(e));
    cudaFree(d);
}
int main()
{
    int sms = 148;
    run_stage2<80, 15, 0, 0, 1>(sms);
    run_stage2<80, 15, 0, 0, 2>(sms);
    run_stage2<64, 15, 0, 0, 1>(sms);
    run_stage2<128, 15, 0, 0, 1>(sms);
    run_stage2<160, 15, 0, 0, 1>(sms);
    return 0;
}
