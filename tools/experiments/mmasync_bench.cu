// Legacy mma.sync throughput on sm_100a (TF32 m16n8k8 and BF16 m16n8k16):
// every warp issues 8 independent accumulator chains in a loop.
#include <cstdio>
#include <cuda_runtime.h>

template <int KIND>
__global__ void bench(float *out, int iters)
{
    float c[8][4] = {};
    unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    for (int i = 0; i < iters; i++)
    {
#pragma unroll
        for (int j = 0; j < 8; j++)
        {
            if (KIND == 0)
                asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                             : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                             : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
            else
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                             : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                             : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
        }
    }
    float s = 0;
    for (int j = 0; j < 8; j++)
        s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main()
{
    float *out;
    cudaMalloc(&out, 148 * 8 * 1024 * 4);
    const int iters = 20000;
    for (int kind = 0; kind < 2; kind++)
        for (int warps : {4, 8, 16})
        {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            auto k = kind == 0 ? bench<0> : bench<1>;
            k<<<148 * 2, 32 * warps>>>(out, 100);
            cudaEventRecord(e0);
            k<<<148 * 2, 32 * warps>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double flop_per_mma = kind == 0 ? 16.0 * 8 * 8 * 2 : 16.0 * 8 * 16 * 2;
            const double flops = flop_per_mma * 8 * iters * (148.0 * 2 * warps);
            printf("%s warps/CTA=%2d (2 CTA/SM): %.1f TFLOP/s\n", kind == 0 ? "tf32 m16n8k8 " : "bf16 m16n8k16", warps,
                   flops / (ms * 1e-3) / 1e12);
        }
    return 0;
}
