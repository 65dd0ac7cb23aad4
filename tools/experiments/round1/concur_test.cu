#include <cstdio>
#include <cuda_runtime.h>
__global__ void spin(long long cycles)
{
    long long t0 = clock64();
    while (clock64() - t0 < cycles)
        ;
}
int main()
{
    cudaStream_t a, b;
    cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    spin<<<1, 32, 0, a>>>(1000);
    cudaDeviceSynchronize();
    for (int blocks : {1, 74, 148, 296})
    {
        cudaEventRecord(e0, 0);
        cudaDeviceSynchronize();
        spin<<<blocks, 128, 0, a>>>(10000000);
        spin<<<blocks, 128, 0, b>>>(10000000);
        cudaDeviceSynchronize();
        cudaEventRecord(e1, 0);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        int dev; cudaGetDevice(&dev); int cke; cudaDeviceGetAttribute(&cke, cudaDevAttrConcurrentKernels, dev);
        printf("blocks %d: two 10M-cycle kernels on 2 streams: %.2f ms (one = ~5.1 ms) concurrentKernels=%d\n", blocks, ms, cke);
    }
    return 0;
}
