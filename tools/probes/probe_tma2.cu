#include <cstdio>
#include <vector>
#include <cute/arch/copy_sm90_tma.hpp>
#include <cutlass/arch/barrier.h>
#include <cuda_runtime.h>
#include <cuda.h>
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__global__ void k(const __grid_constant__ CUtensorMap tm, float* out, int bw, int bh) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) { cutlass::arch::ClusterTransactionBarrier::init(&bar, 1); cutlass::arch::fence_barrier_init(); }
    __syncthreads();
    if (threadIdx.x == 0) {
        cutlass::arch::ClusterTransactionBarrier::arrive_and_expect_tx(&bar, bw*bh*4);
        cute::SM90_TMA_LOAD_2D::copy(&tm, &bar, 0, smem, 3, 10);
    }
    cutlass::arch::ClusterTransactionBarrier::wait(&bar, 0);
    float* t = (float*)smem;
    for (int i = threadIdx.x; i < bw*bh; i += blockDim.x) out[i] = t[i];
}
int main() {
    int W = 164, H = 100;
    std::vector<float> h(W*H); for (int i=0;i<W*H;++i) h[i]=float(i);
    float *d,*o; cudaMalloc(&d,W*H*4); cudaMalloc(&o,1<<20); cudaMemcpy(d,h.data(),W*H*4,cudaMemcpyHostToDevice);
    void* p=nullptr; cudaDriverEntryPointQueryResult q{};
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled",&p,cudaEnableDefault,&q);
    printf("entry %p q=%d\n", p, (int)q);
    auto enc=(EncodeTiledFn)p; CUtensorMap tm; int bw=32,bh=8;
    cuuint64_t gd[2]={(cuuint64_t)W,(cuuint64_t)H}; cuuint64_t gs[1]={(cuuint64_t)W*4};
    cuuint32_t box[2]={(cuuint32_t)bw,(cuuint32_t)bh}; cuuint32_t es[2]={1,1};
    CUresult rc=enc(&tm,CU_TENSOR_MAP_DATA_TYPE_FLOAT32,2,d,gd,gs,box,es,CU_TENSOR_MAP_INTERLEAVE_NONE,CU_TENSOR_MAP_SWIZZLE_NONE,CU_TENSOR_MAP_L2_PROMOTION_NONE,CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("rc=%d\n",(int)rc);
    cudaFuncSetAttribute(k,cudaFuncAttributeMaxDynamicSharedMemorySize,100000);
    k<<<1,128,100000>>>(tm,o,bw,bh);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    std::vector<float> r(bw*bh); cudaMemcpy(r.data(),o,bw*bh*4,cudaMemcpyDeviceToHost);
    printf("r0=%g want %g\n", r[0], float(10*W+3));
}
