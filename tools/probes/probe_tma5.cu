#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cute/arch/copy_sm90_tma.hpp>
#include <cutlass/arch/barrier.h>
#include <cuda_runtime.h>
#include <cuda.h>
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__global__ void k(const __grid_constant__ CUtensorMap tm, float* out, int bw, int bh, int getenv_mode) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) { cutlass::arch::ClusterTransactionBarrier::init(&bar, 1); cutlass::arch::fence_barrier_init(); }
    __syncthreads();
    if (threadIdx.x == 0) {
        cutlass::arch::ClusterTransactionBarrier::arrive_and_expect_tx(&bar, bw*bh*4);
        if (getenv_mode == 1) {
            uint32_t d = (uint32_t)__cvta_generic_to_shared(smem), b = (uint32_t)__cvta_generic_to_shared(&bar);
            asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                :: "r"(d), "l"((uint64_t)&tm), "r"(b), "r"(3), "r"(10) : "memory");
        } else
        cute::SM90_TMA_LOAD_2D::copy(&tm, &bar, 0, smem, getenv_mode >= 10 ? getenv_mode - 10 : 3, 10);
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
    auto enc = getenv("DIRECT") ? (EncodeTiledFn)&cuTensorMapEncodeTiled : (EncodeTiledFn)p; CUtensorMap tm; int bw=32,bh=8;
    cuuint64_t gd[2]={(cuuint64_t)W,(cuuint64_t)H}; cuuint64_t gs[1]={(cuuint64_t)W*4};
    cuuint32_t box[2]={(cuuint32_t)bw,(cuuint32_t)bh}; cuuint32_t es[2]={1,1};
    CUresult rc=enc(&tm,CU_TENSOR_MAP_DATA_TYPE_FLOAT32,2,d,gd,gs,box,es,CU_TENSOR_MAP_INTERLEAVE_NONE,CU_TENSOR_MAP_SWIZZLE_NONE,CU_TENSOR_MAP_L2_PROMOTION_NONE,CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("rc=%d\n",(int)rc); { const unsigned long long* w=(const unsigned long long*)&tm; for(int i=0;i<16;++i) printf("%016llx%s", w[i], i%4==3?"\n":" "); }
    cudaFuncSetAttribute(k,cudaFuncAttributeMaxDynamicSharedMemorySize,100000);
    int mode = getenv("MODE") ? atoi(getenv("MODE")) : 0;
    if (getenv("CLUSTER")) {
        cudaLaunchConfig_t cfg{}; cfg.gridDim = dim3(1); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = 100000;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        printf("launchEx: %s\n", cudaGetErrorString(cudaLaunchKernelEx(&cfg, k, tm, o, bw, bh, mode)));
    } else k<<<1,128,100000>>>(tm,o,bw,bh,mode);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    std::vector<float> r(bw*bh); cudaMemcpy(r.data(),o,bw*bh*4,cudaMemcpyDeviceToHost);
    printf("r0=%g want %g\n", r[0], float(10*W+3));
}
