// Hardware probe: does a TMA tensor store clip the innermost dimension exactly at
// the tensor extent, or in 16-byte units? Tensor map over rows of pitch 520 fp32
// with inner extent E (508..512); one {32, 4} box stored at x = 480 from smem;
// reports which columns >= 480 of the first row were written.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2506_22969_b200/csrc/device/sm100_ptx.cuh"

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void k(const __grid_constant__ CUtensorMap tm, int x0) {
    __shared__ __align__(128) float tile[4 * 32];
    for (int i = threadIdx.x; i < 128; i += blockDim.x) tile[i] = static_cast<float>(x0 + i % 32);
    sst::ptx::fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
        sst::ptx::tma_store_2d(&tm, tile, x0, 0);
        sst::ptx::bulk_commit();
        sst::ptx::bulk_wait<0>();
    }
}

int main() {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto encode = reinterpret_cast<EncodeTiledFn>(fn);
    const int pitch = 520, rows = 8;
    float* d;
    cudaMalloc(&d, pitch * rows * 4);
    for (int E = 508; E <= 512; ++E) {
        std::vector<float> h(pitch * rows, -1.f);
        cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
        CUtensorMap tm;
        cuuint64_t dim[2] = {static_cast<cuuint64_t>(E), static_cast<cuuint64_t>(rows)};
        cuuint64_t stride[1] = {pitch * 4};
        cuuint32_t box[2] = {32, 4}, es[2] = {1, 1};
        CUresult rc = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dim, stride, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (rc != CUDA_SUCCESS) {
            printf("E=%d encode failed %d\n", E, rc);
            continue;
        }
        k<<<1, 128>>>(tm, 480);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
        int last = -1;
        for (int x = 480; x < pitch; ++x)
            if (h[x] != -1.f) last = x;
        printf("extent E=%d: %s, last written column %d (%s)\n", E, cudaGetErrorString(e), last,
               last == E - 1 ? "exact clip" : "NOT exact");
    }
    return 0;
}
