// Probe: 2D TMA tile load (fp32) into shared memory through the sm100_ptx.cuh
// wrappers, with the tensor map passed as a __grid_constant__ parameter, and
// the driver entry point resolved through cudaGetDriverEntryPoint.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_2506_22969_b200/csrc/device/sm100_ptx.cuh"
#include <cuda_runtime.h>
using namespace sst::ptx;

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ void tma_v2(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__global__ void k(const __grid_constant__ CUtensorMap tm, const CUtensorMap* gtm, float* out, int bw, int bh, int c0, int c1, int mode) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    float* tile = reinterpret_cast<float*>(smem);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    __syncthreads();
    if (threadIdx.x < 32) {
        if (mode == 0) {
            if (threadIdx.x == 0) {
                mbar_arrive_expect_tx(&bar, bw * bh * 4);
                tma_load_2d(tile, &tm, &bar, c0, c1);
            }
        } else if (mode == 2) {
            if (threadIdx.x == 0) {
                mbar_arrive_expect_tx(&bar, bw * bh * 4);
                tma_load_2d(tile, gtm, &bar, c0, c1);
            }
        } else if (mode == 3) {
            if (threadIdx.x == 0) {
                mbar_arrive_expect_tx(&bar, bw * bh * 4);
                tma_v2(tile, &tm, &bar, c0, c1);
            }
        } else {
            if (elect_one()) {
                mbar_arrive_expect_tx(&bar, bw * bh * 4);
                tma_load_2d(tile, &tm, &bar, c0, c1);
            }
        }
    }
    mbar_wait(&bar, 0);
    for (int i = threadIdx.x; i < bw * bh; i += blockDim.x) out[i] = tile[i];
}

int main(int argc, char** argv) {
    int W = 164, H = 100;
    std::vector<float> h(W * H);
    for (int i = 0; i < W * H; ++i) h[i] = float(i);
    float *d, *o;
    cudaMalloc(&d, W * H * 4);
    cudaMalloc(&o, 1 << 20);
    cudaMemcpy(d, h.data(), W * H * 4, cudaMemcpyHostToDevice);
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<EncodeTiledFn>(p);
    CUtensorMap tm;
    int bw = 132, bh = 66;
    cuuint64_t gd[2] = {(cuuint64_t)W, (cuuint64_t)H};
    cuuint64_t gs[1] = {(cuuint64_t)W * 4};
    cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)bh};
    cuuint32_t es[2] = {1, 1};
    CUresult rc = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, gd, gs, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode rc=%d\n", (int)rc);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    CUtensorMap* gtm; cudaMalloc(&gtm, sizeof(CUtensorMap)); cudaMemcpy(gtm, &tm, sizeof(tm), cudaMemcpyHostToDevice);
    int mode0 = argc > 1 ? atoi(argv[1]) : 0;
    if (argc > 2) { bw = atoi(argv[2]); bh = atoi(argv[3]);
      cuuint32_t box2[2] = {(cuuint32_t)bw, (cuuint32_t)bh};
      rc = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, gd, gs, box2, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      printf("re-encode box %d x %d rc=%d\n", bw, bh, (int)rc);
      cudaMemcpy(gtm, &tm, sizeof(tm), cudaMemcpyHostToDevice);
    }
    for (int mode = mode0; mode <= mode0; ++mode) {
        k<<<1, 128, 100000>>>(tm, gtm, o, bw, bh, 3, 10, mode);
        cudaError_t e = cudaDeviceSynchronize();
        printf("mode %d: %s\n", mode, cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
        std::vector<float> r(bw * bh);
        cudaMemcpy(r.data(), o, bw * bh * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int y = 0; y < bh; ++y)
            for (int x = 0; x < bw; ++x) {
                int gx = x + 3, gy = y + 10;
                float want = (gx < W && gy < H) ? float(gy * W + gx) : 0.f;
                bad += r[y * bw + x] != want;
            }
        printf("mode %d mismatches %d\n", mode, bad);
    }
    return 0;
}
