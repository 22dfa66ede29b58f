// stencil_kernel.cuh — one time step of a compiled 2:4-sparse stencil operator
// on sm_100a. The reference's hot loop (proj/core/src/emulator.cpp:134-193,
// tiled_sparse_matmul with the b_entry provider, scattered through
// output_position, layout.cpp:190-209) becomes, per CTA batch of
// TXB x TYB output tiles (tile = 16 x 8 outputs, D row m = dx*8 + dy):
//
//   warp 0      TMA producer: grid patch (+halo, zero-filled outside) -> smem,
//               NP-deep ring so several patches are in flight per SM
//   warps 2-5   gather: B''[q, tile] = patch[tile_origin + koff[q]] (the
//               memory map of layout.cpp:162-188), fp32 -> fp16 (RNE, the
//               reference round16 rounding), into the UMMA MN-major operand
//   warp 1      MMA issuer: tcgen05.mma.sp.cta_group::1.kind::f16, A'' from
//               smem (compressed, K-major), metadata from TMEM, D in TMEM
//   warps 6-9   epilogue: tcgen05.ld -> 128B-swizzled smem staging -> TMA
//               bulk store through a tensor map clipped to the interior, so
//               the boundary ring and ragged edges need no masking
//
// MMA column n <-> tile: output box c (32 x-cells = tiles tx = 2c, 2c+1) owns
// columns [c*2*TYB, (c+1)*2*TYB), n = c*2*TYB + 2*ty + (tx & 1), so one
// tcgen05.ld per box feeds one TMA store.
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <cstdint>

#include "sm100_ptx.cuh"

namespace sst {

constexpr int kThreads = 320;
constexpr int kGatherWarp0 = 2, kGatherWarps = 4;
constexpr int kEpiWarp0 = 6, kEpiWarps = 4;
constexpr int kTileW = 16, kTileH = 8;  // r1, r2
constexpr int kTXB = 8;                 // tiles per batch along x (128 outputs)
constexpr int kBoxW = 32;               // output box width (128 B, SWIZZLE_128B)
constexpr uint32_t kTmemCols = 256;
constexpr uint32_t kEpiBarrier = 1;     // named barrier of the 4 epilogue warps

struct StepParams {
    const uint4* a_img;        // A'' smem image (fp16), nks * 4096 bytes
    const uint32_t* e_words;   // [nks][128]
    const int32_t* gsrc;       // [nks][32] patch byte offset of the lane's B'' row
    const int32_t* gdst;       // [nks][32] byte offset of that row in an 8-tile group
    float* dst;                // output storage buffer (right-edge columns, see epilogue)
    int64_t row_pitch, plane_pitch;  // storage pitches (elements)
    int32_t left_pad;
    int32_t gx, gy, gz;        // logical extents
    int32_t r;                 // radius
    int32_t slow_lo, slow_hi;  // window over the slowest axis (y in 2D, z in 3D), interior coords
    int32_t y_end;             // interior rows (gy - 2r)
    int32_t nbx, nby, nbz, nbatch;
    int32_t k_pad, nks;
    int32_t patch_w, patch_h, patch_planes;
    int32_t debug_mode;        // ablation bits (profiling only): 1 no stores, 2 no gather, 4 no MMA
};

struct SmemLayout {
    uint32_t a, b, b_stride, p, p_stride, s, s_stride, gsrc, gdst, bars, tmem_slot, total;
};

__host__ __device__ inline uint32_t align_up(uint32_t v, uint32_t a) { return (v + a - 1) / a * a; }

template <int TYB, int NP>
__host__ __device__ inline SmemLayout smem_layout(int nks, int k_pad, int patch_w, int patch_h,
                                                  int planes) {
    constexpr int N = kTXB * TYB;
    SmemLayout L{};
    uint32_t o = 0;
    L.a = o;
    o += static_cast<uint32_t>(nks) * 4096u;
    L.b_stride = align_up(static_cast<uint32_t>(k_pad) * N * 2u, 1024);
    L.b = o = align_up(o, 1024);
    o += 2 * L.b_stride;
    L.s_stride = align_up(static_cast<uint32_t>(kBoxW * kTileH * TYB) * 4u, 1024);
    L.s = o = align_up(o, 1024);
    o += 2 * L.s_stride;
    L.p_stride = align_up(static_cast<uint32_t>(patch_w * patch_h * planes) * 4u, 128);
    L.p = o = align_up(o, 128);
    o += NP * L.p_stride;
    L.gsrc = o = align_up(o, 16);
    o += static_cast<uint32_t>(nks) * 32u * 4u;
    L.gdst = o;
    o += static_cast<uint32_t>(nks) * 32u * 4u;
    L.bars = o = align_up(o, 8);
    o += (2 * NP + 8) * 8;
    L.tmem_slot = o;
    o += 16;
    L.total = align_up(o, 128);
    return L;
}

// tile (column n of the MMA) -> (tx, ty) of the batch
template <int TYB>
__host__ __device__ inline void tile_of_column(int n, int& tx, int& ty) {
    const int c = n / (2 * TYB), m = n % (2 * TYB);
    ty = m / 2;
    tx = 2 * c + (m & 1);
}

template <int DIMS, int TYB, int NP>
__global__ void __launch_bounds__(kThreads, 1)
    stencil_step_kernel(const __grid_constant__ CUtensorMap tmap_in,
                        const __grid_constant__ CUtensorMap tmap_out, const StepParams p) {
    constexpr int N = kTXB * TYB;
    constexpr int CW = 2 * TYB;          // MMA columns per output box
    constexpr int NBOX = kTXB / 2;       // output boxes per batch
    constexpr int NGROUP = N / 8;        // 8-tile B'' groups
    constexpr int GPW = NGROUP >= kGatherWarps ? NGROUP / kGatherWarps : 1;
    static_assert(N % 16 == 0 && N <= 128, "UMMA N for M=128");
    static_assert(NGROUP % kGatherWarps == 0 || NGROUP < kGatherWarps, "group split");
    using namespace ptx;

    extern __shared__ __align__(1024) uint8_t smem[];
    const SmemLayout L = smem_layout<TYB, NP>(p.nks, p.k_pad, p.patch_w, p.patch_h, p.patch_planes);
    uint8_t* sA = smem + L.a;
    uint8_t* sB = smem + L.b;  // 2 stages
    uint8_t* sS = smem + L.s;  // 2 output staging boxes
    uint8_t* sP = smem + L.p;  // NP stages
    int32_t* sGsrc = reinterpret_cast<int32_t*>(smem + L.gsrc);
    int32_t* sGdst = reinterpret_cast<int32_t*>(smem + L.gdst);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* patch_full = bars;
    uint64_t* patch_empty = bars + NP;
    uint64_t* b_full = bars + 2 * NP;
    uint64_t* b_empty = b_full + 2;
    uint64_t* d_full = b_full + 4;
    uint64_t* d_empty = b_full + 6;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L.tmem_slot);

    const int warp = threadIdx.x / 32;
    const uint32_t lane = lane_id();

    if (threadIdx.x == 0) {
        for (int s = 0; s < NP; ++s) {
            mbar_init(&patch_full[s], 1);
            mbar_init(&patch_empty[s], kGatherWarps);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&b_full[s], kGatherWarps);
            mbar_init(&b_empty[s], 1);
            mbar_init(&d_full[s], 1);
            mbar_init(&d_empty[s], kEpiWarps);
        }
        fence_mbar_init();
        tma_prefetch_desc(&tmap_in);
        tma_prefetch_desc(&tmap_out);
    }
    if (warp == 1) tmem_alloc(tmem_slot, kTmemCols);
    {  // constant operands: A'' image, gather tables
        const int n16 = p.nks * 4096 / 16;
        uint4* dstA = reinterpret_cast<uint4*>(sA);
        for (int i = threadIdx.x; i < n16; i += kThreads) dstA[i] = p.a_img[i];
        for (int i = threadIdx.x; i < p.nks * 32; i += kThreads) {
            sGsrc[i] = p.gsrc[i];
            sGdst[i] = p.gdst[i];
        }
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t e_col = 2 * N;  // metadata columns after the two accumulators

    if (warp >= kEpiWarp0) {  // sparse metadata -> TMEM (each warp its lane quarter)
        const uint32_t q = static_cast<uint32_t>(warp % 4);
        for (int ks = 0; ks < p.nks; ++ks)
            tmem_st_32x32b_x1(tmem + ((q * 32u) << 16) + e_col + ks,
                              p.e_words[ks * 128 + q * 32 + lane]);
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    const int nbx = p.nbx, nby = p.nby;
    auto batch_coords = [&](int b, int& X0, int& Y0, int& Z0) {
        X0 = (b % nbx) * (kTXB * kTileW);
        Y0 = ((b / nbx) % nby) * (TYB * kTileH) + (DIMS == 2 ? p.slow_lo : 0);
        Z0 = b / (nbx * nby) + (DIMS == 3 ? p.slow_lo : 0);
    };

    if (warp == 0) {
        // ------------------------------------------------------ TMA producer
        if (elect_one()) {
            const uint32_t pbytes = static_cast<uint32_t>(p.patch_w * p.patch_h * p.patch_planes) * 4u;
            int it = 0;
            for (int b = blockIdx.x; b < p.nbatch; b += gridDim.x, ++it) {
                const int s = it % NP;
                const uint32_t ph = (it / NP) & 1;
                int X0, Y0, Z0;
                batch_coords(b, X0, Y0, Z0);
                mbar_wait(&patch_empty[s], ph ^ 1);
                mbar_arrive_expect_tx(&patch_full[s], pbytes);
                // storage column X0 is 16-byte aligned (TMA requirement); the
                // window origin sits left_pad cells into the patch (gsrc has it)
                void* dst = sP + s * L.p_stride;
                if (DIMS == 2)
                    tma_load_2d(dst, &tmap_in, &patch_full[s], X0, Y0);
                else
                    tma_load_3d(dst, &tmap_in, &patch_full[s], X0, Y0, Z0);
            }
        }
    } else if (warp == 1) {
        // -------------------------------------------------------- MMA issuer
        const uint32_t idesc = make_idesc_f16(128, N, true, 0, 1);
        const uint32_t b_sbo = static_cast<uint32_t>(p.k_pad) * 16u;
        const uint32_t a0 = smem_u32(sA);
        int it = 0;
        for (int b = blockIdx.x; b < p.nbatch; b += gridDim.x, ++it) {
            const int s = it & 1;
            const uint32_t ph = (it >> 1) & 1;
            mbar_wait(&b_full[s], ph);
            mbar_wait(&d_empty[s], ph ^ 1);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t b0 = smem_u32(sB + s * L.b_stride);
                const int nks = (p.debug_mode & 4) ? 1 : p.nks;
                for (int ks = 0; ks < nks; ++ks) {
                    const uint64_t ad = make_smem_desc(a0 + ks * 4096u, 128, 256);
                    const uint64_t bd = make_smem_desc(b0 + ks * 512u, 128, b_sbo);
                    const uint32_t ea = tmem + e_col + static_cast<uint32_t>(ks);
                    mma_sp_f16(tmem + static_cast<uint32_t>(s * N), ad, bd, ea & ~1u,
                               idesc | (ea & 1u), ks > 0 ? 1u : 0u);
                }
                mma_commit(&b_empty[s]);
                mma_commit(&d_full[s]);
            }
            __syncwarp();
        }
    } else if (warp < kGatherWarp0 + kGatherWarps) {
        // ------------------------------------------------------------ gather
        // warp gw owns 8-tile groups g = gw + 4*gi; lane -> one B'' row of the
        // 32-row sweep j; 8 tiles per 16-byte MN-major store
        const int gw = warp - kGatherWarp0;
        const bool active = gw < NGROUP;
        int32_t toff[GPW][8];  // patch byte offsets of the 8 tile origins of each group
#pragma unroll
        for (int gi = 0; gi < GPW; ++gi)
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                int tx, ty;
                tile_of_column<TYB>((gw + kGatherWarps * gi) * 8 + t, tx, ty);
                toff[gi][t] = (ty * kTileH * p.patch_w + tx * kTileW) * 4;
            }
        const uint32_t gstride = static_cast<uint32_t>(p.k_pad) * 16u;  // bytes per 8-tile group
        int it = 0;
        for (int b = blockIdx.x; b < p.nbatch; b += gridDim.x, ++it) {
            const int ps = it % NP;
            const uint32_t pph = (it / NP) & 1;
            const int s = it & 1;
            const uint32_t ph = (it >> 1) & 1;
            mbar_wait(&patch_full[ps], pph);
            mbar_wait(&b_empty[s], ph ^ 1);
            const uint32_t pbase = smem_u32(sP + ps * L.p_stride);
            const uint32_t bbase = smem_u32(sB + s * L.b_stride);
            const int nks = (active && !(p.debug_mode & 2)) ? p.nks : 0;
#pragma unroll 1
            for (int j = 0; j < nks; ++j) {
                const uint32_t src = pbase + static_cast<uint32_t>(sGsrc[j * 32 + lane]);
                const uint32_t dst = bbase + static_cast<uint32_t>(sGdst[j * 32 + lane]);
#pragma unroll
                for (int gi = 0; gi < GPW; ++gi) {
                    float v[8];
#pragma unroll
                    for (int t = 0; t < 8; ++t)
                        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v[t]) : "r"(src + toff[gi][t]));
                    uint32_t h[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const __half2 hv = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
                        h[i] = *reinterpret_cast<const uint32_t*>(&hv);
                    }
                    const uint32_t d = dst + static_cast<uint32_t>(gw + kGatherWarps * gi) * gstride;
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(d), "r"(h[0]),
                                 "r"(h[1]), "r"(h[2]), "r"(h[3])
                                 : "memory");
                }
            }
            fence_proxy_async_smem();  // generic-proxy writes -> tensor-core reads
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&b_full[s]);
                mbar_arrive(&patch_empty[ps]);
            }
        }
    } else {
        // ---------------------------------------------------------- epilogue
        const uint32_t q = static_cast<uint32_t>(warp % 4);
        const int etid = threadIdx.x - kEpiWarp0 * 32;  // 0..127
        const uint32_t dy = lane % 8, w4 = (lane / 8) * 4;
        const uint32_t s0 = smem_u32(sS);
        int it = 0, nbox = 0;
        for (int b = blockIdx.x; b < p.nbatch; b += gridDim.x, ++it) {
            const int s = it & 1;
            const uint32_t ph = (it >> 1) & 1;
            int X0, Y0, Z0;
            batch_coords(b, X0, Y0, Z0);
            // TMA clips the innermost dimension at 16-byte granularity, so the
            // store map ends at ox4 = ox & ~3 (the last 16-byte boundary of the
            // interior) and the <= 3 interior columns [ox4, ox) of the right-edge
            // box are written with plain stores; the boundary ring is never touched.
            const int ox = p.gx - 2 * p.r, ox4 = ox & ~3;
            const int dxl = static_cast<int>(q) * 4 + static_cast<int>(lane / 8);
            const int y_lim = DIMS == 2 ? p.slow_hi : p.y_end;
            mbar_wait(&d_full[s], ph);
            tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < NBOX; ++c, ++nbox) {
                uint32_t v[CW];
                const uint32_t taddr = tmem + ((q * 32u) << 16) + static_cast<uint32_t>(s * N + c * CW);
                if constexpr (CW == 16) {
                    tmem_ld_32x32b_x16(taddr, v);
                } else if constexpr (CW == 8) {
                    tmem_ld_32x32b_x8(taddr, v);
                } else {
                    tmem_ld_32x32b_x4(taddr, v);
                }
                tmem_wait_ld();
                if (c == NBOX - 1) {  // accumulator fully read: hand it back to the MMA warp
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&d_empty[s]);
                }
                if (p.debug_mode & 1) continue;
                const int bx0 = X0 + c * kBoxW;  // interior x of the box
                if (bx0 + kBoxW > ox4 && bx0 < ox) {
#pragma unroll
                    for (int i = 0; i < CW; ++i) {
                        const int xr = bx0 + (i & 1) * kTileW + dxl;
                        const int yr = Y0 + (i / 2) * kTileH + static_cast<int>(dy);
                        if (xr >= ox4 && xr < ox && yr < y_lim)
                            p.dst[(DIMS == 3 ? static_cast<int64_t>(Z0 + p.r) * p.plane_pitch : 0) +
                                  static_cast<int64_t>(yr + p.r) * p.row_pitch + p.left_pad + p.r + xr] =
                                __uint_as_float(v[i]);
                    }
                }
                if (bx0 >= ox4) continue;  // nothing for the TMA store in this box
                const uint32_t stage = s0 + static_cast<uint32_t>(nbox & 1) * L.s_stride;
                if (etid == 0) bulk_wait_read<1>();  // the box staged here two boxes ago is read
                named_bar_sync(kEpiBarrier, kEpiWarps * 32);
#pragma unroll
                for (int i = 0; i < CW; ++i) {
                    // local output (x, y) of D row m = 32q + lane in tile (2c + (i&1), i/2)
                    const uint32_t y = static_cast<uint32_t>(i / 2) * kTileH + dy;
                    const uint32_t chunk = (static_cast<uint32_t>(i & 1) * 4u + q) ^ dy;
                    asm volatile("st.shared.b32 [%0], %1;" ::"r"(stage + y * 128u + chunk * 16u + w4),
                                 "r"(v[i])
                                 : "memory");
                }
                fence_proxy_async_smem();
                named_bar_sync(kEpiBarrier, kEpiWarps * 32);
                if (etid == 0) {
                    if (DIMS == 2)
                        tma_store_2d(&tmap_out, sS + (nbox & 1) * L.s_stride, X0 + c * kBoxW,
                                     Y0 - p.slow_lo);  // map starts at the window
                    else
                        tma_store_3d(&tmap_out, sS + (nbox & 1) * L.s_stride, X0 + c * kBoxW, Y0, Z0);
                    bulk_commit();
                }
            }
        }
        if (etid == 0) bulk_wait<0>();  // stores globally complete before the CTA retires
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, kTmemCols);
    }
}

}  // namespace sst
