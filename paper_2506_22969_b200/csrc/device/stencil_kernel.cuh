// stencil_kernel.cuh — one time step of a compiled 2:4-sparse stencil operator
// on sm_100a (2D, and the monolithic 3D variant). The reference's hot loop
// (proj/core/src/emulator.cpp:134-193, tiled_sparse_matmul with the b_entry
// provider, scattered through output_position, layout.cpp:190-209) becomes,
// per CTA batch of 8 x TYB output tiles (tile = 16 x 8 outputs, D row m = dx*8 + dy):
//
//   warp 0      TMA producer: grid patch (+halo, zero-filled outside) -> smem,
//               NP-deep ring so several patches are in flight per SM
//   warps 2-5   gather: B''[q, tile] = patch[tile_origin + koff[q]] (the
//               memory map of layout.cpp:162-188), fp32 -> fp16 (RNE, the
//               reference round16 rounding), into the UMMA MN-major operand
//   warp 1      MMA issuer: tcgen05.mma.sp.cta_group::1.kind::f16, A'' from
//               smem (compressed, K-major), metadata from TMEM, D in TMEM
//   warps 6-9   epilogue: tcgen05.ld -> 128B-swizzled smem staging -> TMA
//               bulk store through a tensor map clipped to the interior
//
// mbarrier handshakes between roles, double-buffered B operand and TMEM
// accumulator, persistent CTAs (one per SM) striding over batches.
#pragma once

#include "stencil_common.cuh"

namespace sst {

struct SmemLayout {
    uint32_t a, b, b_stride, p, p_stride, s, s_stride, gsrc, gdst, bars, tmem_slot, total;
};

__host__ __device__ inline uint32_t align_up(uint32_t v, uint32_t a) { return (v + a - 1) / a * a; }

// Shared-memory carve-up; np / nbb / ns = patch, B'' and output-staging ring
// depths, nbars mbarriers.
template <int TYB>
__host__ __device__ inline SmemLayout smem_layout_generic(int nks, int k_pad, int patch_w, int patch_h,
                                                          int planes, int np, int nbb, int nbars,
                                                          int ns = kStageBufs, bool a_in_tmem = false) {
    constexpr int N = kTXB * TYB;
    SmemLayout L{};
    uint32_t o = 0;
    L.a = o;
    o += a_in_tmem ? 0u : static_cast<uint32_t>(nks) * 4096u;
    L.b_stride = align_up(static_cast<uint32_t>(k_pad) * N * 2u, 1024);
    L.b = o = align_up(o, 1024);
    o += nbb * L.b_stride;
    L.s_stride = align_up(static_cast<uint32_t>(kBoxW * kTileH * TYB) * 4u, 1024);
    L.s = o = align_up(o, 1024);
    o += ns * (kTXB / 2) * L.s_stride;
    L.p_stride = align_up(static_cast<uint32_t>(patch_w * patch_h * planes) * 4u, 128);
    L.p = o = align_up(o, 128);
    o += np * L.p_stride;
    L.gsrc = o = align_up(o, 16);
    o += static_cast<uint32_t>(k_pad) * 4u;
    L.gdst = o;
    o += static_cast<uint32_t>(k_pad) * 4u;
    L.bars = o = align_up(o, 8);
    o += nbars * 8;
    L.tmem_slot = o;
    o += 16;
    L.total = align_up(o, 128);
    return L;
}

template <int TYB, int NP, bool AT>
__host__ __device__ inline SmemLayout smem_layout(int nks, int k_pad, int patch_w, int patch_h,
                                                  int planes) {
    return smem_layout_generic<TYB>(nks, k_pad, patch_w, patch_h, planes, NP, 2, 2 * NP + 8, kStageBufs, AT);
}

// AT: compressed A'' in TMEM (tcgen05.mma.sp [a-tmem] form) instead of smem.
template <int DIMS, int TYB, int NP, bool AT>
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
    const SmemLayout L = smem_layout<TYB, NP, AT>(p.nks, p.k_pad, p.patch_w, p.patch_h, p.patch_planes);
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
    const unsigned long long t_start = p.trace ? global_ns() : 0ull;

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
    if (warp == 1) tmem_alloc(tmem_slot, static_cast<uint32_t>(p.tmem_cols));
    stage_constants<AT>(p, sA, sB, sGsrc, sGdst);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // TMEM: two accumulators, the metadata columns, then (AT) the A'' operand
    const TmemCols tc = tmem_budget(2 * N, static_cast<uint32_t>(p.nks), AT);
    const uint32_t e_col = tc.e_col;
    if (warp >= kEpiWarp0) {
        store_metadata<AT>(p, sB, tmem, e_col, static_cast<uint32_t>(warp % 4), lane);
        if constexpr (AT) store_a_tmem(p, sB, tmem, tc.a_col, static_cast<uint32_t>(warp % 4), lane);
    }
    fence_proxy_async_smem();  // scratch (generic writes / reads) is reused by TMA below
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // everything above touches only the plan's constants: it overlaps the previous
    // time step's tail under PDL. The grid buffers are read / written only below.
    grid_dep_wait();
    grid_dep_launch();
    const unsigned long long t_main = p.trace ? global_ns() : 0ull;

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
                    tma_load_2d(dst, &tmap_in, &patch_full[s], X0 + p.load_x0, Y0);
                else
                    tma_load_3d(dst, &tmap_in, &patch_full[s], X0 + p.load_x0, Y0, Z0);
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
                    const uint64_t bd = make_smem_desc(b0 + ks * 512u, 128, b_sbo);
                    const uint32_t ea = tmem + e_col + static_cast<uint32_t>(ks);
                    if constexpr (AT) {
                        mma_sp_f16_ts(tmem + static_cast<uint32_t>(s * N), tmem + tc.a_col + ks * 8u, bd,
                                      ea & ~1u, idesc | (ea & 1u), ks > 0 ? 1u : 0u);
                    } else {
                        const uint64_t ad = make_smem_desc(a0 + ks * 4096u, 128, 256);
                        mma_sp_f16(tmem + static_cast<uint32_t>(s * N), ad, bd, ea & ~1u,
                                   idesc | (ea & 1u), ks > 0 ? 1u : 0u);
                    }
                }
                mma_commit(&b_empty[s]);
                mma_commit(&d_full[s]);
            }
            __syncwarp();
        }
    } else if (warp < kGatherWarp0 + kGatherWarps) {
        // ------------------------------------------------------------ gather
        const int gw = warp - kGatherWarp0;
        const bool active = gw < NGROUP;
        int32_t toff[GPW][8];
        tile_offsets<TYB, GPW>(gw, p.patch_w, toff);
        const uint32_t gstride = static_cast<uint32_t>(p.k_pad) * 16u;  // bytes per 8-tile group
        int it = 0;
        for (int b = blockIdx.x; b < p.nbatch; b += gridDim.x, ++it) {
            const int ps = it % NP;
            const uint32_t pph = (it / NP) & 1;
            const int s = it & 1;
            const uint32_t ph = (it >> 1) & 1;
            mbar_wait(&patch_full[ps], pph);
            mbar_wait(&b_empty[s], ph ^ 1);
            const int nsweeps = (active && !(p.debug_mode & 2)) ? p.k_pad / 32 : 0;
            gather_batch<GPW>(smem_u32(sP + ps * L.p_stride), smem_u32(sB + s * L.b_stride), sGsrc,
                              sGdst, nsweeps, gw, gstride, lane, toff);
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
        int it = 0;
        for (int b = blockIdx.x; b < p.nbatch; b += gridDim.x, ++it) {
            const int s = it & 1;
            const uint32_t ph = (it >> 1) & 1;
            int X0, Y0, Z0;
            batch_coords(b, X0, Y0, Z0);
            mbar_wait(&d_full[s], ph);
            tc_fence_after();
            uint32_t v[NBOX][CW];
            tmem_load_batch<TYB>(tmem + ((q * 32u) << 16) + static_cast<uint32_t>(s * N), v);
            tc_fence_before();  // accumulator read: hand it back to the MMA warp
            __syncwarp();
            if (lane == 0) mbar_arrive(&d_empty[s]);
            if (p.debug_mode & 1) continue;
            store_batch<DIMS, TYB, kStageBufs>(p, &tmap_out, v, sS, L.s_stride, it, X0, Y0, Z0, q, lane, etid);
        }
        if (etid == 0) bulk_wait<0>();  // stores globally complete before the CTA retires
    }

    tc_fence_before();
    __syncthreads();
    if (p.trace && threadIdx.x == 0) {
        unsigned long long* t = p.trace + 4 * blockIdx.x;
        t[0] = smid();
        t[1] = t_start;
        t[2] = t_main;
        t[3] = global_ns();
    }
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, static_cast<uint32_t>(p.tmem_cols));
    }
}

}  // namespace sst
