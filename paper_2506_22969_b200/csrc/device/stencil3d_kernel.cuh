// stencil3d_kernel.cuh — z-streaming variant of the step kernel for 3D stencils.
//
// A 3D stencil's A'' is z-major (expand_units, convert.cpp:376-396): KZ slices of
// C columns, slice dz holding the weights of input plane z = dz of the window.
// The output plane zo is therefore sum_dz A_dz * B(zo + dz), where B(z) is the
// 2D-window gather of ONE input plane. Instead of gathering a kz-plane window per
// output plane (kz times the gather and smem traffic), a CTA walks a run of
// output planes of one (x, y) column and, per input plane z:
//
//   TMA    one plane patch (ring of NP)           warp 0
//   gather B(z) once (K = C rounded to 32)        warps 2-5
//   MMA    D(z - dz) += A_dz * B(z), dz = 0..KZ-1  warp 1 (accumulators live in a
//          TMEM ring of NACC = KZ + 1 slots; D(z - KZ + 1) completes each plane)
//   store  completed D planes                      warps 6-9
//
// Work split: output units (column, zo) in column-major order are cut into one
// contiguous range per CTA (perfect balance); a range re-enters the pipeline
// (2r extra planes) only where it starts a new column.
#pragma once

#include "stencil_kernel.cuh"

namespace sst {

// Right-edge ring cache (see kEdgeRing in stencil_common.cuh): one slot per
// gathered input plane, ring_slots<NP, NB, NACC>() deep. The PRODUCER fills slot
// it % slots when it issues plane it; slot reuse is safe by pipeline depth: the
// producer issues plane it + slots only after the gather of plane it + slots - NP
// (patch_empty), which waited (b_empty) for the MMA of plane it + slots - NP - NB,
// which waited (d_empty) for the epilogue to release output it + slots - NP - NB -
// NACC; with slots > NP + NB + NACC that is past output it - R + 1, so the last
// reader of slot it (output it - R, center plane it) is done.
template <int NP, int NB, int NACC>
__host__ __device__ constexpr int ring_slots() {
    return NP + NB + NACC + 1 <= 16 ? 16 : 32;
}

// elem: patch element bytes (4 fp32 storage, 2 binary16 inter-step storage). A ring
// slot is 16 bytes per output row in both cases (4 fp32 or 8 binary16 cells).
template <int TYB, int NP, int KZ, int NB, int NACC, int NS, bool AT>
__host__ __device__ inline SmemLayout smem_layout_stream(int nks, int k_pad, int patch_w, int patch_h,
                                                         int elem = 4) {
    constexpr int kRingSlots = ring_slots<NP, NB, NACC>();
    static_assert(kRingSlots > NP + NB + NACC, "ring cache slots vs pipeline depth");
    SmemLayout L = smem_layout_generic<TYB>(nks, k_pad, patch_w, patch_h, 1, NP, NB,
                                            2 * NP + 2 * NB + 2 * NACC + kRingSlots, NS, AT, elem);
    L.ring = align_up(L.total, 16);
    L.total = align_up(L.ring + static_cast<uint32_t>(kRingSlots * TYB * kTileH * 4 * 4), 128);
    return L;
}

// Iterates the runs of a CTA's unit range: calls fn(band, zo_a, zo_b) for each run
// (window-relative output planes, inclusive). Units are ordered z-chunk-major:
// u = (zc * nby + band) * L + zl for chunks of L = zchunk planes (the last one
// shorter), so at any time all groups work inside one slab of ~L planes
// (locality for DRAM pages and L2; the y halo shared by consecutive bands of a
// group hits in L2), at the cost of 2r re-entry planes per L outputs. zchunk = 0:
// one chunk (runs are whole columns).
template <class Fn>
__device__ __forceinline__ void for_each_run(int u0, int u1, int ozw, int nby, int zchunk, Fn&& fn) {
    const int L = zchunk > 0 && zchunk < ozw ? zchunk : ozw;
    const int nzc = (ozw + L - 1) / L;
    for (int u = u0; u < u1;) {
        const int zc = min(u / (nby * L), nzc - 1);
        const int Lc = zc == nzc - 1 ? ozw - zc * L : L;
        const int rem = u - nby * L * zc;
        const int band = rem / Lc, zl = rem % Lc;
        const int len = min(u1 - u, Lc - zl);
        fn(band, zc * L + zl, zc * L + zl + len - 1);
        u += len;
    }
}

// NB: B'' ring depth, NACC (> KZ): accumulator ring, NS: output staging buffers,
// AT: compressed A'' in TMEM instead of smem (frees smem and its bandwidth: with
// N = 32 the per-MMA A reads were the largest smem stream of the 3D kernel).
// PEER: the slab P2P halo stores are compiled in (launched only when p.peer_mask != 0)
// HIN / HOUT: the input / output grid is binary16 storage (SST_PREC_F16 runs keep steps
// 1 .. T-1 in binary16, see typed2d.cuh): binary16 patches are gathered by copying the
// bits, binary16 outputs are rounded RNE in the epilogue. The right-edge ring cache
// always holds the OUTPUT storage's ring chunk (maps.ring[p.src] then maps the output
// buffer: its ring cells are constant and equal to the input's): 4 fp32 or 8 binary16
// cells per row, 16 bytes either way.
template <int TYB, int NP, int KZ, int NB, int NACC, int NS, bool AT, bool PEER = false, bool HIN = false,
          bool HOUT = false>
__global__ void __launch_bounds__(kThreads, 1)
    stencil3d_stream_kernel(const __grid_constant__ MapSet maps, const StepParams p) {
    constexpr int N = kTXB * TYB;
    constexpr int CW = 2 * TYB;
    constexpr int NBOX = kTXB / 2;
    constexpr int NGROUP = N / 8;
    constexpr int GPW = NGROUP >= kGatherWarps ? NGROUP / kGatherWarps : 1;
    constexpr int R = (KZ - 1) / 2;
    constexpr int kRingSlots = ring_slots<NP, NB, NACC>();
    static_assert(NACC > KZ, "one accumulator beyond the KZ open ones");
    static_assert(N % 16 == 0 && N <= 128, "UMMA N for M=128");
    static_assert(NACC * N <= 320, "accumulator ring must leave TMEM room for metadata / A''");
    constexpr int ELEM = HIN ? 2 : 4;   // patch element bytes
    constexpr int RW = HOUT ? 8 : 4;    // cells per 16-byte output chunk (ring cache row)
    using namespace ptx;

    extern __shared__ __align__(1024) uint8_t smem[];
    const SmemLayout L =
        smem_layout_stream<TYB, NP, KZ, NB, NACC, NS, AT>(p.nks, p.k_pad, p.patch_w, p.patch_h, ELEM);
    uint8_t* sA = smem + L.a;
    uint8_t* sB = smem + L.b;
    uint8_t* sS = smem + L.s;
    uint8_t* sP = smem + L.p;
    int32_t* sGsrc = reinterpret_cast<int32_t*>(smem + L.gsrc);
    int32_t* sGdst = reinterpret_cast<int32_t*>(smem + L.gdst);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* patch_full = bars;
    uint64_t* patch_empty = bars + NP;
    uint64_t* b_full = bars + 2 * NP;
    uint64_t* b_empty = b_full + NB;
    uint64_t* d_full = b_full + 2 * NB;
    uint64_t* d_empty = d_full + NACC;
    uint64_t* ring_full = d_empty + NACC;  // [kRingSlots]
    uint8_t* sRing = smem + L.ring;  // [kRingSlots][TYB*8 rows][16 bytes]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L.tmem_slot);

    const int warp = threadIdx.x / 32;
    const uint32_t lane = lane_id();
    const unsigned long long t_start = p.trace ? global_ns() : 0ull;
    const int ksz = p.k_pad / 32;  // K steps per z slice

    if (threadIdx.x == 0) {
        for (int s = 0; s < NP; ++s) {
            mbar_init(&patch_full[s], 1);
            mbar_init(&patch_empty[s], kGatherWarps);
        }
        for (int s = 0; s < NB; ++s) {
            mbar_init(&b_full[s], kGatherWarps);
            mbar_init(&b_empty[s], 1);
        }
        for (int s = 0; s < NACC; ++s) {
            mbar_init(&d_full[s], 1);
            mbar_init(&d_empty[s], kEpiWarps);
        }
        for (int s = 0; s < kRingSlots; ++s) mbar_init(&ring_full[s], 1);
        fence_mbar_init();
        tma_prefetch_desc(&maps.in[p.src]);
        tma_prefetch_desc(&maps.out[p.src ^ 1]);
        tma_prefetch_desc(&maps.ring[p.src]);
    }
    if (warp == 1) tmem_alloc(tmem_slot, static_cast<uint32_t>(p.tmem_cols));
    uint64_t* pbar = reinterpret_cast<uint64_t*>(smem + L.pbar);
    if (threadIdx.x == 0) {
        mbar_init(pbar, 1);
        fence_mbar_init();
        stage_constants_issue<AT>(p, sA, sB, sGsrc, sGdst, pbar);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    mbar_wait(pbar, 0);  // constants in smem
    const unsigned long long t_mid = p.trace ? global_ns() : 0ull;  // constants staged, TMEM allocated
    const uint32_t tmem = *tmem_slot;
    const TmemCols tc = tmem_budget(NACC * N, static_cast<uint32_t>(p.nks), AT);
    const uint32_t e_col = tc.e_col;  // metadata after the accumulator ring, then A'' (AT)
    if (warp >= kEpiWarp0) {
        store_metadata<AT>(p, sB, tmem, e_col, static_cast<uint32_t>(warp % 4), lane);
        if constexpr (AT) store_a_tmem(p, sB, tmem, tc.a_col, static_cast<uint32_t>(warp % 4), lane);
    }
    fence_proxy_async_smem();  // scratch (generic writes / reads) is reused by TMA below
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    grid_dep_wait();  // grid buffers only below (PDL: the prologue overlaps the previous step)
    grid_dep_launch();
    const unsigned long long t_main = p.trace ? global_ns() : 0ull;

    // Work split. The grid is (groups x nbx) CTAs: CTA = (group, bx). All CTAs of a
    // group walk the same contiguous range of (by, output plane) units, one per x
    // column bx, so at any time the x-adjacent columns of a row band are in flight
    // together: their patch rows are contiguous in HBM (DRAM page locality) and the
    // x halos they share hit in L2.
    const CUtensorMap* tmap_in = &maps.in[p.src];  // one time step per launch
    const CUtensorMap* tmap_out = &maps.out[p.src ^ 1];
    const int ozw = p.slow_hi - p.slow_lo;
    const int bx = blockIdx.x % p.nbx, grp = blockIdx.x / p.nbx, ngrp = gridDim.x / p.nbx;
    const int64_t units = static_cast<int64_t>(p.nby) * ozw;
    const int u0 = static_cast<int>(units * grp / ngrp);
    const int u1 = static_cast<int>(units * (grp + 1) / ngrp);
    auto col_xy = [&](int by, int& X0, int& Y0) {
        X0 = bx * (kTXB * kTileW);
        Y0 = by * (TYB * kTileH);
    };

    if (warp == 0 && !(dbg(p) & 32)) {
        // ------------------------------------------------------ TMA producer
        if (elect_one()) {
            const uint32_t pbytes = static_cast<uint32_t>(p.patch_w * p.patch_h * ELEM);
            const int ox = p.gx - 2 * p.r, oxc = ox & ~(RW - 1);
            const bool edge = oxc != ox && bx * (kTXB * kTileW) + kTXB * kTileW > ox && !(dbg(p) & 24);
            int it = 0;
            for_each_run(u0, u1, ozw, p.nby, p.zchunk, [&](int col, int zo_a, int zo_b) {
                int X0, Y0;
                col_xy(col, X0, Y0);
                // input (storage) planes of outputs zo_a..zo_b: zo_a .. zo_b + 2R
                for (int z = p.slow_lo + zo_a; z <= p.slow_lo + zo_b + 2 * R; ++z, ++it) {
                    const int s = it % NP;
                    if (dbg(p) & 16) {  // TMA-only: the producer recycles its own ring
                        if (it >= NP) mbar_wait(&patch_full[s], ((it / NP) - 1) & 1);
                    } else {
                        mbar_wait(&patch_empty[s], ((it / NP) & 1) ^ 1);
                    }
                    mbar_arrive_expect_tx(&patch_full[s], pbytes);
                    tma_load_3d(sP + s * L.p_stride, tmap_in, &patch_full[s], X0 + p.load_x0, Y0, z);
                    if (edge) {  // right-edge chunk [oxc, oxc + RW) of the TYB*8 output rows
                        const int rs = it % kRingSlots;
                        mbar_arrive_expect_tx(&ring_full[rs], static_cast<uint32_t>(TYB * kTileH * 16));
                        tma_load_3d(sRing + rs * (TYB * kTileH * 16), &maps.ring[p.src], &ring_full[rs],
                                    static_cast<int>(p.left_pad) + p.r + oxc, Y0 + p.r, z);
                    }
                }
            });
            if (dbg(p) & 16)
                for (int j = (it > NP ? it - NP : 0); j < it; ++j) mbar_wait(&patch_full[j % NP], (j / NP) & 1);
        }
    } else if (dbg(p) & 16) {
        // TMA-only ablation: the other roles idle
    } else if ((dbg(p) & 32) && warp < kEpiWarp0) {
        // store-only ablation: only the epilogue runs (writes zeros)
    } else if (warp == 1) {
        // -------------------------------------------------------- MMA issuer
        const uint32_t idesc = make_idesc_f16(128, N, true, 0, 1);
        const uint32_t b_sbo = static_cast<uint32_t>(p.k_pad) * 16u;
        const uint32_t a0 = smem_u32(sA);
        int it = 0, obase = 0;
        for_each_run(u0, u1, ozw, p.nby, p.zchunk, [&](int col, int zo_a, int zo_b) {
            (void)col;
            for (int zi = zo_a; zi <= zo_b + 2 * R; ++zi, ++it) {  // window-relative input plane
                const int s = it % NB;
                mbar_wait(&b_full[s], (it / NB) & 1);
                // a new accumulator starts at dz = 0 (zo = zi): wait until it is drained
                if (zi <= zo_b) {
                    const int o = obase + (zi - zo_a);
                    mbar_wait(&d_empty[o % NACC], ((o / NACC) & 1) ^ 1);
                }
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t b0 = smem_u32(sB + s * L.b_stride);
#pragma unroll
                    // K step outer, z slice inner: consecutive MMAs go to the KZ different
                    // accumulators (independent), not KZ chains of dependent ones
                    const int nk = (dbg(p) & 4) ? 1 : ksz;
                    for (int ks = 0; ks < nk; ++ks) {
                        const uint64_t bd = make_smem_desc(b0 + ks * 512u, 128, b_sbo);
#pragma unroll
                        for (int dz = 0; dz < KZ; ++dz) {
                            const int zo = zi - dz;
                            if (zo < zo_a || zo > zo_b) continue;
                            const int slot = (obase + (zo - zo_a)) % NACC;
                            const int kk = dz * ksz + ks;  // A'' / metadata K step
                            const uint32_t ea = tmem + e_col + static_cast<uint32_t>(kk);
                            const uint32_t acc = (dz > 0 || ks > 0) ? 1u : 0u;
                            if constexpr (AT) {
                                mma_sp_f16_ts(tmem + static_cast<uint32_t>(slot * N),
                                              tmem + tc.a_col + static_cast<uint32_t>(kk) * 8u, bd, ea & ~1u,
                                              idesc | (ea & 1u), acc);
                            } else {
                                const uint64_t ad = make_smem_desc(a0 + kk * 4096u, 128, 256);
                                mma_sp_f16(tmem + static_cast<uint32_t>(slot * N), ad, bd, ea & ~1u,
                                           idesc | (ea & 1u), acc);
                            }
                        }
                    }
                    mma_commit(&b_empty[s]);
                    const int zdone = zi - 2 * R;  // its last contribution was just issued
                    if (zdone >= zo_a && zdone <= zo_b) mma_commit(&d_full[(obase + zdone - zo_a) % NACC]);
                }
                __syncwarp();
            }
            obase += zo_b - zo_a + 1;
        });
    } else if (warp < kGatherWarp0 + kGatherWarps) {
        // ------------------------------------------------------------ gather
        const int gw = warp - kGatherWarp0;
        const bool active = gw < NGROUP;
        int32_t toff[GPW][8];
        tile_offsets<TYB, GPW, ELEM>(gw, p.patch_w, toff);
        const uint32_t gstride = static_cast<uint32_t>(p.k_pad) * 16u;
        const int nsweeps = (active && !(dbg(p) & 2)) ? ksz : 0;
        int it = 0;
        for_each_run(u0, u1, ozw, p.nby, p.zchunk, [&](int col, int zo_a, int zo_b) {
            (void)col;
            for (int zi = zo_a; zi <= zo_b + 2 * R; ++zi, ++it) {
                const int ps = it % NP, s = it % NB;
                mbar_wait(&patch_full[ps], (it / NP) & 1);
                mbar_wait(&b_empty[s], ((it / NB) & 1) ^ 1);
                gather_batch<GPW, HIN>(smem_u32(sP + ps * L.p_stride), smem_u32(sB + s * L.b_stride),
                                       sGsrc, sGdst, nsweeps, gw, gstride, lane, toff, p.lo_sweep0);

                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&b_full[s]);
                if (lane == 0) mbar_arrive(&patch_empty[ps]);
            }
        });
    } else {
        // ---------------------------------------------------------- epilogue
        const uint32_t q = static_cast<uint32_t>(warp % 4);
        const int etid = threadIdx.x - kEpiWarp0 * 32;
        int o = 0, it_base = 0;  // it_base: gather iteration of the run's first input plane
        const int ox = p.gx - 2 * p.r;
        const bool edge = (ox & (RW - 1)) != 0 && bx * (kTXB * kTileW) + kTXB * kTileW > ox && !(dbg(p) & 24);
        for_each_run(u0, u1, ozw, p.nby, p.zchunk, [&](int col, int zo_a, int zo_b) {
            int X0, Y0;
            col_xy(col, X0, Y0);
            for (int zo = zo_a; zo <= zo_b; ++zo, ++o) {
                const int slot = o % NACC;
                uint32_t v[NBOX][CW];
                if (dbg(p) & 32) {
#pragma unroll
                    for (int c = 0; c < NBOX; ++c)
#pragma unroll
                        for (int i = 0; i < CW; ++i) v[c][i] = 0u;
                } else {
                    mbar_wait(&d_full[slot], (o / NACC) & 1);
                    tc_fence_after();
                    tmem_load_batch<TYB>(tmem + ((q * 32u) << 16) + static_cast<uint32_t>(slot * N), v);
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&d_empty[slot]);
                }
                const uint8_t* ring = nullptr;
                if (edge && !(dbg(p) & 32)) {  // center input plane of output zo
                    const int ci = it_base + (zo - zo_a) + R;
                    mbar_wait(&ring_full[ci % kRingSlots], (ci / kRingSlots) & 1);
                    ring = sRing + (ci % kRingSlots) * (TYB * kTileH * 16);
                }
                if constexpr (HOUT) {
                    if (!(dbg(p) & 1))
                        store_batch_h<3, TYB, NS, kEdgeRing, PEER>(
                            p, tmap_out, reinterpret_cast<__half*>(buf_of(p, p.src ^ 1)), v, sS, L.s_stride, o, X0,
                            Y0, p.slow_lo + zo, q, lane, etid, reinterpret_cast<const __half*>(ring),
                            (PEER && (p.peer_mask & 1)) ? &p.peer_maps->up[p.src ^ 1] : nullptr,
                            (PEER && (p.peer_mask & 2)) ? &p.peer_maps->down[p.src ^ 1] : nullptr);
                } else if (!(dbg(p) & 1))
                    store_batch<3, TYB, NS, kEdgeRing, PEER>(
                        p, tmap_out, buf_of(p, p.src ^ 1), v, sS, L.s_stride, o, X0, Y0, p.slow_lo + zo, q, lane,
                        etid, reinterpret_cast<const float*>(ring), (p.peer_mask & 1) ? &p.peer_maps->up[p.src ^ 1] : nullptr,
                        (p.peer_mask & 2) ? &p.peer_maps->down[p.src ^ 1] : nullptr);
            }
            it_base += zo_b - zo_a + 1 + 2 * R;
        });
        if (etid == 0) bulk_wait<0>();
    }

    tc_fence_before();
    __syncthreads();
    if (p.trace && threadIdx.x == 0) {
        unsigned long long* t = p.trace + 4 * blockIdx.x;
        t[0] = smid();
        t[1] = t_start;
        t[2] = (dbg(p) & 1024) ? t_mid : t_main;  // profiling: prologue split
        t[3] = global_ns();
    }
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, static_cast<uint32_t>(p.tmem_cols));
    }
}

}  // namespace sst
