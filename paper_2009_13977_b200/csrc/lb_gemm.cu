// Persistent tcgen05 3xTF32 GEMM for the large-batch path (see lb.h).
//
//   D[M x N] = alpha * sum_seg A_seg[M x K] B_seg^T + beta * C     (fp32 exact-ish)
//
// One CTA per SM (148 on B200), 8 warps:
//   warp 0      TMA producer: per 32-wide K block one expect_tx and four tensor
//               copies (A hi/lo 128x32, B hi/lo 256x32, 128-byte swizzle) into
//               a 2-deep ring of 96 KB stages
//   warp 1      MMA issuer (lane 0): per K block 4 x {A_lo B_hi, A_hi B_lo,
//               A_hi B_hi} tcgen05.mma.kind::tf32 128x256x8 into a TMEM
//               accumulator; tcgen05.commit frees the stage / hands the tile to
//               the epilogue
//   warp 2      TMEM allocator (512 columns = two 128x256 fp32 accumulators,
//               so the epilogue of tile i overlaps the MMAs of tile i+1)
//   warps 4-7   epilogue: tcgen05.ld 32x32b (lane = row), alpha/beta, RN split,
//               coalesced row stores through a per-warp smem transpose, plus an
//               optional transposed split copy (lanes = consecutive rows, so
//               those stores are coalesced straight from registers)
// Tiles (z, split, n, m) are dealt round-robin over the persistent CTAs, m
// fastest, so CTAs running together share the B tile in L2.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cudaTypedefs.h>

#include "lb.h"

namespace fasthb {
namespace lb {
namespace {

constexpr int A_TILE = BM * BK * 4;             // 16 KB
constexpr int B_TILE = BN * BK * 4;             // 32 KB
constexpr int STAGE = 2 * A_TILE + 2 * B_TILE;  // 96 KB
constexpr int EPI_PITCH = 36;                   // floats per staged row
constexpr int EPI_BYTES = 4 * 32 * EPI_PITCH * 4;
constexpr int SMEM_BYTES = STAGES * STAGE + EPI_BYTES + 256 + 1024;
constexpr int TMEM_COLS = 512;

struct Params {
    CUtensorMap ta_hi[3], ta_lo[3], tb_hi[3], tb_lo[3];
    int M, N, nseg, ksplit, nz, mt, nt, total, kb_per_split, tile_m;
    int nkb[3], tot_kb;
    int a_row0[3], a_col0[3], b_row0[3], b_col0[3];
    int z_a_row, z_a_col, z_b_row, z_b_col;
    int64_t z_out;
    float alpha, beta;
    const float *c_hi, *c_lo;
    int64_t ldc;
    float* d_f32;
    int64_t ldd;
    float *d_hi, *d_lo;
    int64_t lds;
    int split_trunc, c_single;
    float *t_hi, *t_lo;
    int64_t ldt;
    float* partial;
    int debug_swap;
};

__device__ __forceinline__ uint32_t su32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mb_init(uint32_t a, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(n) : "memory");
}
__device__ __forceinline__ void mb_expect(uint32_t a, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
                 : "memory");
}
// Relaxed arrives: the epilogue signals "accumulator read back" (its
// tcgen05.ld already waited); a release arrive would stall on the warp's
// outstanding global stores (MEMBAR) before signalling.
__device__ __forceinline__ void mb_arrive(uint32_t a) {
    asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
#ifndef LB_HANG_DEBUG
__device__ __forceinline__ void mb_wait(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred P;\nLW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        "@!P bra LW_%=;\n}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}
#else  // bounded wait: report the stuck barrier and trap (debug builds only)
__device__ __forceinline__ void mb_wait(uint32_t a, uint32_t parity) {
    for (long long i = 0;; ++i) {
        uint32_t ok;
        asm volatile(
            "{\n.reg .pred P;\nmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\nselp.u32 %0, 1, 0, P;\n}\n"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
        if (ok) return;
        if (i == (1ll << 22)) {
            uint32_t rk;
            asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rk));
            printf("LB hang: block %d rank %u warp %d lane %d bar 0x%x parity %u\n", blockIdx.x, rk,
                   (int)(threadIdx.x >> 5), (int)(threadIdx.x & 31), a, parity);
            __trap();
        }
    }
}
#endif
template <bool PAIR>
__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap* m, int c0, int c1, uint32_t bar) {
    if constexpr (PAIR)  // the mbarrier may sit in the peer (leader) CTA
        asm volatile(
            "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                dst),
            "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(bar)
            : "memory");
    else
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                dst),
            "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(bar)
            : "memory");
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, uint32_t rank) {
    uint32_t o;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(rank));
    return o;
}
__device__ __forceinline__ void mb_arrive_cluster(uint32_t a) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// UMMA shared-memory descriptor, sm_100 version field = 1.  layout 2: 128-byte
// swizzle (K-major operands); layout 1: 128-byte swizzle with 32-byte atoms, the
// only MN-major layout tf32 accepts (4-deep K groups of 128-byte rows)
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint64_t layout = 2) {
    return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (layout << 61);
}
template <bool PAIR>
__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    if constexpr (PAIR)
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
            "l"(a), "l"(b), "r"(idesc), "r"(acc)
            : "memory");
    else
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
            "l"(a), "l"(b), "r"(idesc), "r"(acc)
            : "memory");
}
// commit: arrive on `bar` once the issued MMAs complete (both CTAs of a pair)
template <bool PAIR>
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    if constexpr (PAIR)
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                bar),
            "h"((uint16_t)3)
            : "memory");
    else
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                     : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
          "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
          "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float rn_hi(float x) {  // round to nearest tf32 (10-bit mantissa)
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
}
__device__ __forceinline__ float tr_hi(float x) {  // what the tensor core reads of x
    return __uint_as_float(__float_as_uint(x) & 0xffffe000u);
}

struct TileInfo {
    int m0, n0, split, z, kb_lo, kb_hi;
};
__device__ __forceinline__ TileInfo decode(const Params& p, int t) {
    TileInfo ti;
    const int mi = t % p.mt;
    int r = t / p.mt;
    const int ni = r % p.nt;
    r /= p.nt;
    ti.split = r % p.ksplit;
    ti.z = r / p.ksplit;
    ti.m0 = mi * p.tile_m;
    ti.n0 = ni * BN;
    ti.kb_lo = ti.split * p.kb_per_split;
    ti.kb_hi = min(p.tot_kb, ti.kb_lo + p.kb_per_split);
    return ti;
}

template <bool A_MN, bool B_MN, bool PAIR>
__global__ void __launch_bounds__(256, 1) gemm_kernel(const __grid_constant__ Params p) {
    // PAIR: a 2-CTA cluster runs one 256 x 256 tile with tcgen05.mma.cta_group::2;
    // each CTA loads its 128 A rows and its half (128 rows) of the B tile
    constexpr int CM = PAIR ? 2 : 1;
    constexpr int BNC = BN / CM;                // B rows (N) per CTA
    constexpr int B_T = BNC * BK * 4;
    constexpr int STG = 2 * A_TILE + 2 * B_T;   // 96 KB single, 64 KB pair
    constexpr int NST = PAIR ? 3 : 2;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    float* epi = reinterpret_cast<float*>(smem + NST * STG);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NST * STG + EPI_BYTES);
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * NST + 4);
    const uint32_t full0 = su32(bars), empty0 = su32(bars + NST);
    const uint32_t tfull0 = su32(bars + 2 * NST), tempty0 = su32(bars + 2 * NST + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t rank = 0;
    if constexpr (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const bool leader = rank == 0;
    const int cid = PAIR ? (int)blockIdx.x / 2 : (int)blockIdx.x;
    const int ncl = PAIR ? (int)gridDim.x / 2 : (int)gridDim.x;
    const bool dual = p.total <= ncl;  // one tile per CTA (pair): both accumulators on it
#ifdef LB_HANG_DEBUG
    if (PAIR && threadIdx.x == 0 && blockIdx.x < 2)
        printf("LB pair: block %d rank %u full0 0x%x mapa0 0x%x mapa1 0x%x\n", blockIdx.x, rank, su32(smem),
               mapa_u32(su32(smem), 0), mapa_u32(su32(smem), 1));
#endif

    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) {
            mb_init(full0 + 8 * s, 1);
            mb_init(empty0 + 8 * s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            mb_init(tfull0 + 8 * a, 1);
            mb_init(tempty0 + 8 * a, 4 * CM);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int sg = 0; sg < p.nseg; ++sg) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.ta_hi[sg])) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.ta_lo[sg])) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tb_hi[sg])) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tb_lo[sg])) : "memory");
        }
    }
    if (warp == 2) {
        if constexpr (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_holder)),
                         "r"(TMEM_COLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_holder)),
                         "r"(TMEM_COLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
    }
    fence_before();
    if constexpr (PAIR)
        cluster_sync();
    else
        __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_holder;

    if (warp == 0) {
        // ---------------- TMA producer ----------------
        int stage = 0;
        uint32_t phase = 0;
        for (int t = cid; t < p.total; t += ncl) {
            const TileInfo ti = decode(p, t);
            for (int kb = ti.kb_lo; kb < ti.kb_hi; ++kb) {
                int sg = 0, kbase = 0;
                while (sg + 1 < p.nseg && kb >= kbase + p.nkb[sg]) kbase += p.nkb[sg++];
                const int k0 = (kb - kbase) * BK;
                if (lane == 0) {
                    mb_wait(empty0 + 8 * stage, phase ^ 1);
                    uint32_t fb = full0 + 8 * stage;
                    if (leader) mb_expect(fb, STG * CM);  // the pair's bytes land on the leader's barrier
                    if constexpr (PAIR) fb = (p.debug_swap & 4) ? (fb & 0xFEFFFFFFu) : mapa_u32(fb, 0);
                    const uint32_t base = su32(smem + stage * STG);
                    if constexpr (!A_MN) {
                        const int ar = p.a_row0[sg] + ti.z * p.z_a_row + ti.m0 + (int)rank * BM;
                        const int ac = p.a_col0[sg] + ti.z * p.z_a_col + k0;
                        tma2d<PAIR>(base, &p.ta_hi[sg], ac, ar, fb);
                        tma2d<PAIR>(base + A_TILE, &p.ta_lo[sg], ac, ar, fb);
                    } else {
                        // K x M storage (rows k, columns m): boxes of (32 m) x (32 k)
                        const int ar = p.a_row0[sg] + ti.z * p.z_a_row + k0;
                        const int ac = p.a_col0[sg] + ti.z * p.z_a_col + ti.m0 + (int)rank * BM;
#pragma unroll
                        for (int c = 0; c < BM / 32; ++c) {
                            tma2d<PAIR>(base + c * (BK * 128), &p.ta_hi[sg], ac + 32 * c, ar, fb);
                            tma2d<PAIR>(base + A_TILE + c * (BK * 128), &p.ta_lo[sg], ac + 32 * c, ar, fb);
                        }
                    }
                    if constexpr (!B_MN) {
                        const int br = p.b_row0[sg] + ti.z * p.z_b_row + ti.n0 + (int)rank * BNC;
                        const int bc = p.b_col0[sg] + ti.z * p.z_b_col + k0;
                        tma2d<PAIR>(base + 2 * A_TILE, &p.tb_hi[sg], bc, br, fb);
                        tma2d<PAIR>(base + 2 * A_TILE + B_T, &p.tb_lo[sg], bc, br, fb);
                    } else {
                        // K x N storage: boxes of (32 n) x (32 k), chunk c at c * 4 KB
                        const int br = p.b_row0[sg] + ti.z * p.z_b_row + k0;
                        const int bc = p.b_col0[sg] + ti.z * p.z_b_col + ti.n0 + (int)rank * BNC;
#pragma unroll
                        for (int c = 0; c < BNC / 32; ++c) {
                            tma2d<PAIR>(base + 2 * A_TILE + c * (BK * 128), &p.tb_hi[sg], bc + 32 * c, br, fb);
                            tma2d<PAIR>(base + 2 * A_TILE + B_T + c * (BK * 128), &p.tb_lo[sg], bc + 32 * c, br, fb);
                        }
                    }
                }
                __syncwarp();
                if (++stage == NST) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1 && leader) {
        // ---------------- MMA issuer ----------------
        // instruction descriptor: D f32, A/B tf32, A K-major, B K- or MN-major, N=256, M=128
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((A_MN ? 1u : 0u) << 15) |
                               ((B_MN && !(p.debug_swap & 2) ? 1u : 0u) << 16) |
                               ((uint32_t)(BN >> 3) << 17) | ((uint32_t)((BM * CM) >> 4) << 24);
        uint32_t b_lbo = 0, b_sbo = 1024;
        const uint64_t b_layout = B_MN ? 1 : 2;
        if (B_MN) {
            b_lbo = BK * 128;  // stride between 32-wide N chunks
            b_sbo = 512;       // stride between 4-deep K groups
            if (p.debug_swap & 1) {
                b_lbo = 512;
                b_sbo = BK * 128;
            }
        }
        int stage = 0;
        uint32_t phase = 0;
        int it = 0;
        for (int t = cid; t < p.total; t += ncl, ++it) {
            const TileInfo ti = decode(p, t);
            const int acc = dual ? 0 : (it & 1);
            mb_wait(tempty0 + 8 * acc, ((it >> 1) & 1) ^ 1);
            fence_after();
            for (int kb = ti.kb_lo; kb < ti.kb_hi; ++kb) {
                // dual: K blocks alternate between the two accumulators (halves the
                // truncating accumulation chain; the epilogue adds them in RN fp32)
                const int ab = dual ? ((kb - ti.kb_lo) & 1) : acc;
                const uint32_t dtm = tmem + ab * BN;
                const bool fresh = dual ? (kb - ti.kb_lo < 2) : (kb == ti.kb_lo);
                mb_wait(full0 + 8 * stage, phase);
                fence_after();
                if (lane == 0) {
                    const uint32_t base = su32(smem + stage * STG);
                    const uint32_t ah = base, al = base + A_TILE;
                    const uint32_t bh = base + 2 * A_TILE, bl = bh + B_T;
#pragma unroll
                    for (int ks = 0; ks < BK / 8; ++ks) {
                        // MN-major operands: 32-byte-atom swizzle, 32-wide chunks 4 KB apart,
                        // 4-deep K groups 512 B apart; one MMA K step = 8 rows = 1 KB
                        const uint64_t dah = A_MN ? sdesc(ah + ks * 1024, BK * 128, 512, 1) : sdesc(ah + ks * 32, 0, 1024);
                        const uint64_t dal = A_MN ? sdesc(al + ks * 1024, BK * 128, 512, 1) : sdesc(al + ks * 32, 0, 1024);
                        const uint32_t boff = B_MN ? ks * 1024 : ks * 32;
                        const uint64_t dbh = sdesc(bh + boff, b_lbo, b_sbo, b_layout);
                        const uint64_t dbl = sdesc(bl + boff, b_lbo, b_sbo, b_layout);
                        const uint32_t first = (fresh && ks == 0) ? 0u : 1u;
                        mma_tf32<PAIR>(dtm, dal, dbh, idesc, first);
                        mma_tf32<PAIR>(dtm, dah, dbl, idesc, 1u);
                        mma_tf32<PAIR>(dtm, dah, dbh, idesc, 1u);
                    }
                    umma_commit<PAIR>(empty0 + 8 * stage);
                }
                __syncwarp();
                if (++stage == NST) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (lane == 0) umma_commit<PAIR>(tfull0 + 8 * acc);
            __syncwarp();
        }
    } else if (warp >= 4) {
        // ---------------- epilogue ----------------
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        float* st = epi + q * 32 * EPI_PITCH;
        int it = 0;
        for (int t = cid; t < p.total; t += ncl, ++it) {
            const TileInfo ti = decode(p, t);
            const int acc = dual ? 0 : (it & 1);
            const bool two = dual && ti.kb_hi - ti.kb_lo > 1;
            mb_wait(tfull0 + 8 * acc, (it >> 1) & 1);
            fence_after();
            const int mrow0 = ti.m0 + (int)rank * BM;  // this CTA's 128 rows of the tile
            const int row_t = q * 32 + lane;           // this lane's row
            const int64_t grow_l = (int64_t)ti.z * p.z_out + mrow0 + row_t;
            for (int c = 0; c < BN / 32; ++c) {
                // C operand of this chunk first: 16 independent 16-byte loads in
                // flight per lane while the accumulator is read back
                float4 chv[8], clv[8];
                if (p.c_hi && !p.partial) {
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int grow = mrow0 + q * 32 + i * 4 + (lane >> 3);
                        const int gcol = ti.n0 + c * 32 + (lane & 7) * 4;
                        if (grow < p.M && gcol < p.N) {
                            const int64_t off = ((int64_t)ti.z * p.z_out + grow) * p.ldc + gcol;
                            chv[i] = __ldcs(reinterpret_cast<const float4*>(p.c_hi + off));
                            if (!p.c_single) clv[i] = __ldcs(reinterpret_cast<const float4*>(p.c_lo + off));
                        }
                    }
                }
                float v[32];
                tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + acc * BN + c * 32, v);
                if (two) {
                    float v1[32];
                    tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + BN + c * 32, v1);
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] += v1[j];
                }
                const int ncol0 = ti.n0 + c * 32;
                if (p.t_hi && mrow0 + row_t < p.M) {
                    // transposed split copy: element (n, row) at t[n * ldt + row]
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        if (ncol0 + j < p.N) {
                            const float y = p.alpha * v[j];
                            const float h = rn_hi(y);
                            p.t_hi[(int64_t)(ncol0 + j) * p.ldt + grow_l] = h;
                            p.t_lo[(int64_t)(ncol0 + j) * p.ldt + grow_l] = y - h;
                        }
                    }
                }
                if (c == BN / 32 - 1) {  // accumulator fully read: hand it back to the MMA warp
                    fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        if constexpr (PAIR)
                            mb_arrive_cluster(mapa_u32(tempty0 + 8 * acc, 0));
                        else
                            mb_arrive(tempty0 + 8 * acc);
                    }
                }
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                    *reinterpret_cast<float4*>(st + lane * EPI_PITCH + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                __syncwarp();
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int r = i * 4 + (lane >> 3);
                    const int cc = (lane & 7) * 4;
                    const int grow = mrow0 + q * 32 + r;
                    const int gcol = ncol0 + cc;
                    if (grow < p.M && gcol < p.N) {
                        float4 a = *reinterpret_cast<const float4*>(st + r * EPI_PITCH + cc);
                        a.x *= p.alpha;
                        a.y *= p.alpha;
                        a.z *= p.alpha;
                        a.w *= p.alpha;
                        if (p.partial) {
                            float* dst = p.partial + (((int64_t)ti.z * p.ksplit + ti.split) * p.M + grow) * p.N + gcol;
                            *reinterpret_cast<float4*>(dst) = a;
                        } else {
                            const int64_t gr = (int64_t)ti.z * p.z_out + grow;
                            if (p.c_hi) {
                                float4 c = chv[i];
                                if (!p.c_single) {
                                    const float4 cl = clv[i];
                                    c = make_float4(c.x + cl.x, c.y + cl.y, c.z + cl.z, c.w + cl.w);
                                }
                                a.x += p.beta * c.x;
                                a.y += p.beta * c.y;
                                a.z += p.beta * c.z;
                                a.w += p.beta * c.w;
                            }
                            if (p.d_f32) *reinterpret_cast<float4*>(p.d_f32 + gr * p.ldd + gcol) = a;
                            if (p.d_hi) {
                                const float4 h = p.split_trunc ? make_float4(tr_hi(a.x), tr_hi(a.y), tr_hi(a.z), tr_hi(a.w))
                                                               : make_float4(rn_hi(a.x), rn_hi(a.y), rn_hi(a.z), rn_hi(a.w));
                                if (p.split_trunc) {  // (x, x - trunc(x))
                                    *reinterpret_cast<float4*>(p.d_hi + gr * p.lds + gcol) = a;
                                    *reinterpret_cast<float4*>(p.d_lo + gr * p.lds + gcol) =
                                        make_float4(a.x - h.x, a.y - h.y, a.z - h.z, a.w - h.w);
                                } else {
                                    *reinterpret_cast<float4*>(p.d_hi + gr * p.lds + gcol) = h;
                                    *reinterpret_cast<float4*>(p.d_lo + gr * p.lds + gcol) =
                                        make_float4(a.x - h.x, a.y - h.y, a.z - h.z, a.w - h.w);
                                }
                            }
                        }
                    }
                }
                __syncwarp();
            }
        }
    }
    fence_before();
    if constexpr (PAIR)
        cluster_sync();
    else
        __syncthreads();
    fence_after();
    if (warp == 2) {
        if constexpr (PAIR)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }
    return fn;
}

// 2-D map over a row-major rows x cols fp32 matrix (pitch ld), box (bc, br), 128-byte swizzle
// (32-byte swizzle atoms for MN-major operands)
bool make_map(CUtensorMap* m, const float* ptr, int64_t rows, int64_t cols, int64_t ld, int bc, int br,
              bool atom32 = false) {
    auto fn = encode_fn();
    if (!fn || !ptr || (reinterpret_cast<uintptr_t>(ptr) & 15) || (ld * 4) % 16) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
    cuuint32_t box[2] = {(cuuint32_t)bc, (cuuint32_t)br};
    cuuint32_t es[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE,
              atom32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

namespace {
bool use_pair(int M) {
    // CTA pairs (256-row tiles) from M = 512 on (B-row products run 64 pairs)
    const int pair_env = getenv("FASTH_LB_PAIR") ? atoi(getenv("FASTH_LB_PAIR")) : -1;
    const int pair_min = getenv("FASTH_LB_PAIR_MIN") ? atoi(getenv("FASTH_LB_PAIR_MIN")) : 512;
    return pair_env >= 0 ? (pair_env != 0 && M > BM) : M >= pair_min;
}

// Split-K reduction with the full epilogue: D = sum_s P[z][s] (+ beta C), written
// fp32 and/or split (one float4 per thread).
__global__ void reduce_epilogue_kernel(const float4* __restrict__ part, int ks, int nz, int M, int N, int64_t z_out,
                                       float beta, const float* __restrict__ c_hi, const float* __restrict__ c_lo,
                                       int c_single, int64_t ldc, float* __restrict__ d_f32, int64_t ldd,
                                       float* __restrict__ d_hi, float* __restrict__ d_lo, int64_t lds,
                                       int split_trunc) {
    const int n4 = N / 4;
    const int64_t per = (int64_t)M * n4, total = per * nz;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t z = e / per, w = e % per;
        const int r = (int)(w / n4), c = (int)(w % n4) * 4;
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int k = 0; k < ks; ++k) {
            const float4 v = __ldcs(part + (z * ks + k) * per + w);
            a.x += v.x, a.y += v.y, a.z += v.z, a.w += v.w;
        }
        const int64_t gr = z * z_out + r;
        if (c_hi) {
            float4 cv = *reinterpret_cast<const float4*>(c_hi + gr * ldc + c);
            if (!c_single) {
                const float4 cl = *reinterpret_cast<const float4*>(c_lo + gr * ldc + c);
                cv.x += cl.x, cv.y += cl.y, cv.z += cl.z, cv.w += cl.w;
            }
            a.x += beta * cv.x, a.y += beta * cv.y, a.z += beta * cv.z, a.w += beta * cv.w;
        }
        if (d_f32) *reinterpret_cast<float4*>(d_f32 + gr * ldd + c) = a;
        if (d_hi) {
            const float4 h = split_trunc ? make_float4(tr_hi(a.x), tr_hi(a.y), tr_hi(a.z), tr_hi(a.w))
                                         : make_float4(rn_hi(a.x), rn_hi(a.y), rn_hi(a.z), rn_hi(a.w));
            *reinterpret_cast<float4*>(d_hi + gr * lds + c) = split_trunc ? a : h;
            *reinterpret_cast<float4*>(d_lo + gr * lds + c) = make_float4(a.x - h.x, a.y - h.y, a.z - h.z, a.w - h.w);
        }
    }
}
}  // namespace

cudaError_t gemm_launch(Gemm& g, cudaStream_t s, int num_sms);

// Front end: a product with too few output tiles to fill the GPU (small batch)
// runs split K into g.split_scratch and reduces with the full epilogue.
cudaError_t gemm(Gemm& g, cudaStream_t s, int num_sms) {
    if (g.split_scratch && !g.partial && !g.t_hi) {
        const bool pair = use_pair(g.M);
        const int tile_m = pair ? 2 * BM : BM;
        const int nz = std::max(1, g.nz);
        const int tiles = nz * ((g.M + tile_m - 1) / tile_m) * ((g.N + BN - 1) / BN);
        const int units = pair ? std::max(num_sms / 2, 1) : std::max(num_sms, 1);
        int tot_kb = 0;
        for (int sg = 0; sg < g.nseg; ++sg) tot_kb += (g.seg[sg].K + BK - 1) / BK;
        if (tiles * 2 <= units && tot_kb >= 4) {
            const int64_t fit = g.split_scratch_floats / ((int64_t)nz * g.M * g.N);
            const int ks = (int)std::min<int64_t>({(int64_t)units / tiles, (int64_t)tot_kb / 2, 64, fit});
            if (ks >= 2) {
                Gemm q = g;
                q.partial = g.split_scratch;
                q.ksplit = ks;
                q.c_hi = q.c_lo = nullptr;
                q.d_f32 = q.d_hi = q.d_lo = nullptr;
                cudaError_t e = gemm_launch(q, s, num_sms);
                if (e != cudaSuccess) return e;
                const int64_t work = (int64_t)nz * g.M * (g.N / 4);
                const int grid = (int)std::min<int64_t>((work + 255) / 256, (int64_t)num_sms * 8);
                g.launched = 2;
                reduce_epilogue_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<const float4*>(g.split_scratch), q.ksplit,
                                                            nz, g.M, g.N, g.z_out, g.beta, g.c_hi, g.c_lo,
                                                            g.c_single, g.ldc, g.d_f32, g.ldd, g.d_hi, g.d_lo,
                                                            g.lds, g.split_trunc);
                return cudaGetLastError();
            }
        }
    }
    g.launched = 1;
    return gemm_launch(g, s, num_sms);
}

cudaError_t gemm_launch(Gemm& g, cudaStream_t s, int num_sms) {
    if (g.M <= 0 || g.N <= 0 || g.nseg < 1 || g.nseg > 3 || g.N % 4) return cudaErrorInvalidValue;
    if (g.t_hi && g.c_hi) return cudaErrorInvalidValue;  // the transposed copy carries no C term
    Params p{};
    p.M = g.M;
    p.N = g.N;
    p.nseg = g.nseg;
    const bool pair = use_pair(g.M);
    int tot_kb = 0;
    for (int sg = 0; sg < g.nseg; ++sg) {
        const Segment& S = g.seg[sg];
        if (S.K <= 0) return cudaErrorInvalidValue;
        p.nkb[sg] = (S.K + BK - 1) / BK;
        tot_kb += p.nkb[sg];
        p.a_row0[sg] = S.a_row0;
        p.a_col0[sg] = S.a_col0;
        p.b_row0[sg] = S.b_row0;
        p.b_col0[sg] = S.b_col0;
        bool ok = g.a_mn ? make_map(&p.ta_hi[sg], S.A.hi, S.A.rows, S.A.cols, S.A.ld, 32, BK, true) &&
                               make_map(&p.ta_lo[sg], S.A.lo, S.A.rows, S.A.cols, S.A.ld, 32, BK, true)
                         : make_map(&p.ta_hi[sg], S.A.hi, S.A.rows, S.A.cols, S.A.ld, BK, BM) &&
                               make_map(&p.ta_lo[sg], S.A.lo, S.A.rows, S.A.cols, S.A.ld, BK, BM);
        if (!g.b_mn)
            ok = ok && make_map(&p.tb_hi[sg], S.B.hi, S.B.rows, S.B.cols, S.B.ld, BK, pair ? BN / 2 : BN) &&
                 make_map(&p.tb_lo[sg], S.B.lo, S.B.rows, S.B.cols, S.B.ld, BK, pair ? BN / 2 : BN);
        else
            ok = ok && make_map(&p.tb_hi[sg], S.B.hi, S.B.rows, S.B.cols, S.B.ld, 32, BK, true) &&
                 make_map(&p.tb_lo[sg], S.B.lo, S.B.rows, S.B.cols, S.B.ld, 32, BK, true);
        if (!ok) return cudaErrorInvalidValue;
    }
    p.tot_kb = tot_kb;
    const bool part = g.partial != nullptr;
    p.ksplit = part ? std::max(1, std::min(g.ksplit, tot_kb)) : 1;
    p.kb_per_split = (tot_kb + p.ksplit - 1) / p.ksplit;
    p.ksplit = (tot_kb + p.kb_per_split - 1) / p.kb_per_split;  // no empty splits
    g.ksplit = p.ksplit;
    p.nz = std::max(1, g.nz);
    p.tile_m = pair ? 2 * BM : BM;
    p.mt = (g.M + p.tile_m - 1) / p.tile_m;
    p.nt = (g.N + BN - 1) / BN;
    p.total = p.nz * p.ksplit * p.mt * p.nt;
    p.z_a_row = g.z_a_row;
    p.z_a_col = g.z_a_col;
    p.z_b_row = g.z_b_row;
    p.z_b_col = g.z_b_col;
    p.z_out = g.z_out;
    p.alpha = g.alpha;
    p.beta = g.beta;
    p.c_hi = g.c_hi;
    p.c_lo = g.c_lo;
    p.ldc = g.ldc;
    p.d_f32 = g.d_f32;
    p.ldd = g.ldd;
    p.d_hi = g.d_hi;
    p.d_lo = g.d_lo;
    p.lds = g.lds;
    p.split_trunc = g.split_trunc ? 1 : 0;
    p.c_single = g.c_single ? 1 : 0;
    p.t_hi = g.t_hi;
    p.t_lo = g.t_lo;
    p.ldt = g.ldt;
    p.partial = g.partial;
    p.debug_swap = g.debug_swap;
    const int which = (g.b_mn ? 1 : 0) + (pair ? 2 : 0) + (g.a_mn ? 4 : 0);
    void (*kern)(Params) = nullptr;
    switch (which) {
        case 0: kern = gemm_kernel<false, false, false>; break;
        case 1: kern = gemm_kernel<false, true, false>; break;
        case 2: kern = gemm_kernel<false, false, true>; break;
        case 3: kern = gemm_kernel<false, true, true>; break;
        case 4: kern = gemm_kernel<true, false, false>; break;
        case 5: kern = gemm_kernel<true, true, false>; break;
        case 6: kern = gemm_kernel<true, false, true>; break;
        default: kern = gemm_kernel<true, true, true>; break;
    }
    if (cudaError_t e = ensure_smem(reinterpret_cast<const void*>(kern), SMEM_BYTES); e != cudaSuccess) return e;
    const int units = pair ? std::max(num_sms / 2, 1) : std::max(num_sms, 1);
    const int grid = std::min(p.total, units) * (pair ? 2 : 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3(256, 1, 1);
    cfg.dynamicSmemBytes = SMEM_BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = pair ? 2 : 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, p);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace lb
}  // namespace fasthb
