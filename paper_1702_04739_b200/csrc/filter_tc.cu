// K3tc: Boruvka candidate filter on the 5th-gen tensor cores (sm_100a).
//
// Same contract as boruvka_filter_kernel (per row: best approximate squared
// distance a1 to a column of another component, its column j1, and the
// second best a2), computed from a 3-term FP16 split of the centred, scaled
// points: y*2^s = hi + lo (hi = fp16(y 2^s), lo = fp16(y 2^s - hi)), and
//   <y_i, y_j> 2^2s ~ hi_i.hi_j + hi_i.lo_j + lo_i.hi_j
// evaluated by tcgen05.mma kind::f16 with FP32 accumulation in TMEM.
// Operand images are pre-swizzled in HBM in the UMMA K-major SWIZZLE_128B
// layout (one 16 KB image per 128 points per part), so a plain 1-D bulk copy
// (cp.async.bulk, TMA engine) lands them ready for the MMA descriptors.
//
// CTA = 256 rows (two 128-row blocks, A resident in smem) x all 128-column
// tiles.  Warp 0: bulk-copy producer; warp 1: TMEM allocation + MMA issue
// (one elected lane); warps 2-9: epilogue, one thread per row reading its
// 128 accumulator columns with tcgen05.ld and keeping (a1, j1, a2).
// Accumulators are double buffered in TMEM (2 x 256 columns) so the MMA of
// tile t+1 overlaps the epilogue of tile t.  Each row keeps its TC_K best
// (a, j) in registers -- a candidate list (sorted, lexicographic (a, j)) and
// the bound lb every unlisted column satisfies (a >= lb) -- so later Boruvka
// rounds can take a row's minimum from its list while the listed columns
// stay in other components, and launch the filter only for the 256-row
// blocks (blk_flag) holding rows whose list ran out.  d <= 64: one 64-wide K atom,
// A resident; d > 64: every stage streams one K atom of A (both row blocks)
// and of the tile, accumulating the atoms in TMEM.
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"
#include "prof.h"

namespace isoc {

constexpr int TC_BM = 128;          // rows per block = TMEM lanes
constexpr int TC_BN = 128;          // columns per tile
constexpr int TC_STAGES = 4;
constexpr int TC_EPI = 16;          // epilogue warps (2 threads per row, 64 columns each)
constexpr int TC_THREADS = 64 + 32 * TC_EPI;
constexpr int TC_PART = 16384;      // bytes of one 128 x 64 fp16 image
constexpr int TC_META = 8;
constexpr int TC_MS = 4;            // metadata ring slots
constexpr int TC_K = FILTER_LIST_K;  // candidate list length per row (kernels.h)

// Resident-A layout (d <= 64: one 64-wide K atom) and streaming layout
// (d > 64: each stage carries one K atom of both row blocks and the tile).
template <bool STREAM>
struct TcSmemT {
    uint8_t A[2][2][TC_PART];            // [row block][hi/lo]
    uint8_t B[TC_STAGES][2][TC_PART];    // [stage][hi/lo]
    int32_t mcomp[TC_MS][TC_BN];         // column metadata ring (bulk-copied by the producer)
    float mnorm[TC_MS][TC_BN];
    float xla[(TC_K + 1) * 2 * TC_BM];   // second-half lists of each row
    int32_t xlj[(TC_K + 1) * 2 * TC_BM];
    uint64_t full[TC_STAGES];
    uint64_t empty[TC_STAGES];
    uint64_t afull;
    uint64_t tfull[2];
    uint64_t tempty[2];
    uint64_t mfull[TC_MS];
    uint64_t mempty[TC_MS];
    uint32_t tmem_base;
};
constexpr int TC_SSTAGES = 2;            // streaming stages (96 KB each)
template <>
struct TcSmemT<true> {
    uint8_t S[TC_SSTAGES][6][TC_PART];   // [stage][A blk0 hi, lo, A blk1 hi, lo, B hi, lo]
    int32_t mcomp[TC_MS][TC_BN];
    float mnorm[TC_MS][TC_BN];
    float xla[(TC_K + 1) * 2 * TC_BM];
    int32_t xlj[(TC_K + 1) * 2 * TC_BM];
    uint64_t full[TC_STAGES];
    uint64_t empty[TC_STAGES];
    uint64_t afull;
    uint64_t tfull[2];
    uint64_t tempty[2];
    uint64_t mfull[TC_MS];
    uint64_t mempty[TC_MS];
    uint32_t tmem_base;
};
using TcSmem = TcSmemT<false>;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// explicit shared-memory vector loads (the dynamic-smem struct is reached
// through an aligned generic pointer, which would otherwise become LD.E)
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];\n" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ int4 lds_i4(uint32_t a) {
    int4 v;
    asm volatile("ld.shared.v4.s32 {%0,%1,%2,%3}, [%4];\n" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// K-major SWIZZLE_128B UMMA shared-memory descriptor (version 1, LBO 16 B,
// SBO = 8 rows x 128 B)
__device__ __forceinline__ uint64_t umma_desc(const void* p) {
    const uint64_t addr = smem_u32(p);
    return ((addr >> 4) & 0x3FFFull) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

// kind::f16, FP16 x FP16 -> FP32, both K-major, M = 128, N = 128
constexpr uint32_t TC_IDESC = (1u << 4) | ((uint32_t)(TC_BN >> 3) << 17) | ((uint32_t)(TC_BM >> 4) << 24);

__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(TC_IDESC), "r"(accum));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
          "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
          "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Each row keeps TC_KL = TC_K + 1 entries: the TC_K it reports and one more,
// whose value is the bound lb of every column outside the list (a value
// that falls off the end is >= it).  Branch-free insertion of (a, j) into
// the sorted list (strict <: among equal values the earlier -- smaller --
// column stays first).
constexpr int TC_KL = TC_K + 1;
__device__ __forceinline__ void list_insert(float a, int32_t j, float (&la)[TC_KL], int32_t (&lj)[TC_KL]) {
    float x = a;
    int32_t xj = j;
#pragma unroll
    for (int p = 0; p < TC_KL; ++p) {
        const bool lt = x < la[p];
        const float ta = la[p];
        const int32_t tj = lj[p];
        la[p] = lt ? x : ta;
        lj[p] = lt ? xj : tj;
        x = lt ? ta : x;
        xj = lt ? tj : xj;
    }
}

// lexicographic (a, j) insertion for merging two lists whose columns interleave
__device__ __forceinline__ void list_insert_lex(float a, int32_t j, float (&la)[TC_KL], int32_t (&lj)[TC_KL]) {
    float x = a;
    int32_t xj = j;
#pragma unroll
    for (int p = 0; p < TC_KL; ++p) {
        const bool lt = x < la[p] || (x == la[p] && xj >= 0 && (lj[p] < 0 || xj < lj[p]));
        const float ta = la[p];
        const int32_t tj = lj[p];
        la[p] = lt ? x : ta;
        lj[p] = lt ? xj : tj;
        x = lt ? ta : x;
        xj = lt ? tj : xj;
    }
}

template <bool STREAM>
__global__ void __launch_bounds__(TC_THREADS, 1)
filter_tc_kernel(const uint8_t* __restrict__ img, const float* __restrict__ ny,
                 const int32_t* __restrict__ comp, int64_t n, int64_t row_lo, int64_t row_hi,
                 float kscale, float* __restrict__ out_la, int32_t* __restrict__ out_lj,
                 float* __restrict__ out_lb, const uint8_t* __restrict__ imgA,
                 const int32_t* __restrict__ rows_map, int64_t nmap, int KA) {
    // rows_map != nullptr: gathered mode -- the CTA's 256 rows are
    // rows_map[256 * blockIdx.x + 0..255] (global ids, < nmap valid) and their
    // A operands come from the gathered image imgA (built by tc_gather_kernel)
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    TcSmemT<STREAM>& sm = *reinterpret_cast<TcSmemT<STREAM>*>(
        reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023)));
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t blk0 = row_lo / TC_BM + 2 * (int64_t)blockIdx.x;   // first 128-row block
    const int64_t ntiles = (n + TC_BN - 1) / TC_BN;
    const int64_t nblocks_total = (n + TC_BM - 1) / TC_BM;

    if (tid == 0) {
        for (int s = 0; s < TC_STAGES; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], 1);
        }
        mbar_init(&sm.afull, 1);
        for (int s = 0; s < 2; ++s) {
            mbar_init(&sm.tfull[s], 1);
            mbar_init(&sm.tempty[s], TC_EPI);
        }
        for (int s = 0; s < TC_MS; ++s) {
            mbar_init(&sm.mfull[s], 1);
            mbar_init(&sm.mempty[s], TC_EPI);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
            smem_u32(&sm.tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = sm.tmem_base;

    if (warp == 0) {
        // ------------------------------------------------ producer
        if (lane == 0) {
          if constexpr (!STREAM) {
            mbar_expect_tx(&sm.afull, 4 * TC_PART);
            for (int r = 0; r < 2; ++r) {
                const int64_t b = (blk0 + r < nblocks_total) ? blk0 + r : nblocks_total - 1;
                const uint8_t* asrc = rows_map ? imgA + (2 * (int64_t)blockIdx.x + r) * 2 * (int64_t)TC_PART
                                               : img + b * 2 * (int64_t)TC_PART;
                bulk_g2s(sm.A[r][0], asrc, TC_PART, &sm.afull);
                bulk_g2s(sm.A[r][1], asrc + TC_PART, TC_PART, &sm.afull);
            }
          }
            int64_t q = 0;   // stage uses (streaming)
            for (int64_t t = 0; t < ntiles; ++t) {
              if constexpr (!STREAM) {
                const int s = (int)(t % TC_STAGES);
                const uint32_t ph = (uint32_t)((t / TC_STAGES) & 1);
                if (t >= TC_STAGES) mbar_wait(&sm.empty[s], ph ^ 1);
                mbar_expect_tx(&sm.full[s], 2 * TC_PART);
                // hi and lo images of a block are adjacent: one 32 KB copy
                bulk_g2s(sm.B[s][0], img + (t * 2) * (int64_t)TC_PART, 2 * TC_PART, &sm.full[s]);
              } else {
                // one stage per K atom: both row blocks' A atom and the tile's B atom
                for (int a = 0; a < KA; ++a, ++q) {
                    const int s = (int)(q % TC_SSTAGES);
                    const uint32_t ph = (uint32_t)((q / TC_SSTAGES) & 1);
                    if (q >= TC_SSTAGES) mbar_wait(&sm.empty[s], ph ^ 1);
                    mbar_expect_tx(&sm.full[s], 6 * TC_PART);
                    for (int r = 0; r < 2; ++r) {
                        const int64_t b = (blk0 + r < nblocks_total) ? blk0 + r : nblocks_total - 1;
                        const uint8_t* asrc =
                            rows_map ? imgA + (((2 * (int64_t)blockIdx.x + r) * KA + a) * 2) * (int64_t)TC_PART
                                     : img + ((b * KA + a) * 2) * (int64_t)TC_PART;
                        bulk_g2s(sm.S[s][2 * r + 0], asrc, TC_PART, &sm.full[s]);
                        bulk_g2s(sm.S[s][2 * r + 1], asrc + TC_PART, TC_PART, &sm.full[s]);
                    }
                    bulk_g2s(sm.S[s][4], img + ((t * KA + a) * 2 + 0) * (int64_t)TC_PART, TC_PART, &sm.full[s]);
                    bulk_g2s(sm.S[s][5], img + ((t * KA + a) * 2 + 1) * (int64_t)TC_PART, TC_PART, &sm.full[s]);
                }
              }
                // the tile's column components and norms for the epilogue
                const int ms = (int)(t % TC_MS);
                const uint32_t mph = (uint32_t)((t / TC_MS) & 1);
                if (t >= TC_MS) mbar_wait(&sm.mempty[ms], mph ^ 1);
                mbar_expect_tx(&sm.mfull[ms], 2 * TC_BN * 4);
                bulk_g2s(sm.mcomp[ms], comp + t * TC_BN, TC_BN * 4, &sm.mfull[ms]);
                bulk_g2s(sm.mnorm[ms], ny + t * TC_BN, TC_BN * 4, &sm.mfull[ms]);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            if constexpr (!STREAM) mbar_wait(&sm.afull, 0);
            int64_t q = 0;
            for (int64_t t = 0; t < ntiles; ++t) {
                const int as = (int)(t & 1);
                if (t >= 2) mbar_wait(&sm.tempty[as], (uint32_t)(((t >> 1) - 1) & 1));
              if constexpr (!STREAM) {
                const int s = (int)(t % TC_STAGES);
                const uint32_t ph = (uint32_t)((t / TC_STAGES) & 1);
                mbar_wait(&sm.full[s], ph);
                asm volatile("tcgen05.fence::after_thread_sync;\n");
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    const uint32_t dcol = tmem + (uint32_t)(as * 256 + r * 128);
#pragma unroll
                    for (int step = 0; step < 12; ++step) {
                        const int pass = step >> 2, kk = step & 3;
                        // pass 0: hi.hi, 1: hi.lo, 2: lo.hi
                        const uint64_t da = umma_desc(sm.A[r][pass == 2 ? 1 : 0]) + (uint64_t)(kk * 2);
                        const uint64_t db = umma_desc(sm.B[s][pass == 1 ? 1 : 0]) + (uint64_t)(kk * 2);
                        umma_f16(dcol, da, db, step > 0 ? 1u : 0u);
                    }
                }
                umma_commit(&sm.empty[s]);
              } else {
                for (int a = 0; a < KA; ++a, ++q) {
                    const int s = (int)(q % TC_SSTAGES);
                    const uint32_t ph = (uint32_t)((q / TC_SSTAGES) & 1);
                    mbar_wait(&sm.full[s], ph);
                    asm volatile("tcgen05.fence::after_thread_sync;\n");
#pragma unroll
                    for (int r = 0; r < 2; ++r) {
                        const uint32_t dcol = tmem + (uint32_t)(as * 256 + r * 128);
#pragma unroll
                        for (int step = 0; step < 12; ++step) {
                            const int pass = step >> 2, kk = step & 3;
                            const uint64_t da = umma_desc(sm.S[s][2 * r + (pass == 2 ? 1 : 0)]) + (uint64_t)(kk * 2);
                            const uint64_t db = umma_desc(sm.S[s][4 + (pass == 1 ? 1 : 0)]) + (uint64_t)(kk * 2);
                            umma_f16(dcol, da, db, (a > 0 || step > 0) ? 1u : 0u);
                        }
                    }
                    umma_commit(&sm.empty[s]);
                }
              }
                umma_commit(&sm.tfull[as]);
            }
        }
    } else {
        // ------------------------------------------------ epilogue
        // warp e = warp - 2 (0..15): TMEM lane quarter warp & 3, row block
        // (e >> 3), column half (e >> 2) & 1; a row's two threads combine at
        // the end.  The row norm is added after the minimum (rounding is
        // monotone, so min / second min commute with + rn).
        const int e = warp - 2;
        const int q = warp & 3;
        const int r = e >> 3;
        const int hcol = (e >> 2) & 1;
        const int lrow = q * 32 + lane;
        int64_t row;
        bool live;
        if (rows_map) {
            const int64_t g = 256 * (int64_t)blockIdx.x + r * TC_BM + lrow;
            live = g < nmap;
            row = live ? rows_map[g] : -1;
        } else {
            row = (blk0 + r) * TC_BM + lrow;
            live = row >= row_lo && row < row_hi;
        }
        const int32_t rc = live ? comp[row] : -2;
        float la[TC_KL];
        int32_t lj[TC_KL];
#pragma unroll
        for (int p = 0; p < TC_KL; ++p) { la[p] = INFINITY; lj[p] = -1; }
        for (int64_t t = 0; t < ntiles; ++t) {
            const int as = (int)(t & 1);
            const int ms = (int)(t % TC_MS);
            mbar_wait(&sm.mfull[ms], (uint32_t)((t / TC_MS) & 1));
            mbar_wait(&sm.tfull[as], (uint32_t)((t >> 1) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;\n");
            const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(as * 256 + r * 128 + hcol * 64);
#pragma unroll 1
            for (int c = 0; c < 2; ++c) {
                float v[32];
                tmem_ld32(tbase + (uint32_t)(c * 32), v);
                const int lc0 = hcol * 64 + c * 32;
                // masked estimates and their chunk minimum; the list can only
                // change if some value is below its last entry
                float m = INFINITY;
#pragma unroll
                for (int i4 = 0; i4 < 8; ++i4) {
                    const float4 cn4 = lds_f4(smem_u32(&sm.mnorm[ms][lc0 + 4 * i4]));
                    const int4 cc4 = lds_i4(smem_u32(&sm.mcomp[ms][lc0 + 4 * i4]));
                    const float cn[4] = {cn4.x, cn4.y, cn4.z, cn4.w};
                    const int32_t cc[4] = {cc4.x, cc4.y, cc4.z, cc4.w};
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int i = 4 * i4 + u;
                        const float a = fmaf(kscale, v[i], cn[u]);
                        v[i] = (cc[u] != rc) ? a : INFINITY;
                        m = fminf(m, v[i]);
                    }
                }
                // per value: a warp runs an insertion only when one of its 32
                // rows has that value below its list end (a per-chunk gate
                // would run all 32 whenever any row's chunk qualifies)
                if (m < la[TC_KL - 1]) {
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (v[i] < la[TC_KL - 1]) list_insert(v[i], (int32_t)(t * TC_BN + lc0 + i), la, lj);
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;\n");
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&sm.tempty[as]);
                mbar_arrive(&sm.mempty[ms]);
            }
        }
        // the two column halves of a row merge through shared memory (the
        // operand stages are free once every MMA has completed: each thread
        // waited on the last tile's tfull)
        const int slot = r * TC_BM + lrow;
        float* xla = sm.xla;
        int32_t* xlj = sm.xlj;
        if (hcol == 1) {
#pragma unroll
            for (int p = 0; p < TC_KL; ++p) {
                xla[p * 2 * TC_BM + slot] = la[p];
                xlj[p * 2 * TC_BM + slot] = lj[p];
            }
        }
        asm volatile("bar.sync 1, %0;\n" ::"n"(32 * TC_EPI) : "memory");
        if (hcol == 0 && live) {
#pragma unroll
            for (int p = 0; p < TC_KL; ++p) list_insert_lex(xla[p * 2 * TC_BM + slot], xlj[p * 2 * TC_BM + slot], la, lj);
            const float lb = la[TC_K];
            // the row norm is added after the minimum (rounding is monotone)
            const float rn = ny[row];
            const int64_t li = row - row_lo;
#pragma unroll
            for (int p = 0; p < TC_K; ++p) {
                out_la[li * TC_K + p] = la[p] + rn;
                out_lj[li * TC_K + p] = lj[p];
            }
            out_lb[li] = lb + rn;
        }
    }
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
    }
}

// Pre-swizzled FP16 split images: img[(block * 2 + part) * 16 KB], part 0 = hi,
// 1 = lo; element (r, k) of a block at (r/8)*1024 + (r%8)*128 + ((k/8)^(r%8))*16 + (k%8)*2.
__global__ void tc_image_kernel(const float* __restrict__ YT, int64_t npad, int d, int KA, float scale,
                                int64_t nblocks, uint8_t* __restrict__ img) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // one (point, k) pair
    if (idx >= nblocks * TC_BM * 64 * KA) return;
    const int kg = (int)(idx % (64 * KA));
    const int64_t p = idx / (64 * KA);
    const int a = kg >> 6, k = kg & 63;
    const int64_t b = p / TC_BM;
    const int r = (int)(p % TC_BM);
    const float y = (kg < d && p < npad) ? YT[(int64_t)kg * npad + p] * scale : 0.f;
    const __half hi = __float2half_rn(y);
    const __half lo = __float2half_rn(y - __half2float(hi));
    const int64_t off = (int64_t)(r >> 3) * 1024 + (r & 7) * 128 + (((k >> 3) ^ (r & 7)) << 4) + (k & 7) * 2;
    *reinterpret_cast<__half*>(img + ((b * KA + a) * 2 + 0) * (int64_t)TC_PART + off) = hi;
    *reinterpret_cast<__half*>(img + ((b * KA + a) * 2 + 1) * (int64_t)TC_PART + off) = lo;
}

// Gathered A images for the rows of rows_map: row g of the gathered image is
// row rows_map[g] of img, 16-byte chunks re-swizzled for the new row slot.
__global__ void tc_gather_kernel(const uint8_t* __restrict__ img, const int32_t* __restrict__ rows_map,
                                 const int32_t* __restrict__ nmap_dev, int KA, uint8_t* __restrict__ imgA) {
    const int64_t nmap = *nmap_dev;
    const int64_t total = (nmap + 255) / 256 * 256 * KA * 2 * 8;   // (row, atom, part, chunk)
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(e & 7);
        const int part = (int)((e >> 3) & 1);
        const int64_t ra = e >> 4;
        const int a = (int)(ra % KA);
        const int64_t g = ra / KA;
        const int rd = (int)(g % TC_BM);
        const int64_t bd = g / TC_BM;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (g < nmap) {
            const int64_t src = rows_map[g];
            const int rs = (int)(src % TC_BM);
            const int64_t bs = src / TC_BM;
            const uint8_t* p = img + ((bs * KA + a) * 2 + part) * (int64_t)TC_PART + (rs >> 3) * 1024 +
                               (rs & 7) * 128 + ((c ^ (rs & 7)) << 4);
            v = *reinterpret_cast<const uint4*>(p);
        }
        uint8_t* q = imgA + ((bd * KA + a) * 2 + part) * (int64_t)TC_PART + (rd >> 3) * 1024 + (rd & 7) * 128 +
                     ((c ^ (rd & 7)) << 4);
        *reinterpret_cast<uint4*>(q) = v;
    }
}

size_t tc_image_bytes(int64_t n, int d) {
    const int64_t nblocks = (n + TC_BM - 1) / TC_BM;
    const int KA = (d + 63) / 64;
    return (size_t)nblocks * KA * 2 * TC_PART;
}

cudaError_t launch_tc_image(const float* YT, int64_t npad, int d, float scale, int64_t n, uint8_t* img,
                            cudaStream_t st) {
    const int64_t nblocks = (n + TC_BM - 1) / TC_BM;
    const int KA = (d + 63) / 64;
    const int64_t total = nblocks * TC_BM * 64 * KA;
    tc_image_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(YT, npad, d, KA, scale, nblocks, img);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_filter_tc(const uint8_t* img, const float* ny, const int32_t* comp, int64_t n, int d,
                             int64_t lo, int64_t hi, float kscale, float* la, int32_t* lj, float* lb,
                             const int32_t* rows_map, const int32_t* nmap_dev, int64_t nmap, uint8_t* imgA,
                             cudaStream_t st) {
    if (hi <= lo) return cudaSuccess;
    const int KA = (d + 63) / 64;
    unsigned grid = (unsigned)filter_tc_blocks(lo, hi);
    if (rows_map) {
        if (nmap <= 0) return cudaSuccess;
        grid = (unsigned)((nmap + 255) / 256);
        tc_gather_kernel<<<148 * 4, 256, 0, st>>>(img, rows_map, nmap_dev, KA, imgA);
        note_launch();
    }
    const int pid = prof_begin(PK_FILTER, st);
    cudaError_t e;
    if (KA == 1) {
        const size_t smem = sizeof(TcSmemT<false>) + 1024;
        e = ensure_max_dyn_smem((const void*)filter_tc_kernel<false>, (size_t)((int)smem));
        if (e != cudaSuccess) return e;
        filter_tc_kernel<false><<<grid, TC_THREADS, smem, st>>>(img, ny, comp, n, lo, hi, kscale, la, lj, lb,
                                                                 imgA, rows_map, nmap, 1);
    } else {
        const size_t smem = sizeof(TcSmemT<true>) + 1024;
        e = ensure_max_dyn_smem((const void*)filter_tc_kernel<true>, (size_t)((int)smem));
        if (e != cudaSuccess) return e;
        filter_tc_kernel<true><<<grid, TC_THREADS, smem, st>>>(img, ny, comp, n, lo, hi, kscale, la, lj, lb,
                                                                imgA, rows_map, nmap, KA);
    }
    prof_end(pid, st);
    note_launch();
    return cudaGetLastError();
}

int64_t filter_tc_blocks(int64_t lo, int64_t hi) {
    const int64_t b_lo = lo / TC_BM, b_hi = (hi + TC_BM - 1) / TC_BM;
    return (b_hi - b_lo + 1) / 2;
}

}  // namespace isoc
