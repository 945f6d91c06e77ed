// qm_tma.cuh -- TMA bulk-copy pipeline for the streaming elementwise kernels.
//
// The streaming kernels move 8 (fp32) or 16 (fp64) bytes per sample and do
// ~35 issue slots of math per sample, so at full HBM bandwidth each SM must
// keep ~40 KB of loads in flight while its warps compute.  With plain LDG the
// bytes in flight are capped by registers (the math needs ~70 of them); here
// the bytes in flight live in shared memory instead:
//
//   * one persistent CTA per SM: a producer warp + NC consumer warps;
//   * a ring of S stages of TILE bytes; the producer's elected lane waits for a
//     stage to be free (mbarrier "empty"), then issues one
//     cp.async.bulk global->shared (UBLKCP) completing on mbarrier "full";
//   * consumers wait on "full", map the tile IN PLACE in shared memory
//     (LDS.128 -> math -> STS.128), then, after a consumer-only named barrier,
//     one elected consumer issues cp.async.bulk shared->global for the tile,
//     waits for the bulk read of shared memory and arrives on "empty".
//
// The producer runs up to S tiles ahead, so S * TILE bytes per SM are in
// flight no matter how many registers the math uses.
//
// Two pipelines live here: tma_stream_map (the in-place design above, kept for
// A/B runs, QM_STREAM_PATH=tma) and tma_load_map (below; the default): input by
// TMA, stage released per warp right after its LDS, output by streaming stores.
#pragma once
#include "qm_math.cuh"

namespace qm {

// Programmatic dependent launch (the streaming maps are launched with it, qm_lib.cu):
// let the next grid on the stream launch now (its CTAs take SMs as ours exit and
// wait below), and wait for every prior grid to complete -- with its memory
// visible -- before this grid's first global access.  No-ops for a normal launch.
__device__ __forceinline__ void pdl_begin()
{
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}


QM_DEV uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

QM_DEV void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
// called by a whole warp: one elected lane initialises the barrier (predicated,
// no branch -- the kernels then have no divergent branch at all)
QM_DEV void mbar_init_elect(uint64_t *bar, uint32_t count)
{
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\t"
                 "@P mbarrier.init.shared::cta.b64 [%0], %1;\n\t}"
                 :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
QM_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
QM_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

QM_DEV void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
QM_DEV void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}
QM_DEV void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}"
        :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}
QM_DEV void bulk_g2s(void *dst_smem, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_u32(dst_smem)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// The producer's per-tile issue, run by ALL 32 lanes of the producer warp: one
// lane chosen by elect.sync arms the stage's "full" barrier with the byte count
// and issues the bulk copy, both predicated inside one asm block -- no branch, so
// the producer contributes no divergent branch (P:551's argument, measured by ncu).
QM_DEV void elect_tma_load(uint64_t *bar, void *dst_smem, const void *src, uint32_t bytes)
{
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "elect.sync _|P, 0xffffffff;\n\t"
        "@P mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %3;\n\t"
        "@P cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%1], [%2], %3, [%0];\n\t}"
        :: "r"(smem_u32(bar)), "r"(smem_u32(dst_smem)), "l"(src), "r"(bytes) : "memory");
}

QM_DEV void bulk_s2g(void *dst, const void *src_smem, uint32_t bytes)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 :: "l"(dst), "r"(smem_u32(src_smem)), "r"(bytes) : "memory");
}
QM_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
QM_DEV void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
QM_DEV void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
QM_DEV void consumer_bar(int nthreads) { asm volatile("bar.sync 1, %0;" :: "r"(nthreads) : "memory"); }

// Persistent pipelined map over `ntiles` full tiles of TILE_ELEMS elements of
// type T.  OP::tile(T *smem_tile, int ctid, int nct) maps one tile in place;
// it is called by all consumer threads (ctid in [0, nct)) of the CTA.
template <typename T, int TILE_ELEMS, int STAGES, int NC, typename OP>
__device__ __forceinline__ void tma_stream_map(const T *__restrict__ in, T *__restrict__ out, int64_t ntiles, OP op)
{
    constexpr uint32_t TILE_BYTES = TILE_ELEMS * sizeof(T);
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T *tiles = reinterpret_cast<T *>(smem_raw);
    __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init_elect(&full[s], 1); mbar_init_elect(&empty[s], 1); }
        fence_mbar_init();
    }
    pdl_begin();
    __syncthreads();

    const int64_t first = blockIdx.x, step = gridDim.x;
    if (warp == 0) {
        // ---------------- producer (all lanes; one elected lane issues)
        int s = 0;
        uint32_t ph = 0;
        int64_t k = 0;
        for (int64_t t = first; t < ntiles; t += step, ++k) {
            if (k >= STAGES) mbar_wait(&empty[s], ph ^ 1);
            elect_tma_load(&full[s], tiles + (size_t)s * TILE_ELEMS, in + t * TILE_ELEMS, TILE_BYTES);
            if (++s == STAGES) { s = 0; ph ^= 1; }
        }
    } else {
        // ---------------- consumers
        const int ctid = threadIdx.x - 32;
        int s = 0, prev = -1;
        uint32_t ph = 0;
        for (int64_t t = first; t < ntiles; t += step) {
            mbar_wait(&full[s], ph);
            T *tile = tiles + (size_t)s * TILE_ELEMS;
            op.tile(tile, ctid, NC * 32);
            fence_proxy_async();                 // generic-proxy smem writes -> async proxy
            consumer_bar(NC * 32);
            if (ctid == 0) {
                bulk_s2g(out + t * TILE_ELEMS, tile, TILE_BYTES);
                bulk_commit();
                // release the PREVIOUS stage once its bulk store has read shared
                // memory (keeps this warp from waiting on the store just issued)
                if (prev >= 0) {
                    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                    mbar_arrive(&empty[prev]);
                }
                prev = s;
            }
            if (++s == STAGES) { s = 0; ph ^= 1; }
        }
        if (ctid == 0) bulk_wait_all();           // global writes complete before exit
    }
}

}  // namespace qm

namespace qm {

// ----------------------------------------------------------------------------
// TMA-in / STG-out pipeline ("load map").  Same producer as tma_stream_map, but
// the consumers do not write the tile back into shared memory:
//
//   * each consumer warp owns a contiguous 1/NC slice of a tile; it waits on
//     "full", reads its slice into registers (LDS.128, PER vectors per lane),
//     and its lane 0 arrives on "empty" (count NC) at once -- the stage goes
//     back to the producer before the math, not after the tile's store;
//   * the warp then maps its registers and writes them with 128-bit streaming
//     stores (st.global.cs) straight to global memory: stores need no
//     completion, so nothing of the output is held in shared memory;
//   * no CTA-wide barrier per tile: a warp that finishes its slice goes on to
//     the next tile without waiting for the other warps.
//
// OP::map_slice<PER>(V a[PER]) maps a lane's PER 16-byte vectors in place; with
// R > 1 outputs per input, OP::map_slice<PER>(a, b[R PER]) fills b instead.
template <typename V, int TILE_VECS, int STAGES, int NC, typename OP, int R = 1>
__device__ __forceinline__ void tma_load_map(const V *__restrict__ in, V *__restrict__ out, int64_t ntiles, OP op)
{
    static_assert(sizeof(V) == 16, "16-byte vectors");
    static_assert(TILE_VECS % (32 * NC) == 0, "tile must split evenly over the consumer warps");
    constexpr int PER = TILE_VECS / (32 * NC);
    constexpr uint32_t TILE_BYTES = TILE_VECS * 16;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    V *tiles = reinterpret_cast<V *>(smem_raw);
    __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init_elect(&full[s], 1); mbar_init_elect(&empty[s], NC); }
        fence_mbar_init();
    }
    pdl_begin();
    __syncthreads();

    const int64_t first = blockIdx.x, step = gridDim.x;
    if (warp == 0) {   // producer: all 32 lanes run the loop, one elected lane issues (no divergence)
        int s = 0;
        uint32_t ph = 0;
        int64_t k = 0;
        for (int64_t t = first; t < ntiles; t += step, ++k) {
            if (k >= STAGES) mbar_wait(&empty[s], ph ^ 1);
            elect_tma_load(&full[s], tiles + (size_t)s * TILE_VECS, in + t * TILE_VECS, TILE_BYTES);
            if (++s == STAGES) { s = 0; ph ^= 1; }
        }
        return;
    }
    const int w = warp - 1;
    const int off = w * (PER * 32) + lane;
    int s = 0;
    uint32_t ph = 0;
    for (int64_t t = first; t < ntiles; t += step) {
        mbar_wait(&full[s], ph);
        const V *tile = tiles + (size_t)s * TILE_VECS + off;
        V a[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j) a[j] = tile[32 * j];
        // WAR across proxies: the generic-proxy reads of this stage must be
        // ordered before the producer's next async-proxy (TMA) write into it
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if constexpr (R == 1) {
            op.template map_slice<PER>(a);
            V *o = out + t * TILE_VECS + off;
#pragma unroll
            for (int j = 0; j < PER; ++j) st_stream(o + 32 * j, a[j]);
        } else {
            // R output vectors per input vector (input vector i -> outputs R i .. R i + R - 1)
            V b[R * PER];
            op.template map_slice<PER>(a, b);
            V *o = out + (size_t)R * (t * TILE_VECS + off);
#pragma unroll
            for (int j = 0; j < PER; ++j)
#pragma unroll
                for (int r = 0; r < R; ++r) st_stream(o + R * 32 * j + r, b[R * j + r]);
        }
        if (++s == STAGES) { s = 0; ph ^= 1; }
    }
}

}  // namespace qm
