// fs_scan.cuh -- tile-ordered prefix sums for the queue-order kernels
// (fs_order.cuh) and K1's ordered job list: decoupled look-back over dynamic
// tile ids, block scans.
#pragma once
#include "fs_device.cuh"

#define FS_OT_THREADS 256
#define FS_OT_ITEMS 8
#define FS_OT_TILE (FS_OT_THREADS * FS_OT_ITEMS)
#define FS_RS_BINS 256
#define FS_RS_MAXPASS 4
#define FS_LB_EPOCH_MASK 0xffffffu
#define FS_LB_VALUE_MASK ((1ull << 38) - 1)

// Per-fill device counters (zeroed by one memset per fill).
struct OrderCtl {
    int32_t tile[8];      // dynamic tile ids, one per look-back launch
    int32_t njobs;        // |B| (k_match_fast's appends)
    int32_t na;           // |A| (k_merge_a's last tile)
    int32_t pad_[6];
};
enum { OT_UPKEEP = 0, OT_MERGE_A = 1 };

// ---------------------------------------------------------------- look-back
// Tile status word: [63:62] flag (1 aggregate, 2 inclusive prefix), [61:38]
// launch epoch, [37:0] value.  Words of other launches read as "not yet".
__device__ __forceinline__ unsigned long long lb_word(uint32_t flag, uint32_t epoch, int64_t v) {
    return ((unsigned long long)flag << 62) | ((unsigned long long)(epoch & FS_LB_EPOCH_MASK) << 38) |
           ((unsigned long long)v & FS_LB_VALUE_MASK);
}
__device__ __forceinline__ void lb_store(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long lb_load(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Exclusive prefix of `agg` over tiles 0..tile-1 by one warp: 32
// predecessors' words per step (the nearest inclusive prefix ends the walk),
// so a tile whose predecessors have only published aggregates walks back 32
// tiles per round trip.  Tile ids must be handed out in launch order (dynamic
// ids) so every predecessor is running or done.  Call with all 32 lanes of
// one warp; every lane returns the exclusive prefix.
__device__ inline int64_t warp_lookback(unsigned long long *st, int32_t tile, uint32_t epoch, int64_t agg, int lane) {
    if (tile == 0) {
        if (lane == 0) lb_store(st, lb_word(2, epoch, agg));
        return 0;
    }
    if (lane == 0) lb_store(st + tile, lb_word(1, epoch, agg));
    const uint32_t ep = epoch & FS_LB_EPOCH_MASK;
    int64_t excl = 0;
    int32_t top = tile - 1;  // lane l reads tile top - l
    while (true) {
        const int32_t k = top - lane;
        unsigned long long w = 0;
        uint32_t flag = 2;   // lanes past tile 0 read as an empty inclusive word
        if (k >= 0) {
            do {
                w = lb_load(st + k);
                flag = (uint32_t)(w >> 62);
                if ((uint32_t)((w >> 38) & FS_LB_EPOCH_MASK) != ep) flag = 0;
            } while (flag == 0);
        }
        const unsigned incl = __ballot_sync(FS_FULL, flag == 2);
        const int stop = incl ? __ffs(incl) - 1 : 31;  // nearest inclusive word (or the whole window)
        int64_t v = (k >= 0 && lane <= stop) ? (int64_t)(w & FS_LB_VALUE_MASK) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FS_FULL, v, o);
        excl += v;
        if (incl) break;
        top -= 32;
    }
    if (lane == 0) lb_store(st + tile, lb_word(2, epoch, excl + agg));
    return excl;
}

__device__ __forceinline__ int32_t dyn_tile(int32_t *ctr) {
    __shared__ int32_t t;
    if (threadIdx.x == 0) t = atomicAdd(ctr, 1);
    __syncthreads();
    const int32_t v = t;
    __syncthreads();
    return v;
}

// Block-wide exclusive scan of one int per thread (256 threads); returns the
// thread's exclusive prefix, *total the block sum.
__device__ inline int32_t block_excl_scan256(int32_t v, int32_t *total) {
    __shared__ int32_t ws[FS_OT_THREADS / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(FS_FULL, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    int32_t wbase = 0, tot = 0;
#pragma unroll
    for (int k = 0; k < FS_OT_THREADS / 32; k++) {
        const int32_t s = ws[k];
        if (k < warp) wbase += s;
        tot += s;
    }
    __syncthreads();
    *total = tot;
    return wbase + x - v;
}

