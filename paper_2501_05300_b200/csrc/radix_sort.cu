// radix_sort.cu -- hand-written stable LSD radix sort of (uint64 key, uint32 value) pairs.
//
// Per 8-bit digit pass: (1) per-tile 256-bin histograms stored digit-major, (2) one exclusive
// scan over all (digit, tile) counts gives every tile's output offset per digit, (3) a stable
// scatter: each tile ranks its keys per digit in input order (warp match + per-warp counts,
// chunk by chunk) and writes key/value to offset + rank.  Deterministic; no atomics in global
// memory.  Used for the Morton/level particle sort (north_star (a)) and the contact-key sorts.
#include "common.cuh"

namespace {
constexpr int RS_THREADS = 256;
constexpr int RS_ITEMS = 16;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;
constexpr int RS_WARPS = RS_THREADS / 32;

__global__ void k_rs_hist(const uint64_t *__restrict__ keys, int64_t n, int shift, uint32_t *__restrict__ hist,
                          int64_t ntiles)
{
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * RS_TILE;
#pragma unroll 4
    for (int k = 0; k < RS_ITEMS; k++) {
        int64_t i = base + (int64_t)k * RS_THREADS + threadIdx.x;
        if (i < n) atomicAdd(&h[(keys[i] >> shift) & 0xFF], 1u);
    }
    __syncthreads();
    hist[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

__global__ void k_rs_scatter(const uint64_t *__restrict__ kin, const uint32_t *__restrict__ vin,
                             uint64_t *__restrict__ kout, uint32_t *__restrict__ vout, int64_t n, int shift,
                             const uint32_t *__restrict__ offs, int64_t ntiles)
{
    __shared__ uint32_t running[256];
    __shared__ uint32_t whist[RS_WARPS][256];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    running[threadIdx.x] = offs[(int64_t)threadIdx.x * ntiles + blockIdx.x];
    for (int q = 0; q < RS_WARPS; q++) whist[q][threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * RS_TILE;
    const unsigned lt = (1u << lane) - 1u;
    for (int k = 0; k < RS_ITEMS; k++) {
        int64_t i = base + (int64_t)k * RS_THREADS + threadIdx.x;
        const bool valid = i < n;
        uint64_t key = valid ? kin[i] : 0;
        uint32_t val = valid ? vin[i] : 0;
        uint32_t d = valid ? (uint32_t)((key >> shift) & 0xFF) : 256u + lane;   // invalid: unique
        unsigned peers = __match_any_sync(0xffffffffu, d);
        uint32_t rank_w = __popc(peers & lt);
        if (valid && rank_w == 0) whist[w][d] = __popc(peers);
        __syncthreads();
        if (valid) {
            uint32_t pre = 0;
            for (int q = 0; q < w; q++) pre += whist[q][d];
            uint32_t dst = running[d] + pre + rank_w;
            kout[dst] = key;
            vout[dst] = val;
        }
        __syncthreads();
        uint32_t tot = 0;
        for (int q = 0; q < RS_WARPS; q++) { tot += whist[q][threadIdx.x]; whist[q][threadIdx.x] = 0; }
        running[threadIdx.x] += tot;
        __syncthreads();
    }
}
}  // namespace

size_t sort_temp_bytes(int64_t n)
{
    int64_t ntiles = (n + RS_TILE - 1) / RS_TILE;
    int64_t m = 256 * ntiles;
    return (size_t)(m + 1) * sizeof(uint32_t) + scan_temp_bytes(m) + 512;
}

void radix_sort_u64(uint64_t *keys[2], uint32_t *vals[2], int64_t n, int nbits, void *temp, cudaStream_t s,
                    long long *launches)
{
    if (n <= 1) return;
    int64_t ntiles = (n + RS_TILE - 1) / RS_TILE;
    int64_t m = 256 * ntiles;
    uint32_t *hist = (uint32_t *)temp;
    void *stemp = (void *)((char *)temp + (((size_t)(m + 1) * sizeof(uint32_t) + 255) & ~(size_t)255));
    int passes = (nbits + 7) / 8;
    int cur = 0;
    for (int p = 0; p < passes; p++) {
        int shift = 8 * p;
        k_rs_hist<<<(unsigned)ntiles, RS_THREADS, 0, s>>>(keys[cur], n, shift, hist, ntiles);
        scan_u32(hist, hist, m, stemp, s, launches);
        k_rs_scatter<<<(unsigned)ntiles, RS_THREADS, 0, s>>>(keys[cur], vals[cur], keys[cur ^ 1], vals[cur ^ 1], n,
                                                             shift, hist, ntiles);
        if (launches) *launches += 2;
        cur ^= 1;
    }
    if (cur != 0) {
        cudaMemcpyAsync(keys[0], keys[1], n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s);
        cudaMemcpyAsync(vals[0], vals[1], n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s);
    }
}
