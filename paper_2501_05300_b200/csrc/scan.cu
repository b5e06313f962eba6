// scan.cu -- deterministic exclusive prefix sum of uint32 (reduce-then-scan, 3 kernels).
// Used for contact compaction (candidate flags -> contact index), incidence CSR offsets and
// the radix sort's digit offsets.  Tile = 256 threads x 16 items.
#include "common.cuh"

namespace {
constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 16;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v)
{
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// block-wide exclusive scan of one value per thread; returns the exclusive prefix, total in *tot
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t *tot)
{
    __shared__ uint32_t wsum[SCAN_THREADS / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t inc = warp_incl_scan(v);
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    if (w == 0) {
        uint32_t s = lane < SCAN_THREADS / 32 ? wsum[lane] : 0u;
        s = warp_incl_scan(s);
        if (lane < SCAN_THREADS / 32) wsum[lane] = s;
    }
    __syncthreads();
    uint32_t base = w > 0 ? wsum[w - 1] : 0u;
    *tot = wsum[SCAN_THREADS / 32 - 1];
    __syncthreads();
    return base + inc - v;
}

__global__ void k_scan_reduce(const uint32_t *__restrict__ in, int64_t n, uint32_t *__restrict__ part)
{
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; k++) {
        int64_t i = base + (int64_t)k * SCAN_THREADS + threadIdx.x;
        if (i < n) s += in[i];
    }
    uint32_t tot;
    block_excl_scan(s, &tot);
    if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

__global__ void k_scan_partials(uint32_t *part, int64_t nb, uint32_t *total_out)
{
    uint32_t carry = 0;
    for (int64_t b0 = 0; b0 < nb; b0 += SCAN_THREADS) {
        int64_t i = b0 + threadIdx.x;
        uint32_t v = i < nb ? part[i] : 0u;
        uint32_t tot;
        uint32_t ex = block_excl_scan(v, &tot);
        if (i < nb) part[i] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) *total_out = carry;
}

__global__ void k_scan_down(const uint32_t *in, uint32_t *out, int64_t n, const uint32_t *__restrict__ part)
{
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    uint32_t v[SCAN_ITEMS];
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; k++) {
        int64_t i = base + k;
        v[k] = i < n ? in[i] : 0u;
        s += v[k];
    }
    uint32_t tot;
    uint32_t ex = block_excl_scan(s, &tot) + part[blockIdx.x];
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; k++) {
        int64_t i = base + k;
        if (i < n) out[i] = ex;
        ex += v[k];
    }
}
}  // namespace

size_t scan_temp_bytes(int64_t n)
{
    int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
    return (size_t)(nb + 1) * sizeof(uint32_t) + 256;
}

void scan_u32(const uint32_t *in, uint32_t *out, int64_t n, void *temp, cudaStream_t s, long long *launches)
{
    int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
    uint32_t *part = (uint32_t *)temp;
    if (n == 0) {
        cudaMemsetAsync(out, 0, sizeof(uint32_t), s);
        return;
    }
    k_scan_reduce<<<(unsigned)nb, SCAN_THREADS, 0, s>>>(in, n, part);
    k_scan_partials<<<1, SCAN_THREADS, 0, s>>>(part, nb, out + n);
    k_scan_down<<<(unsigned)nb, SCAN_THREADS, 0, s>>>(in, out, n, part);
    if (launches) *launches += 3;
}
