// dist.h -- transports of the x-slab domain decomposition.
//
// A rank owns the particles of its slab [slab_lo, slab_hi) and holds ghost copies of its two
// neighbours' particles within the band width W of the shared faces.  Two collectives carry
// the whole decomposition:
//   exchange   -- point-to-point with the left (rank-1) and right (rank+1) neighbours: the
//                 ghost band states at rebuild, the ghost velocities after every sweep;
//   allreduce  -- a handful of per-step scalars (impact trigger, NaN flag, rebuild trigger,
//                 report sums, int64 plate reactions).
// NcclTransport runs one process per GPU over NCCL (libnccl is opened at run time, the one
// torch already loaded when present).  LoopTransport runs G ranks as G host threads of one
// process (the same device or several), exchanging with cudaMemcpyAsync after host barriers:
// it exercises every line of the decomposition on a single GPU without kernels that wait on
// one another.
#pragma once
#include <cuda_runtime.h>

#include <condition_variable>
#include <mutex>
#include <string>
#include <vector>

struct Transport {
    int rank = 0, G = 1;
    virtual ~Transport() {}
    // send[k]/recv[k], k = 0 left neighbour, 1 right neighbour; byte counts agreed beforehand
    // (0 -> nothing moves in that direction).  Stream-ordered on s.
    virtual bool exchange(const void *const send[2], const size_t sbytes[2], void *const recv[2], const size_t rbytes[2],
                          cudaStream_t s, std::string &err) = 0;
    // host-side reductions (op 0 sum, 1 max) over all ranks; the caller has synchronised s
    virtual bool allreduce_f64(double *v, int n, int op, cudaStream_t s, std::string &err) = 0;
    virtual bool allreduce_i64(long long *v, int n, int op, cudaStream_t s, std::string &err) = 0;
    // exchange() only enqueues stream-ordered work (no host synchronisation): it can be captured
    // in a CUDA graph
    virtual bool graph_safe() const { return false; }
};

Transport *make_nccl_transport(int rank, int G, const void *unique_id, std::string &err);
bool nccl_unique_id(void *out128, std::string &err);

struct LoopGroup {
    int G;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    long long generation = 0;
    struct Slot {
        const void *send[2] = {nullptr, nullptr};
        cudaEvent_t ready = nullptr, done = nullptr;
        double red[64];
        long long redi[64];
    };
    std::vector<Slot> slot;
    explicit LoopGroup(int g) : G(g), slot(g) {}
    void barrier()
    {
        std::unique_lock<std::mutex> lk(m);
        const long long gen = generation;
        if (++arrived == G) {
            arrived = 0;
            generation++;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen; });
        }
    }
};

Transport *make_loop_transport(int rank, LoopGroup *grp, std::string &err);

// dist.cu kernels
void launch_slab_flags(int64_t n, const double4 *pos, double lo, double hi, uint32_t *flag, cudaStream_t s);
void launch_band_flags(int64_t n, const double4 *pos, double lo_band, double hi_band, int use_lo, int use_hi,
                       uint32_t *flag_lo, uint32_t *flag_hi, cudaStream_t s);
void launch_compact_idx(int64_t n, const uint32_t *flag, const uint32_t *scan, uint32_t *out, cudaStream_t s);
void launch_gather_state(int64_t n, const uint32_t *idx, const double4 *pos, const double4 *vel, const double4 *ang,
                         const uint32_t *gid, double4 *opos, double4 *ovel, double4 *oang, uint32_t *ogid, cudaStream_t s);
void launch_pack_band(int64_t n, const uint32_t *idx, const double4 *pos, const double4 *vel, const double4 *ang,
                      const uint32_t *gid, double4 *buf, cudaStream_t s);
void launch_unpack_band(int64_t n, const double4 *buf, double4 *pos, double4 *vel, double4 *ang, uint32_t *gid,
                        cudaStream_t s);
void launch_pack_halo(int64_t n, const uint32_t *idx, const double4 *vel, const double4 *ang, double4 *buf, cudaStream_t s);
void launch_unpack_halo(int64_t n, const uint32_t *idx, const double4 *buf, double4 *vel, double4 *ang, cudaStream_t s);
void launch_inv_perm(int64_t n, const uint32_t *perm, uint32_t *inv, cudaStream_t s);
void launch_map_idx(int64_t n, const uint32_t *in, uint32_t offset, const uint32_t *inv, uint32_t *out, cudaStream_t s);
void launch_gid_keys(int64_t n, const uint32_t *gid, const uint8_t *own, uint64_t *keys, uint32_t *vals, cudaStream_t s);
void launch_own_flags(int64_t n, const uint32_t *perm, uint32_t n_own, uint8_t *own, cudaStream_t s);
void launch_keys_to_u32(int64_t n, const uint64_t *keys, uint32_t *out, cudaStream_t s);
