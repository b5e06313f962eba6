// dist.cu -- x-slab decomposition transports and data-movement kernels (see dist.h).
#include <dlfcn.h>

#include <cstring>
#include <mutex>

#include <nccl.h>

#include "common.cuh"
#include "dist.h"

// ------------------------------------------------------------------ NCCL (opened at run time)
namespace {
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
};

NcclApi &nccl(std::string &err)
{
    static NcclApi api;
    static bool tried = false;
    static std::mutex mu;                 // contexts may be created from several host threads
    std::lock_guard<std::mutex> lock(mu);
    if (tried) {
        if (!api.ok) err = "libnccl.so.2 could not be loaded";
        return api;
    }
    tried = true;
    // the copy torch already loaded (same soname) first, then the loader's search path
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        err = std::string("dlopen libnccl.so.2: ") + dlerror();
        return api;
    }
#define SYM(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, "nccl" #f))
    SYM(GetUniqueId); SYM(CommInitRank); SYM(CommDestroy); SYM(Send); SYM(Recv); SYM(AllReduce);
    SYM(GroupStart); SYM(GroupEnd); SYM(GetErrorString);
#undef SYM
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv && api.AllReduce &&
             api.GroupStart && api.GroupEnd && api.GetErrorString;
    if (!api.ok) err = "libnccl.so.2 lacks a required symbol";
    return api;
}

struct NcclTransport : Transport {
    ncclComm_t comm = nullptr;
    NcclApi *api = nullptr;
    double *dbuf = nullptr;
    long long *ibuf = nullptr;
    ~NcclTransport() override
    {
        if (comm) api->CommDestroy(comm);
        if (dbuf) cudaFree(dbuf);
        if (ibuf) cudaFree(ibuf);
    }
    bool check(ncclResult_t r, std::string &err, const char *what)
    {
        if (r == ncclSuccess) return true;
        err = std::string(what) + ": " + api->GetErrorString(r);
        return false;
    }
    bool exchange(const void *const send[2], const size_t sbytes[2], void *const recv[2], const size_t rbytes[2],
                  cudaStream_t s, std::string &err) override
    {
        const int nb[2] = {rank - 1, rank + 1};
        if (!check(api->GroupStart(), err, "ncclGroupStart")) return false;
        for (int k = 0; k < 2; k++) {
            if (nb[k] < 0 || nb[k] >= G) continue;
            if (sbytes[k] && !check(api->Send(send[k], sbytes[k], ncclChar, nb[k], comm, s), err, "ncclSend")) return false;
            if (rbytes[k] && !check(api->Recv(recv[k], rbytes[k], ncclChar, nb[k], comm, s), err, "ncclRecv")) return false;
        }
        return check(api->GroupEnd(), err, "ncclGroupEnd");
    }
    template <class T>
    bool allreduce(T *v, int n, int op, cudaStream_t s, std::string &err, T *dev, ncclDataType_t ty)
    {
        if (cudaMemcpyAsync(dev, v, n * sizeof(T), cudaMemcpyHostToDevice, s) != cudaSuccess) { err = "H2D"; return false; }
        if (!check(api->AllReduce(dev, dev, n, ty, op ? ncclMax : ncclSum, comm, s), err, "ncclAllReduce")) return false;
        if (cudaMemcpyAsync(v, dev, n * sizeof(T), cudaMemcpyDeviceToHost, s) != cudaSuccess) { err = "D2H"; return false; }
        if (cudaStreamSynchronize(s) != cudaSuccess) { err = "sync after allreduce"; return false; }
        return true;
    }
    bool allreduce_f64(double *v, int n, int op, cudaStream_t s, std::string &err) override
    {
        return allreduce<double>(v, n, op, s, err, dbuf, ncclFloat64);
    }
    bool graph_safe() const override { return true; }   // grouped ncclSend/ncclRecv: stream-ordered
    bool allreduce_i64(long long *v, int n, int op, cudaStream_t s, std::string &err) override
    {
        return allreduce<long long>(v, n, op, s, err, ibuf, ncclInt64);
    }
};

struct LoopTransport : Transport {
    LoopGroup *g = nullptr;
    ~LoopTransport() override
    {
        auto &sl = g->slot[rank];
        if (sl.ready) cudaEventDestroy(sl.ready);
        if (sl.done) cudaEventDestroy(sl.done);
        sl.ready = sl.done = nullptr;
    }
    bool exchange(const void *const send[2], const size_t sbytes[2], void *const recv[2], const size_t rbytes[2],
                  cudaStream_t s, std::string &err) override
    {
        auto &me = g->slot[rank];
        me.send[0] = send[0];
        me.send[1] = send[1];
        cudaEventRecord(me.ready, s);
        g->barrier();
        // my left neighbour's "right" buffer is meant for me, and vice versa
        if (rank > 0 && rbytes[0]) {
            cudaStreamWaitEvent(s, g->slot[rank - 1].ready, 0);
            cudaMemcpyAsync(recv[0], g->slot[rank - 1].send[1], rbytes[0], cudaMemcpyDeviceToDevice, s);
        }
        if (rank < G - 1 && rbytes[1]) {
            cudaStreamWaitEvent(s, g->slot[rank + 1].ready, 0);
            cudaMemcpyAsync(recv[1], g->slot[rank + 1].send[0], rbytes[1], cudaMemcpyDeviceToDevice, s);
        }
        cudaEventRecord(me.done, s);
        g->barrier();
        // my send buffers are reusable once the neighbours' copies are done
        if (rank > 0) cudaStreamWaitEvent(s, g->slot[rank - 1].done, 0);
        if (rank < G - 1) cudaStreamWaitEvent(s, g->slot[rank + 1].done, 0);
        if (cudaGetLastError() != cudaSuccess) { err = "loopback exchange failed"; return false; }
        return true;
    }
    template <class T>
    bool allreduce(T *v, int n, int op, T *(*field)(LoopGroup::Slot &), std::string &err)
    {
        if (n > 64) { err = "loopback allreduce: n > 64"; return false; }
        std::memcpy(field(g->slot[rank]), v, n * sizeof(T));
        g->barrier();
        for (int k = 0; k < n; k++) {
            T a = field(g->slot[0])[k];
            for (int r = 1; r < G; r++) {
                const T b = field(g->slot[r])[k];
                a = op ? (b > a ? b : a) : a + b;      // rank order: identical on every rank
            }
            v[k] = a;
        }
        g->barrier();
        return true;
    }
    bool allreduce_f64(double *v, int n, int op, cudaStream_t, std::string &err) override
    {
        return allreduce<double>(v, n, op, [](LoopGroup::Slot &s) { return s.red; }, err);
    }
    bool allreduce_i64(long long *v, int n, int op, cudaStream_t, std::string &err) override
    {
        return allreduce<long long>(v, n, op, [](LoopGroup::Slot &s) { return s.redi; }, err);
    }
};
}  // namespace

bool nccl_unique_id(void *out128, std::string &err)
{
    NcclApi &api = nccl(err);
    if (!api.ok) return false;
    ncclUniqueId id;
    if (api.GetUniqueId(&id) != ncclSuccess) { err = "ncclGetUniqueId failed"; return false; }
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out128, &id, 128);
    return true;
}

Transport *make_nccl_transport(int rank, int G, const void *unique_id, std::string &err)
{
    NcclApi &api = nccl(err);
    if (!api.ok) return nullptr;
    if (!unique_id) { err = "world_size > 1 over NCCL needs nccl_unique_id"; return nullptr; }
    auto *t = new NcclTransport();
    t->rank = rank;
    t->G = G;
    t->api = &api;
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    if (cudaMalloc(&t->dbuf, 64 * sizeof(double)) != cudaSuccess || cudaMalloc(&t->ibuf, 64 * sizeof(long long)) != cudaSuccess) {
        err = "cudaMalloc for the NCCL scalars failed";
        delete t;
        return nullptr;
    }
    const ncclResult_t r = api.CommInitRank(&t->comm, G, id, rank);
    if (r != ncclSuccess) {
        err = std::string("ncclCommInitRank: ") + api.GetErrorString(r);
        t->comm = nullptr;
        delete t;
        return nullptr;
    }
    return t;
}

Transport *make_loop_transport(int rank, LoopGroup *grp, std::string &err)
{
    if (!grp || rank < 0 || rank >= grp->G) { err = "bad loopback group / rank"; return nullptr; }
    auto *t = new LoopTransport();
    t->rank = rank;
    t->G = grp->G;
    t->g = grp;
    auto &sl = grp->slot[rank];
    if (cudaEventCreateWithFlags(&sl.ready, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming) != cudaSuccess) {
        err = "cudaEventCreate failed";
        delete t;
        return nullptr;
    }
    return t;
}

// ------------------------------------------------------------------ kernels
#define GRID(n) (unsigned)(((n) + 255) / 256), 256, 0, s

// ------------------------------------------------------------------ history hand-over
// A contact's impulse history is authoritative on a rank that owns one of its bodies (that rank
// has held the contact since it formed).  At every rebuild each rank sends each neighbour the
// authoritative entries whose bodies the neighbour will hold, so a contact that enters a rank's
// local set -- a particle migrating, or a pair drifting into the ghost band -- arrives with its
// history and every rank warm-starts it from the same impulses (bit-identity).
__global__ void k_hist_auth(int64_t nh, const uint32_t *__restrict__ vals, const uint2 *__restrict__ cand,
                            const uint8_t *__restrict__ own, uint8_t *__restrict__ auth)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nh) return;
    const uint2 ij = cand[vals[t]];
    auth[t] = (own[ij.x] || (!(ij.y & PARTNER_EXT) && own[ij.y])) ? 1 : 0;
}
__global__ void k_gid_list(int64_t n, const uint32_t *__restrict__ idx, const uint32_t *__restrict__ gid,
                           uint64_t *__restrict__ out)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) out[t] = gid[idx ? idx[t] : t];
}
__device__ __forceinline__ bool in_sorted(const uint64_t *__restrict__ a, int64_t n, uint64_t v)
{
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo < n && a[lo] == v;
}
__global__ void k_hist_select(int64_t nh, const uint64_t *__restrict__ hkey, const uint8_t *__restrict__ auth,
                              const uint64_t *__restrict__ B, int64_t nB, uint32_t *__restrict__ flag)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nh) return;
    const uint64_t k = hkey[t];
    const uint32_t ga = (uint32_t)(k >> 32), gb = (uint32_t)k;
    const bool ext = gb >= PLATE_KEY_BASE;                 // walls and plates: the particle alone
    flag[t] = (auth[t] && in_sorted(B, nB, ga) && (ext || in_sorted(B, nB, gb))) ? 1u : 0u;
}
struct __align__(16) HistRec { unsigned long long key, pad; P4 a, b; };
__global__ void k_hist_pack(int64_t n, const uint32_t *__restrict__ idx, const uint64_t *__restrict__ hkey,
                            const P4 *__restrict__ hPa, const P4 *__restrict__ hPb, HistRec *__restrict__ out)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const uint32_t i = idx[t];
    out[t] = HistRec{hkey[i], 0ull, hPa[i], hPb[i]};
}
__global__ void k_hist_unpack(int64_t n, const HistRec *__restrict__ in, uint64_t *__restrict__ key,
                              uint32_t *__restrict__ val, uint32_t val0, P4 *__restrict__ Pa, P4 *__restrict__ Pb)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const HistRec r = in[t];
    key[t] = r.key;
    val[t] = val0 + (uint32_t)t;
    Pa[t] = r.a;
    Pb[t] = r.b;
}
__global__ void k_iota_keys(int64_t n, const uint64_t *__restrict__ hkey, uint64_t *__restrict__ key,
                            uint32_t *__restrict__ val)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) { key[t] = hkey[t]; val[t] = (uint32_t)t; }
}
// after a stable sort of (key, entry index): keep the last entry of each key (received entries
// were appended after the rank's own, so they win); output compacted in key order
__global__ void k_hist_last(int64_t n, const uint64_t *__restrict__ key, uint32_t *__restrict__ flag)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) flag[t] = (t + 1 == n || key[t + 1] != key[t]) ? 1u : 0u;
}
__global__ void k_hist_emit(int64_t n, const uint32_t *__restrict__ flag, const uint32_t *__restrict__ scan,
                            const uint64_t *__restrict__ key, const uint32_t *__restrict__ val,
                            const P4 *__restrict__ Pa, const P4 *__restrict__ Pb, uint64_t *__restrict__ okey,
                            P4 *__restrict__ oPa, P4 *__restrict__ oPb)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n || !flag[t]) return;
    const uint32_t o = scan[t], v = val[t];
    okey[o] = key[t];
    oPa[o] = Pa[v];
    oPb[o] = Pb[v];
}
#define G256(n) (unsigned)(((n) + 255) / 256), 256, 0, s
void launch_hist_auth(int64_t nh, const uint32_t *vals, const uint2 *cand, const uint8_t *own, uint8_t *auth, cudaStream_t s)
{ if (nh) k_hist_auth<<<G256(nh)>>>(nh, vals, cand, own, auth); }
void launch_gid_list(int64_t n, const uint32_t *idx, const uint32_t *gid, uint64_t *out, cudaStream_t s)
{ if (n) k_gid_list<<<G256(n)>>>(n, idx, gid, out); }
void launch_hist_select(int64_t nh, const uint64_t *hkey, const uint8_t *auth, const uint64_t *B, int64_t nB, uint32_t *flag,
                        cudaStream_t s)
{ if (nh) k_hist_select<<<G256(nh)>>>(nh, hkey, auth, B, nB, flag); }
void launch_hist_pack(int64_t n, const uint32_t *idx, const uint64_t *hkey, const P4 *hPa, const P4 *hPb, void *out,
                      cudaStream_t s)
{ if (n) k_hist_pack<<<G256(n)>>>(n, idx, hkey, hPa, hPb, (HistRec *)out); }
void launch_hist_unpack(int64_t n, const void *in, uint64_t *key, uint32_t *val, uint32_t val0, P4 *Pa, P4 *Pb,
                        cudaStream_t s)
{ if (n) k_hist_unpack<<<G256(n)>>>(n, (const HistRec *)in, key, val, val0, Pa, Pb); }
void launch_iota_keys(int64_t n, const uint64_t *hkey, uint64_t *key, uint32_t *val, cudaStream_t s)
{ if (n) k_iota_keys<<<G256(n)>>>(n, hkey, key, val); }
void launch_hist_last(int64_t n, const uint64_t *key, uint32_t *flag, cudaStream_t s)
{ if (n) k_hist_last<<<G256(n)>>>(n, key, flag); }
void launch_hist_emit(int64_t n, const uint32_t *flag, const uint32_t *scan, const uint64_t *key, const uint32_t *val,
                      const P4 *Pa, const P4 *Pb, uint64_t *okey, P4 *oPa, P4 *oPb, cudaStream_t s)
{ if (n) k_hist_emit<<<G256(n)>>>(n, flag, scan, key, val, Pa, Pb, okey, oPa, oPb); }
#undef G256

// histogram of the owned particles' x over [lo, hi) in nb bins (outside: edge bins)
__global__ void k_hist_x(int64_t n, const uint8_t *__restrict__ own, const double4 *__restrict__ pos, double lo,
                         double hi, int nb, unsigned long long *__restrict__ hist)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || (own && !own[i])) return;
    int b = (int)floor((pos[i].x - lo) / (hi - lo) * nb);
    b = b < 0 ? 0 : (b >= nb ? nb - 1 : b);
    atomicAdd(&hist[b], 1ull);
}
void launch_hist_x(int64_t n, const uint8_t *own, const double4 *pos, double lo, double hi, int nb,
                   unsigned long long *hist, cudaStream_t s)
{
    cudaMemsetAsync(hist, 0, nb * sizeof(unsigned long long), s);
    if (n) k_hist_x<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, own, pos, lo, hi, nb, hist);
}

__global__ void k_slab_flags(int64_t n, const double4 *__restrict__ pos, double lo, double hi, uint32_t *__restrict__ flag)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) { const double x = pos[i].x; flag[i] = (x >= lo && x < hi) ? 1u : 0u; }
}

__global__ void k_band_flags(int64_t n, const double4 *__restrict__ pos, double lo_band, double hi_band, int use_lo,
                             int use_hi, uint32_t *__restrict__ flo, uint32_t *__restrict__ fhi)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double x = pos[i].x;
    flo[i] = (use_lo && x < lo_band) ? 1u : 0u;
    fhi[i] = (use_hi && x >= hi_band) ? 1u : 0u;
}

__global__ void k_compact_idx(int64_t n, const uint32_t *__restrict__ flag, const uint32_t *__restrict__ scan,
                              uint32_t *__restrict__ out)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && flag[i]) out[scan[i]] = (uint32_t)i;
}

__global__ void k_gather_state(int64_t n, const uint32_t *__restrict__ idx, const double4 *__restrict__ pos,
                               const double4 *__restrict__ vel, const double4 *__restrict__ ang,
                               const uint32_t *__restrict__ gid, double4 *__restrict__ opos, double4 *__restrict__ ovel,
                               double4 *__restrict__ oang, uint32_t *__restrict__ ogid)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const uint32_t i = idx[k];
    opos[k] = pos[i];
    ovel[k] = vel[i];
    oang[k] = ang[i];
    ogid[k] = gid[i];
}

// band record: pos, vel, ang, (gid bits, 0, 0, 0) -- 128 B per particle
__global__ void k_pack_band(int64_t n, const uint32_t *__restrict__ idx, const double4 *__restrict__ pos,
                            const double4 *__restrict__ vel, const double4 *__restrict__ ang,
                            const uint32_t *__restrict__ gid, double4 *__restrict__ buf)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const uint32_t i = idx[k];
    buf[4 * k] = pos[i];
    buf[4 * k + 1] = vel[i];
    buf[4 * k + 2] = ang[i];
    buf[4 * k + 3] = make_double4(__longlong_as_double((long long)gid[i]), 0.0, 0.0, 0.0);
}

__global__ void k_unpack_band(int64_t n, const double4 *__restrict__ buf, double4 *__restrict__ pos,
                              double4 *__restrict__ vel, double4 *__restrict__ ang, uint32_t *__restrict__ gid)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    pos[k] = buf[4 * k];
    vel[k] = buf[4 * k + 1];
    ang[k] = buf[4 * k + 2];
    gid[k] = (uint32_t)__double_as_longlong(buf[4 * k + 3].x);
}

__global__ void k_pack_halo(int64_t n, const uint32_t *__restrict__ idx, const double4 *__restrict__ vel,
                            const double4 *__restrict__ ang, double4 *__restrict__ buf)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const uint32_t i = idx[k];
    buf[2 * k] = vel[i];
    buf[2 * k + 1] = ang[i];
}

__global__ void k_unpack_halo(int64_t n, const uint32_t *__restrict__ idx, const double4 *__restrict__ buf,
                              double4 *__restrict__ vel, double4 *__restrict__ ang)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const uint32_t i = idx[k];
    vel[i] = buf[2 * k];
    ang[i] = buf[2 * k + 1];
}

__global__ void k_inv_perm(int64_t n, const uint32_t *__restrict__ perm, uint32_t *__restrict__ inv)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) inv[perm[i]] = (uint32_t)i;
}

__global__ void k_map_idx(int64_t n, const uint32_t *__restrict__ in, uint32_t offset, const uint32_t *__restrict__ inv,
                          uint32_t *__restrict__ out)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) out[k] = inv[(in ? in[k] : (uint32_t)k) + offset];
}

// owned gids first (ghosts get a key above every gid)
__global__ void k_gid_keys(int64_t n, const uint32_t *__restrict__ gid, const uint8_t *__restrict__ own,
                           uint64_t *__restrict__ keys, uint32_t *__restrict__ vals)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) { keys[i] = own[i] ? (uint64_t)gid[i] : (1ull << 32); vals[i] = (uint32_t)i; }
}

// after the rebuild's sort (perm: new -> old), owned iff the old index was in the owned block
__global__ void k_own_flags(int64_t n, const uint32_t *__restrict__ perm, uint32_t n_own, uint8_t *__restrict__ own)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) own[i] = perm[i] < n_own ? 1 : 0;
}

__global__ void k_keys_to_u32(int64_t n, const uint64_t *__restrict__ keys, uint32_t *__restrict__ out)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (uint32_t)keys[i];
}

void launch_slab_flags(int64_t n, const double4 *pos, double lo, double hi, uint32_t *flag, cudaStream_t s)
{ if (n) k_slab_flags<<<GRID(n)>>>(n, pos, lo, hi, flag); }
void launch_band_flags(int64_t n, const double4 *pos, double lo_band, double hi_band, int use_lo, int use_hi,
                       uint32_t *flag_lo, uint32_t *flag_hi, cudaStream_t s)
{ if (n) k_band_flags<<<GRID(n)>>>(n, pos, lo_band, hi_band, use_lo, use_hi, flag_lo, flag_hi); }
void launch_compact_idx(int64_t n, const uint32_t *flag, const uint32_t *scan, uint32_t *out, cudaStream_t s)
{ if (n) k_compact_idx<<<GRID(n)>>>(n, flag, scan, out); }
void launch_gather_state(int64_t n, const uint32_t *idx, const double4 *pos, const double4 *vel, const double4 *ang,
                         const uint32_t *gid, double4 *opos, double4 *ovel, double4 *oang, uint32_t *ogid, cudaStream_t s)
{ if (n) k_gather_state<<<GRID(n)>>>(n, idx, pos, vel, ang, gid, opos, ovel, oang, ogid); }
void launch_pack_band(int64_t n, const uint32_t *idx, const double4 *pos, const double4 *vel, const double4 *ang,
                      const uint32_t *gid, double4 *buf, cudaStream_t s)
{ if (n) k_pack_band<<<GRID(n)>>>(n, idx, pos, vel, ang, gid, buf); }
void launch_unpack_band(int64_t n, const double4 *buf, double4 *pos, double4 *vel, double4 *ang, uint32_t *gid,
                        cudaStream_t s)
{ if (n) k_unpack_band<<<GRID(n)>>>(n, buf, pos, vel, ang, gid); }
void launch_pack_halo(int64_t n, const uint32_t *idx, const double4 *vel, const double4 *ang, double4 *buf, cudaStream_t s)
{ if (n) k_pack_halo<<<GRID(n)>>>(n, idx, vel, ang, buf); }
void launch_unpack_halo(int64_t n, const uint32_t *idx, const double4 *buf, double4 *vel, double4 *ang, cudaStream_t s)
{ if (n) k_unpack_halo<<<GRID(n)>>>(n, idx, buf, vel, ang); }
void launch_inv_perm(int64_t n, const uint32_t *perm, uint32_t *inv, cudaStream_t s)
{ if (n) k_inv_perm<<<GRID(n)>>>(n, perm, inv); }
void launch_map_idx(int64_t n, const uint32_t *in, uint32_t offset, const uint32_t *inv, uint32_t *out, cudaStream_t s)
{ if (n) k_map_idx<<<GRID(n)>>>(n, in, offset, inv, out); }
void launch_gid_keys(int64_t n, const uint32_t *gid, const uint8_t *own, uint64_t *keys, uint32_t *vals, cudaStream_t s)
{ if (n) k_gid_keys<<<GRID(n)>>>(n, gid, own, keys, vals); }
void launch_own_flags(int64_t n, const uint32_t *perm, uint32_t n_own, uint8_t *own, cudaStream_t s)
{ if (n) k_own_flags<<<GRID(n)>>>(n, perm, n_own, own); }
void launch_keys_to_u32(int64_t n, const uint64_t *keys, uint32_t *out, cudaStream_t s)
{ if (n) k_keys_to_u32<<<GRID(n)>>>(n, keys, out); }
