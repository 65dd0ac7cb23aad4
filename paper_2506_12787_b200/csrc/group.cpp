// Multi-GPU render inside the library: one context per
// device, the scene and the MLP weights replicated, the batch of positions split
// contiguously (B / P per device, the first B % P one more), no inter-device
// dependency while rendering, and one exchange: the outputs to the root device.
//
// The reference renders one position per call (train::render_at,
// training.cpp:189-195) and has no multi-device path; this is the batched caller
// side of that boundary, built on the public C ABI (swr_render /
// swr_render_device per device).
//
// * swr_group_render (host buffers): every device renders its shard straight into
//   its slice of the caller's buffers, one host thread per device; no collective.
// * swr_group_render_device (device buffers on the root): the root scatters each
//   shard's positions peer to peer, every device renders its shard chunk by chunk,
//   and each chunk is sent to the root as soon as it is rendered -- NCCL
//   point-to-point (ncclSend / ncclRecv in a group, one communicator per device from
//   ncclCommInitAll) on a per-device communication stream, so the transfer of chunk
//   k overlaps the rendering of chunk k + 1. The root's own shard renders in place.
//   A device listed twice (the single-GPU test arrangement) cannot join an NCCL
//   communicator; such groups move the chunks with peer copies instead.
// * swr_comm_* / swr_render_gather: the same gather between processes (one process
//   per GPU under torchrun), over a communicator made from an ncclUniqueId.
//
// NCCL is loaded at first use (dlopen "libnccl.so.2": the copy a host process such
// as torch already loaded, else the system one).
#include "swr.h"
#include "swr_internal.h"

#include <nccl.h>

#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <thread>

namespace
{
using namespace swr;

struct Nccl
{
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t *, int, const int *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;

    void check(ncclResult_t r, const char *what) const
    {
        if (r != ncclSuccess)
            throw std::runtime_error(std::string("NCCL ") + what + ": " + GetErrorString(r));
    }
};

const Nccl &nccl()
{
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h)
            throw std::runtime_error(std::string("cannot load libnccl.so.2: ") + dlerror());
        auto get = [&](const char *name) {
            void *f = dlsym(h, name);
            if (!f)
                throw std::runtime_error(std::string("libnccl.so.2 lacks ") + name);
            return f;
        };
        n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(get("ncclGetUniqueId"));
        n.CommInitAll = reinterpret_cast<decltype(n.CommInitAll)>(get("ncclCommInitAll"));
        n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(get("ncclCommInitRank"));
        n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(get("ncclCommDestroy"));
        n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(get("ncclGroupStart"));
        n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(get("ncclGroupEnd"));
        n.Send = reinterpret_cast<decltype(n.Send)>(get("ncclSend"));
        n.Recv = reinterpret_cast<decltype(n.Recv)>(get("ncclRecv"));
        n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(get("ncclGetErrorString"));
    });
    if (!n.Send)
        throw std::runtime_error("NCCL unavailable");
    return n;
}

// the group / communicator paths use host threads, several devices and NCCL
// groups: not capturable into a CUDA graph (swr_render_device per context is)
void refuse_capture(cudaStream_t user)
{
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(user, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone)
        throw std::invalid_argument("multi-GPU renders cannot be captured into a CUDA graph "
                                    "(capture swr_render_device on each context instead)");
}

void api(int rc)
{
    if (rc == SWR_OK)
        return;
    const std::string msg = swr_last_error();
    if (rc == SWR_EINVAL)
        throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

// contiguous shard of rank r: B / P each, the first B % P ranks one more (the same
// split as shard.py's shard_range, so in-process and per-process sharding agree)
void shard(int64_t B, int P, int r, int64_t &start, int64_t &count)
{
    const int64_t base = B / P, extra = B % P;
    start = r * base + std::min<int64_t>(r, extra);
    count = base + (r < extra ? 1 : 0);
}

struct Dev
{
    swr_ctx *ctx = nullptr;
    int device = 0;
    cudaStream_t render = nullptr, comm = nullptr;
    cudaEvent_t rendered[2]{}, sent[2]{};
    float *pos = nullptr;           // this shard's positions (non-root)
    float *stage[2]{};              // two spectrum chunk buffers (non-root)
    double *pooled = nullptr, *rssi = nullptr, *ang = nullptr; // whole-shard heads (non-root)
    int32_t *rc = nullptr;
    int64_t cap_pos = 0, cap_chunk = 0;
};

void free_dev(Dev &d)
{
    if (d.render)
    {
        cudaSetDevice(d.device);
        cudaStreamSynchronize(d.render);
        cudaStreamSynchronize(d.comm);
    }
    for (void *p : {(void *)d.pos, (void *)d.stage[0], (void *)d.stage[1], (void *)d.pooled, (void *)d.rssi,
                    (void *)d.ang, (void *)d.rc})
        if (p)
            cudaFree(p);
    for (int i = 0; i < 2; i++)
    {
        if (d.rendered[i])
            cudaEventDestroy(d.rendered[i]);
        if (d.sent[i])
            cudaEventDestroy(d.sent[i]);
    }
    if (d.render)
        cudaStreamDestroy(d.render);
    if (d.comm)
        cudaStreamDestroy(d.comm);
}

template <class T>
T *dmalloc(size_t count)
{
    void *p = nullptr;
    check_cuda(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)), "cudaMalloc");
    return static_cast<T *>(p);
}
} // namespace

struct swr_group
{
    std::vector<Dev> dev;
    bool own = false;        // contexts created (and destroyed) by the group
    bool use_nccl = false;   // all devices distinct: NCCL point-to-point; else peer copies
    std::vector<ncclComm_t> comms;
    int H = 0, W = 0;
    std::mutex mu;           // one render call at a time per group
};

struct swr_comm
{
    swr_ctx *ctx = nullptr;
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0, device = 0;
    cudaStream_t st = nullptr;
    cudaEvent_t rendered[2]{}, sent[2]{};
    float *stage[2]{};
    int64_t cap_chunk = 0;
};

namespace
{
void init_group(swr_group &g)
{
    const int P = int(g.dev.size());
    swr_scene_info i0{};
    api(swr_scene_get_info(g.dev[0].ctx, &i0));
    g.H = i0.n_elevation;
    g.W = i0.n_azimuth;
    std::vector<int> ids;
    for (auto &d : g.dev)
    {
        swr_scene_info info{};
        api(swr_scene_get_info(d.ctx, &info));
        if (info.n_elevation != g.H || info.n_azimuth != g.W || info.n != i0.n)
            throw std::invalid_argument("group contexts hold different scenes");
        ids.push_back(d.device);
        check_cuda(cudaSetDevice(d.device), "cudaSetDevice");
        check_cuda(cudaStreamCreateWithFlags(&d.render, cudaStreamNonBlocking), "stream");
        check_cuda(cudaStreamCreateWithFlags(&d.comm, cudaStreamNonBlocking), "stream");
        for (int k = 0; k < 2; k++)
        {
            check_cuda(cudaEventCreateWithFlags(&d.rendered[k], cudaEventDisableTiming), "event");
            check_cuda(cudaEventCreateWithFlags(&d.sent[k], cudaEventDisableTiming), "event");
        }
    }
    std::vector<int> sorted = ids;
    std::sort(sorted.begin(), sorted.end());
    g.use_nccl = P > 1 && std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
    if (g.use_nccl)
    {
        // peers reach each other's memory for the position scatter
        for (int a : ids)
            for (int b : ids)
                if (a != b)
                {
                    int ok = 0;
                    cudaDeviceCanAccessPeer(&ok, a, b);
                    if (ok)
                    {
                        cudaSetDevice(a);
                        const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
                        if (e == cudaErrorPeerAccessAlreadyEnabled)
                            cudaGetLastError();
                        else
                            check_cuda(e, "peer access");
                    }
                }
        g.comms.assign(P, nullptr);
        nccl().check(nccl().CommInitAll(g.comms.data(), P, ids.data()), "ncclCommInitAll");
    }
}

void destroy_group(swr_group *g)
{
    if (!g)
        return;
    for (auto &d : g->dev)
        free_dev(d);
    for (auto c : g->comms)
        if (c)
            nccl().CommDestroy(c);
    if (g->own)
        for (auto &d : g->dev)
            swr_scene_destroy(d.ctx);
    delete g;
}
} // namespace

extern "C" {

int swr_group_create(swr_ctx *const *ctxs, int n, swr_group **out)
{
    return swr_guarded([&] {
        if (!ctxs || !out || n < 1)
            throw std::invalid_argument("group needs at least one context");
        *out = nullptr;
        auto *g = new swr_group();
        try
        {
            for (int i = 0; i < n; i++)
            {
                if (!ctxs[i])
                    throw std::invalid_argument("null context");
                Dev d;
                d.ctx = ctxs[i];
                double dv = 0;
                api(swr_get_option(ctxs[i], "device", &dv));
                d.device = int(dv);
                g->dev.push_back(d);
            }
            init_group(*g);
        }
        catch (...)
        {
            destroy_group(g);
            throw;
        }
        *out = g;
    });
}

int swr_group_create_wrfc(const char *path, const int *devices, int n_dev, swr_group **out)
{
    return swr_guarded([&] {
        if (!path || !devices || !out || n_dev < 1)
            throw std::invalid_argument("group needs a path and at least one device");
        *out = nullptr;
        std::vector<swr_ctx *> ctxs;
        try
        {
            for (int i = 0; i < n_dev; i++)
            {
                swr_ctx *c = nullptr;
                api(swr_scene_create_wrfc(path, devices[i], &c));
                ctxs.push_back(c);
            }
            swr_group *g = nullptr;
            api(swr_group_create(ctxs.data(), n_dev, &g));
            g->own = true;
            *out = g;
        }
        catch (...)
        {
            for (auto c : ctxs)
                swr_scene_destroy(c);
            throw;
        }
    });
}

void swr_group_destroy(swr_group *g) { destroy_group(g); }

int swr_group_size(swr_group *g, int *n)
{
    return swr_guarded([&] {
        if (!g || !n)
            throw std::invalid_argument("null argument");
        *n = int(g->dev.size());
    });
}

int swr_group_context(swr_group *g, int i, swr_ctx **out)
{
    return swr_guarded([&] {
        if (!g || !out || i < 0 || i >= int(g->dev.size()))
            throw std::invalid_argument("no such group member");
        *out = g->dev[size_t(i)].ctx;
    });
}

int swr_group_render(swr_group *g, const float *pos_m, int64_t B, uint32_t flags, float *spectra, double *pooled,
                     double *rssi, int32_t *aoa_rc, double *aoa_ang)
{
    return swr_guarded([&] {
        if (!g || B < 0 || (B > 0 && !pos_m))
            throw std::invalid_argument("bad group render arguments");
        std::lock_guard<std::mutex> lk(g->mu);
        const int P = int(g->dev.size());
        const size_t per = size_t(2) * g->H * g->W;
        std::vector<int> rc(size_t(P), SWR_OK);
        std::vector<std::string> err(static_cast<size_t>(P));
        std::vector<std::thread> th;
        for (int r = 0; r < P; r++)
            th.emplace_back([&, r] {
                int64_t s0, n;
                shard(B, P, r, s0, n);
                if (n == 0)
                    return;
                rc[size_t(r)] = swr_render(g->dev[size_t(r)].ctx, pos_m + 3 * s0, n, flags,
                                           spectra ? spectra + per * s0 : nullptr, pooled ? pooled + s0 : nullptr,
                                           rssi ? rssi + s0 : nullptr, aoa_rc ? aoa_rc + 2 * s0 : nullptr,
                                           aoa_ang ? aoa_ang + 2 * s0 : nullptr);
                if (rc[size_t(r)] != SWR_OK)
                    err[size_t(r)] = swr_last_error();
            });
        for (auto &t : th)
            t.join();
        for (int r = 0; r < P; r++)
            if (rc[size_t(r)] != SWR_OK)
            {
                if (rc[size_t(r)] == SWR_EINVAL)
                    throw std::invalid_argument("device " + std::to_string(g->dev[size_t(r)].device) + ": " +
                                                err[size_t(r)]);
                throw std::runtime_error("device " + std::to_string(g->dev[size_t(r)].device) + ": " +
                                         err[size_t(r)]);
            }
    });
}

int swr_group_render_device(swr_group *g, const float *d_pos, int64_t B, uint32_t flags, float *d_spec,
                            double *d_pooled, double *d_rssi, int32_t *d_aoa_rc, double *d_aoa_ang, void *stream)
{
    return swr_guarded([&] {
        if (!g || B < 0 || (B > 0 && !d_pos))
            throw std::invalid_argument("bad group render arguments");
        if (B == 0)
            return;
        std::lock_guard<std::mutex> lk(g->mu);
        const int P = int(g->dev.size());
        Dev &root = g->dev[0];
        const size_t per = size_t(2) * g->H * g->W;
        const bool want_spec = (flags & SWR_OUT_SPECTRA) && d_spec;
        const bool want_pooled = (flags & SWR_OUT_POOLED) && d_pooled, want_rssi = (flags & SWR_OUT_RSSI) && d_rssi;
        const bool want_aoa = (flags & SWR_OUT_AOA) && (d_aoa_rc || d_aoa_ang);
        cudaStream_t user = (cudaStream_t)stream;
        refuse_capture(user);
        // everything starts after the work already queued on the caller's stream
        check_cuda(cudaSetDevice(root.device), "cudaSetDevice");
        cudaEvent_t start;
        check_cuda(cudaEventCreateWithFlags(&start, cudaEventDisableTiming), "event");
        check_cuda(cudaEventRecord(start, user), "event");

        // per-device staging and the position scatter
        std::vector<int64_t> s0(static_cast<size_t>(P)), cnt(static_cast<size_t>(P)), chunk(static_cast<size_t>(P));
        int64_t rounds = 0;
        for (int r = 0; r < P; r++)
        {
            Dev &d = g->dev[size_t(r)];
            shard(B, P, r, s0[size_t(r)], cnt[size_t(r)]);
            double ch = 256;
            api(swr_get_option(d.ctx, "chunk", &ch));
            chunk[size_t(r)] = std::max<int64_t>(1, int64_t(ch));
            rounds = std::max(rounds, (cnt[size_t(r)] + chunk[size_t(r)] - 1) / chunk[size_t(r)]);
            check_cuda(cudaSetDevice(d.device), "cudaSetDevice");
            check_cuda(cudaStreamWaitEvent(d.render, start, 0), "wait");
            if (r == 0)
                check_cuda(cudaStreamWaitEvent(d.comm, start, 0), "wait"); // receives land in the caller's buffers
            if (r == 0 || cnt[size_t(r)] == 0)
                continue;
            if (d.cap_pos < cnt[size_t(r)])
            {
                for (void *p : {(void *)d.pos, (void *)d.pooled, (void *)d.rssi, (void *)d.ang, (void *)d.rc})
                    if (p)
                        cudaFree(p);
                d.pos = dmalloc<float>(size_t(3) * cnt[size_t(r)]);
                d.pooled = dmalloc<double>(cnt[size_t(r)]);
                d.rssi = dmalloc<double>(cnt[size_t(r)]);
                d.ang = dmalloc<double>(size_t(2) * cnt[size_t(r)]);
                d.rc = dmalloc<int32_t>(size_t(2) * cnt[size_t(r)]);
                d.cap_pos = cnt[size_t(r)];
            }
            if (want_spec && d.cap_chunk < chunk[size_t(r)])
            {
                for (auto &p : d.stage)
                {
                    if (p)
                        cudaFree(p);
                    p = dmalloc<float>(per * chunk[size_t(r)]);
                }
                d.cap_chunk = chunk[size_t(r)];
            }
            check_cuda(cudaMemcpyPeerAsync(d.pos, d.device, d_pos + 3 * s0[size_t(r)], root.device,
                                           sizeof(float) * 3 * cnt[size_t(r)], d.render),
                       "position scatter");
        }

        auto move = [&](void *dst, const void *src, size_t bytes, int r, ncclComm_t comm_r) {
            // chunk of device r -> root, on r's communication stream (peer copy when NCCL is not used)
            Dev &d = g->dev[size_t(r)];
            if (g->use_nccl)
            {
                nccl().check(nccl().Send(src, bytes, ncclUint8, 0, comm_r, d.comm), "send");
                nccl().check(nccl().Recv(dst, bytes, ncclUint8, r, g->comms[0], root.comm), "recv");
            }
            else
                check_cuda(cudaMemcpyPeerAsync(dst, root.device, src, d.device, bytes, d.comm), "peer copy");
        };

        // round k: every device renders its chunk k (the root in place), then the
        // non-root chunks go to the root on the communication streams
        for (int64_t k = 0; k < rounds; k++)
        {
            for (int r = 0; r < P; r++)
            {
                Dev &d = g->dev[size_t(r)];
                const int64_t c0 = k * chunk[size_t(r)];
                if (c0 >= cnt[size_t(r)])
                    continue;
                const int64_t n = std::min(chunk[size_t(r)], cnt[size_t(r)] - c0);
                check_cuda(cudaSetDevice(d.device), "cudaSetDevice");
                const int64_t b = s0[size_t(r)] + c0; // global position index
                if (r == 0)
                {
                    api(swr_render_device(d.ctx, d_pos + 3 * b, n, flags, want_spec ? d_spec + per * b : nullptr,
                                          want_pooled ? d_pooled + b : nullptr, want_rssi ? d_rssi + b : nullptr,
                                          d_aoa_rc ? d_aoa_rc + 2 * b : nullptr, d_aoa_ang ? d_aoa_ang + 2 * b : nullptr,
                                          d.render));
                    continue;
                }
                float *st = want_spec ? d.stage[k & 1] : nullptr;
                if (k >= 2 && want_spec)
                    check_cuda(cudaStreamWaitEvent(d.render, d.sent[k & 1], 0), "wait"); // buffer free again
                api(swr_render_device(d.ctx, d.pos + 3 * c0, n, flags, st, d.pooled + c0, d.rssi + c0, d.rc + 2 * c0,
                                      d.ang + 2 * c0, d.render));
                check_cuda(cudaEventRecord(d.rendered[k & 1], d.render), "event");
                check_cuda(cudaStreamWaitEvent(d.comm, d.rendered[k & 1], 0), "wait");
            }
            if (!want_spec)
                continue;
            if (g->use_nccl)
                nccl().check(nccl().GroupStart(), "group start");
            for (int r = 1; r < P; r++)
            {
                Dev &d = g->dev[size_t(r)];
                const int64_t c0 = k * chunk[size_t(r)];
                if (c0 >= cnt[size_t(r)])
                    continue;
                const int64_t n = std::min(chunk[size_t(r)], cnt[size_t(r)] - c0);
                move(d_spec + per * (s0[size_t(r)] + c0), d.stage[k & 1], sizeof(float) * per * size_t(n), r,
                     g->use_nccl ? g->comms[size_t(r)] : nullptr);
            }
            if (g->use_nccl)
                nccl().check(nccl().GroupEnd(), "group end");
            for (int r = 1; r < P; r++)
            {
                Dev &d = g->dev[size_t(r)];
                if (k * chunk[size_t(r)] >= cnt[size_t(r)])
                    continue;
                check_cuda(cudaSetDevice(d.device), "cudaSetDevice");
                check_cuda(cudaEventRecord(d.sent[k & 1], d.comm), "event");
            }
        }
        // the heads outputs of every non-root shard: one transfer per array
        if (g->use_nccl)
            nccl().check(nccl().GroupStart(), "group start");
        for (int r = 1; r < P; r++)
        {
            Dev &d = g->dev[size_t(r)];
            const int64_t n = cnt[size_t(r)], b = s0[size_t(r)];
            if (n == 0)
                continue;
            check_cuda(cudaSetDevice(d.device), "cudaSetDevice");
            cudaEvent_t done;
            check_cuda(cudaEventCreateWithFlags(&done, cudaEventDisableTiming), "event");
            check_cuda(cudaEventRecord(done, d.render), "event");
            check_cuda(cudaStreamWaitEvent(d.comm, done, 0), "wait");
            cudaEventDestroy(done);
            const ncclComm_t cr = g->use_nccl ? g->comms[size_t(r)] : nullptr;
            if (want_pooled)
                move(d_pooled + b, d.pooled, sizeof(double) * size_t(n), r, cr);
            if (want_rssi)
                move(d_rssi + b, d.rssi, sizeof(double) * size_t(n), r, cr);
            if (want_aoa && d_aoa_rc)
                move(d_aoa_rc + 2 * b, d.rc, sizeof(int32_t) * 2 * size_t(n), r, cr);
            if (want_aoa && d_aoa_ang)
                move(d_aoa_ang + 2 * b, d.ang, sizeof(double) * 2 * size_t(n), r, cr);
        }
        if (g->use_nccl)
            nccl().check(nccl().GroupEnd(), "group end");
        // the caller's stream resumes once the root has rendered its shard and received the rest
        auto join = [&](int dev_of, cudaStream_t from) {
            check_cuda(cudaSetDevice(dev_of), "cudaSetDevice");
            cudaEvent_t e;
            check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
            check_cuda(cudaEventRecord(e, from), "event");
            check_cuda(cudaSetDevice(root.device), "cudaSetDevice");
            check_cuda(cudaStreamWaitEvent(user, e, 0), "wait");
            check_cuda(cudaEventDestroy(e), "event");
        };
        join(root.device, root.render);
        if (g->use_nccl)
            join(root.device, root.comm);
        else
            for (int r = 1; r < P; r++)
                join(g->dev[size_t(r)].device, g->dev[size_t(r)].comm);
        check_cuda(cudaEventDestroy(start), "event");
    });
}

// ---- between processes (one process per GPU): the same chunked gather to rank 0

int swr_nccl_unique_id(void *id128)
{
    return swr_guarded([&] {
        if (!id128)
            throw std::invalid_argument("null id buffer");
        static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
        ncclUniqueId id;
        nccl().check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(id128, &id, sizeof(id));
    });
}

int swr_comm_create(swr_ctx *ctx, const void *id128, int nranks, int rank, swr_comm **out)
{
    return swr_guarded([&] {
        if (!ctx || !id128 || !out || nranks < 1 || rank < 0 || rank >= nranks)
            throw std::invalid_argument("bad communicator arguments");
        *out = nullptr;
        auto c = std::make_unique<swr_comm>();
        c->ctx = ctx;
        c->nranks = nranks;
        c->rank = rank;
        double dv = 0;
        api(swr_get_option(ctx, "device", &dv));
        c->device = int(dv);
        check_cuda(cudaSetDevice(c->device), "cudaSetDevice");
        ncclUniqueId id;
        std::memcpy(&id, id128, sizeof(id));
        nccl().check(nccl().CommInitRank(&c->comm, nranks, id, rank), "ncclCommInitRank");
        check_cuda(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking), "stream");
        for (int k = 0; k < 2; k++)
        {
            check_cuda(cudaEventCreateWithFlags(&c->rendered[k], cudaEventDisableTiming), "event");
            check_cuda(cudaEventCreateWithFlags(&c->sent[k], cudaEventDisableTiming), "event");
        }
        *out = c.release();
    });
}

void swr_comm_destroy(swr_comm *c)
{
    if (!c)
        return;
    cudaSetDevice(c->device);
    if (c->st)
    {
        cudaStreamSynchronize(c->st);
        cudaStreamDestroy(c->st);
    }
    for (int k = 0; k < 2; k++)
    {
        if (c->rendered[k])
            cudaEventDestroy(c->rendered[k]);
        if (c->sent[k])
            cudaEventDestroy(c->sent[k]);
        if (c->stage[k])
            cudaFree(c->stage[k]);
    }
    if (c->comm)
        nccl().CommDestroy(c->comm);
    delete c;
}

int swr_render_gather(swr_comm *cm, const float *d_pos, const int64_t *counts, uint32_t flags, float *d_spec_root,
                      double *d_pooled_root, void *stream)
{
    return swr_guarded([&] {
        if (!cm || !counts)
            throw std::invalid_argument("null argument");
        const int R = cm->nranks, me = cm->rank;
        std::vector<int64_t> start(size_t(R) + 1, 0);
        for (int r = 0; r < R; r++)
        {
            if (counts[r] < 0)
                throw std::invalid_argument("negative shard");
            start[size_t(r) + 1] = start[size_t(r)] + counts[r];
        }
        const int64_t n_me = counts[me];
        if (n_me > 0 && !d_pos)
            throw std::invalid_argument("null positions");
        if (me == 0 && (flags & SWR_OUT_SPECTRA) && !d_spec_root)
            throw std::invalid_argument("rank 0 needs the gathered spectra buffer");
        swr_scene_info info{};
        api(swr_scene_get_info(cm->ctx, &info));
        const size_t per = size_t(2) * info.n_elevation * info.n_azimuth;
        double ch = 256;
        api(swr_get_option(cm->ctx, "chunk", &ch));
        const int64_t chunk = std::max<int64_t>(1, int64_t(ch));
        cudaStream_t user = (cudaStream_t)stream;
        refuse_capture(user);
        check_cuda(cudaSetDevice(cm->device), "cudaSetDevice");
        const bool spec = flags & SWR_OUT_SPECTRA;
        {
            // the communication stream starts after the caller's queued work
            cudaEvent_t e;
            check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
            check_cuda(cudaEventRecord(e, user), "event");
            check_cuda(cudaStreamWaitEvent(cm->st, e, 0), "wait");
            cudaEventDestroy(e);
        }
        if (me != 0 && spec && cm->cap_chunk < chunk)
        {
            for (auto &p : cm->stage)
            {
                if (p)
                    cudaFree(p);
                p = dmalloc<float>(per * chunk);
            }
            cm->cap_chunk = chunk;
        }
        int64_t rounds = 0;
        for (int r = 0; r < R; r++)
            rounds = std::max(rounds, (counts[r] + chunk - 1) / chunk);
        const uint32_t fl = flags & (SWR_OUT_SPECTRA | SWR_OUT_POOLED);
        for (int64_t k = 0; k < rounds; k++)
        {
            const int64_t c0 = k * chunk, n = std::min(chunk, n_me - c0);
            if (n > 0)
            {
                if (me == 0)
                    api(swr_render_device(cm->ctx, d_pos + 3 * c0, n, fl, spec ? d_spec_root + per * c0 : nullptr,
                                          d_pooled_root ? d_pooled_root + c0 : nullptr, nullptr, nullptr, nullptr,
                                          user));
                else
                {
                    if (k >= 2 && spec)
                        check_cuda(cudaStreamWaitEvent(user, cm->sent[k & 1], 0), "wait");
                    api(swr_render_device(cm->ctx, d_pos + 3 * c0, n, fl, spec ? cm->stage[k & 1] : nullptr, nullptr,
                                          nullptr, nullptr, nullptr, user));
                    check_cuda(cudaEventRecord(cm->rendered[k & 1], user), "event");
                    check_cuda(cudaStreamWaitEvent(cm->st, cm->rendered[k & 1], 0), "wait");
                }
            }
            if (!spec)
                continue;
            nccl().check(nccl().GroupStart(), "group start");
            if (me == 0)
            {
                for (int r = 1; r < R; r++)
                {
                    const int64_t m = std::min(chunk, counts[r] - c0);
                    if (m > 0)
                        nccl().check(nccl().Recv(d_spec_root + per * (start[size_t(r)] + c0), sizeof(float) * per * m,
                                                 ncclUint8, r, cm->comm, cm->st),
                                     "recv");
                }
            }
            else if (n > 0)
                nccl().check(nccl().Send(cm->stage[k & 1], sizeof(float) * per * n, ncclUint8, 0, cm->comm, cm->st),
                             "send");
            nccl().check(nccl().GroupEnd(), "group end");
            if (me != 0 && n > 0)
                check_cuda(cudaEventRecord(cm->sent[k & 1], cm->st), "event");
        }
        {
            // the caller's stream resumes after this rank's sends (or rank 0's receives)
            cudaEvent_t e;
            check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
            check_cuda(cudaEventRecord(e, cm->st), "event");
            check_cuda(cudaStreamWaitEvent(user, e, 0), "wait");
            cudaEventDestroy(e);
        }
    });
}

} // extern "C"
