// comm.cpp -- NCCL and loopback implementations of comm.h.
#include "comm.h"

#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <tuple>
#include <vector>

namespace qsb {

namespace {

using Clock = std::chrono::steady_clock;

double ms_since(Clock::time_point t0)
{
    return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

// Poll a stream until it drained: spin briefly, then sleep in 50 us steps.
// `poll` returns 0 while healthy, else an error (already in err).
template <class F>
int poll_stream(cudaStream_t s, double timeout_ms, std::string &err, F poll)
{
    const auto t0 = Clock::now();
    for (int it = 0;; it++) {
        const cudaError_t q = cudaStreamQuery(s);
        if (q == cudaSuccess) return 0;
        if (q != cudaErrorNotReady) {
            cudaGetLastError();
            err = std::string("cudaStreamQuery: ") + cudaGetErrorString(q);
            return 1;
        }
        if (poll()) return 1;
        if (ms_since(t0) > timeout_ms) {
            err = "timed out after " + std::to_string((long long)timeout_ms) +
                  " ms waiting for the device (communication never completed: SPMD call mismatch or a dead peer?)";
            return 1;
        }
        if (it > 2000) std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
}

// ------------------------------------------------------------------ NCCL
class NcclComm : public Comm {
public:
    ncclComm_t comm = nullptr;
    bool aborted = false;

    // non-blocking communicator: an NCCL call may return ncclInProgress;
    // the next call is allowed once the async state left ncclInProgress
    int settle(ncclResult_t r, const char *what, std::string &err)
    {
        const auto t0 = Clock::now();
        while (r == ncclInProgress) {
            if (ncclCommGetAsyncError(comm, &r) != ncclSuccess) break;
            if (r != ncclInProgress) break;
            if (ms_since(t0) > timeout_ms) {
                err = std::string(what) + ": timed out in ncclInProgress";
                abort();
                return 1;
            }
            std::this_thread::yield();
        }
        if (r != ncclSuccess) {
            err = std::string(what) + ": " + ncclGetErrorString(r);
            abort();
            return 1;
        }
        return 0;
    }
    int group_start(std::string &err) override { return settle(ncclGroupStart(), "ncclGroupStart", err); }
    int group_end(std::string &err) override { return settle(ncclGroupEnd(), "ncclGroupEnd", err); }
    int send(const void *buf, size_t bytes, int peer, cudaStream_t s, std::string &err) override
    {
        return settle(ncclSend(buf, bytes, ncclUint8, peer, comm, s), "ncclSend", err);
    }
    int recv(void *buf, size_t bytes, int peer, cudaStream_t s, std::string &err) override
    {
        return settle(ncclRecv(buf, bytes, ncclUint8, peer, comm, s), "ncclRecv", err);
    }
    int all_gather(const double *snd, double *rcv, size_t count, cudaStream_t s, std::string &err) override
    {
        return settle(ncclAllGather(snd, rcv, count, ncclDouble, comm, s), "ncclAllGather", err);
    }
    int wait(cudaStream_t s, double tmo, std::string &err) override
    {
        const int r = poll_stream(s, tmo, err, [&]() {
            ncclResult_t st = ncclSuccess;
            if (ncclCommGetAsyncError(comm, &st) != ncclSuccess || (st != ncclSuccess && st != ncclInProgress)) {
                err = std::string("NCCL async error: ") + ncclGetErrorString(st);
                return 1;
            }
            return 0;
        });
        if (r) abort();
        return r;
    }
    void abort() override
    {
        if (comm && !aborted) ncclCommAbort(comm);
        aborted = true;
    }
    ~NcclComm() override
    {
        if (!comm || aborted) return;
        ncclResult_t r = ncclCommFinalize(comm);
        const auto t0 = Clock::now();
        while (r == ncclInProgress && ms_since(t0) < 10e3) {
            if (ncclCommGetAsyncError(comm, &r) != ncclSuccess) break;
            std::this_thread::yield();
        }
        if (r == ncclSuccess) ncclCommDestroy(comm);
        else ncclCommAbort(comm);
    }
};

// -------------------------------------------------------------- loopback
struct Msg {
    const void *buf;
    size_t bytes;
    cudaEvent_t ready;  // recorded on the sender's stream at its group end
};

struct Hub {
    std::mutex mu;
    std::condition_variable cv;
    int n = 0;
    int refs = 0;
    bool aborted = false;
    std::map<std::tuple<int, int, uint64_t>, Msg> msgs;          // (src, dst, seq)
    std::map<std::tuple<int, int, uint64_t>, cudaEvent_t> done;  // receiver's copy enqueued
    std::vector<uint64_t> sseq, rseq;                            // n x n counters
};

std::mutex g_hubs_mu;
std::map<std::string, std::shared_ptr<Hub>> g_hubs;

class LoopbackComm : public Comm {
public:
    std::shared_ptr<Hub> hub;
    std::string id;
    struct Op {
        void *buf;
        size_t bytes;
        int peer;
        cudaStream_t s;
    };
    std::vector<Op> sends, recvs;
    int depth = 0;

    int group_start(std::string &) override
    {
        depth++;
        return 0;
    }
    int group_end(std::string &err) override
    {
        if (depth == 0) {
            err = "group_end without group_start";
            return 1;
        }
        if (--depth > 0) return 0;
        std::vector<Op> S, R;
        S.swap(sends);
        R.swap(recvs);
        return run(S, R, err);
    }
    int send(const void *buf, size_t bytes, int peer, cudaStream_t s, std::string &err) override
    {
        if (peer < 0 || peer >= size) { err = "send: peer out of range"; return 1; }
        sends.push_back({const_cast<void *>(buf), bytes, peer, s});
        return depth ? 0 : flush_single(err);
    }
    int recv(void *buf, size_t bytes, int peer, cudaStream_t s, std::string &err) override
    {
        if (peer < 0 || peer >= size) { err = "recv: peer out of range"; return 1; }
        recvs.push_back({buf, bytes, peer, s});
        return depth ? 0 : flush_single(err);
    }
    int flush_single(std::string &err)
    {
        std::vector<Op> S, R;
        S.swap(sends);
        R.swap(recvs);
        return run(S, R, err);
    }
    int all_gather(const double *snd, double *rcv, size_t count, cudaStream_t s, std::string &err) override
    {
        group_start(err);
        for (int p = 0; p < size; p++) {
            sends.push_back({const_cast<double *>(snd), count * sizeof(double), p, s});
            recvs.push_back({rcv + (size_t)p * count, count * sizeof(double), p, s});
        }
        return group_end(err);
    }
    // every send registered first (so peers never wait on each other in a
    // cycle), then each recv waits for its matching send and enqueues the
    // copy on the receiver's stream, then each send waits until its copy is
    // enqueued and orders the sender's stream after it
    int run(const std::vector<Op> &S, const std::vector<Op> &R, std::string &err)
    {
        Hub &h = *hub;
        const int me = rank, n = size;
        std::vector<uint64_t> sq(S.size());
        for (size_t i = 0; i < S.size(); i++) {
            cudaEvent_t e;
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess || cudaEventRecord(e, S[i].s) != cudaSuccess) {
                cudaGetLastError();
                err = "loopback: event record failed";
                return 1;
            }
            std::lock_guard<std::mutex> g(h.mu);
            sq[i] = h.sseq[(size_t)me * n + S[i].peer]++;
            h.msgs[std::make_tuple(me, S[i].peer, sq[i])] = Msg{S[i].buf, S[i].bytes, e};
        }
        h.cv.notify_all();
        const auto deadline = Clock::now() + std::chrono::microseconds((long long)(timeout_ms * 1e3));
        for (const Op &r : R) {
            Msg m{};
            uint64_t q;
            {
                std::unique_lock<std::mutex> g(h.mu);
                q = h.rseq[(size_t)r.peer * n + me]++;
                const auto key = std::make_tuple(r.peer, me, q);
                if (!h.cv.wait_until(g, deadline, [&]() { return h.aborted || h.msgs.count(key); })) {
                    err = "loopback: timed out waiting for rank " + std::to_string(r.peer) +
                          "'s send (SPMD call mismatch?)";
                    return 1;
                }
                if (h.aborted) {
                    err = "loopback: communicator aborted";
                    return 1;
                }
                m = h.msgs[key];
                h.msgs.erase(key);
            }
            if (m.bytes != r.bytes) {
                err = "loopback: rank " + std::to_string(r.peer) + " sent " + std::to_string(m.bytes) + " bytes, recv expects " +
                      std::to_string(r.bytes);
                return 1;
            }
            cudaEvent_t d;
            if (cudaStreamWaitEvent(r.s, m.ready, 0) != cudaSuccess ||
                (r.bytes && cudaMemcpyAsync(r.buf, m.buf, r.bytes, cudaMemcpyDeviceToDevice, r.s) != cudaSuccess) ||
                cudaEventCreateWithFlags(&d, cudaEventDisableTiming) != cudaSuccess || cudaEventRecord(d, r.s) != cudaSuccess) {
                cudaGetLastError();
                err = "loopback: copy enqueue failed";
                return 1;
            }
            cudaEventDestroy(m.ready);
            {
                std::lock_guard<std::mutex> g(h.mu);
                h.done[std::make_tuple(r.peer, me, q)] = d;
            }
            h.cv.notify_all();
        }
        for (size_t i = 0; i < S.size(); i++) {
            cudaEvent_t d;
            {
                std::unique_lock<std::mutex> g(h.mu);
                const auto key = std::make_tuple(me, S[i].peer, sq[i]);
                if (!h.cv.wait_until(g, deadline, [&]() { return h.aborted || h.done.count(key); })) {
                    err = "loopback: timed out waiting for rank " + std::to_string(S[i].peer) +
                          "'s recv (SPMD call mismatch?)";
                    return 1;
                }
                if (h.aborted) {
                    err = "loopback: communicator aborted";
                    return 1;
                }
                d = h.done[key];
                h.done.erase(key);
            }
            if (cudaStreamWaitEvent(S[i].s, d, 0) != cudaSuccess) {
                cudaGetLastError();
                err = "loopback: stream wait failed";
                return 1;
            }
            cudaEventDestroy(d);
        }
        return 0;
    }
    int wait(cudaStream_t s, double tmo, std::string &err) override
    {
        return poll_stream(s, tmo, err, [&]() {
            if (hub->aborted) {
                err = "loopback: communicator aborted";
                return 1;
            }
            return 0;
        });
    }
    void abort() override
    {
        {
            std::lock_guard<std::mutex> g(hub->mu);
            hub->aborted = true;
        }
        hub->cv.notify_all();
    }
    ~LoopbackComm() override
    {
        std::lock_guard<std::mutex> g(g_hubs_mu);
        if (--hub->refs == 0) g_hubs.erase(id);
    }
};

}  // namespace

Comm *make_nccl_comm(const void *id128, int nranks, int rank, double timeout_ms, std::string &err)
{
    NcclComm *c = new NcclComm();
    c->rank = rank;
    c->size = nranks;
    c->timeout_ms = timeout_ms;
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.blocking = 0;  // calls return while in progress: the host can poll errors and time out
    ncclResult_t r = ncclCommInitRankConfig(&c->comm, nranks, id, rank, &cfg);
    if (r != ncclSuccess && r != ncclInProgress) {
        err = std::string("ncclCommInitRankConfig: ") + ncclGetErrorString(r);
        c->comm = nullptr;
        delete c;
        return nullptr;
    }
    if (c->settle(r, "ncclCommInitRankConfig", err)) {
        delete c;
        return nullptr;
    }
    return c;
}

void new_loopback_id(void *out128)
{
    static std::mutex mu;
    static uint64_t next = 1;
    uint64_t v[16] = {0};
    {
        std::lock_guard<std::mutex> g(mu);
        v[0] = 0x716c6f6f70626b31ULL;  // tag
        v[1] = next++;
        v[2] = (uint64_t)Clock::now().time_since_epoch().count();
    }
    std::memcpy(out128, v, 128);
}

Comm *make_loopback_comm(const void *id128, int nranks, int rank, double timeout_ms, std::string &err)
{
    std::string id((const char *)id128, 128);
    std::shared_ptr<Hub> h;
    {
        std::lock_guard<std::mutex> g(g_hubs_mu);
        auto it = g_hubs.find(id);
        if (it == g_hubs.end()) {
            h = std::make_shared<Hub>();
            h->n = nranks;
            h->sseq.assign((size_t)nranks * nranks, 0);
            h->rseq.assign((size_t)nranks * nranks, 0);
            g_hubs[id] = h;
        } else {
            h = it->second;
            if (h->n != nranks) {
                err = "loopback: rank count differs from the hub's";
                return nullptr;
            }
        }
        h->refs++;
    }
    LoopbackComm *c = new LoopbackComm();
    c->hub = h;
    c->id = id;
    c->rank = rank;
    c->size = nranks;
    c->timeout_ms = timeout_ms;
    return c;
}

}  // namespace qsb
