// comm.h -- the exchange transport of the SPMD (one context per rank) mode.
//
// The runtime's exchange engine (runtime.cpp exec_exchange / exec_pairwise,
// the cross-rank readouts) is written once against this interface; two
// transports implement it:
//   NcclComm     -- NCCL over NVLink/NVSwitch, one process per GPU
//                   ("a buffer for each MPI process ... split the
//                   MPI send"), non-blocking communicator with async-error
//                   polling and a timeout (an SPMD call mismatch returns
//                   QSIM_ERR_COMM instead of hanging);
//   LoopbackComm -- P ranks in P host threads of ONE process on ONE GPU, a
//                   send/recv pair becomes a device copy on the receiver's
//                   stream.  It runs the unchanged NCCL-branch code of the
//                   runtime (pieces, pack/unpack, pairwise combine, gathers)
//                   where only one GPU is available.
// Semantics follow NCCL: inside group_start/group_end, sends and recvs to a
// peer match in posting order; the transfer is ordered on the given stream
// (work enqueued on it before group_end is complete before data leaves, work
// enqueued after group_end sees the received data and may reuse the send
// buffers).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>

namespace qsb {

class Comm {
public:
    virtual ~Comm() {}
    // 0 on success, else an error message in err (the context is then poisoned)
    virtual int group_start(std::string &err) = 0;
    virtual int group_end(std::string &err) = 0;
    virtual int send(const void *buf, size_t bytes, int peer, cudaStream_t s, std::string &err) = 0;
    virtual int recv(void *buf, size_t bytes, int peer, cudaStream_t s, std::string &err) = 0;
    // recv[r * count + j] = rank r's send[j] (doubles)
    virtual int all_gather(const double *send, double *recv, size_t count, cudaStream_t s, std::string &err) = 0;
    // Wait until every operation enqueued on `s` completed, polling the
    // transport's asynchronous error state; gives up after timeout_ms
    // (then aborts the communicator).  0: done.
    virtual int wait(cudaStream_t s, double timeout_ms, std::string &err) = 0;
    virtual void abort() = 0;
    int rank = 0, size = 1;
    double timeout_ms = 600e3;  // blocking host waits of the transport (qsim option comm_timeout_ms)
};

// NCCL communicator from a 128-byte ncclUniqueId; nullptr + err on failure
Comm *make_nccl_comm(const void *id128, int nranks, int rank, double timeout_ms, std::string &err);
// Loopback: ranks of one hub (qsim_get_loopback_id) in threads of this process
Comm *make_loopback_comm(const void *id128, int nranks, int rank, double timeout_ms, std::string &err);
// fresh loopback hub id (128 bytes)
void new_loopback_id(void *out128);

}  // namespace qsb
