// comm.hpp — the engine's collectives, one rank per process (one process per GPU).
//
// Two transports behind one interface:
//  * NCCL (adsb_comm_init): collectives are enqueued on the engine's streams
//    and run over NVLink / NVSwitch without a host round trip;
//  * host callbacks (adsb_comm_init_host): the caller supplies all-reduce /
//    all-gather over host memory (e.g. torch.distributed with gloo). The
//    engine stages device buffers through pinned memory and calls them from
//    the calling thread. Used to run the multi-rank code paths where NCCL
//    ranks cannot be had (several ranks on one GPU, CPU-only transports); no
//    device kernel ever waits on another rank, so ranks sharing a GPU are safe.
//
// Every rank must issue the same collectives in the same order; the engine's
// sizing decisions that feed them (batch sizes, epoch counts) are made
// rank-invariant through comm_allreduce_host (engine.cu).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "common.hpp"

#define ADSB_NCCL(call)                                                                   \
    do {                                                                                  \
        ncclResult_t _r = (call);                                                         \
        if (_r != ncclSuccess)                                                            \
            ::adsb::fail(ADSB_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(_r)); \
    } while (0)

struct adsb_comm {
    ncclComm_t comm = nullptr;           // NCCL transport (nullptr: host callbacks)
    adsb_host_collectives host{};        // host transport
    void* user = nullptr;
    int nranks = 1;
    int rank = 0;
    int device = 0;
    // pinned staging for the host transport (grown on demand)
    void* staging = nullptr;
    size_t staging_bytes = 0;
    ~adsb_comm();
};

namespace adsb {

enum class RedOp : int { kSum = ADSB_REDUCE_SUM, kMax = ADSB_REDUCE_MAX, kMin = ADSB_REDUCE_MIN };

// In-place all-reduce of `count` device u32 (sum) on `stream`.
void comm_allreduce_u32_sum(adsb_comm* c, uint32_t* dev, size_t count, cudaStream_t stream);
// In-place all-reduce of host u64 values (used for sizing decisions and scalars).
void comm_allreduce_host(adsb_comm* c, uint64_t* host, size_t count, RedOp op, cudaStream_t stream);
// recv[r * count + i] = rank r's send[i], device buffers, on `stream`.
void comm_allgather_u64(adsb_comm* c, const unsigned long long* send, unsigned long long* recv, size_t count,
                        cudaStream_t stream);

}  // namespace adsb
