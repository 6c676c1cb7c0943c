// comm.cpp — NCCL and host-callback transports of the engine's collectives (comm.hpp).
#include "comm.hpp"

#include <cstring>

#include "device.cuh"

adsb_comm::~adsb_comm() {
    if (comm) ncclCommDestroy(comm);
    if (staging) cudaFreeHost(staging);
}

namespace adsb {
namespace {

void* staging(adsb_comm* c, size_t bytes) {
    if (c->staging_bytes < bytes) {
        if (c->staging) ADSB_CUDA(cudaFreeHost(c->staging));
        c->staging = nullptr;
        const size_t want = bytes + bytes / 4 + 4096;
        ADSB_CUDA(cudaMallocHost(&c->staging, want));
        c->staging_bytes = want;
    }
    return c->staging;
}

void host_call(int rc, const char* what) {
    if (rc != 0) fail(ADSB_ERR_NCCL, std::string("host collective ") + what + " failed (" + std::to_string(rc) + ")");
}

}  // namespace

void comm_allreduce_u32_sum(adsb_comm* c, uint32_t* dev, size_t count, cudaStream_t stream) {
    if (!c || c->nranks == 1 || count == 0) return;
    if (c->comm) {
        ADSB_NCCL(ncclAllReduce(dev, dev, count, ncclUint32, ncclSum, c->comm, stream));
        return;
    }
    auto* h = static_cast<uint32_t*>(staging(c, count * sizeof(uint32_t)));
    ADSB_CUDA(cudaMemcpyAsync(h, dev, count * sizeof(uint32_t), cudaMemcpyDeviceToHost, stream));
    ADSB_CUDA(cudaStreamSynchronize(stream));
    host_call(c->host.allreduce_u32_sum(c->user, h, count), "allreduce_u32_sum");
    ADSB_CUDA(cudaMemcpyAsync(dev, h, count * sizeof(uint32_t), cudaMemcpyHostToDevice, stream));
    ADSB_CUDA(cudaStreamSynchronize(stream));  // the staging buffer is reused by the next call
}

void comm_allreduce_host(adsb_comm* c, uint64_t* host, size_t count, RedOp op, cudaStream_t stream) {
    if (!c || c->nranks == 1 || count == 0) return;
    if (c->comm) {
        auto* pinned = static_cast<uint64_t*>(staging(c, count * sizeof(uint64_t)));
        void* dev = nullptr;
        ADSB_CUDA(cudaMallocAsync(&dev, count * sizeof(uint64_t), stream));
        std::memcpy(pinned, host, count * sizeof(uint64_t));
        ADSB_CUDA(cudaMemcpyAsync(dev, pinned, count * sizeof(uint64_t), cudaMemcpyHostToDevice, stream));
        const ncclRedOp_t nop = op == RedOp::kSum ? ncclSum : op == RedOp::kMax ? ncclMax : ncclMin;
        ADSB_NCCL(ncclAllReduce(dev, dev, count, ncclUint64, nop, c->comm, stream));
        ADSB_CUDA(cudaMemcpyAsync(pinned, dev, count * sizeof(uint64_t), cudaMemcpyDeviceToHost, stream));
        ADSB_CUDA(cudaFreeAsync(dev, stream));
        ADSB_CUDA(cudaStreamSynchronize(stream));
        std::memcpy(host, pinned, count * sizeof(uint64_t));
        return;
    }
    host_call(c->host.allreduce_u64(c->user, host, count, static_cast<int>(op)), "allreduce_u64");
}

void comm_allgather_u64(adsb_comm* c, const unsigned long long* send, unsigned long long* recv, size_t count,
                        cudaStream_t stream) {
    if (!c || c->nranks == 1) {
        if (count && recv != send)
            ADSB_CUDA(cudaMemcpyAsync(recv, send, count * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, stream));
        return;
    }
    if (count == 0) return;
    if (c->comm) {
        ADSB_NCCL(ncclAllGather(send, recv, count, ncclUint64, c->comm, stream));
        return;
    }
    const size_t W = static_cast<size_t>(c->nranks);
    auto* h = static_cast<uint64_t*>(staging(c, (W + 1) * count * sizeof(uint64_t)));
    uint64_t* mine = h + W * count;
    ADSB_CUDA(cudaMemcpyAsync(mine, send, count * sizeof(uint64_t), cudaMemcpyDeviceToHost, stream));
    ADSB_CUDA(cudaStreamSynchronize(stream));
    host_call(c->host.allgather_u64(c->user, mine, h, count), "allgather_u64");
    ADSB_CUDA(cudaMemcpyAsync(recv, h, W * count * sizeof(uint64_t), cudaMemcpyHostToDevice, stream));
    ADSB_CUDA(cudaStreamSynchronize(stream));
}

}  // namespace adsb
