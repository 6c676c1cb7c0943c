// comm.hpp — one NCCL communicator per process (one process per GPU).
#pragma once

#include <nccl.h>

#include <string>

#include "common.hpp"

#define ADSB_NCCL(call)                                                                   \
    do {                                                                                  \
        ncclResult_t _r = (call);                                                         \
        if (_r != ncclSuccess)                                                            \
            ::adsb::fail(ADSB_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(_r)); \
    } while (0)

struct adsb_comm {
    ncclComm_t comm = nullptr;
    int nranks = 1;
    int rank = 0;
    int device = 0;
};
