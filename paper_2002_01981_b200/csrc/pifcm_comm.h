// pifcm_comm.h -- the context's communicator (comm.cu).  Internal.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/pifcm.h"

namespace pifcm {

struct Comm {
    enum Kind { NONE = 0, NCCL = 1, HOST = 2 } kind = NONE;
    int rank = 0, world = 1;
    void *nccl = nullptr;      // ncclComm_t
    pifcm_host_coll host{};    // HOST: caller's collectives
    void *buf = nullptr;       // device scratch of the fitness all-gather
    size_t buf_bytes = 0;
};

void dist_range(int P, int world, int rank, int *p0, int *p1);
int comm_unique_id(uint8_t *id, std::string &err);
int comm_init(Comm &c, int device, const pifcm_dist *d, const pifcm_host_coll *hc, std::string &err);
void comm_free(Comm &c);
int comm_allgather_fitness(Comm &c, double *fit, int P, cudaStream_t st, std::string &err);
int comm_broadcast(Comm &c, void *buf, size_t bytes, int root, cudaStream_t st, std::string &err);

}  // namespace pifcm
