// p2p.cu -- the z-slab exchange over peer memory (NVLink / NVSwitch) instead
// of host-driven collectives.
//
// Ranks map each other's state buffers, gathered-record buffers and arrival
// flags (CUDA IPC, pifcm_peer_*).  After a slab step, k_p2p_put stores the
// slab's boundary planes straight into the neighbours' halo planes and its
// per-chunk records into every rank's gathered buffer (rank-major slots, the
// canonical order of k_slab_finalize), then -- once all its blocks' stores
// are fenced system-wide -- raises this rank's arrival flag on every rank.
// k_p2p_wait spins (acquire, system scope) until every rank's flag reached the
// epoch.  One barrier per iteration; no host round trip, no NCCL call.
#include <cuda_runtime.h>
#include <stdint.h>

#include "pifcm_internal.cuh"

namespace pifcm {

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned *p, unsigned v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void k_p2p_put(P2PPut a) {
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nth = (long long)gridDim.x * blockDim.x;
    // the H boundary planes -> the neighbours' H halo planes (P states each)
    const long long hp = (long long)a.H * a.plane;
    if (a.lo_dst) {
        const long long n = hp * a.P;
        for (long long i = tid; i < n; i += nth) {
            const long long p = i / hp, k = i - p * hp;
            a.lo_dst[p * a.lo_state + k] = a.src[p * a.state + hp + k];                        // first H local planes
        }
    }
    if (a.hi_dst) {
        const long long n = hp * a.P;
        for (long long i = tid; i < n; i += nth) {
            const long long p = i / hp, k = i - p * hp;
            a.hi_dst[p * a.hi_state + k] = a.src[p * a.state + (long long)a.nz * a.plane + k];  // last H local planes
        }
    }
    // this rank's records -> slot [rank] of every rank's gathered buffer
    if (a.rec_src) {
        const long long n = (long long)a.P * a.nrec * kNR;
        for (int w = 0; w < a.world; ++w) {
            double *dst = a.rec_dst[w];
            for (long long i = tid; i < n; i += nth) {
                const long long p = i / ((long long)a.nrec * kNR), k = i - p * (long long)a.nrec * kNR;
                dst[((long long)a.rank * a.P + p) * (long long)a.nrec_max * kNR + k] = a.rec_src[i];
            }
        }
    }
    // all blocks' stores visible system-wide, then the last block raises the flags
    __threadfence_system();
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0) last = atomicAdd(a.counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last && threadIdx.x == 0) {
        *a.counter = 0u;
        __threadfence_system();
        for (int w = 0; w < a.world; ++w) st_release_sys(a.flags[w] + a.rank, a.epoch);
    }
}

cudaError_t launch_p2p_put(const P2PPut &a, cudaStream_t st) {
    long long n = a.plane * a.P;
    const long long nr = (long long)a.P * a.nrec * kNR;
    if (nr > n) n = nr;
    long long b = (n + 255) / 256;
    if (b > 148 * 2) b = 148 * 2;
    if (b < 1) b = 1;
    k_p2p_put<<<(int)b, 256, 0, st>>>(a);
    return cudaGetLastError();
}

// Wait until every rank raised its flag to `epoch` (bounded: ~20 s, then the
// status word reports PIFCM_ECUDA instead of hanging the device).
__global__ void k_p2p_wait(const unsigned *flags, int world, unsigned epoch, int *status) {
    if (threadIdx.x != 0) return;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int w = 0; w < world; ++w) {
        while (ld_acquire_sys(flags + w) < epoch) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > 20ull * 1000000000ull) {
                if (status) atomicExch(status, (int)PIFCM_ECUDA);
                return;
            }
            __nanosleep(200);
        }
    }
}

cudaError_t launch_p2p_wait(const unsigned *flags, int world, unsigned epoch, int *status, cudaStream_t st) {
    k_p2p_wait<<<1, 32, 0, st>>>(flags, world, epoch, status);
    return cudaGetLastError();
}

}  // namespace pifcm
