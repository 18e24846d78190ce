// Multi-GPU communication of the distributed BDDC-PCG: NCCL over
// NVLink/NVSwitch, one rank per B200. NCCL is loaded at run time (dlopen of
// libnccl.so.2, preferring the copy torch already mapped), so the single-GPU library
// carries no NCCL link dependency.
//
// Per PCG iteration the distributed path issues (all on the solve stream):
//   halo exchange of u0 and of p   grouped ncclSend/ncclRecv with the neighbour ranks
//   interface exchange of h_i      grouped ncclSend/ncclRecv with the neighbour ranks
//   gather of the c_i (r_c)        in-place ncclAllGather (padded per rank)
//   3 scalar reductions            in-place ncclAllGather of one partial per rank, summed
//                                  in rank order by the consuming kernel (deterministic,
//                                  identical on every rank)
#pragma once

#include <vector>

#include "common.cuh"

namespace bddc_b200 {

// 128-byte ncclUniqueId (rank 0 creates it; the caller broadcasts it).
void nccl_unique_id(char out[128]);

class Comm {
public:
    Comm(const char id[128], int rank, int world);  // the device must be current
    ~Comm();
    Comm(const Comm&) = delete;
    Comm& operator=(const Comm&) = delete;

    int rank() const { return rank_; }
    int world() const { return world_; }
    // buf holds world * per_rank doubles; this rank's block is buf + rank * per_rank.
    void allgather_inplace(double* buf, std::size_t per_rank, cudaStream_t s);
    // For peer k: send sendbuf[soff[k], soff[k+1]) and receive into recvbase[roff[k], roff[k+1]).
    void exchange(const std::vector<int>& peers, const double* sendbuf, const std::vector<std::int32_t>& soff,
                  double* recvbase, const std::vector<std::int32_t>& roff, cudaStream_t s);

private:
    void* comm_ = nullptr;
    int rank_ = 0, world_ = 1;
};

// dst[k] = src[idx[k]], k < n
void launch_pack(int n, const std::int32_t* idx, const double* src, double* dst, cudaStream_t s);
// out[slot] = sum(part[0..n)) (fixed order), optionally sqrt
void launch_reduce_to(const double* part, int n, double* out, bool take_sqrt, cudaStream_t s);

}  // namespace bddc_b200
