// Multi-GPU communication of the distributed BDDC-PCG, one rank per B200.
// NCCL is loaded at run time (dlopen of libnccl.so.2, preferring the copy torch already
// mapped), so the single-GPU library carries no NCCL link dependency; it serves the setup
// (A_ci gather, IPC handle exchange) and the BDDC_P2P=0 fallback.
//
// Per PCG iteration the distributed path exchanges: the halo of u0, the c_i (r_c), the
// shared-interface h_i, p.q, r.r, and r.z with the halo of z. By default these ride on the
// producing / consuming kernels (fused_comm.cuh, LL format over the IPC mappings below);
// BDDC_FUSED_EX=0 uses the single-CTA flag-based exchange kernels declared here, BDDC_P2P=0
// grouped ncclSend/ncclRecv and in-place ncclAllGather. Scalars are gathered as one partial
// per rank and summed in rank order by the consumer (deterministic, identical on every rank).
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

// ---------------------------------------------------------------------------------------
// Peer-memory exchanges over NVLink / NVSwitch (the default on a multi-GPU box; NCCL stays
// the fallback, BDDC_P2P=0). Every rank maps the peers' receive buffers with CUDA IPC; one
// single-CTA kernel per exchange stores this rank's values straight into the peers' buffers,
// publishes a sequence number in each peer's flag array (st.release.sys after a system
// fence) and then waits (ld.acquire.sys) for the flags of the ranks it receives from. The
// puts precede the wait inside one kernel on every rank, so no rank ever waits on a rank
// that is waiting on it; a bounded spin traps instead of hanging the GPU.
constexpr int kMaxPeers = 64;
constexpr int kFlagTypes = 12;

struct PeerPut {
    double* dst;            // peer memory (IPC mapping), already offset
    std::uint64_t* flag;    // the peer's flag slot for (type, this rank)
    std::int32_t off, cnt;  // values idx[off .. off+cnt) (or src[off ..] when idx is null)
};

struct ExchangeDesc {
    std::int32_t n_put = 0, n_wait = 0;
    std::uint64_t* seq = nullptr;       // device counter of this exchange type (graph-capturable)
    unsigned long long* stats = nullptr;  // diagnostics: {count, total ns, wait ns} (null: off)
    const std::int32_t* idx = nullptr;  // pack indices into src, or null for contiguous
    // the puts flattened over all peers (one parallel loop): value i goes from
    // src[item_src[i]] to item_dst[i] (peer memory)
    std::int32_t n_items = 0;
    double* const* item_dst = nullptr;
    const std::int32_t* item_src = nullptr;
    PeerPut put[kMaxPeers];
    std::uint64_t* wait[kMaxPeers];     // this rank's flag slots to wait on
};

class PeerLinks {
public:
    // Collective over `comm`: exports the local buffers (device allocations, in the same
    // order on every rank) and maps every peer's copies.
    PeerLinks(Comm& comm, const std::vector<void*>& exports);
    ~PeerLinks();
    PeerLinks(const PeerLinks&) = delete;
    PeerLinks& operator=(const PeerLinks&) = delete;
    void* peer(int rank, int buffer) const { return ptrs_[static_cast<std::size_t>(rank) * nbuf_ + buffer]; }

private:
    std::vector<void*> ptrs_;  // [rank][buffer]; own rank = the local pointer
    int nbuf_ = 0, rank_ = 0, world_ = 1;
};

// One exchange: seq = ++*desc->seq, puts per desc, system fence, flags = seq, then wait for
// the incoming flags. part != null: first reduces part[0..grid) (fixed order) into src[slot]
// (scalar gathers).
void launch_exchange(const ExchangeDesc& desc, double* src, const double* part, int grid, int slot,
                     cudaStream_t s);
// Two exchanges fused in one launch (e.g. the halo of z together with the r.z gather): the
// scalar reduction (if any) feeds desc2's src2.
void launch_exchange2(const ExchangeDesc& desc1, double* src1, const ExchangeDesc& desc2, double* src2,
                      const double* part, int grid, int slot, cudaStream_t s);

// dst[k] = src[idx[k]], k < n
void launch_pack(int n, const std::int32_t* idx, const double* src, double* dst, cudaStream_t s);
// out[slot] = sum(part[0..n)) (fixed order), optionally sqrt
void launch_reduce_to(const double* part, int n, double* out, bool take_sqrt, cudaStream_t s);

}  // namespace bddc_b200
