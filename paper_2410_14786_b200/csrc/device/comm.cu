#include "comm.cuh"

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

namespace bddc_b200 {
namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // torch's copy, if mapped
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = std::string("cannot load libnccl.so.2: ") + dlerror();
            return;
        }
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::decay_t<decltype(fn)>>(dlsym(h, name));
            if (!fn && err.empty()) err = std::string("libnccl.so.2 lacks ") + name;
        };
        sym(api.GetUniqueId, "ncclGetUniqueId");
        sym(api.CommInitRank, "ncclCommInitRank");
        sym(api.CommDestroy, "ncclCommDestroy");
        sym(api.AllGather, "ncclAllGather");
        sym(api.Send, "ncclSend");
        sym(api.Recv, "ncclRecv");
        sym(api.GroupStart, "ncclGroupStart");
        sym(api.GroupEnd, "ncclGroupEnd");
        sym(api.GetErrorString, "ncclGetErrorString");
    });
    if (!err.empty()) throw std::runtime_error(err);
    return api;
}

void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw std::runtime_error(std::string("NCCL error in ") + what + ": " + nccl().GetErrorString(r));
}

__global__ void pack_kernel(int n, const std::int32_t* __restrict__ idx, const double* __restrict__ src,
                            double* __restrict__ dst) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) dst[k] = src[idx[k]];
}

__global__ void reduce_to_kernel(const double* part, int n, double* out, int take_sqrt) {
    __shared__ double scratch[8];
    double v = 0.0;
#pragma unroll 8  // independent loads in flight; the sum order is unchanged
    for (int i = threadIdx.x; i < n; i += blockDim.x) v += part[i];
    v = block_sum<256>(v, scratch);
    if (threadIdx.x == 0) *out = take_sqrt ? sqrt(v) : v;
}

}  // namespace

void nccl_unique_id(char out[128]) {
    ncclUniqueId id;
    check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    std::memcpy(out, &id, 128);
}

Comm::Comm(const char id[128], int rank, int world) : rank_(rank), world_(world) {
    ncclUniqueId uid;
    std::memcpy(&uid, id, 128);
    ncclComm_t c = nullptr;
    check(nccl().CommInitRank(&c, world, uid, rank), "ncclCommInitRank");
    comm_ = c;
}

Comm::~Comm() {
    if (comm_) nccl().CommDestroy(static_cast<ncclComm_t>(comm_));
}

void Comm::allgather_inplace(double* buf, std::size_t per_rank, cudaStream_t s) {
    check(nccl().AllGather(buf + static_cast<std::size_t>(rank_) * per_rank, buf, per_rank, ncclDouble,
                           static_cast<ncclComm_t>(comm_), s),
          "ncclAllGather");
}

void Comm::exchange(const std::vector<int>& peers, const double* sendbuf, const std::vector<std::int32_t>& soff,
                    double* recvbase, const std::vector<std::int32_t>& roff, cudaStream_t s) {
    if (peers.empty()) return;
    const NcclApi& api = nccl();
    auto c = static_cast<ncclComm_t>(comm_);
    check(api.GroupStart(), "ncclGroupStart");
    for (std::size_t k = 0; k < peers.size(); ++k) {
        const std::size_t ns = soff[k + 1] - soff[k], nr = roff[k + 1] - roff[k];
        if (ns) check(api.Send(sendbuf + soff[k], ns, ncclDouble, peers[k], c, s), "ncclSend");
        if (nr) check(api.Recv(recvbase + roff[k], nr, ncclDouble, peers[k], c, s), "ncclRecv");
    }
    check(api.GroupEnd(), "ncclGroupEnd");
}

namespace {

__device__ __forceinline__ void st_release_sys(std::uint64_t* p, std::uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ std::uint64_t ld_acquire_sys(const std::uint64_t* p) {
    std::uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

constexpr int kExThreads = 512;

// value i of D goes from src[item_src[i]] to item_dst[i] (peer memory). Four items per thread
// in flight: the index, pointer and value loads of a round issue back to back instead of one
// dependent chain per item (the put loop of a single CTA is latency-bound otherwise).
template <int THREADS>
__device__ __forceinline__ void put_items(const ExchangeDesc& D, const double* src) {
    const int n = D.n_items;
    for (int i0 = static_cast<int>(threadIdx.x); i0 < n; i0 += 4 * THREADS) {
        int si[4];
        double* di[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int i = i0 + q * THREADS;
            si[q] = i < n ? __ldg(D.item_src + i) : 0;
            di[q] = i < n ? D.item_dst[i] : nullptr;
        }
        double v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = di[q] ? __ldcg(src + si[q]) : 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (di[q]) *di[q] = v[q];
    }
}

// The descriptors travel as __grid_constant__ kernel parameters (constant bank: no dependent
// global loads before the first put).
struct ExchangeArgs {
    ExchangeDesc d[2];
    double* src[2];
    const double* part;
    int grid, slot, nd;
};


__device__ __forceinline__ void wait_all(const ExchangeDesc& D, std::uint64_t seq, int lane_base) {
    const int w = static_cast<int>(threadIdx.x) - lane_base;
    if (w >= 0 && w < D.n_wait) {
        const std::uint64_t* f = D.wait[w];
        std::uint64_t t0 = 0, t = 0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        while (ld_acquire_sys(f) < seq) {
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > 20000000000ull) __trap();  // no peer progress for 20 s: fail loudly, never hang
        }
    }
}

// The flags are released after the CTA barrier: bar.sync orders every thread's peer stores
// before the flag stores, each flag published by its own thread with a system-scope release
// (PTX release cumulativity).
__global__ void __launch_bounds__(kExThreads) exchange_kernel(const __grid_constant__ ExchangeArgs A) {
    __shared__ double scratch[kExThreads / 32];
    __shared__ std::uint64_t seq_s[2];
    const ExchangeDesc& D1 = A.d[0];
    const ExchangeDesc& D2 = A.d[1];
    const bool two = A.nd > 1;
    std::uint64_t t_start = 0, t_wait = 0, t_end = 0;
    if (D1.stats) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    if (threadIdx.x == 0) {  // every rank runs the same exchanges in the same order
        seq_s[0] = *D1.seq + 1;
        *D1.seq = seq_s[0];
        if (two) {
            seq_s[1] = *D2.seq + 1;
            *D2.seq = seq_s[1];
        }
    }
    double* const dst_scalar = two ? A.src[1] : A.src[0];
    if (A.part) {  // scalar gather: this rank's total first (fixed order)
        double v = 0.0;
        for (int i = threadIdx.x; i < A.grid; i += blockDim.x) v += A.part[i];
        v = block_sum<kExThreads>(v, scratch);
        if (threadIdx.x == 0) dst_scalar[A.slot] = v;
    }
    __syncthreads();
    put_items<kExThreads>(D1, A.src[0]);
    if (two) put_items<kExThreads>(D2, A.src[1]);
    __syncthreads();
    if (static_cast<int>(threadIdx.x) < D1.n_put) st_release_sys(D1.put[threadIdx.x].flag, seq_s[0]);
    if (two && threadIdx.x >= kMaxPeers && static_cast<int>(threadIdx.x) - kMaxPeers < D2.n_put)
        st_release_sys(D2.put[threadIdx.x - kMaxPeers].flag, seq_s[1]);
    if (D1.stats) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_wait));
    wait_all(D1, seq_s[0], 0);
    if (two) wait_all(D2, seq_s[1], kMaxPeers);
    __syncthreads();
    if (D1.stats && threadIdx.x == 0) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        D1.stats[0] += 1;
        D1.stats[1] += t_end - t_start;
        D1.stats[2] += t_end - t_wait;
    }
}

}  // namespace

PeerLinks::PeerLinks(Comm& comm, const std::vector<void*>& exports)
    : nbuf_(static_cast<int>(exports.size())), rank_(comm.rank()), world_(comm.world()) {
    const std::size_t hb = sizeof(cudaIpcMemHandle_t);
    const std::size_t per = (hb * exports.size() + 7) / 8;  // doubles per rank
    std::vector<double> host(per * world_, 0.0);
    for (std::size_t b = 0; b < exports.size(); ++b) {
        cudaIpcMemHandle_t h;
        BDDC_CUDA(cudaIpcGetMemHandle(&h, exports[b]));
        std::memcpy(reinterpret_cast<char*>(host.data() + per * rank_) + b * hb, &h, hb);
    }
    double* dev = nullptr;
    BDDC_CUDA(cudaMalloc(&dev, sizeof(double) * host.size()));
    BDDC_CUDA(cudaMemcpy(dev, host.data(), sizeof(double) * host.size(), cudaMemcpyHostToDevice));
    comm.allgather_inplace(dev, per, nullptr);
    BDDC_CUDA(cudaDeviceSynchronize());
    BDDC_CUDA(cudaMemcpy(host.data(), dev, sizeof(double) * host.size(), cudaMemcpyDeviceToHost));
    cudaFree(dev);
    ptrs_.assign(static_cast<std::size_t>(world_) * nbuf_, nullptr);
    for (int q = 0; q < world_; ++q)
        for (int b = 0; b < nbuf_; ++b) {
            if (q == rank_) {
                ptrs_[static_cast<std::size_t>(q) * nbuf_ + b] = exports[b];
                continue;
            }
            cudaIpcMemHandle_t h;
            std::memcpy(&h, reinterpret_cast<const char*>(host.data() + per * q) + b * hb, hb);
            void* p = nullptr;
            BDDC_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
            ptrs_[static_cast<std::size_t>(q) * nbuf_ + b] = p;
        }
}

PeerLinks::~PeerLinks() {
    for (int q = 0; q < world_; ++q)
        if (q != rank_)
            for (int b = 0; b < nbuf_; ++b)
                if (void* p = ptrs_[static_cast<std::size_t>(q) * nbuf_ + b]) cudaIpcCloseMemHandle(p);
}

void launch_exchange(const ExchangeDesc& desc, double* src, const double* part, int grid, int slot,
                     cudaStream_t s) {
    ExchangeArgs A{};
    A.d[0] = desc;
    A.src[0] = src;
    A.part = part;
    A.grid = grid;
    A.slot = slot;
    A.nd = 1;
    exchange_kernel<<<1, kExThreads, 0, s>>>(A);
    BDDC_LAUNCHED();
}

void launch_exchange2(const ExchangeDesc& desc1, double* src1, const ExchangeDesc& desc2, double* src2,
                      const double* part, int grid, int slot, cudaStream_t s) {
    ExchangeArgs A{};
    A.d[0] = desc1;
    A.d[1] = desc2;
    A.src[0] = src1;
    A.src[1] = src2;
    A.part = part;
    A.grid = grid;
    A.slot = slot;
    A.nd = 2;
    exchange_kernel<<<1, kExThreads, 0, s>>>(A);
    BDDC_LAUNCHED();
}

void launch_pack(int n, const std::int32_t* idx, const double* src, double* dst, cudaStream_t s) {
    if (n <= 0) return;
    pack_kernel<<<std::min(148 * 4, (n + 255) / 256), 256, 0, s>>>(n, idx, src, dst);
    BDDC_LAUNCHED();
}

void launch_reduce_to(const double* part, int n, double* out, bool take_sqrt, cudaStream_t s) {
    reduce_to_kernel<<<1, 256, 0, s>>>(part, n, out, take_sqrt ? 1 : 0);
    BDDC_LAUNCHED();
}

}  // namespace bddc_b200
