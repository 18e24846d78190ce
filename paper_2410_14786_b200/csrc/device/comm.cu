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
