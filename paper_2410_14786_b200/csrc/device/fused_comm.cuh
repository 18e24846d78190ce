// Peer-memory exchanges fused into the producing and consuming kernels (multi-GPU), in a
// low-latency ("LL") format: every value travels as two 8-byte words {tag:32 | half of the
// value:32}, stored straight into the peer's LL buffer (CUDA-IPC mapping, device/comm.cu) by the
// CTA that computed it. An aligned 8-byte store is single-copy atomic, so a reader that sees
// the expected tag in both words holds the value: no fences, no flags, no separate exchange
// launch. The transfer overlaps the rest of the producer grid and the launch of the consumer;
// the consumer polls only the entries it actually reads, where it reads them.
//
// Tags: one device counter per exchange type. Every CTA of the producer reads it (tag =
// counter + 1) before taking its grid ticket; the last CTA (threadFenceReduction pattern)
// stores the new counter, so the consumer kernel (next in stream order) reads the tag the
// local producer used — every rank runs the same exchanges in the same order. Scalar
// reductions: the last CTA sums the grid partials (fixed order) into red[slot] and sends that
// one value. A 20 s bounded poll traps instead of hanging the GPU.
#pragma once

#include "comm.cuh"

namespace bddc_b200 {

using ll_word = unsigned long long;

struct Publish {
    std::uint64_t* seq = nullptr;  // this exchange's tag counter; null = nothing to publish
    unsigned int* ticket = nullptr;
    // vector values, bucketed by producing CTA: CTA b sends items [cta_ptr[b], cta_ptr[b+1]),
    // item i = src[item_src[i]] -> the LL word pair at item_dst[i] (peer memory)
    const std::int32_t* cta_ptr = nullptr;
    const std::int32_t* item_src = nullptr;
    ll_word* const* item_dst = nullptr;
    const double* src = nullptr;
    // scalar (optional): part[0..grid) summed into red[slot], sent to sc_dst[0..n_sc)
    const double* part = nullptr;
    double* red = nullptr;
    int grid = 0, slot = 0;
    ll_word* const* sc_dst = nullptr;
    int n_sc = 0;
    unsigned long long* trace = nullptr;  // diagnostics (BDDC_FUSED_TRACE): event ring, see trace_event
    int kid = 0;                          // kernel id in the trace
};

// diagnostics: trace[0] counts events; event i = {kid * 4 + what, globaltimer} at trace[1 + 2i]
__device__ __forceinline__ std::uint64_t gtimer() {
    std::uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void trace_event(unsigned long long* trace, int id, std::uint64_t t) {
    const unsigned long long i = atomicAdd(trace, 1ull);
    if (i < (1ull << 20)) {
        trace[1 + 2 * i] = static_cast<unsigned long long>(id);
        trace[2 + 2 * i] = t;
    }
}

__device__ __forceinline__ void ll_store(ll_word* w, double v, std::uint32_t tag) {
    const ll_word bits = static_cast<ll_word>(__double_as_longlong(v));
    const ll_word t = static_cast<ll_word>(tag) << 32;
    const ll_word lo = t | (bits & 0xffffffffull), hi = t | (bits >> 32);
    asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(w), "l"(lo), "l"(hi) : "memory");
}

__device__ __forceinline__ void ll_load_pair(const ll_word* w, ll_word& lo, ll_word& hi) {
    asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(w) : "memory");
}

// Poll one LL value until both words carry `tag`.
__device__ __forceinline__ double ll_get(const ll_word* w, std::uint32_t tag) {
    ll_word lo, hi;
    ll_load_pair(w, lo, hi);
    if (static_cast<std::uint32_t>(lo >> 32) != tag || static_cast<std::uint32_t>(hi >> 32) != tag) {
        const std::uint64_t t0 = gtimer();
        for (int spin = 1;; ++spin) {
            ll_load_pair(w, lo, hi);
            if (static_cast<std::uint32_t>(lo >> 32) == tag && static_cast<std::uint32_t>(hi >> 32) == tag) break;
            if ((spin & 1023) == 0 && gtimer() - t0 > 20000000000ull) __trap();  // no peer progress for 20 s
        }
    }
    return __longlong_as_double(static_cast<long long>((hi << 32) | (lo & 0xffffffffull)));
}

// The tag a consumer expects: the local producer of this exchange already stored it.
__device__ __forceinline__ std::uint32_t ll_tag(const std::uint64_t* seq) {
    return static_cast<std::uint32_t>(__ldcg(reinterpret_cast<const unsigned long long*>(seq)));
}

// Call from EVERY thread of every CTA of the producer grid, after its last global writes.
// Returns true in the grid's last CTA (after its tail: red[slot] holds the reduced scalar).
template <int THREADS>
__device__ __forceinline__ bool publish(const Publish& P) {
    if (P.seq == nullptr) return false;
    __shared__ int last_s;
    __shared__ double red_s[THREADS / 32];
    const std::uint64_t t_in = P.trace ? gtimer() : 0;
    const std::uint32_t last = ll_tag(P.seq);
    const std::uint32_t tag = last == 0xffffffffu ? 1u : last + 1u;  // never 0 (the buffers start zeroed)
    __syncthreads();  // this CTA's outputs are written
    if (threadIdx.x == 0) {
        fence_acq_rel_gpu();  // local writes only (the peer stores follow: no wait for NVLink acks)
        last_s = atomicAdd(P.ticket, 1u) == gridDim.x * gridDim.y * gridDim.z - 1;
    }
    __syncthreads();
    if (P.cta_ptr) {  // this CTA's own values, straight to the peers
        const int b = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
        const int i1 = __ldg(P.cta_ptr + b + 1);
        for (int i = __ldg(P.cta_ptr + b) + static_cast<int>(threadIdx.x); i < i1; i += THREADS)
            ll_store(P.item_dst[i], __ldcg(P.src + __ldg(P.item_src + i)), tag);
    }
    if (!last_s) return false;
    if (threadIdx.x == 0) {
        *P.seq = tag;  // every CTA has read the old value (before its ticket)
        *P.ticket = 0u;
        if (P.trace) trace_event(P.trace, P.kid * 4 + 2, t_in);
    }
    if (P.part) {
        fence_acq_rel_gpu();  // every other CTA's partial is visible to the last one
        double v = 0.0;
#pragma unroll 8  // independent loads in flight; the sum order is unchanged
        for (int i = threadIdx.x; i < P.grid; i += THREADS) v += __ldcg(P.part + i);
        v = block_sum<THREADS>(v, red_s);
        if (threadIdx.x == 0) P.red[P.slot] = v;
        if (static_cast<int>(threadIdx.x) < P.n_sc) ll_store(P.sc_dst[threadIdx.x], v, tag);
    }
    if (P.trace && threadIdx.x == 0) trace_event(P.trace, P.kid * 4 + 3, gtimer());
    __syncthreads();
    return true;
}

}  // namespace bddc_b200
