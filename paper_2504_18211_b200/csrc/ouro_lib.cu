// ouro_lib.cu -- libouro_b200: heap construction, driver-phase kernels and the
// C-ABI of include/ouro.h (everything except the GPU-free config half, which is
// ouro_config.cpp).  sm_100a only.
//
// The hot path itself is the header-only device allocator in
// include/ouro_device.cuh; the kernels here are (a) the paper's driver phases
// (alloc / write / verify / free) as batch
// launchers, (b) construction (new_arena + allocator init, SPEC.md:45-53,
// 244-251), (c) quiescent stats / canonical digest / disjointness audit
// (SURVEY.md §8c), (d) mixed churn (BASELINE configs[3]),
// (e) the single-warp op-script runner used for oracle parity, and (f) atomic
// micro-benchmarks that give the roofline denominators.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cub/cub.cuh>
#include <vector>

#include "../../include/ouro.h"
#include "../../include/ouro_device.cuh"
#include "ouro_internal.h"

using namespace ouro_dev;
using ouro_host::Geometry;

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            std::fprintf(stderr, "ouro: %s failed: %s (%s:%d)\n", #x, cudaGetErrorString(e_), \
                         __FILE__, __LINE__);                                          \
            return OURO_ERR_CUDA;                                                      \
        }                                                                              \
    } while (0)

namespace {

constexpr int kBlock = 256;
constexpr size_t kSmHintBytes = 256 * 32 * 8;
// Launch shape of the malloc/free/churn drivers (one request per thread, requests
// independent), per heap; new heaps start from the process default
// (ouro_set_launch_shape).  op_waves = 0: one thread per request (grid = n /
// block); op_waves = w >= 1: persistent grid of w x (resident CTAs per SM) x SMs
// that grid-strides over the requests (measured slower).
std::atomic<int> g_def_block{256};
std::atomic<int> g_def_waves{0};
template <class Kern>
unsigned op_grid(const ouro_heap* H, Kern kern, u64 n) {
    const u64 need = std::max<u64>(1, (n + H->op_block - 1) / H->op_block);
    if (H->op_waves <= 0) return (unsigned)need;
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, H->device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, H->op_block, 0);
    const u64 cap = (u64)std::max(1, per_sm) * (u64)std::max(1, sms) * (u64)H->op_waves;
    return (unsigned)std::min(need, cap);
}

// Every host entry point that touches a heap runs on the heap's device and
// restores the caller's current device on return (several heaps on several
// devices may be driven from one host thread, or one heap per host thread).
struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) { prev = -1; ok = false; return; }
        if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;
};
#define OURO_BIND(H)                                   \
    DeviceGuard dev_guard_((H)->device);               \
    if (!dev_guard_.ok) return OURO_ERR_CUDA

// Scoped device buffer / event / stream: released on every return path.
struct DevBuf {
    void* p = nullptr;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { if (p) cudaFree(p); }
    cudaError_t alloc(size_t bytes) { return cudaMalloc(&p, std::max<size_t>(bytes, 16)); }
    template <class T> T* as() const { return static_cast<T*>(p); }
};
struct Events {
    std::vector<cudaEvent_t> ev;
    ~Events() { for (auto e : ev) cudaEventDestroy(e); }
    cudaError_t create(size_t n) {
        for (size_t i = 0; i < n; ++i) {
            cudaEvent_t e;
            const cudaError_t r = cudaEventCreate(&e);
            if (r != cudaSuccess) return r;
            ev.push_back(e);
        }
        return cudaSuccess;
    }
};
struct Stream {
    cudaStream_t s = nullptr;
    ~Stream() { if (s) cudaStreamDestroy(s); }
};

__host__ __device__ inline u64 mix64h(u64 x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
__host__ __device__ inline u64 hmix(u64 a, u64 b) { return mix64h(a * 0x9E3779B97F4A7C15ull + mix64h(b)); }
__host__ __device__ inline u64 pattern_base(u64 seed, u64 slot, u32 it) {
    return mix64h(seed ^ (slot * 0xD1B54A32D192ED03ull) ^ ((u64)it * 0x8CB92BA72F3D8DD7ull));
}
__host__ __device__ inline u64 pattern_word(u64 base, u64 w) { return base ^ (w * 0x9E3779B97F4A7C15ull) ^ (w << 7); }

u64 next_pow2(u64 v) { return v <= 1 ? 1 : (1ull << (64 - __builtin_clzll(v - 1))); }
cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
unsigned grid_for(u64 n) { return (unsigned)std::max<u64>(1, (n + kBlock - 1) / kBlock); }

// ----------------------------------------------------------- construction ----
__global__ void k_fill_ring(u64* slots, u64 R, u64 cap, int mode, u32 first_chunk, u32 ppc, u32 page_bits) {
    for (u64 t = blockIdx.x * (u64)blockDim.x + threadIdx.x; t < R; t += (u64)gridDim.x * blockDim.x) {
        u64 v = 0;
        if (t < cap) {
            u32 val;
            if (mode == 0) val = (u32)t;
            else val = ((first_chunk + (u32)(t / ppc)) << page_bits) | (u32)(t % ppc);
            v = (1ull << 32) | val;
        }
        slots[t] = v;
    }
}

// Prefill a virtual queue's first segments (consecutive chunks from `seg0`).
__global__ void k_fill_segments(uint8_t* heap, u32 chunk_shift, u32 seg0, u64 S, u32 hdr, u64 cap,
                                u32 first_chunk, u32 ppc, u32 page_bits) {
    for (u64 t = blockIdx.x * (u64)blockDim.x + threadIdx.x; t < cap; t += (u64)gridDim.x * blockDim.x) {
        const u32 c = seg0 + (u32)(t / S);
        u64* w = reinterpret_cast<u64*>(heap + ((u64)c << chunk_shift));
        const u32 val = ((first_chunk + (u32)(t / ppc)) << page_bits) | (u32)(t % ppc);
        w[hdr + t % S] = ((u64)vtag_seg(t / S) << 32) | val;
    }
}
__global__ void k_vl_headers(uint8_t* heap, u32 chunk_shift, u32 seg0, u32 m) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    u64* w = reinterpret_cast<u64*>(heap + ((u64)(seg0 + i) << chunk_shift));
    w[0] = (i + 1 < m) ? (((u64)(i + 1) << 32) | (seg0 + i + 1)) : NONE_LINK;
    w[1] = (1ull << 32) | ((i + 1 < m) ? 1ull : 0ull);  // in-linked flag | retire counter (link event)
}
// Page-kind chunk headers: Reserved segment storage or Assigned(k) fully free.
__global__ void k_init_pq_chunks(ouro_heap_view v, const u32* pq) {
    const u32 c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= v.N) return;
    const u32* start = pq;
    const u32* n = pq + v.K;
    const u32* s = pq + 2 * v.K;
    u32 k = 0;
    while (k + 1 < v.K && c >= start[k] + n[k]) ++k;
    u64* row = bm_row(v, c);
    if (c - start[k] < s[k]) {
        v.meta[c] = mk_meta(0, ST_RESERVED, 0);
        return;
    }
    v.meta[c] = mk_meta(1, k + 1, ppc_of(v, k));  // bitmap all-zero = all free
    (void)row;
}

// ------------------------------------------------------------ driver phases ----
// (Forcing 32 registers for 8 blocks/SM was measured slower: the spills cost
// more than the extra warps gain, profiles/r1_ncu_summary.md.)
// 6 resident blocks per SM (<= 40 registers): the blocks of an OOM storm only
// wait out their retry rounds, so residency sets how many waves the storm takes
// (pq1g 8 KiB alloc 297 -> 276 us, cq1g 595 -> 496 us; served sizes unchanged).
#ifndef OURO_ALLOC_MIN_BLOCKS
#define OURO_ALLOC_MIN_BLOCKS 6
#endif
template <int KIND, int FL, class SZ = u32>
__global__ void __launch_bounds__(kBlock, OURO_ALLOC_MIN_BLOCKS) k_alloc(ouro_heap_view v, u64 n, u64 uniform, const SZ* sizes, void** out) {
#if OURO_STORM_STATS
    const u64 tk0 = clock64();
#endif
    ouro_block_init(v);
#if OURO_STORM_STATS
    const u64 tk1 = clock64();
#endif
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i - threadIdx.x % 32 < n; i += stride) {
        const u32 lanes = __ballot_sync(0xFFFFFFFFu, i < n);
        if (i < n) out[i] = ouro_malloc_t<KIND, FL>(v, sizes ? sizes[i] : uniform, nullptr, lanes);
    }
#if OURO_STORM_STATS
    if ((threadIdx.x & 31) == 0) {
        OURO_DBG(20, 1);
        OURO_DBG(21, tk1 - tk0);
        OURO_DBG(22, clock64() - tk1);
        if (threadIdx.x == 0) { OURO_DBG(23, 1); u64 g; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g)); OURO_DBG(24, g >> 10); }
    }
#endif
}
template <int KIND, int FL>
__global__ void __launch_bounds__(kBlock) k_free(ouro_heap_view v, u64 n, void* const* ptrs) {
    ouro_block_init();
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i - threadIdx.x % 32 < n; i += stride) {
        const u32 lanes = __ballot_sync(0xFFFFFFFFu, i < n);
        if (i < n) ouro_free_t<KIND, FL>(v, ptrs[i], lanes);
    }
}

__device__ __forceinline__ u64 region_len(const ouro_heap_view& v, const void* p) {
    const u64 off = (u64)((const uint8_t*)p - v.base);
    const u32 c = (u32)(off >> v.chunk_shift);
    if (v.kind == KIND_PAGE) {
        // static partition: the class is arithmetic (as in free_impl), no header load
        const u32 k = c < v.pq_n0 ? 0u : 1u + (c - v.pq_n0) / v.pq_q;
        return k < v.K ? 1ull << (v.min_shift + k) : 0ull;
    }
    const u32 st = m_state(v.meta[c]);
    if (st == 0 || st > v.K) return 0;
    return 1ull << (v.min_shift + st - 1);
}

#ifndef OURO_PAT_RUN
#define OURO_PAT_RUN 2
#endif
// Pattern writer / verifier.  Warp w covers the slot group
// {g + k*G : lane k < 32}, G = ceil(n / 32): regions under 512 B are done by
// their own lane (16 B vector accesses), regions of >= 512 B by the whole warp
// (16 B per lane, 512 B coalesced per access).  Striding a group over the slot
// range spreads the live slots of an OOM-heavy launch -- the first ones (8 KiB:
// 13 104 of 2^20) -- over thousands of warps; with a warp per 32 consecutive
// slots, ~400 warps did all of that work one page after another (verify ran at
// ~0.4 TB/s; now 8 KiB write 4.0 TB/s, verify 2.3 TB/s).  Lanes work in runs of
// OURO_PAT_RUN consecutive slots so small regions still coalesce in pairs (runs
// of 1 / 2 / 4 / 8, 16 B write: 0.9 / 1.4 / 1.4 / 1.4 TB/s; 8 KiB: 4.0 / 4.0 /
// 3.3 / 2.4 TB/s).
// lanes in runs of kPatRun consecutive slots (so small regions coalesce per run),
// the 32 / kPatRun runs of a warp strided Q slots apart over the slot range
constexpr u32 kPatRun = OURO_PAT_RUN;
#ifndef OURO_PAT_BATCH
#define OURO_PAT_BATCH 4
#endif
constexpr u32 kPatBatch = OURO_PAT_BATCH;
// 4 resident blocks (<= 64 registers): the batched verify would otherwise take
// ~100 registers and run at half the occupancy.
#ifndef OURO_PAT_MIN_BLOCKS
#define OURO_PAT_MIN_BLOCKS 4
#endif
__device__ __forceinline__ u64 slot_of(u64 g, u32 lane, u64 Q) {
    return g * kPatRun + (lane % kPatRun) + (u64)(lane / kPatRun) * Q;
}
template <bool VERIFY>
__device__ __forceinline__ void pattern_body(const ouro_heap_view& v, u64 n, void* const* ptrs, u64 seed, u32 it,
                                             u64* result) {
    const u32 lane = threadIdx.x & 31;
    const u64 nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
    const u64 runs = 32 / kPatRun;                                        // lane runs per warp
    const u64 Q = ((n + runs - 1) / runs + kPatRun - 1) / kPatRun * kPatRun;  // slots per run column
    const u64 G = Q / kPatRun;
    u64 bad = 0;
    for (u64 g = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; g < G; g += nwarps) {
        const u64 i = slot_of(g, lane, Q);
        void* p = i < n ? ptrs[i] : nullptr;
        const u64 len = p ? region_len(v, p) : 0;
        if (len && len < 512) {
            const u64 b = pattern_base(seed, i, it);
            u64* w = reinterpret_cast<u64*>(p);
            u64 nb = 0;
            for (u64 j = 0; j < len / 8; j += 2) {
                if (VERIFY) {
                    const ulonglong2 x = reinterpret_cast<const ulonglong2*>(w)[j / 2];
                    nb += (x.x != pattern_word(b, j)) + (x.y != pattern_word(b, j + 1));
                } else {
                    reinterpret_cast<ulonglong2*>(w)[j / 2] =
                        make_ulonglong2(pattern_word(b, j), pattern_word(b, j + 1));
                }
            }
            if (VERIFY && nb) { bad += nb; atomicMin(&result[1], i); }
        }
        u32 todo = __ballot_sync(0xFFFFFFFFu, len >= 512);
        while (todo) {
            const u32 src = __ffs(todo) - 1;
            todo &= todo - 1;
            u64* w = reinterpret_cast<u64*>(__shfl_sync(0xFFFFFFFFu, (u64)p, src));
            const u64 L = __shfl_sync(0xFFFFFFFFu, len, src);
            const u64 slot = slot_of(g, src, Q);
            const u64 b = pattern_base(seed, slot, it);
            u64 nb = 0;
            // verify: kPatBatch 512 B steps per pass, all loads issued before the
            // compares -- that many 16 B loads in flight per lane instead of one
            // (pq1g 2-8 KiB verify 2.2-2.3 -> 2.8-3.0 TB/s, cq1g 4.3-4.5 -> 5.8-5.9 TB/s;
            // profiles/r2/pattern_ab.txt).  Stores need no batching.
            const u64 words = L / 8;
            if constexpr (VERIFY) {
                for (u64 j0 = 2 * lane; j0 < words; j0 += 64 * kPatBatch) {
                    ulonglong2 x[kPatBatch];
#pragma unroll
                    for (u32 u = 0; u < kPatBatch; ++u)
                        if (j0 + 64 * u < words) x[u] = reinterpret_cast<const ulonglong2*>(w)[(j0 + 64 * u) / 2];
#pragma unroll
                    for (u32 u = 0; u < kPatBatch; ++u) {
                        const u64 j = j0 + 64 * u;
                        if (j < words) nb += (x[u].x != pattern_word(b, j)) + (x[u].y != pattern_word(b, j + 1));
                    }
                }
            } else {
                for (u64 j = 2 * lane; j < words; j += 64)
                    reinterpret_cast<ulonglong2*>(w)[j / 2] = make_ulonglong2(pattern_word(b, j), pattern_word(b, j + 1));
            }
            if (VERIFY && nb) { bad += nb; atomicMin(&result[1], slot); }
        }
    }
    if (VERIFY) {
        for (int o = 16; o; o >>= 1) bad += __shfl_xor_sync(0xFFFFFFFFu, bad, o);
        if (lane == 0 && bad) atomicAdd(&result[0], bad);
    }
}
// Separate kernels: the verifier is held to 4 resident blocks' registers, the
// writer compiles to ~40 on its own.
template <bool VERIFY>
__global__ void __launch_bounds__(kBlock) k_pattern(ouro_heap_view v, u64 n, void* const* ptrs, u64 seed, u32 it,
                                                    u64* result) {
    pattern_body<VERIFY>(v, n, ptrs, seed, it, result);
}
template <>
__global__ void __launch_bounds__(kBlock, OURO_PAT_MIN_BLOCKS) k_pattern<true>(ouro_heap_view v, u64 n,
                                                                               void* const* ptrs, u64 seed, u32 it,
                                                                               u64* result) {
    pattern_body<true>(v, n, ptrs, seed, it, result);
}
unsigned pattern_grid(u64 n) { return (unsigned)std::max<u64>(1, ((n + 31) / 32 + 7) / 8); }  // ~one group per warp

__global__ void k_count(u64 n, void* const* ptrs, u64* count) {
    const u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x;
    const bool live = i < n && ptrs[i] != nullptr;
    const u32 b = __ballot_sync(0xFFFFFFFFu, live);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(count, (u64)__popc(b));
}

// ------------------------------------------------------------------- audit ----
__global__ void k_audit_collect(ouro_heap_view v, u64 n, void* const* ptrs, u64* offs, u64* lens, u64* res,
                                unsigned long long* idx) {
    const u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x;
    if (i >= n || !ptrs[i]) return;
    const u64 off = (u64)((uint8_t*)ptrs[i] - v.base);
    atomicAdd(&res[0], 1ull);
    if (off >= v.heap_bytes) { atomicAdd(&res[1], 1ull); return; }
    const u32 c = (u32)(off >> v.chunk_shift);
    const u32 st = m_state(v.meta[c]);
    if (st == 0 || st > v.K) { atomicAdd(&res[1], 1ull); return; }
    const u32 k = st - 1;
    const u64 len = 1ull << (v.min_shift + k);
    if (off & (len - 1)) atomicAdd(&res[2], 1ull);
    const u32 p = (u32)((off & (v.chunk_bytes - 1)) >> (v.min_shift + k));
    if (!((bm_row(v, c)[p >> 6] >> (p & 63)) & 1ull)) atomicAdd(&res[4], 1ull);  // must be marked allocated
    atomicAdd(&res[5], len);
    const u64 j = atomicAdd(idx, 1ull);
    offs[j] = off;
    lens[j] = len;
}
__global__ void k_audit_neighbours(u64 m, const u64* offs, const u64* lens, u64* res) {
    const u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x;
    if (i + 1 >= m) return;
    if (offs[i] + lens[i] > offs[i + 1]) atomicAdd(&res[3], 1ull);
}

// ------------------------------------------------------------------- churn ----
template <int KIND, int FL>
__device__ __forceinline__ void churn_slot(const ouro_heap_view& v, u64 t, bool in, u32 r, u64 seed, void** slots,
                                           uint8_t* touched, u64* res) {
    const u64 h = mix64h(seed ^ (t << 32) ^ r);
    void* s = in ? slots[t] : nullptr;
    const bool do_free = in && s && (h & 1);
    const bool do_malloc = in && !s;
    const u32 fm = __ballot_sync(0xFFFFFFFFu, do_free);
    const u32 mm = __ballot_sync(0xFFFFFFFFu, do_malloc);
    if (!in) return;
    u32 ev_ok = 0, ev_fail = 0, ev_free = 0, ev_reuse = 0, ev_bad = 0;
    if (do_free) {
        ouro_free_t<KIND, FL>(v, s, fm);
        slots[t] = nullptr;
        ev_free = 1;
    } else if (do_malloc) {
        void* p = ouro_malloc_t<KIND, FL>(v, 8 + (h >> 1) % 4089, nullptr, mm);
        if (p) {
            *reinterpret_cast<u64*>(p) = mix64h(t ^ seed);
            slots[t] = p;
            ev_ok = 1;
            const u64 g = (u64)((uint8_t*)p - v.base) >> v.min_shift;
            const u32 old = atomicOr(reinterpret_cast<u32*>(touched) + (g >> 5), 1u << (g & 31));
            ev_reuse = (old >> (g & 31)) & 1u;
        } else {
            ev_fail = 1;
        }
    } else {
        ev_bad = *reinterpret_cast<const u64*>(s) != mix64h(t ^ seed);
    }
    const u32 m = __activemask();
    const u32 lane = lane_id();
    const u32 a = __ballot_sync(m, ev_ok), b = __ballot_sync(m, ev_fail), c = __ballot_sync(m, ev_free);
    const u32 d = __ballot_sync(m, ev_reuse), e = __ballot_sync(m, ev_bad);
    if (lane == (u32)(__ffs(m) - 1)) {
        if (a) atomicAdd(&res[0], (u64)__popc(a));
        if (b) atomicAdd(&res[1], (u64)__popc(b));
        if (c) atomicAdd(&res[2], (u64)__popc(c));
        if (d) atomicAdd(&res[3], (u64)__popc(d));
        if (e) atomicAdd(&res[4], (u64)__popc(e));
    }
}
#ifndef OURO_CHURN_MIN_BLOCKS
#define OURO_CHURN_MIN_BLOCKS 5
#endif
// 5 resident blocks (<= 48 registers): left free, the compiler takes 62-64 for the
// churn loop plus the retry rounds and the kernel loses a fifth of its warps.
template <int KIND, int FL>
__global__ void __launch_bounds__(kBlock, OURO_CHURN_MIN_BLOCKS) k_churn(ouro_heap_view v, u64 n, u32 r, u64 seed, void** slots,
                                                  uint8_t* touched, u64* res) {
    ouro_block_init(v);
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 t = blockIdx.x * (u64)blockDim.x + threadIdx.x; t - threadIdx.x % 32 < n; t += stride)
        churn_slot<KIND, FL>(v, t, t < n, r, seed, slots, touched, res);
}

// --------------------------------------------------------- op-script runner ----
template <int KIND, int FL>
__global__ void k_script(ouro_heap_view v, const ouro_script_step* steps, u32 nsteps, u64* out_off, int* out_st) {
    ouro_block_init();
    const u32 lane = threadIdx.x;
    for (u32 s = 0; s < nsteps; ++s) {
        const ouro_script_step& st = steps[s];
        out_off[s * 32 + lane] = ~0ull;
        out_st[s * 32 + lane] = -1;
        __syncwarp();
        const u32 lanes = st.lane_mask;
        if ((lanes >> lane) & 1u) {
            if (st.op == 0 || st.op == 2) {
                int status;
                void* p = st.op == 0 ? ouro_malloc_t<KIND, FL>(v, st.arg[lane], &status, lanes)
                                     : ouro_malloc_coalesced_t<KIND, FL>(v, st.arg[lane], &status, lanes);
                out_off[s * 32 + lane] = p ? (u64)((uint8_t*)p - v.base) : ~0ull;
                out_st[s * 32 + lane] = status;
            } else {
                const u64 a = st.arg[lane];
                u64 off;
                if (a >> 63) off = a & ~(1ull << 63);
                else off = a < (u64)s * 32 ? out_off[a] : ~0ull;
                if (off == ~0ull) off = ~1ull;
                out_st[s * 32 + lane] = ouro_free_t<KIND, FL>(v, v.base + off, lanes);
            }
        }
        __syncwarp();
    }
}

// --------------------------------------------------------------- digest ----
struct DigestDev {
    u64 header_hash;
    u64 queue_hash;
    u64 live_pages;
    u64 assigned_total;
    u32 bad;
    u32 pad;
    u64 class_chunks[OURO_MAX_CLASSES];
    u64 class_queued_live[OURO_MAX_CLASSES];
    u64 class_live_pages[OURO_MAX_CLASSES];
};

__global__ void k_digest_headers(ouro_heap_view v, DigestDev* d, u32* where) {
    const u32 c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= v.N) return;
    const u64 m = v.meta[c];
    const u32 st = m_state(m);
    const u64* b = bm_row(v, c);
    u64 bh = 0, pc = 0, any = 0;
    for (u32 w = 0; w < v.Wmax; ++w) {
        bh = hmix(bh ^ w, b[w]);
        pc += __popcll(b[w]);
        any |= b[w];
    }
    atomicAdd(&d->header_hash, v.kind == OURO_KIND_PAGE ? hmix(hmix(c, m), bh) : hmix(m & 0xFFFFFFFFFFull, bh));
    if (st == ST_RESERVED) return;
    if (st == ST_UNASSIGNED) {
        if (m_free(m) != 0 || any) atomicOr(&d->bad, 1u);
        return;
    }
    if (st > v.K) { atomicOr(&d->bad, 2u); return; }
    const u32 k = st - 1;
    atomicAdd(where + c, 1u);
    atomicAdd(&d->assigned_total, 1ull);
    atomicAdd(&d->class_chunks[k], 1ull);
    const u64 live = ppc_of(v, k) - m_free(m);
    atomicAdd(&d->class_live_pages[k], live);
    atomicAdd(&d->live_pages, live);
    if (ppc_of(v, k) - pc != m_free(m)) atomicOr(&d->bad, 4u);  // allocated bits = live pages
}

// Value of ticket t in a quiescent queue (segment table for virtual flavours).
__device__ __forceinline__ bool ticket_value(const ouro_heap_view& v, const ouro_queue_dev& Q, const u32* segtab,
                                             u64 seg_first, u64 t, u32* out) {
    u64 x;
    if (Q.flavor == FL_ARRAY) {
        x = Q.slots[t & Q.ring_mask];
    } else {
        const u64 S = Q.flavor == FL_VA ? v.S_va : v.S_vl;
        const u64 s = t / S;
        const u32 c = segtab[s - seg_first];
        if (c == NONE) return false;
        x = chunk_words(v, c)[(Q.flavor == FL_VA ? 0 : 2) + t % S];
    }
    *out = (u32)x;
    return true;
}

// mode 0: pool / private pool (where[c]++), 1: page-kind class k, 2: chunk-kind class k
__global__ void k_digest_queue(ouro_heap_view v, const ouro_queue_dev* Qp, const u32* segtab, u64 seg_first, int mode,
                               u32 k, DigestDev* d, u32* where, u32* entries) {
    const ouro_queue_dev& Q = *Qp;
    const u64 n = Q.tail - Q.head;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        u32 x;
        if (!ticket_value(v, Q, segtab, seg_first, Q.head + i, &x)) { atomicOr(&d->bad, 8u); continue; }
        if (mode == 0) {
            if (x < v.N) atomicAdd(where + x, 1u);
            else atomicOr(&d->bad, 16u);
        } else if (mode == 1) {
            atomicAdd(&d->queue_hash, hmix(k + 1, x));
            atomicAdd(&d->class_queued_live[k], 1ull);
        } else {
            const u32 c = x & v.cmask;
            const u32 glow = v.chunk_bits >= 32 ? 0u : x >> v.chunk_bits;
            const u64 m = v.meta[c];
            if (m_state(m) == k + 1 && (m_gen(m) & v.gmask) == glow) {
                atomicAdd(entries + c, 1u);
                atomicAdd(&d->class_queued_live[k], 1ull);
            }
        }
    }
}

// ------------------------------------------------------- atomic peaks ----
__global__ void k_atom_distinct32(u32* a, u64 words, u32 iters) {
    const u64 tid = blockIdx.x * (u64)blockDim.x + threadIdx.x;
    const u64 stride = (u64)gridDim.x * blockDim.x;
    u32 acc = 0;
    for (u32 r = 0; r < iters; ++r) {
        const u64 idx = ((tid + r * stride) * 8) % words;  // one 4 B counter per 32 B sector
        acc += atomicAdd(a + idx, 1u);
    }
    if (acc == 0xFFFFFFFFu) a[0] = acc;
}
__global__ void k_atom_distinct_cas64(u64* a, u64 words, u32 iters) {
    const u64 tid = blockIdx.x * (u64)blockDim.x + threadIdx.x;
    const u64 stride = (u64)gridDim.x * blockDim.x;
    u64 acc = 0;
    for (u32 r = 0; r < iters; ++r) {
        const u64 idx = ((tid + r * stride) * 4) % words;
        const u64 old = a[idx];
        acc += atomicCAS(a + idx, old, old + 1);
    }
    if (acc == ~0ull) a[0] = acc;
}
__global__ void k_atom_same_warp(u64* a, u32 iters) {
    u64 acc = 0;
    for (u32 r = 0; r < iters; ++r) {
        u64 x = 0;
        if ((threadIdx.x & 31) == 0) x = atomicAdd(a, 1ull);
        acc += __shfl_sync(0xFFFFFFFFu, x, 0);
    }
    if (acc == ~0ull) a[1] = acc;
}
// One leader lane per block loads ONE word back to back, each load's address
// depending on the previous result: the retry-round poll pattern of an OOM storm.
__global__ void k_hot_poll(const u64* a, u32 iters, u64* cyc) {
    if (threadIdx.x) return;
    u64 acc = 0;
    const u64 c0 = clock64();
    for (u32 r = 0; r < iters; ++r) acc += ld_rlx(a + (acc >> 63));
    if (acc == 12345) cyc[1] = acc;  // consume before the clock read
    atomicAdd(cyc, clock64() - c0);
}
__global__ void k_atom_same_lane(u64* a, u32 iters) {
    u64 acc = 0;
    for (u32 r = 0; r < iters; ++r) {
        u64 x;
        asm volatile("atom.relaxed.gpu.global.add.u64 %0, [%1], %2;" : "=l"(x) : "l"(a), "l"((u64)(threadIdx.x + r)) : "memory");
        acc += x;
    }
    if (acc == ~0ull) a[1] = acc;
}

// ------------------------------------------------------------ variant switch ----
#define OURO_VSWITCH(H, FN, ...)                                            \
    switch ((H)->cfg.allocator_kind * 3 + (H)->cfg.queue_flavor) {          \
    case 0: FN<0, 0>(__VA_ARGS__); break;                                   \
    case 1: FN<0, 1>(__VA_ARGS__); break;                                   \
    case 2: FN<0, 2>(__VA_ARGS__); break;                                   \
    case 3: FN<1, 0>(__VA_ARGS__); break;                                   \
    case 4: FN<1, 1>(__VA_ARGS__); break;                                   \
    default: FN<1, 2>(__VA_ARGS__); break;                                  \
    }

template <int K, int F>
void launch_alloc(ouro_heap* H, u64 n, u64 uni, const u32* sizes, void** out, cudaStream_t st) {
    k_alloc<K, F><<<op_grid(H, k_alloc<K, F>, n), H->op_block, 0, st>>>(H->view, n, uni, sizes, out);
}
template <int K, int F>
void launch_alloc16(ouro_heap* H, u64 n, const uint16_t* sizes, void** out, cudaStream_t st) {
    k_alloc<K, F, uint16_t><<<op_grid(H, k_alloc<K, F, uint16_t>, n), H->op_block, 0, st>>>(H->view, n, 0, sizes, out);
}
template <int K, int F>
void launch_free(ouro_heap* H, u64 n, void* const* p, cudaStream_t st) {
    k_free<K, F><<<op_grid(H, k_free<K, F>, n), H->op_block, 0, st>>>(H->view, n, p);
}
template <int K, int F>
void launch_churn(ouro_heap* H, u64 n, u32 r, u64 seed, void** slots, u64* res, cudaStream_t st) {
    k_churn<K, F><<<op_grid(H, k_churn<K, F>, n), H->op_block, 0, st>>>(H->view, n, r, seed, slots, H->d_touched, res);
}
template <int K, int F>
void launch_script(ouro_heap* H, const ouro_script_step* s, u32 n, u64* o, int* st) {
    k_script<K, F><<<1, 32>>>(H->view, s, n, o, st);
}

// ---------------------------------------------------------- heap building ----
void* dalloc(ouro_heap* H, size_t bytes) {
    void* p = nullptr;
    if (cudaMalloc(&p, std::max<size_t>(bytes, 16)) != cudaSuccess) return nullptr;
    H->owned.push_back(p);
    return p;
}

// Allocate every device structure once (sizes depend only on the config).
ouro_status plan(ouro_heap* H) {
    const Geometry& g = H->g;
    const u32 N = g.N, K = g.K;
    H->nq = 2 * K + 1;
    H->hq.assign(H->nq, ouro_queue_dev{});
    H->pq_start.assign(K, 0);
    H->pq_n.assign(K, 0);
    H->pq_s.assign(K, 0);
    const u64 S_va = g.chunk / 8, S_vl = g.chunk / 8 - 2;
    auto init_q = [&](ouro_queue_dev& q, u32 flavor, u64 cap, int seg_src) -> bool {
        q.flavor = flavor;
        q.cap = cap;
        q.seg_src = seg_src;
        if (flavor == FL_ARRAY) {
            const u64 R = next_pow2(std::max<u64>(cap, 1));
            q.ring_shift = (u32)__builtin_ctzll(R);
            q.ring_mask = R - 1;
            q.slots = static_cast<u64*>(dalloc(H, R * 8));
            return q.slots != nullptr;
        }
        if (flavor == FL_VA) {
            q.D = (u32)((cap + S_va - 1) / S_va + 2);
            q.dir = static_cast<u64*>(dalloc(H, (size_t)q.D * 8));
            q.dcnt = static_cast<u32*>(dalloc(H, (size_t)q.D * 4));
            return q.dir && q.dcnt;
        }
        // VirtualList creation ring: at least twice the segments that the tickets
        // of every resident thread (< 2^19 on B200) can span, so a ring entry
        // outlives the enqueuers of its segment (256 at 64 KiB chunks; 16 Ki
        // entries at 1 KiB chunks, where thousands of segments are in flight).
        const u64 R = std::max<u64>(OURO_VL_RECENT, next_pow2(2 * ((1ull << 19) / S_vl + 2)));
        q.vl_rmask = R - 1;
        q.vl_recent = static_cast<u64*>(dalloc(H, R * 8));
        return q.vl_recent != nullptr;
    };
    const u32 fl = H->cfg.queue_flavor;
    if (H->cfg.allocator_kind == OURO_KIND_PAGE) {
        u32 at = 0;
        for (u32 k = 0; k < K; ++k) {
            H->pq_n[k] = N / K + (k == 0 ? N % K : 0);
            H->pq_start[k] = at;
            at += H->pq_n[k];
        }
        for (u32 k = 0; k < K; ++k) {
            const u64 ppc = g.ppc(k);
            u32 s = 0;
            if (fl != FL_ARRAY) {  // gap G1: self-hosted segment reserve
                const u64 Sx = fl == FL_VA ? S_va : S_vl;
                for (s = 0; s <= H->pq_n[k]; ++s) {
                    const u64 cap = (u64)(H->pq_n[k] - s) * ppc;
                    const u64 need = cap == 0 ? 0 : (cap + Sx - 1) / Sx + 2;
                    if (need <= s) break;
                }
            }
            H->pq_s[k] = s;
            const u64 cap = (u64)(H->pq_n[k] - s) * ppc;
            if (fl == FL_ARRAY) {
                if (!init_q(H->hq[k], FL_ARRAY, cap, -1)) return OURO_ERR_CUDA;
            } else {
                if (!init_q(H->hq[K + 1 + k], FL_ARRAY, std::max<u32>(s, 1), -1)) return OURO_ERR_CUDA;
                if (!init_q(H->hq[k], fl, cap, (int)(K + 1 + k))) return OURO_ERR_CUDA;
            }
        }
        if (!init_q(H->hq[K], FL_ARRAY, 1, -1)) return OURO_ERR_CUDA;
        H->d_pq = static_cast<u32*>(dalloc(H, 3 * K * 4));
        if (!H->d_pq) return OURO_ERR_CUDA;
    } else {
        if (!init_q(H->hq[K], FL_ARRAY, N, -1)) return OURO_ERR_CUDA;
        for (u32 k = 0; k < K; ++k)
            if (!init_q(H->hq[k], fl, 2ull * N, (int)K)) return OURO_ERR_CUDA;
        H->floor_F = fl == FL_ARRAY ? 0 : (int64_t)std::min<u32>(K, N / 8);
    }
    return OURO_OK;
}

// (Re)initialise all contents: freshly constructed heap.
ouro_status fill(ouro_heap* H, cudaStream_t st) {
    const Geometry& g = H->g;
    const u32 N = g.N, K = g.K;
    const u32 fl = H->cfg.queue_flavor;
    const u64 S_va = g.chunk / 8, S_vl = g.chunk / 8 - 2;
    CK(cudaMemsetAsync(H->d_meta, 0, (size_t)N * 8, st));
    CK(cudaMemsetAsync(H->d_bitmap, 0, (size_t)N * g.Wmax * 8, st));
    CK(cudaMemsetAsync(H->d_assigned, 0, (size_t)K * 4, st));
    CK(cudaMemsetAsync(H->d_ctr, 0, (size_t)OURO_CTR_SHARDS * (2 * K + OURO_CTR_N) * 8, st));
    CK(cudaMemsetAsync(H->d_sticky, 0, 8, st));
    CK(cudaMemsetAsync(H->d_sm_hint, 0, kSmHintBytes, st));
    if (H->d_touched) CK(cudaMemsetAsync(H->d_touched, 0, g.heap / g.minp / 8 + 8, st));
    for (auto& q : H->hq) {
        q.count = 0; q.head = 0; q.tail = 0; q.seg_live = 0; q.seg_hwm = 0;
        q.vl_head = q.vl_tail = ((u64)0 << 32) | NONE;
        for (auto& r : q.vl_deq) r = NONE_LINK;
        q.vl_front = 0;
        if (q.flavor == FL_VL && q.vl_recent) CK(cudaMemsetAsync(q.vl_recent, 0xFF, (q.vl_rmask + 1) * 8, st));
    }
    auto ring_fill = [&](ouro_queue_dev& q, u64 cap, int mode, u32 first, u32 ppc) -> ouro_status {
        const u64 R = q.ring_mask + 1;
        k_fill_ring<<<std::min<u64>((R + kBlock - 1) / kBlock, 148 * 64), kBlock, 0, st>>>(q.slots, R, cap, mode, first, ppc, g.page_bits);
        CK(cudaGetLastError());
        q.count = (int64_t)cap;
        q.tail = cap;
        return OURO_OK;
    };
    auto dir_init = [&](ouro_queue_dev& q, u32 m, u32 seg0) -> ouro_status {
        std::vector<u64> dir(q.D);
        for (u32 i = 0; i < q.D; ++i) dir[i] = ((u64)i << 32) | (i < m ? seg0 + i : NONE);
        CK(cudaMemcpyAsync(q.dir, dir.data(), (size_t)q.D * 8, cudaMemcpyHostToDevice, st));
        CK(cudaMemsetAsync(q.dcnt, 0, (size_t)q.D * 4, st));
        CK(cudaStreamSynchronize(st));
        return OURO_OK;
    };
    if (H->cfg.allocator_kind == OURO_KIND_PAGE) {
        std::vector<u32> pq(3 * K);
        for (u32 k = 0; k < K; ++k) { pq[k] = H->pq_start[k]; pq[K + k] = H->pq_n[k]; pq[2 * K + k] = H->pq_s[k]; }
        CK(cudaMemcpyAsync(H->d_pq, pq.data(), 3 * K * 4, cudaMemcpyHostToDevice, st));
        k_init_pq_chunks<<<grid_for(N), kBlock, 0, st>>>(H->view, H->d_pq);
        CK(cudaGetLastError());
        for (u32 k = 0; k < K; ++k) {
            const u32 ppc = g.ppc(k);
            const u32 s = H->pq_s[k];
            const u64 cap = (u64)(H->pq_n[k] - s) * ppc;
            const u32 first = H->pq_start[k] + s;
            if (fl == FL_ARRAY) {
                if (ring_fill(H->hq[k], cap, 1, first, ppc) != OURO_OK) return OURO_ERR_CUDA;
                continue;
            }
            ouro_queue_dev& q = H->hq[k];
            ouro_queue_dev& P = H->hq[K + 1 + k];
            const u64 Sx = fl == FL_VA ? S_va : S_vl;
            const u32 m = (u32)((cap + Sx - 1) / Sx);
            const u32 seg0 = H->pq_start[k];
            // every segment chunk of the class, prefilled or in the private pool, starts
            // zeroed: recycled ones are never zeroed again (seg_acquire_zero)
            if (s) CK(cudaMemsetAsync(H->d_heap + ((u64)seg0 << g.chunk_shift), 0, (size_t)s << g.chunk_shift, st));
            if (cap) {
                k_fill_segments<<<std::min<u64>((cap + kBlock - 1) / kBlock, 148 * 64), kBlock, 0, st>>>(
                    H->d_heap, g.chunk_shift, seg0, Sx, fl == FL_VA ? 0 : 2, cap, first, ppc, g.page_bits);
                CK(cudaGetLastError());
            }
            q.count = (int64_t)cap;
            q.tail = cap;
            q.seg_live = q.seg_hwm = m;
            if (fl == FL_VA) {
                if (dir_init(q, m, seg0) != OURO_OK) return OURO_ERR_CUDA;
            } else if (m) {
                k_vl_headers<<<grid_for(m), kBlock, 0, st>>>(H->d_heap, g.chunk_shift, seg0, m);
                CK(cudaGetLastError());
                q.vl_head = ((u64)0 << 32) | seg0;
                q.vl_tail = ((u64)(m - 1) << 32) | (seg0 + m - 1);
                const u64 R = q.vl_rmask + 1;
                std::vector<u64> ring(R, NONE_LINK);
                for (u64 i = m > R ? m - R : 0; i < m; ++i) ring[i & q.vl_rmask] = (i << 32) | (seg0 + i);
                CK(cudaMemcpyAsync(q.vl_recent, ring.data(), R * 8, cudaMemcpyHostToDevice, st));
                CK(cudaStreamSynchronize(st));
                for (u32 i = 0; i < std::min<u32>(m, OURO_VL_RECENT); ++i)
                    q.vl_deq[i] = ((u64)i << 32) | (seg0 + i);
                q.vl_front = std::min<u32>(m, OURO_VL_RECENT) - 1;
            }
            // private segment pool: reserve chunks not used by the prefill
            std::vector<u64> ps(P.ring_mask + 1, 0);
            for (u32 i = m; i < s; ++i) ps[i - m] = (1ull << 32) | (seg0 + i);
            CK(cudaMemcpyAsync(P.slots, ps.data(), ps.size() * 8, cudaMemcpyHostToDevice, st));
            CK(cudaStreamSynchronize(st));
            P.count = (int64_t)(s - m);
            P.tail = s - m;
        }
        if (ring_fill(H->hq[K], 0, 0, 0, 1) != OURO_OK) return OURO_ERR_CUDA;
    } else {
        if (ring_fill(H->hq[K], N, 0, 0, 1) != OURO_OK) return OURO_ERR_CUDA;
        for (u32 k = 0; k < K; ++k) {
            ouro_queue_dev& q = H->hq[k];
            if (fl == FL_ARRAY) CK(cudaMemsetAsync(q.slots, 0, (q.ring_mask + 1) * 8, st));
            else if (fl == FL_VA && dir_init(q, 0, 0) != OURO_OK) return OURO_ERR_CUDA;
        }
    }
    CK(cudaMemcpyAsync(H->d_q, H->hq.data(), H->nq * sizeof(ouro_queue_dev), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    return OURO_OK;
}

void make_view(ouro_heap* H) {
    const Geometry& g = H->g;
    ouro_heap_view& v = H->view;
    std::memset(&v, 0, sizeof(v));
    v.base = H->d_heap;
    v.meta = H->d_meta;
    v.bitmap = H->d_bitmap;
    v.assigned = H->d_assigned;
    v.q = H->d_q;
    v.ctr = H->d_ctr;
    v.sticky = H->d_sticky;
    v.sm_hint = H->d_sm_hint;
    v.heap_bytes = g.heap;
    v.chunk_bytes = g.chunk;
    v.S_va = g.chunk / 8;
    v.S_vl = g.chunk / 8 - 2;
    v.floor_F = H->floor_F;
    v.spin_limit = 1ull << 22;
    v.N = g.N;
    v.K = g.K;
    v.page_bits = g.page_bits;
    v.chunk_bits = g.chunk_bits;
    v.chunk_shift = g.chunk_shift;
    v.min_shift = g.min_shift;
    v.Wmax = g.Wmax;
    v.gmask = g.gmask;
    v.cmask = g.cmask;
    v.kind = H->cfg.allocator_kind;
    v.flavor = H->cfg.queue_flavor;
    v.backoff = H->cfg.backoff;
    v.max_retries = H->cfg.max_retries;
    v.sleep_base_ns = H->cfg.sleep_base_ns;
    v.sleep_cap_ns = H->cfg.sleep_cap_ns;
    v.checks = 0;
    if (H->cfg.allocator_kind == OURO_KIND_PAGE) {
        v.pq_n0 = H->pq_n.empty() ? g.N : H->pq_n[0];
        v.pq_q = g.N / g.K;
        for (u32 k = 0; k < g.K && k < 32; ++k) v.pq_s[k] = H->pq_s[k];
    }
}

// Quiescent canonical digest + per-class recount (device passes, host finish).
ouro_status compute_digest(ouro_heap* H, ouro_digest* out, DigestDev* hd_out, std::vector<ouro_queue_dev>* qs_out,
                           cudaStream_t st) {
    const Geometry& g = H->g;
    const u32 N = g.N, K = g.K;
    DevBuf d_buf, where_buf, entries_buf;
    CK(d_buf.alloc(sizeof(DigestDev)));
    CK(where_buf.alloc((size_t)N * 4));
    CK(entries_buf.alloc((size_t)N * 4));
    DigestDev* d = d_buf.as<DigestDev>();
    u32* where = where_buf.as<u32>();
    u32* entries = entries_buf.as<u32>();
    CK(cudaMemsetAsync(d, 0, sizeof(DigestDev), st));
    CK(cudaMemsetAsync(where, 0, (size_t)N * 4, st));
    CK(cudaMemsetAsync(entries, 0, (size_t)N * 4, st));
    std::vector<ouro_queue_dev> qs(H->nq);
    CK(cudaMemcpyAsync(qs.data(), H->d_q, H->nq * sizeof(ouro_queue_dev), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    k_digest_headers<<<grid_for(N), kBlock, 0, st>>>(H->view, d, where);
    CK(cudaGetLastError());
    std::vector<u32> host_where_add(N, 0);
    bool host_bad = false;
    const u64 S_va = g.chunk / 8, S_vl = g.chunk / 8 - 2;
    // segment table of a quiescent virtual queue (seq-indexed chunk ids)
    auto segtab_of = [&](const ouro_queue_dev& q, std::vector<u32>& tab, u64& first) -> ouro_status {
        tab.clear();
        first = 0;
        if (q.flavor == FL_ARRAY || q.tail == q.head) return OURO_OK;
        const u64 Sx = q.flavor == FL_VA ? S_va : S_vl;
        const u64 s0 = q.head / Sx, s1 = (q.tail - 1) / Sx;
        first = s0;
        tab.assign(s1 - s0 + 1, NONE);
        if (q.flavor == FL_VA) {
            std::vector<u64> dir(q.D);
            CK(cudaMemcpy(dir.data(), q.dir, (size_t)q.D * 8, cudaMemcpyDeviceToHost));
            for (u64 s = s0; s <= s1; ++s) {
                const u64 e = dir[s % q.D];
                if ((u32)(e >> 32) == (u32)s) tab[s - s0] = (u32)e;
            }
        } else {
            u32 cur = (u32)q.vl_head;
            u32 i = (u32)(q.vl_head >> 32);
            u64 guard = 0;
            while (cur != NONE && guard++ < (1ull << 26)) {
                const u64 s = s0 + (u32)(i - (u32)s0);
                if (s > s1) break;
                if (s >= s0) tab[s - s0] = cur;
                u64 nx;
                CK(cudaMemcpy(&nx, H->d_heap + ((u64)cur << g.chunk_shift), 8, cudaMemcpyDeviceToHost));
                cur = nx == NONE_LINK ? NONE : (u32)nx;
                ++i;
            }
        }
        return OURO_OK;
    };
    auto count_segments = [&](const ouro_queue_dev& q) -> ouro_status {
        if (q.flavor == FL_VA) {
            std::vector<u64> dir(q.D);
            CK(cudaMemcpy(dir.data(), q.dir, (size_t)q.D * 8, cudaMemcpyDeviceToHost));
            for (u32 i = 0; i < q.D; ++i)
                if ((u32)dir[i] != NONE) { if ((u32)dir[i] < N) host_where_add[(u32)dir[i]]++; else host_bad = true; }
        } else if (q.flavor == FL_VL) {
            u32 cur = (u32)q.vl_head;
            u64 guard = 0;
            while (cur != NONE && guard++ < (1ull << 26)) {
                if (cur < N) host_where_add[cur]++; else { host_bad = true; break; }
                u64 nx;
                CK(cudaMemcpy(&nx, H->d_heap + ((u64)cur << g.chunk_shift), 8, cudaMemcpyDeviceToHost));
                cur = nx == NONE_LINK ? NONE : (u32)nx;
            }
        }
        return OURO_OK;
    };
    auto run_queue = [&](u32 qi, int mode, u32 k) -> ouro_status {
        const ouro_queue_dev& q = qs[qi];
        const u64 n = q.tail - q.head;
        if (n == 0) return OURO_OK;
        std::vector<u32> tab;
        u64 first;
        if (segtab_of(q, tab, first) != OURO_OK) return OURO_ERR_CUDA;
        DevBuf dtab_buf;
        u32* dtab = nullptr;
        if (!tab.empty()) {
            CK(dtab_buf.alloc(tab.size() * 4));
            dtab = dtab_buf.as<u32>();
            CK(cudaMemcpy(dtab, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice));
        }
        k_digest_queue<<<(unsigned)std::min<u64>((n + kBlock - 1) / kBlock, 148 * 32), kBlock, 0, st>>>(
            H->view, H->d_q + qi, dtab, first, mode, k, d, where, entries);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(st));
        return OURO_OK;
    };
    if (H->cfg.allocator_kind == OURO_KIND_CHUNK) {
        if (run_queue(K, 0, 0) != OURO_OK) return OURO_ERR_CUDA;
        for (u32 k = 0; k < K; ++k) {
            if (count_segments(qs[k]) != OURO_OK) return OURO_ERR_CUDA;
            if (run_queue(k, 2, k) != OURO_OK) return OURO_ERR_CUDA;
        }
    } else {
        for (u32 k = 0; k < K; ++k) {
            if (H->cfg.queue_flavor != FL_ARRAY) {
                if (count_segments(qs[k]) != OURO_OK) return OURO_ERR_CUDA;
                if (run_queue(K + 1 + k, 0, 0) != OURO_OK) return OURO_ERR_CUDA;
            }
            if (run_queue(k, 1, k) != OURO_OK) return OURO_ERR_CUDA;
        }
    }
    DigestDev hd;
    std::vector<u32> hw(N), he(N);
    std::vector<u64> meta(N);
    CK(cudaMemcpyAsync(&hd, d, sizeof(hd), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hw.data(), where, (size_t)N * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(he.data(), entries, (size_t)N * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(meta.data(), H->d_meta, (size_t)N * 8, cudaMemcpyDeviceToHost, st));
    u32 sticky[2];
    CK(cudaMemcpyAsync(sticky, H->d_sticky, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    bool ok = hd.bad == 0 && !host_bad;
    const bool dbg = std::getenv("OURO_DIGEST_DEBUG") != nullptr;
    if (dbg && !ok) std::fprintf(stderr, "digest: dev bad %u host_bad %d\n", (unsigned)hd.bad, (int)host_bad);
    int shown = 0;
    for (u32 c = 0; c < N; ++c) {
        if (hw[c] + host_where_add[c] != 1) {
            ok = false;
            if (dbg && shown++ < 16)
                std::fprintf(stderr, "digest: chunk %u where %u segments %u meta %016llx\n", c, hw[c],
                             host_where_add[c], (unsigned long long)meta[c]);
        }
        if (H->cfg.allocator_kind == OURO_KIND_CHUNK) {
            const u32 s8 = (u32)(meta[c] >> 32) & 0xFF;
            const bool has_free = s8 >= 1 && s8 <= K && (u32)meta[c] > 0;
            if (he[c] != (has_free ? 1u : 0u)) ok = false;
        }
    }
    std::memset(out, 0, sizeof(*out));
    out->num_chunks = N;
    out->num_classes = K;
    out->partition_ok = ok ? 1 : 0;
    out->sticky_mask = sticky[1];
    out->live_pages = hd.live_pages;
    out->unassigned_chunks = N - hd.assigned_total;
    out->header_hash = hd.header_hash;
    out->queue_hash = hd.queue_hash;
    for (u32 k = 0; k < K; ++k) {
        out->class_chunks[k] = hd.class_chunks[k];
        out->class_queued_live[k] = hd.class_queued_live[k];
        out->class_live_pages[k] = hd.class_live_pages[k];
    }
    if (hd_out) *hd_out = hd;
    if (qs_out) *qs_out = qs;
    return OURO_OK;
}

}  // namespace

// =================================================================== C ABI ====
extern "C" {

ouro_status ouro_heap_create(const ouro_config* cfg, int device, ouro_heap** out) {
    if (!cfg || !out) return OURO_ERR_USAGE;
    ouro_host::Geometry g;
    if (ouro_host::geometry(cfg, &g) != OURO_OK) return OURO_ERR_CONFIG;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || ndev <= device) return OURO_ERR_CUDA;
    DeviceGuard dev_guard_(device);  // the caller's current device is restored on return
    if (!dev_guard_.ok) return OURO_ERR_CUDA;
    auto* H = new ouro_heap();
    H->cfg = *cfg;
    H->g = g;
    H->device = device;
    H->op_block = g_def_block.load();
    H->op_waves = g_def_waves.load();
    auto fail = [&](ouro_status s) { ouro_heap_destroy(H); return s; };
    H->d_heap = static_cast<uint8_t*>(dalloc(H, g.heap));
    H->d_meta = static_cast<u64*>(dalloc(H, (size_t)g.N * 8));
    H->d_bitmap = static_cast<u64*>(dalloc(H, (size_t)g.N * g.Wmax * 8));
    H->d_assigned = static_cast<u32*>(dalloc(H, (size_t)g.K * 4));
    H->d_ctr = static_cast<u64*>(dalloc(H, (size_t)OURO_CTR_SHARDS * (2 * g.K + OURO_CTR_N) * 8));
    H->d_sticky = static_cast<u32*>(dalloc(H, 8));
    H->d_sm_hint = static_cast<u64*>(dalloc(H, kSmHintBytes));
    if (!H->d_heap || !H->d_meta || !H->d_bitmap || !H->d_assigned || !H->d_ctr || !H->d_sticky || !H->d_sm_hint)
        return fail(OURO_ERR_CUDA);
    if (plan(H) != OURO_OK) return fail(OURO_ERR_CUDA);
    H->d_q = static_cast<ouro_queue_dev*>(dalloc(H, H->nq * sizeof(ouro_queue_dev)));
    if (!H->d_q) return fail(OURO_ERR_CUDA);
    make_view(H);
    const ouro_status s = fill(H, 0);
    if (s != OURO_OK) return fail(s);
    *out = H;
    return OURO_OK;
}

ouro_status ouro_heap_destroy(ouro_heap* H) {
    if (!H) return OURO_ERR_USAGE;
    DeviceGuard dev_guard_(H->device);
    for (void* p : H->owned) cudaFree(p);
    if (H->d_touched) cudaFree(H->d_touched);
    delete H;
    return OURO_OK;
}

ouro_status ouro_heap_reset(ouro_heap* H, void* stream) {
    if (!H) return OURO_ERR_USAGE;
    OURO_BIND(H);
    CK(cudaStreamSynchronize(S(stream)));
    return fill(H, S(stream));
}

size_t ouro_heap_view_size(void) { return sizeof(ouro_heap_view); }

ouro_status ouro_set_launch_shape(int block_threads, int waves) {
    if (block_threads < 32 || block_threads > kBlock || block_threads % 32 || waves < 0) return OURO_ERR_USAGE;
    g_def_block = block_threads;
    g_def_waves = waves;
    return OURO_OK;
}

ouro_status ouro_heap_set_launch_shape(ouro_heap* H, int block_threads, int waves) {
    if (!H || block_threads < 32 || block_threads > kBlock || block_threads % 32 || waves < 0) return OURO_ERR_USAGE;
    H->op_block = block_threads;
    H->op_waves = waves;
    return OURO_OK;
}

ouro_status ouro_heap_set_checks(ouro_heap* H, int on) {
    if (!H) return OURO_ERR_USAGE;
    H->view.checks = on ? 1u : 0u;
    return OURO_OK;
}

ouro_status ouro_heap_set_spin_limit(ouro_heap* H, uint64_t limit) {
    if (!H || limit == 0) return OURO_ERR_USAGE;
    H->view.spin_limit = limit;
    return OURO_OK;
}

ouro_status ouro_heap_debug_add_count(ouro_heap* H, uint32_t qi, int64_t delta) {
    if (!H || qi >= H->nq) return OURO_ERR_USAGE;
    OURO_BIND(H);
    CK(cudaDeviceSynchronize());
    int64_t c;
    CK(cudaMemcpy(&c, &(H->d_q + qi)->count, 8, cudaMemcpyDeviceToHost));
    c += delta;
    CK(cudaMemcpy(&(H->d_q + qi)->count, &c, 8, cudaMemcpyHostToDevice));
    return OURO_OK;
}

ouro_status ouro_heap_get_view(const ouro_heap* H, void* out, size_t size) {
    if (!H || !out || size < sizeof(ouro_heap_view)) return OURO_ERR_USAGE;
    std::memcpy(out, &H->view, sizeof(ouro_heap_view));
    return OURO_OK;
}

ouro_status ouro_heap_config(const ouro_heap* H, ouro_config* cfg, ouro_geometry* geo) {
    if (!H) return OURO_ERR_USAGE;
    if (cfg) *cfg = H->cfg;
    if (geo) return ouro_config_geometry(&H->cfg, geo);
    return OURO_OK;
}

uint64_t ouro_heap_base(const ouro_heap* H) { return H ? (uint64_t)(uintptr_t)H->d_heap : 0; }

ouro_status ouro_page_region(ouro_heap* H, uint32_t h, uint64_t* offset, uint64_t* len) {
    if (!H) return OURO_ERR_USAGE;
    const Geometry& g = H->g;
    const u64 c = (u64)h >> g.page_bits;
    const u32 p = h & ((1u << g.page_bits) - 1u);
    if (c >= g.N) return OURO_ERR_RANGE;
    OURO_BIND(H);
    u64 m;
    CK(cudaMemcpy(&m, H->d_meta + c, 8, cudaMemcpyDeviceToHost));
    const u32 st = (u32)(m >> 32) & 0xFF;
    if (st == 0 || st == 0xFF || st > g.K) return OURO_ERR_INVALID_HANDLE;
    const u32 k = st - 1;
    if (p >= g.ppc(k)) return OURO_ERR_INVALID_HANDLE;
    *offset = (c << g.chunk_shift) + ((u64)p << (g.min_shift + k));
    *len = g.page_bytes(k);
    return OURO_OK;
}

ouro_status ouro_heap_last_error(ouro_heap* H, uint32_t* first, uint32_t* mask, int clear) {
    if (!H) return OURO_ERR_USAGE;
    OURO_BIND(H);
    u32 s[2];
    CK(cudaMemcpy(s, H->d_sticky, 8, cudaMemcpyDeviceToHost));
    if (first) *first = s[0];
    if (mask) *mask = s[1];
    if (clear) CK(cudaMemset(H->d_sticky, 0, 8));
    return OURO_OK;
}

ouro_status ouro_heap_digest(ouro_heap* H, ouro_digest* out, void* stream) {
    if (!H || !out) return OURO_ERR_USAGE;
    OURO_BIND(H);
    CK(cudaStreamSynchronize(S(stream)));
    return compute_digest(H, out, nullptr, nullptr, S(stream));
}

ouro_status ouro_heap_queue_links(ouro_heap* H, uint32_t qi, uint64_t out[4]) {
    if (!H || !out || qi >= H->nq) return OURO_ERR_USAGE;
    OURO_BIND(H);
    CK(cudaDeviceSynchronize());
    const ouro_queue_dev* q = H->d_q + qi;
    CK(cudaMemcpy(&out[0], &q->count, 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&out[1], &q->head, 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&out[2], &q->vl_head, 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&out[3], &q->vl_tail, 8, cudaMemcpyDeviceToHost));
    return OURO_OK;
}

ouro_status ouro_heap_vl_ring(ouro_heap* H, uint32_t qi, uint64_t out[OURO_VL_RECENT]) {
    if (!H || !out || qi >= H->nq) return OURO_ERR_USAGE;
    OURO_BIND(H);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(out, &(H->d_q + qi)->vl_deq[0], 8 * OURO_VL_RECENT, cudaMemcpyDeviceToHost));
    return OURO_OK;
}

ouro_status ouro_heap_stats(ouro_heap* H, ouro_stats* out, void* stream) {
    if (!H || !out) return OURO_ERR_USAGE;
    OURO_BIND(H);
    CK(cudaStreamSynchronize(S(stream)));
    ouro_digest dg;
    DigestDev hd;
    std::vector<ouro_queue_dev> qs;
    const ouro_status s = compute_digest(H, &dg, &hd, &qs, S(stream));
    if (s != OURO_OK) return s;
    const Geometry& g = H->g;
    const size_t per = 2 * g.K + OURO_CTR_N;
    std::vector<u64> shards(OURO_CTR_SHARDS * per), ctr(per, 0);
    u32 sticky[2];
    CK(cudaMemcpy(shards.data(), H->d_ctr, shards.size() * 8, cudaMemcpyDeviceToHost));
    for (size_t s = 0; s < OURO_CTR_SHARDS; ++s)
        for (size_t i = 0; i < per; ++i) ctr[i] += shards[s * per + i];
    CK(cudaMemcpy(sticky, H->d_sticky, 8, cudaMemcpyDeviceToHost));
    std::memset(out, 0, sizeof(*out));
    out->num_classes = g.K;
    out->num_chunks = g.N;
    out->sticky_first = sticky[0];
    out->sticky_mask = sticky[1];
    const u64* c = ctr.data() + 2 * g.K;
    out->stale_drops = c[OURO_CTR_STALE];
    out->double_frees = c[OURO_CTR_DOUBLE_FREE];
    out->invalid_frees = c[OURO_CTR_INVALID_FREE];
    out->bad_sizes = c[OURO_CTR_BAD_SIZE];
    out->timeouts = c[OURO_CTR_TIMEOUT];
    out->corruptions = c[OURO_CTR_CORRUPTION];
    if (H->cfg.allocator_kind == OURO_KIND_CHUNK) out->pool_len = (u64)qs[g.K].count;
    for (u32 k = 0; k < g.K; ++k) {
        ouro_class_stats& cs = out->cls[k];
        cs.page_bytes = g.page_bytes(k);
        cs.pages_per_chunk = g.ppc(k);
        cs.chunks = hd.class_chunks[k];
        cs.live_pages = hd.class_live_pages[k];
        cs.queue_len = (u64)qs[k].count;
        cs.queued_live = hd.class_queued_live[k];
        cs.seg_live = qs[k].seg_live;
        cs.seg_hwm = qs[k].seg_hwm;
        cs.retries = ctr[k];
        cs.ooms = ctr[g.K + k];
    }
    return OURO_OK;
}

ouro_status ouro_launch_alloc(ouro_heap* H, uint64_t n, uint64_t uniform_bytes, const uint32_t* d_sizes, void** d_out,
                              void* stream) {
    if (!H || !d_out) return OURO_ERR_USAGE;
    if (n == 0) return OURO_OK;
    OURO_BIND(H);
    OURO_VSWITCH(H, launch_alloc, H, n, uniform_bytes, d_sizes, d_out, S(stream));
    CK(cudaGetLastError());
    return OURO_OK;
}

ouro_status ouro_launch_alloc_u16(ouro_heap* H, uint64_t n, const uint16_t* d_sizes, void** d_out, void* stream) {
    if (!H || !d_out || !d_sizes) return OURO_ERR_USAGE;
    if (n == 0) return OURO_OK;
    OURO_BIND(H);
    OURO_VSWITCH(H, launch_alloc16, H, n, d_sizes, d_out, S(stream));
    CK(cudaGetLastError());
    return OURO_OK;
}

ouro_status ouro_launch_free(ouro_heap* H, uint64_t n, void* const* d_ptrs, void* stream) {
    if (!H || !d_ptrs) return OURO_ERR_USAGE;
    if (n == 0) return OURO_OK;
    OURO_BIND(H);
    OURO_VSWITCH(H, launch_free, H, n, d_ptrs, S(stream));
    CK(cudaGetLastError());
    return OURO_OK;
}

ouro_status ouro_launch_write(ouro_heap* H, uint64_t n, void* const* d_ptrs, uint64_t seed, uint32_t it, void* stream) {
    if (!H || !d_ptrs) return OURO_ERR_USAGE;
    if (n == 0) return OURO_OK;
    OURO_BIND(H);
    k_pattern<false><<<pattern_grid(n), kBlock, 0, S(stream)>>>(H->view, n, d_ptrs, seed, it, nullptr);
    CK(cudaGetLastError());
    return OURO_OK;
}

ouro_status ouro_launch_verify(ouro_heap* H, uint64_t n, void* const* d_ptrs, uint64_t seed, uint32_t it,
                               uint64_t* d_result, void* stream) {
    if (!H || !d_ptrs || !d_result) return OURO_ERR_USAGE;
    if (n == 0) return OURO_OK;
    OURO_BIND(H);
    k_pattern<true><<<pattern_grid(n), kBlock, 0, S(stream)>>>(H->view, n, d_ptrs, seed, it,
                                                              reinterpret_cast<u64*>(d_result));
    CK(cudaGetLastError());
    return OURO_OK;
}

ouro_status ouro_launch_count(ouro_heap* H, uint64_t n, void* const* d_ptrs, uint64_t* d_count, void* stream) {
    if (!H || !d_ptrs || !d_count) return OURO_ERR_USAGE;
    if (n == 0) return OURO_OK;
    OURO_BIND(H);
    k_count<<<grid_for(n), kBlock, 0, S(stream)>>>(n, d_ptrs, reinterpret_cast<u64*>(d_count));
    CK(cudaGetLastError());
    return OURO_OK;
}

ouro_status ouro_audit(ouro_heap* H, uint64_t n, void* const* d_ptrs, ouro_audit_result* out, void* stream) {
    if (!H || !d_ptrs || !out) return OURO_ERR_USAGE;
    std::memset(out, 0, sizeof(*out));
    if (n == 0) return OURO_OK;
    OURO_BIND(H);
    cudaStream_t st = S(stream);
    DevBuf offs_b, lens_b, offs2_b, lens2_b, res_b, idx_b;
    CK(offs_b.alloc(n * 8));
    CK(lens_b.alloc(n * 8));
    CK(offs2_b.alloc(n * 8));
    CK(lens2_b.alloc(n * 8));
    CK(res_b.alloc(8 * 8));
    CK(idx_b.alloc(8));
    u64 *offs = offs_b.as<u64>(), *lens = lens_b.as<u64>(), *offs2 = offs2_b.as<u64>(), *lens2 = lens2_b.as<u64>();
    u64* res = res_b.as<u64>();
    unsigned long long* idx = idx_b.as<unsigned long long>();
    CK(cudaMemsetAsync(res, 0, 64, st));
    CK(cudaMemsetAsync(idx, 0, 8, st));
    k_audit_collect<<<grid_for(n), kBlock, 0, st>>>(H->view, n, d_ptrs, offs, lens, res, idx);
    CK(cudaGetLastError());
    u64 m = 0;
    CK(cudaMemcpyAsync(&m, idx, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (m > 1) {
        size_t tb = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, offs, offs2, lens, lens2, (int)m, 0, 64, st));
        DevBuf tmp;
        CK(tmp.alloc(tb));
        CK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, offs, offs2, lens, lens2, (int)m, 0, 64, st));
        k_audit_neighbours<<<grid_for(m), kBlock, 0, st>>>(m, offs2, lens2, res);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(st));
    }
    u64 r[8];
    CK(cudaMemcpyAsync(r, res, 64, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    out->live = r[0];
    out->out_of_heap = r[1];
    out->misaligned = r[2];
    out->overlaps = r[3];
    out->not_marked = r[4];
    out->bytes = r[5];
    return OURO_OK;
}

ouro_status ouro_launch_churn(ouro_heap* H, uint64_t n, uint32_t round_begin, uint32_t rounds, uint64_t seed,
                              void** d_slots, uint64_t* d_result, void* stream) {
    if (!H || !d_slots || !d_result) return OURO_ERR_USAGE;
    OURO_BIND(H);
    if (!H->d_touched) {
        const size_t b = H->g.heap / H->g.minp / 8 + 8;
        CK(cudaMalloc(&H->d_touched, b));
        CK(cudaMemset(H->d_touched, 0, b));
    }
    for (uint32_t r = round_begin; r < round_begin + rounds; ++r) {
        OURO_VSWITCH(H, launch_churn, H, n, r, seed, d_slots, reinterpret_cast<u64*>(d_result), S(stream));
    }
    CK(cudaGetLastError());
    return OURO_OK;
}

ouro_status ouro_run_script(ouro_heap* H, const ouro_script_step* steps, uint32_t nsteps, uint64_t* out_offset,
                            int32_t* out_status) {
    if (!H || !steps || !out_offset || !out_status) return OURO_ERR_USAGE;
    OURO_BIND(H);
    DevBuf ds_b, doff_b, dst_b;
    CK(ds_b.alloc((size_t)nsteps * sizeof(ouro_script_step) + 1));
    CK(doff_b.alloc((size_t)nsteps * 32 * 8 + 8));
    CK(dst_b.alloc((size_t)nsteps * 32 * 4 + 4));
    ouro_script_step* ds = ds_b.as<ouro_script_step>();
    u64* doff = doff_b.as<u64>();
    int* dst = dst_b.as<int>();
    CK(cudaMemcpy(ds, steps, (size_t)nsteps * sizeof(ouro_script_step), cudaMemcpyHostToDevice));
    OURO_VSWITCH(H, launch_script, H, ds, nsteps, doff, dst);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(out_offset, doff, (size_t)nsteps * 32 * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(out_status, dst, (size_t)nsteps * 32 * 4, cudaMemcpyDeviceToHost));
    return OURO_OK;
}

// run_trial: host buffers in, host results out.  Every
// launcher status is checked; buffers, events and the stream are released on
// every return path.
ouro_status ouro_run_trial(ouro_heap* H, const ouro_trial_config* tc, ouro_trial_result* out) {
    if (!H || !tc || !out) return OURO_ERR_USAGE;
    if (tc->iterations < 2 || tc->iterations > 64 || tc->num_allocations == 0) return OURO_ERR_USAGE;
    OURO_BIND(H);
    std::memset(out, 0, sizeof(*out));
    const u64 n = tc->num_allocations;
    Stream stream;
    CK(cudaStreamCreateWithFlags(&stream.s, cudaStreamNonBlocking));
    cudaStream_t st = stream.s;
    DevBuf ptrs_b, dsz_b, dres_b;
    CK(ptrs_b.alloc(n * sizeof(void*)));
    if (tc->sizes) CK(dsz_b.alloc(n * 4));
    CK(dres_b.alloc(4 * 8));
    void** ptrs = ptrs_b.as<void*>();
    u32* dsz = tc->sizes ? dsz_b.as<u32>() : nullptr;
    u64* dres = dres_b.as<u64>();
    Events evs;
    CK(evs.create(5));
    cudaEvent_t* ev = evs.ev.data();
    bool verified = true;
#define OURO_TRY(x)                                  \
    do {                                             \
        const ouro_status s_ = (x);                  \
        if (s_ != OURO_OK) return s_;                \
    } while (0)
    for (u32 it = 0; it < tc->iterations; ++it) {
        const u64 init[4] = {0, ~0ull, 0, 0};
        CK(cudaMemcpyAsync(dres, init, 32, cudaMemcpyHostToDevice, st));
        CK(cudaEventRecord(ev[0], st));
        if (tc->sizes) CK(cudaMemcpyAsync(dsz, tc->sizes, n * 4, cudaMemcpyHostToDevice, st));
        OURO_TRY(ouro_launch_alloc(H, n, tc->allocation_bytes, dsz, ptrs, st));
        CK(cudaEventRecord(ev[1], st));
        OURO_TRY(ouro_launch_write(H, n, ptrs, tc->seed, it, st));
        CK(cudaEventRecord(ev[2], st));
        OURO_TRY(ouro_launch_verify(H, n, ptrs, tc->seed, it, reinterpret_cast<uint64_t*>(dres), st));
        OURO_TRY(ouro_launch_count(H, n, ptrs, reinterpret_cast<uint64_t*>(dres + 2), st));
        CK(cudaEventRecord(ev[3], st));
        OURO_TRY(ouro_launch_free(H, n, ptrs, st));
        CK(cudaEventRecord(ev[4], st));
        u64 r[4];
        CK(cudaMemcpyAsync(r, dres, 32, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        float a, w, vv, f;
        CK(cudaEventElapsedTime(&a, ev[0], ev[1]));
        CK(cudaEventElapsedTime(&w, ev[1], ev[2]));
        CK(cudaEventElapsedTime(&vv, ev[2], ev[3]));
        CK(cudaEventElapsedTime(&f, ev[3], ev[4]));
        out->alloc_ms[it] = a;
        out->write_ms[it] = w;
        out->verify_ms[it] = vv;
        out->free_ms[it] = f;
        out->ok_allocs += r[2];
        out->failed_allocs += n - r[2];
        if (r[0] != 0) verified = false;
    }
#undef OURO_TRY
    out->iterations = tc->iterations;
    out->verified = verified ? 1 : 0;
    ouro_trial_means(out->alloc_ms, tc->iterations, &out->mean_all_ms, &out->mean_subsequent_ms);
    double fa;
    ouro_trial_means(out->free_ms, tc->iterations, &fa, &out->mean_subsequent_free_ms);
    out->h2d_bytes = tc->sizes ? n * 4 : 0;
    out->d2h_bytes = 32;
    return OURO_OK;
}

ouro_status ouro_atomic_peak(int device, int mode, double* ops_per_s) {
    if (!ops_per_s) return OURO_ERR_USAGE;
    DeviceGuard dev_guard_(device);
    if (!dev_guard_.ok) return OURO_ERR_CUDA;
    const u64 words = 1ull << 22;  // 32 MiB of u64 / 16 MiB of u32 counters: L2-resident (atomics resolve in L2)
    DevBuf buf_b;
    CK(buf_b.alloc(words * 8));
    void* buf = buf_b.p;
    CK(cudaMemset(buf, 0, words * 8));
    const unsigned blocks = 148 * 8, threads = 256;
    const u32 iters = mode >= 2 ? 64 : 64;
    Events evs;
    CK(evs.create(2));
    cudaEvent_t a = evs.ev[0], b = evs.ev[1];
    auto run = [&]() {
        switch (mode) {
        case 0: k_atom_distinct32<<<blocks, threads>>>((u32*)buf, words * 2, iters); break;
        case 1: k_atom_distinct_cas64<<<blocks, threads>>>((u64*)buf, words, iters); break;
        case 2: k_atom_same_warp<<<blocks, threads>>>((u64*)buf, iters); break;
        case 4: k_hot_poll<<<148 * 6, 32>>>((const u64*)buf, 2048, (u64*)buf + 64); break;
        default: k_atom_same_lane<<<blocks, threads>>>((u64*)buf, iters / 16); break;
        }
    };
    run();
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        CK(cudaEventRecord(a));
        run();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = std::min(best, ms);
    }
    CK(cudaGetLastError());
    double ops = (double)blocks * threads * iters;
    if (mode == 2) ops /= 32.0;
    if (mode == 3) ops = (double)blocks * threads * (iters / 16);
    if (mode == 4) ops = 2048.0;  // loads of ONE poller (all 888 run concurrently): 1 / hot-word latency
    *ops_per_s = ops / (best * 1e-3);
    return OURO_OK;
}

// Event counters of an OURO_STORM_STATS=1 experiment build (zeros otherwise).
ouro_status ouro_debug_counters(uint64_t out[32], int reset) {
    std::memset(out, 0, 32 * 8);
#if OURO_STORM_STATS
    std::vector<u64> h(256 * 32);
    CK(cudaMemcpyFromSymbol(h.data(), g_storm_dbg, h.size() * 8));
    for (size_t i = 0; i < h.size(); ++i) out[i % 32] += h[i];
    if (reset) {
        std::fill(h.begin(), h.end(), 0ull);
        CK(cudaMemcpyToSymbol(g_storm_dbg, h.data(), h.size() * 8));
    }
#else
    (void)reset;
#endif
    return OURO_OK;
}

const char* ouro_build_info(void) {
    return "libouro_b200 sm_100a (" __DATE__ " " __TIME__ ")";
}

}  // extern "C"
