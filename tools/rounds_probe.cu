// rounds_probe.cu -- the allocator's own retry-round loop (ouro_dev::fail_rounds,
// include/ouro_device.cuh) driven in isolation: 4096 x 256 threads, 6 blocks/SM,
// every warp's leader runs max_retries-1 rounds against an empty queue (count = 0),
// like tools/storm_probe.cu mode 6 but with the real code.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -Iinclude -o tools/rounds_probe tools/rounds_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "ouro_device.cuh"

using namespace ouro_dev;

// storm_probe.cu mode 6's loop verbatim, on the heap's queue count
static __device__ __noinline__ u64 pump_rounds(const u64* count, u64* ent, int rounds) {
    volatile u64* ve = ent;
    bool pump = false;
    u64 last = 0, acc = 0;
    { const u64 e0 = *ve; last = (e0 >> 2) + ((e0 >> 1) & 1); }
    for (int r = 0; r < rounds; ++r) {
        asm volatile("fence.sc.cta;" ::: "memory");
        if (pump) {
            const u64 c = ld_rlx(count);
            ++last;
            *ve = (last << 2) | 2u | (c == 0 ? 1u : 0u);
            acc += c;
        } else {
            for (;;) {
                const u64 e = *ve;
                if ((e >> 2) > last) { last = e >> 2; break; }
                if (!(e & 2u)) {
                    if (atomicCAS(ent, e, e | 2u) == e) {
                        pump = true;
                        const u64 c = ld_rlx(count);
                        last = (e >> 2) + 1;
                        *ve = (last << 2) | 2u | (c == 0 ? 1u : 0u);
                        break;
                    }
                    continue;
                }
            }
        }
    }
    if (pump) *ve = (last << 2) | (*ve & 1u);
    return acc;
}

__device__ unsigned long long g_polls[4];
__shared__ unsigned int s_polls[4];
template <int V>
static __device__ __noinline__ u32 copy_loop(ouro_queue_dev* Q, u32 a, u32 maxr, u64* smh) {
    const u64 tag = poll_tag(Q);
    u64* slot = poll_slot(tag);
    u32 need = obs_need(slot, tag), fl = 1u, r, seq = 0, streak = 0, extra = 0;
    bool pump = false;
    for (;;) {
        if (++a >= maxr) { r = (a << 1) | 1u; break; }
        asm volatile("fence.sc.cta;" ::: "memory");
        if (extra) { --extra; atomicAdd(&s_polls[3], 1u); continue; }
        if (!pump) {
            for (u32 spins = 0;;) {
                const u64 e = ld_sh(slot);
                const bool mine = V == 7 ? true : tag_is(e, tag);
                if (mine && (int)(e_seq(e) - need) >= 0) {
                    fl = (u32)e & (1u | kPoolEmpty);
                    const u32 avail = e_seq(e) - need;
                    if ((fl & 1u) && e_streak(e) > avail) extra = avail;
                    need = e_seq(e) + 1u;
                    break;
                }
                if (mine && (e & kPump) && ++spins < kPumpSteal) { poll_wait(); continue; }
                seq = mine ? e_seq(e) : need - 1u;
                streak = mine && (e & 1u) ? e_streak(e) : 0u;
                if (atomicCAS(slot, e, mk_obs(seq, tag, (u32)kPump, streak)) == e) { pump = true; atomicAdd(&s_polls[1], 1u); break; }
                spins = 0;
            }
        }
        if (pump) {
            atomicAdd(&s_polls[0], 1u);
            fl = poll_load(Q, 0, nullptr, 0);
            ++seq;
            streak = (fl & 1u) ? streak + 1u : 0u;
            *reinterpret_cast<volatile u64*>(slot) = mk_obs(seq, tag, (u32)kPump | fl, streak);
            need = seq + 1u;
        }
        if (!(fl & 1u)) { r = a << 1; break; }
    }
    if (pump) *reinterpret_cast<volatile u64*>(slot) = mk_obs(seq, tag, fl, streak);
    return r;
}

// mode 3's loop shape (fixed rounds, pump decided per round) with the allocator's entry format
template <int X>
static __device__ __noinline__ u32 shape3_fmt(ouro_queue_dev* Q, int rounds) {
    const u64 tag = poll_tag(Q);
    u64* slot = poll_slot(tag);
    u32 need = obs_need(slot, tag), seq = 0, acc = 0;
    bool pump = false, done = false;
    for (int r = 0; r < rounds; ++r) {
        if (X == 2 && done) continue;
        asm volatile("fence.sc.cta;" ::: "memory");
        if (pump) {
            const u32 fl = poll_load(Q, 0, nullptr, 0);
            ++seq;
            *reinterpret_cast<volatile u64*>(slot) = mk_obs(seq, tag, (u32)kPump | fl, 0);
            need = seq + 1u;
            acc += fl;
        } else {
            for (;;) {
                const u64 e = ld_sh(slot);
                if (tag_is(e, tag) && (int)(e_seq(e) - need) >= 0) { need = e_seq(e) + 1u; acc += (u32)e & 1u; break; }
                if (!(e & kPump)) {
                    seq = e_seq(e);
                    if (atomicCAS(slot, e, mk_obs(seq, tag, (u32)kPump, 0)) == e) {
                        pump = true;
                        const u32 fl = poll_load(Q, 0, nullptr, 0);
                        ++seq;
                        *reinterpret_cast<volatile u64*>(slot) = mk_obs(seq, tag, (u32)kPump | fl, 0);
                        need = seq + 1u;
                        acc += fl;
                        break;
                    }
                }
            }
        }
        if (X == 1 && acc == 0) break;
        if (X == 2) done = acc == 0;
    }
    if (pump) *reinterpret_cast<volatile u64*>(slot) = mk_obs(seq, tag, 1u, 0);
    return acc;
}

__global__ void __launch_bounds__(256, 6) k_rounds(ouro_heap_view v, int mode) {
    if (mode == 12) {
        ouro_block_init();
        u32 r = 0;
        if (lane_id() == 0) r = shape3_fmt<2>(v.q, 62);
        r = __shfl_sync(0xFFFFFFFFu, r, 0);
        if (r == 12345) v.sticky[0] = 1;
        return;
    }
    if (mode == 11) {
        ouro_block_init();
        u32 r = 0;
        if (lane_id() == 0) r = shape3_fmt<1>(v.q, 62);
        if (lane_id() == 0 && v.max_retries == 1234) r += shape3_fmt<2>(v.q, 62);
        r = __shfl_sync(0xFFFFFFFFu, r, 0);
        if (r == 12345) v.sticky[0] = 1;
        return;
    }
    if (mode == 10) {
        ouro_block_init();
        u32 r = 0;
        if (lane_id() == 0) r = shape3_fmt<0>(v.q, 62);
        r = __shfl_sync(0xFFFFFFFFu, r, 0);
        if (r == 12345) v.sticky[0] = 1;
        return;
    }
    if (mode >= 5) {
        ouro_block_init();
        if (threadIdx.x < 4) s_polls[threadIdx.x] = 0;
        __syncthreads();
        u32 r = 0;
        if (lane_id() == 0)
            r = mode == 5 ? copy_loop<5>(v.q, 1, 64, nullptr) : mode == 7 ? copy_loop<7>(v.q, 1, 64, nullptr)
              : mode == 8 ? copy_loop<8>(v.q, 1, 64, nullptr) : copy_loop<9>(v.q, 1, 64, nullptr);
        r = __shfl_sync(0xFFFFFFFFu, r, 0);
        if (r == 12345) v.sticky[0] = 1;
        __syncthreads();
        if (threadIdx.x < 4) atomicAdd(&g_polls[threadIdx.x], s_polls[threadIdx.x]);
        return;
    }
    if (mode == 4) {
        u32 r = 0;
        if (lane_id() == 0) r = fail_rounds_loop<false, false>(v.q, nullptr, 0, 1, 64, 100, 100000, nullptr);
        r = __shfl_sync(0xFFFFFFFFu, r, 0);
        if (r == 12345) v.sticky[0] = 1;
        return;
    }
    if (mode == 3) {
        __shared__ u64 ent6;
        if (threadIdx.x == 0) ent6 = 0;
        __syncthreads();
        u64 acc = 0;
        if (lane_id() == 0) acc = pump_rounds((const u64*)&v.q->count, &ent6, 62);
        acc = __shfl_sync(0xFFFFFFFFu, acc, 0);
        if (acc == 12345) v.sticky[0] = 1;
        return;
    }
    ouro_block_init();
    const u32 lane = lane_id();
    u32 a = 1, oom = 0;
    if (mode == 1) {  // whole group: as pq_alloc calls it
        if (lane == 0) oom = fail_rounds(v, v.q, nullptr, 0, &a) ? 1u : 0u;
        oom = __shfl_sync(0xFFFFFFFFu, oom, 0);
    }
    if (oom == 12345) v.sticky[0] = oom;
}

int main() {
    ouro_heap_view v{};
    ouro_queue_dev* q;
    cudaMalloc(&q, 2 * sizeof(ouro_queue_dev));
    cudaMemset(q, 0, 2 * sizeof(ouro_queue_dev));
    u32* sticky;
    cudaMalloc(&sticky, 8);
    v.q = q;
    v.sticky = sticky;
    v.max_retries = 64;
    v.backoff = OURO_BACKOFF_FENCE;
    v.K = 1;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaFuncSetAttribute(k_rounds, cudaFuncAttributeMaxDynamicSharedMemorySize, 36 << 10);
    for (int mode : {10, 1}) {
        float best = 1e30f;
        for (int it = 0; it < 5; ++it) {
            cudaEventRecord(a);
            k_rounds<<<4096, 256, mode == 2 ? (36 << 10) : 0>>>(v, mode == 2 ? 1 : mode);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        unsigned long long gp[4] = {0, 0, 0, 0};
        cudaMemcpyFromSymbol(gp, g_polls, 32);
        static const unsigned long long z4[4] = {0, 0, 0, 0};
        cudaMemcpyToSymbol(g_polls, z4, 32);
        printf("mode %d: %.1f us %s  polls/run %llu terms %llu extra-rounds %llu\n", mode, best * 1e3,
               cudaGetErrorString(cudaGetLastError()), gp[0] / 5, gp[1] / 5, gp[2] / 5);
#if OURO_STORM_STATS
        static unsigned long long h[256 * 16], t[16];
        cudaMemcpyFromSymbol(h, g_storm_dbg, sizeof(h));
        for (int i = 0; i < 16; ++i) t[i] = 0;
        for (int i = 0; i < 256 * 16; ++i) t[i % 16] += h[i];
        const char* nm[16] = {"loops", "rounds", "polls", "taken", "polls-as-nonpump", "-", "poll-cyc", "-",
                              "-", "allspins", "lostCAS", "loop-cyc", "fence-cyc", "obs-cyc", "pump-rounds",
                              "pump-cyc"};
        for (int i = 0; i < 16; ++i) if (t[i]) printf("  %s=%llu", nm[i], t[i] / 5);
        printf("\n  cyc/round %.0f poll-cyc %.0f pump-round %.0f polls/round %.3f\n", (double)t[11] / t[1],
               (double)t[6] / t[2], (double)t[15] / (t[14] ? t[14] : 1), (double)t[2] / t[1]);
        cudaMemset(h, 0, 0);
        static unsigned long long z[256 * 16];
        cudaMemcpyToSymbol(g_storm_dbg, z, sizeof(z));
#endif
    }
    return 0;
}
