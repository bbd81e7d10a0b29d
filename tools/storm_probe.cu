// storm_probe.cu -- OOM-storm retry rounds in isolation (no allocator): 2^20
// threads (4096 x 256, 6 blocks/SM like k_alloc), every warp's leader needs
// ROUNDS retry rounds, each = backoff fence + one observation of an empty queue
// whose count word every warp would otherwise poll.  Compares how the
// observation is made:
//   mode 0  each warp loads the hot count word itself
//   mode 1  one self-elected observer warp polls the count and publishes
//           (seq, empty) to R replica lines; every other warp reads the
//           replica of its SM (seq must exceed the one its last round used)
//   mode 2  mode 1 without the per-round fence
// Prints kernel time, the number of observer terms and polls, and the floor
// ROUNDS x waves x hot-load latency for reference.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/storm_probe tools/storm_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

typedef unsigned long long u64;
typedef unsigned int u32;

__device__ __forceinline__ u64 ld_rlx(const u64* p) {
    u64 r;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(r) : "l"(p) : "memory");
    return r;
}
__device__ __forceinline__ void st_rlx(u64* p, u64 v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_weak(u64* p, u64 v) {
    asm volatile("st.global.cg.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u32 smid() { u32 r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }

constexpr int kStride = 32;  // u64 words between replicas (256 B)
struct St {
    u64 count;
    u64 pad0[31];
    u64 own;  // (last seq << 1) | owned
    u64 pad1[31];
    u64 stats[8];  // observer terms, polls, count-load cycles, observer iteration cycles, sampled spins
    u64 pad2[24];
    u64 rep[256 * kStride];
};

// mode 6 body: lane 0 alone, out of line, the other lanes parked (the allocator's shape)
static __device__ __noinline__ u64 pump_rounds(St* s, u64* ent, int rounds, int sleep_ns) {
    volatile u64* ve = ent;
    bool pump = false;
    u64 last = 0, acc = 0;
    { const u64 e0 = *ve; last = (e0 >> 2) + ((e0 >> 1) & 1); }
    for (int r = 0; r < rounds; ++r) {
        asm volatile("fence.sc.cta;" ::: "memory");
        if (pump) {
            const u64 c = ld_rlx(&s->count);
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
                        const u64 c = ld_rlx(&s->count);
                        last = (e >> 2) + 1;
                        *ve = (last << 2) | 2u | (c == 0 ? 1u : 0u);
                        break;
                    }
                    continue;
                }
                if (sleep_ns) __nanosleep(sleep_ns);
            }
        }
    }
    if (pump) *ve = (last << 2) | (*ve & 1u);
    return acc;
}

template <int MODE>
__global__ void __launch_bounds__(256, 6) k_storm(St* s, int rounds, int R, int sleep_ns) {
    const u32 lane = threadIdx.x & 31;
    if (MODE == 0) {
        u64 acc = 0;
        for (int r = 0; r < rounds; ++r) {
            asm volatile("fence.sc.cta;" ::: "memory");
            if (lane == 0) acc += ld_rlx(&s->count + (acc >> 63));
            acc = __shfl_sync(0xFFFFFFFFu, acc, 0);
        }
        if (acc == 12345) s->stats[3] = acc;
        return;
    }
    if (MODE == 6) {
        __shared__ u64 ent6;
        if (threadIdx.x == 0) ent6 = 0;
        __syncthreads();
        u64 acc = 0;
        if (lane == 0) acc = pump_rounds(s, &ent6, rounds, sleep_ns);
        acc = __shfl_sync(0xFFFFFFFFu, acc, 0);
        if (acc == 12345) s->stats[5] = acc;
        return;
    }
    if (MODE == 5) {
        __shared__ u64 ent;
        if (threadIdx.x == 0) ent = 0;
        __syncthreads();
        volatile u64* ve = &ent;
        bool pump = false;
        u64 last = 0, acc = 0, polls = 0, load_cyc = 0, iter_cyc = 0, tprev = 0;
        if (lane == 0) { const u64 e0 = *ve; last = (e0 >> 2) + ((e0 >> 1) & 1); }
        for (int r = 0; r < rounds; ++r) {
            asm volatile("fence.sc.cta;" ::: "memory");
            if (lane == 0) {
                if (pump) {
                    const u64 t = clock64();
                    if (tprev) iter_cyc += t - tprev;
                    tprev = t;
                    const u64 c = ld_rlx(&s->count);
                    load_cyc += clock64() - t;
                    ++last;
                    *ve = (last << 2) | 2u | (c == 0 ? 1u : 0u);
                    ++polls;
                    acc += c;
                } else {
                    for (;;) {
                        const u64 e = *ve;
                        if ((e >> 2) > last) { last = e >> 2; break; }
                        if (!(e & 2u)) {
                            if (atomicCAS(&ent, e, e | 2u) == e) {
                                pump = true;
                                const u64 c = ld_rlx(&s->count);
                                last = (e >> 2) + 1;
                                *ve = (last << 2) | 2u | (c == 0 ? 1u : 0u);
                                ++polls;
                                break;
                            }
                            continue;
                        }
                        if (sleep_ns) __nanosleep(sleep_ns);
                    }
                }
            }
            acc = __shfl_sync(0xFFFFFFFFu, acc, 0);
        }
        if (lane == 0 && pump) {
            *ve = (last << 2) | (*ve & 1u);  // release (pumping flag cleared)
            atomicAdd(&s->stats[0], 1ull);
            atomicAdd(&s->stats[1], polls);
            atomicAdd(&s->stats[2], load_cyc);
            atomicAdd(&s->stats[3], iter_cyc);
        }
        if (acc == 12345) s->stats[5] = acc;
        return;
    }
    u64* rp = &s->rep[(smid() % R) * kStride];
    bool obs = false;
    u64 myseq = 0, last = 0, polls = 0;
    if (lane == 0) last = (ld_rlx(rp) >> 8) + 1;  // first round: a poll issued after the next one completed
    last = __shfl_sync(0xFFFFFFFFu, last, 0);
    u64 tprev = 0, spins_tot = 0, iter_cyc = 0, load_cyc = 0, prev_e = 0;
    bool have_prev = false;
    for (int r = 0; r < rounds; ++r) {
        if (obs && lane == 0) {
            const u64 t = clock64();
            if (tprev) iter_cyc += t - tprev;
            tprev = t;
        }
        if (MODE == 1 || MODE == 3) asm volatile("fence.sc.cta;" ::: "memory");
        u64 e = 0;
        if (!obs) {
            u32 become = 0;
            if (lane == 0) {
                for (u32 spin = 1;; ++spin) {
                    e = ld_rlx(rp);
                    ++spins_tot;
                    if ((e >> 8) > last) break;
                    if (sleep_ns) __nanosleep(sleep_ns);
                    if ((spin & 7) == 0) {
                        const u64 o = ld_rlx(&s->own);
                        if (!(o & 1) && atomicCAS(&s->own, o, o | 1) == o) {
                            myseq = o >> 1;
                            become = 1;
                            break;
                        }
                    }
                }
            }
            become = __shfl_sync(0xFFFFFFFFu, become, 0);
            if (become) {
                obs = true;
                myseq = __shfl_sync(0xFFFFFFFFu, myseq, 0);
                if (lane == 0) atomicAdd(&s->stats[0], 1ull);
            }
        }
        if (obs && MODE == 4) {
            ++myseq;
            long long c = 0;
            u64 c0 = clock64();
            if (lane == 0) c = (long long)ld_rlx(&s->count);   // issued before the previous result's stores
            if (have_prev)
                for (int i = lane; i < R; i += 32) st_rlx(&s->rep[i * kStride], prev_e);
            if (lane == 0) {
                if (c != 12345) load_cyc += clock64() - c0;
                e = (myseq << 8) | (c <= 0 ? 1u : 0u);
            }
            e = __shfl_sync(0xFFFFFFFFu, e, 0);
            prev_e = e;
            have_prev = true;
            ++polls;
        } else if (obs) {
            ++myseq;
            if (lane == 0) {
                const u64 c0 = clock64();
                const long long c = (long long)ld_rlx(&s->count);
                if (c != 12345) load_cyc += clock64() - c0;
                e = (myseq << 8) | (c <= 0 ? 1u : 0u);
            }
            e = __shfl_sync(0xFFFFFFFFu, e, 0);
            if (MODE == 3) {
                for (int i = lane; i < R; i += 32) st_weak(&s->rep[i * kStride], e);
            } else {
                for (int i = lane; i < R; i += 32) st_rlx(&s->rep[i * kStride], e);
            }
            ++polls;
        }
        e = __shfl_sync(0xFFFFFFFFu, e, 0);
        last = e >> 8;
    }
    if (lane == 0 && (threadIdx.x >> 5) == 0 && (blockIdx.x & 63) == 0) atomicAdd(&s->stats[4], spins_tot);
    if (obs && MODE == 4 && have_prev)
        for (int i = lane; i < R; i += 32) st_rlx(&s->rep[i * kStride], prev_e);
    if (obs && lane == 0) {
        atomicExch(&s->own, myseq << 1);
        atomicAdd(&s->stats[1], polls);
        atomicAdd(&s->stats[2], load_cyc);
        atomicAdd(&s->stats[3], iter_cyc);
    }
}

int main(int argc, char** argv) {
    St* s;
    cudaMalloc(&s, sizeof(St));
    const int rounds = 63;
    const unsigned blocks = 4096, threads = 256;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    unsigned nb = blocks, nt = threads;
    int smem = 0;  // dynamic shared memory: 36 KiB forces 6 blocks/SM like k_alloc
    auto run = [&](int mode, int R, int sl) {
        float best = 1e30f;
        u64 st[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int it = 0; it < 5; ++it) {
            cudaMemset(s, 0, sizeof(St));
            cudaEventRecord(a);
            if (mode == 0) k_storm<0><<<nb, nt, smem>>>(s, rounds, R, sl);
            else if (mode == 1) k_storm<1><<<nb, nt, smem>>>(s, rounds, R, sl);
            else if (mode == 2) k_storm<2><<<nb, nt, smem>>>(s, rounds, R, sl);
            else if (mode == 3) k_storm<3><<<nb, nt, smem>>>(s, rounds, R, sl);
            else if (mode == 4) k_storm<4><<<nb, nt, smem>>>(s, rounds, R, sl);
            else if (mode == 5) k_storm<5><<<nb, nt, smem>>>(s, rounds, R, sl);
            else k_storm<6><<<nb, nt, smem>>>(s, rounds, R, sl);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
            cudaMemcpy(st, s->stats, 64, cudaMemcpyDeviceToHost);
        }
        cudaError_t e = cudaGetLastError();
        printf("[smem %d] [%u x %u] mode %d R %3d sleep %4d: %8.1f us  terms %llu polls %llu  count-load %llu cyc  obs-iter %llu cyc  "
               "spins/round %.2f %s\n", smem, nb, nt, mode, R, sl, best * 1e3, st[0], st[1], st[1] ? st[2] / st[1] : 0ull,
               st[1] ? st[3] / st[1] : 0ull, st[4] / (64.0 * 63.0), e == cudaSuccess ? "" : cudaGetErrorString(e));
    };
    run(0, 1, 0);
    for (int R : {32, 64, 148}) run(1, R, 0);
    run(2, 64, 0);
    run(6, 1, 0); run(6, 1, 64);
    cudaFuncSetAttribute(k_storm<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 36 << 10);
    smem = 36 << 10;
    run(6, 1, 0); run(6, 1, 64);
    return 0;
}
