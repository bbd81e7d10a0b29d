// ouro_multi.cpp -- single-process multi-device driver over the C-ABI
// (BASELINE configs[4]): one host thread per device, each with
// its own heap in its own HBM (no pointer crosses devices, so there is no
// collective and no NCCL), a host barrier before every step, CUDA events per
// device.  Aggregate = successful pairs summed over devices / the slowest
// device's alloc + free kernel time (weak scaling, max over devices).
// Uses only the public C-ABI of include/ouro.h plus the CUDA runtime.
#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/ouro.h"

namespace {

class HostBarrier {
   public:
    explicit HostBarrier(unsigned n) : n_(n) {}
    void wait() {
        std::unique_lock<std::mutex> lk(m_);
        const unsigned long long g = gen_;
        if (++waiting_ == n_) {
            waiting_ = 0;
            ++gen_;
            cv_.notify_all();
            return;
        }
        cv_.wait(lk, [&] { return gen_ != g; });
    }

   private:
    std::mutex m_;
    std::condition_variable cv_;
    unsigned n_, waiting_ = 0;
    unsigned long long gen_ = 0;
};

constexpr size_t kFlushBytes = 256u << 20;  // > the 126 MB L2: written before every timed kernel

struct DeviceRun {
    int device = 0;
    ouro_status status = OURO_OK;
    double ms = 0;          // summed alloc + free kernel time over the timed steps
    uint64_t pairs = 0;     // successful pairs over the timed steps
    uint32_t sticky = 0;
};

// One device's share: every barrier is reached even after a failure, so a
// failing device cannot deadlock the others.
void run_device(DeviceRun* R, HostBarrier* bar, const ouro_config* cfg, uint64_t n, const uint32_t* sizes,
                uint32_t nsizes, uint32_t warmup, uint32_t steps) {
    ouro_status st = OURO_OK;
    ouro_heap* H = nullptr;
    void** ptrs = nullptr;
    uint64_t* cnt = nullptr;
    void* flush = nullptr;
    cudaStream_t s = nullptr;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    auto cuda_ok = [&](cudaError_t e) {
        if (e != cudaSuccess && st == OURO_OK) st = OURO_ERR_CUDA;
        return st == OURO_OK;
    };
    if (cuda_ok(cudaSetDevice(R->device))) st = ouro_heap_create(cfg, R->device, &H);
    if (st == OURO_OK) cuda_ok(cudaMalloc(&ptrs, n * sizeof(void*)));
    if (st == OURO_OK) cuda_ok(cudaMalloc(&cnt, 8));
    if (st == OURO_OK) cuda_ok(cudaMalloc(&flush, kFlushBytes));
    if (st == OURO_OK) cuda_ok(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    for (auto& e : ev)
        if (st == OURO_OK) cuda_ok(cudaEventCreate(&e));
    bar->wait();  // every heap built
    for (uint32_t step = 0; step < warmup + steps; ++step) {
        bar->wait();  // start barrier of the step
        if (st != OURO_OK) continue;
        for (uint32_t i = 0; i < nsizes && st == OURO_OK; ++i) {
            cuda_ok(cudaMemsetAsync(cnt, 0, 8, s));
            cuda_ok(cudaMemsetAsync(flush, (int)(i & 0xFF), kFlushBytes, s));
            cuda_ok(cudaEventRecord(ev[0], s));
            if (st == OURO_OK) st = ouro_launch_alloc(H, n, sizes[i], nullptr, ptrs, s);
            cuda_ok(cudaEventRecord(ev[1], s));
            if (st == OURO_OK) st = ouro_launch_count(H, n, ptrs, cnt, s);
            cuda_ok(cudaMemsetAsync(flush, (int)((i + 1) & 0xFF), kFlushBytes, s));
            cuda_ok(cudaEventRecord(ev[2], s));
            if (st == OURO_OK) st = ouro_launch_free(H, n, ptrs, s);
            cuda_ok(cudaEventRecord(ev[3], s));
            uint64_t ok = 0;
            cuda_ok(cudaMemcpyAsync(&ok, cnt, 8, cudaMemcpyDeviceToHost, s));
            cuda_ok(cudaStreamSynchronize(s));
            float a = 0, f = 0;
            cuda_ok(cudaEventElapsedTime(&a, ev[0], ev[1]));
            cuda_ok(cudaEventElapsedTime(&f, ev[2], ev[3]));
            if (step >= warmup) {
                R->ms += (double)a + (double)f;
                R->pairs += ok;
            }
        }
    }
    if (H) {
        uint32_t first = 0, mask = 0;
        if (ouro_heap_last_error(H, &first, &mask, 0) == OURO_OK) R->sticky = first;
    }
    for (auto e : ev)
        if (e) cudaEventDestroy(e);
    if (s) cudaStreamDestroy(s);
    if (flush) cudaFree(flush);
    if (cnt) cudaFree(cnt);
    if (ptrs) cudaFree(ptrs);
    if (H) ouro_heap_destroy(H);
    R->status = st;
}

}  // namespace

extern "C" ouro_status ouro_multi_sweep(const ouro_config* cfg, uint32_t ndev, const int* devices,
                                        uint64_t threads_per_device, const uint32_t* sizes, uint32_t nsizes,
                                        uint32_t warmup, uint32_t steps, ouro_multi_result* out) {
    if (!cfg || !devices || !sizes || !out || ndev == 0 || ndev > OURO_MAX_DEVICES || nsizes == 0 ||
        threads_per_device == 0 || steps == 0)
        return OURO_ERR_USAGE;
    if (ouro_config_validate(cfg, nullptr, 0) != OURO_OK) return OURO_ERR_CONFIG;
    std::memset(out, 0, sizeof(*out));
    int caller = -1;
    cudaGetDevice(&caller);  // left untouched: the workers are separate host threads
    std::vector<DeviceRun> runs(ndev);
    HostBarrier bar(ndev);
    std::vector<std::thread> th;
    for (uint32_t d = 0; d < ndev; ++d) {
        runs[d].device = devices[d];
        th.emplace_back(run_device, &runs[d], &bar, cfg, threads_per_device, sizes, nsizes, warmup, steps);
    }
    for (auto& t : th) t.join();
    ouro_status st = OURO_OK;
    out->ndev = ndev;
    out->verified = 1;
    for (uint32_t d = 0; d < ndev; ++d) {
        if (runs[d].status != OURO_OK && st == OURO_OK) st = runs[d].status;
        if (runs[d].sticky) out->verified = 0;
        out->dev_ms[d] = runs[d].ms;
        out->dev_pairs[d] = runs[d].pairs;
        out->pairs_total += runs[d].pairs;
        out->max_ms = std::max(out->max_ms, runs[d].ms);
    }
    out->pairs_per_s = out->max_ms > 0 ? (double)out->pairs_total / (out->max_ms / 1e3) : 0.0;
    return st;
}
