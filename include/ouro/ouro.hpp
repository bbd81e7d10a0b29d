// ouro/ouro.hpp -- C++20 host API over the C-ABI (include/ouro.h).
//
// Drop-in for the reference's public C++ surface (namespace ouro):
//   QueueFlavor / AllocatorKind / BackoffPolicy   /root/reference/proj/include/ouro/config.hpp:17,21,24
//   HeapConfig (+ validate, num_chunks, ...)      config.hpp:26-52, proj/src/config.cpp:16-42
//   Variant, kAllVariants                         config.hpp:55-69
//   variant_name / variant_from_name              config.hpp:71-73, config.cpp:44-59
//   ConfigError ... CorruptionError               /root/reference/proj/include/ouro/errors.hpp:11-46
// plus the device heap the SPEC describes (new_arena / stats / run_trial,
// SPEC.md:45, 285, 379) as ouro::DeviceHeap.  validate() calls the library's
// ouro_config_validate, so reject set and messages are the reference's.
// Header-only; link with libouro_b200.so.
#pragma once

#include <array>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>

#include "../ouro.h"

namespace ouro {

enum class QueueFlavor : std::uint8_t { Array, VirtualArray, VirtualList };
enum class AllocatorKind : std::uint8_t { Page, Chunk };
enum class BackoffPolicy : std::uint8_t { FenceRetry, SleepRetry };

class ConfigError : public std::runtime_error { public: using std::runtime_error::runtime_error; };
class InvalidHandleError : public std::runtime_error { public: using std::runtime_error::runtime_error; };
class DoubleFreeError : public std::runtime_error { public: using std::runtime_error::runtime_error; };
class RangeError : public std::runtime_error { public: using std::runtime_error::runtime_error; };
class TimeoutError : public std::runtime_error { public: using std::runtime_error::runtime_error; };
class CorruptionError : public std::logic_error { public: using std::logic_error::logic_error; };
class CudaError : public std::runtime_error { public: using std::runtime_error::runtime_error; };

// Map a C-ABI status to the reference's exception taxonomy.
inline void throw_if(ouro_status s, const char* what) {
    if (s == OURO_OK) return;
    std::string m = std::string(what) + ": " + ouro_status_name(s);
    switch (s) {
    case OURO_ERR_CONFIG: throw ConfigError(m);
    case OURO_ERR_INVALID_HANDLE: throw InvalidHandleError(m);
    case OURO_ERR_DOUBLE_FREE: throw DoubleFreeError(m);
    case OURO_ERR_RANGE: throw RangeError(m);
    case OURO_ERR_TIMEOUT: throw TimeoutError(m);
    case OURO_ERR_CORRUPTION: throw CorruptionError(m);
    case OURO_ERR_CUDA: throw CudaError(m);
    default: throw std::runtime_error(m);
    }
}

struct HeapConfig {
    std::uint64_t heap_bytes = 64ull << 20;
    std::uint64_t chunk_bytes = 64ull << 10;
    std::uint64_t min_page_bytes = 16;
    std::uint64_t max_page_bytes = 8192;
    QueueFlavor queue_flavor = QueueFlavor::Array;
    AllocatorKind allocator_kind = AllocatorKind::Page;
    BackoffPolicy backoff = BackoffPolicy::FenceRetry;
    std::uint32_t max_retries = 64;
    std::uint32_t sleep_base_ns = 100;
    std::uint32_t sleep_cap_ns = 100'000;

    ouro_config to_c() const {
        ouro_config c{};
        c.heap_bytes = heap_bytes;
        c.chunk_bytes = chunk_bytes;
        c.min_page_bytes = min_page_bytes;
        c.max_page_bytes = max_page_bytes;
        c.queue_flavor = static_cast<std::uint8_t>(queue_flavor);
        c.allocator_kind = static_cast<std::uint8_t>(allocator_kind);
        c.backoff = static_cast<std::uint8_t>(backoff);
        c.max_retries = max_retries;
        c.sleep_base_ns = sleep_base_ns;
        c.sleep_cap_ns = sleep_cap_ns;
        return c;
    }
    // Throws ConfigError exactly where the reference's validate() does.
    void validate() const {
        char msg[256];
        const ouro_config c = to_c();
        if (ouro_config_validate(&c, msg, sizeof msg) != OURO_OK) throw ConfigError(msg);
    }
    std::uint32_t num_chunks() const { return static_cast<std::uint32_t>(heap_bytes / chunk_bytes); }
    std::uint32_t max_pages_per_chunk() const { return static_cast<std::uint32_t>(chunk_bytes / min_page_bytes); }
};
static_assert(sizeof(HeapConfig) == sizeof(ouro_config), "HeapConfig layout");

struct Variant {
    AllocatorKind kind;
    QueueFlavor flavor;
    bool operator==(const Variant&) const = default;
};

inline constexpr std::array<Variant, 6> kAllVariants = {{
    {AllocatorKind::Page, QueueFlavor::Array},
    {AllocatorKind::Chunk, QueueFlavor::Array},
    {AllocatorKind::Page, QueueFlavor::VirtualArray},
    {AllocatorKind::Chunk, QueueFlavor::VirtualArray},
    {AllocatorKind::Page, QueueFlavor::VirtualList},
    {AllocatorKind::Chunk, QueueFlavor::VirtualList},
}};

inline std::string_view variant_name(Variant v) {
    return ouro_variant_name(static_cast<std::uint8_t>(v.kind), static_cast<std::uint8_t>(v.flavor));
}

inline std::optional<Variant> variant_from_name(std::string_view name) {
    std::uint8_t k, f;
    const std::string s(name);
    if (!ouro_variant_from_name(s.c_str(), &k, &f)) return std::nullopt;
    return Variant{static_cast<AllocatorKind>(k), static_cast<QueueFlavor>(f)};
}

// RAII device heap: new_arena + allocator.  Kernels
// receive view() by value and call ouro_malloc / ouro_free (ouro_device.cuh).
class DeviceHeap {
public:
    explicit DeviceHeap(const HeapConfig& cfg, int device = 0) {
        cfg.validate();
        const ouro_config c = cfg.to_c();
        throw_if(ouro_heap_create(&c, device, &h_), "ouro_heap_create");
    }
    ~DeviceHeap() { if (h_) ouro_heap_destroy(h_); }
    DeviceHeap(const DeviceHeap&) = delete;
    DeviceHeap& operator=(const DeviceHeap&) = delete;

    ouro_heap* get() const { return h_; }
    template <class View>
    View view() const {
        View v;
        throw_if(ouro_heap_get_view(h_, &v, sizeof v), "ouro_heap_get_view");
        return v;
    }
    ouro_stats stats(void* stream = nullptr) const {
        ouro_stats s;
        throw_if(ouro_heap_stats(h_, &s, stream), "ouro_heap_stats");
        return s;
    }
    ouro_digest digest(void* stream = nullptr) const {
        ouro_digest d;
        throw_if(ouro_heap_digest(h_, &d, stream), "ouro_heap_digest");
        return d;
    }
    // Surfaces the sticky device error word as the reference's exception.
    void check_device_errors(bool clear = true) const {
        std::uint32_t first = 0, mask = 0;
        throw_if(ouro_heap_last_error(h_, &first, &mask, clear ? 1 : 0), "ouro_heap_last_error");
        throw_if(static_cast<ouro_status>(first), "device");
    }
    ouro_trial_result run_trial(std::uint64_t n, std::uint64_t bytes, std::uint32_t iterations = 10,
                                std::uint64_t seed = 1) const {
        ouro_trial_config tc{};
        tc.num_allocations = n;
        tc.allocation_bytes = bytes;
        tc.iterations = iterations;
        tc.seed = seed;
        ouro_trial_result r;
        throw_if(ouro_run_trial(h_, &tc, &r), "ouro_run_trial");
        return r;
    }

private:
    ouro_heap* h_ = nullptr;
};

}  // namespace ouro
