// ref_shim.cpp -- C entry points over the reference's OWN config code (TEST INFRASTRUCTURE).
//
// Built by oracle/Makefile together with /root/reference/proj/src/config.cpp,
// compiled where it lies (never copied), into oracle/_ref/libouro_refconfig.so.
// Tests use it to pin the oracle and the product's validate()/variant-name
// behaviour to the reference itself (proj/src/config.cpp:16-59,
// proj/include/ouro/config.hpp:26-73).
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <string_view>

#include "ouro/config.hpp"
#include "ouro/errors.hpp"

extern "C" {

struct ref_config {  // field-for-field HeapConfig
    uint64_t heap_bytes, chunk_bytes, min_page_bytes, max_page_bytes;
    uint8_t queue_flavor, allocator_kind, backoff, reserved0;
    uint32_t max_retries, sleep_base_ns, sleep_cap_ns;
};

static ouro::HeapConfig to_ref(const ref_config* c) {
    ouro::HeapConfig h;
    h.heap_bytes = c->heap_bytes;
    h.chunk_bytes = c->chunk_bytes;
    h.min_page_bytes = c->min_page_bytes;
    h.max_page_bytes = c->max_page_bytes;
    h.queue_flavor = static_cast<ouro::QueueFlavor>(c->queue_flavor);
    h.allocator_kind = static_cast<ouro::AllocatorKind>(c->allocator_kind);
    h.backoff = static_cast<ouro::BackoffPolicy>(c->backoff);
    h.max_retries = c->max_retries;
    h.sleep_base_ns = c->sleep_base_ns;
    h.sleep_cap_ns = c->sleep_cap_ns;
    return h;
}

// 0 = valid, 1 = ConfigError (message copied), 2 = other exception.
int ref_validate(const ref_config* c, char* msg, size_t len) {
    try {
        to_ref(c).validate();
        if (msg && len) msg[0] = 0;
        return 0;
    } catch (const ouro::ConfigError& e) {
        if (msg && len) std::snprintf(msg, len, "%s", e.what());
        return 1;
    } catch (...) {
        return 2;
    }
}

void ref_default(ref_config* c) {
    ouro::HeapConfig h;
    c->heap_bytes = h.heap_bytes;
    c->chunk_bytes = h.chunk_bytes;
    c->min_page_bytes = h.min_page_bytes;
    c->max_page_bytes = h.max_page_bytes;
    c->queue_flavor = static_cast<uint8_t>(h.queue_flavor);
    c->allocator_kind = static_cast<uint8_t>(h.allocator_kind);
    c->backoff = static_cast<uint8_t>(h.backoff);
    c->reserved0 = 0;
    c->max_retries = h.max_retries;
    c->sleep_base_ns = h.sleep_base_ns;
    c->sleep_cap_ns = h.sleep_cap_ns;
}

uint32_t ref_num_chunks(const ref_config* c) { return to_ref(c).num_chunks(); }
uint32_t ref_max_pages_per_chunk(const ref_config* c) { return to_ref(c).max_pages_per_chunk(); }

// Writes the NUL-terminated name; returns its length.
int ref_variant_name(uint8_t kind, uint8_t flavor, char* out, size_t len) {
    ouro::Variant v{static_cast<ouro::AllocatorKind>(kind), static_cast<ouro::QueueFlavor>(flavor)};
    std::string_view s = ouro::variant_name(v);
    std::snprintf(out, len, "%.*s", (int)s.size(), s.data());
    return (int)s.size();
}

int ref_variant_from_name(const char* name, uint8_t* kind, uint8_t* flavor) {
    auto v = ouro::variant_from_name(name);
    if (!v) return 0;
    *kind = static_cast<uint8_t>(v->kind);
    *flavor = static_cast<uint8_t>(v->flavor);
    return 1;
}

int ref_all_variants(uint8_t* kinds, uint8_t* flavors) {
    int i = 0;
    for (auto v : ouro::kAllVariants) {
        kinds[i] = static_cast<uint8_t>(v.kind);
        flavors[i] = static_cast<uint8_t>(v.flavor);
        ++i;
    }
    return i;
}

// Layout facts of the reference struct (sizeof, alignof, field offsets).
void ref_layout(uint64_t* out) {
    out[0] = sizeof(ouro::HeapConfig);
    out[1] = alignof(ouro::HeapConfig);
    out[2] = offsetof(ouro::HeapConfig, queue_flavor);
    out[3] = offsetof(ouro::HeapConfig, allocator_kind);
    out[4] = offsetof(ouro::HeapConfig, backoff);
    out[5] = offsetof(ouro::HeapConfig, max_retries);
    out[6] = offsetof(ouro::HeapConfig, sleep_base_ns);
    out[7] = offsetof(ouro::HeapConfig, sleep_cap_ns);
    out[8] = sizeof(ouro::Variant);
}

}  // extern "C"
