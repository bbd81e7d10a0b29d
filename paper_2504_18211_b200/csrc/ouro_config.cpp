// ouro_config.cpp -- host-side configuration half of the C-ABI (no GPU needed).
//
// Re-implements, from the reference's documented behaviour:
//   HeapConfig defaults          /root/reference/proj/include/ouro/config.hpp:26-38
//   HeapConfig::validate         /root/reference/proj/src/config.cpp:16-42
//   num_chunks / pages per chunk /root/reference/proj/include/ouro/config.hpp:45-51
//   variant_name / from_name     /root/reference/proj/src/config.cpp:44-59
//   size_class_of, handles
//   backoff mapping
// tests/test_config.py checks every rule against the reference's own
// config.cpp (oracle/_ref) and the oracle.
#include <bit>
#include <cstdio>
#include <cstring>

#include "../../include/ouro.h"
#include "ouro_internal.h"

namespace {

bool is_pow2(uint64_t v) { return v != 0 && (v & (v - 1)) == 0; }

ouro_status check(const ouro_config* c, const char** why) {
    if (!c) { *why = "null config"; return OURO_ERR_USAGE; }
    if (!is_pow2(c->heap_bytes) || !is_pow2(c->chunk_bytes) || !is_pow2(c->min_page_bytes) ||
        !is_pow2(c->max_page_bytes)) {
        *why = "heap, chunk and page-class sizes must be powers of two";
        return OURO_ERR_CONFIG;
    }
    if (c->min_page_bytes > c->max_page_bytes) { *why = "min_page_bytes exceeds max_page_bytes"; return OURO_ERR_CONFIG; }
    if (c->max_page_bytes > c->chunk_bytes) { *why = "max_page_bytes exceeds chunk_bytes"; return OURO_ERR_CONFIG; }
    if (c->chunk_bytes > c->heap_bytes) { *why = "chunk_bytes exceeds heap_bytes"; return OURO_ERR_CONFIG; }
    const uint64_t n = c->heap_bytes / c->chunk_bytes;
    if (n > (1ull << 24)) { *why = "more than 2^24 chunks; chunk index does not fit a packed handle"; return OURO_ERR_CONFIG; }
    const unsigned pb = (unsigned)std::countr_zero(c->chunk_bytes / c->min_page_bytes);
    const unsigned cb = n > 1 ? (unsigned)std::bit_width(n - 1) : 0u;
    if (pb + cb > 32) { *why = "chunk/page split does not fit a 32-bit handle"; return OURO_ERR_CONFIG; }
    if (c->max_retries == 0) { *why = "max_retries must be at least 1"; return OURO_ERR_CONFIG; }
    *why = "";
    return OURO_OK;
}

}  // namespace

namespace ouro_host {

ouro_status geometry(const ouro_config* c, Geometry* g) {
    const char* why;
    const ouro_status s = check(c, &why);
    if (s != OURO_OK) return s;
    if (c->queue_flavor > 2 || c->allocator_kind > 1 || c->backoff > 1) return OURO_ERR_CONFIG;
    g->heap = c->heap_bytes;
    g->chunk = c->chunk_bytes;
    g->minp = c->min_page_bytes;
    g->maxp = c->max_page_bytes;
    g->N = (uint32_t)(c->heap_bytes / c->chunk_bytes);
    g->K = (uint32_t)std::countr_zero(g->maxp / g->minp) + 1;
    g->page_bits = (uint32_t)std::countr_zero(g->chunk / g->minp);
    g->chunk_bits = g->N > 1 ? (uint32_t)std::bit_width((uint64_t)g->N - 1) : 0u;
    g->chunk_shift = (uint32_t)std::countr_zero(g->chunk);
    g->min_shift = (uint32_t)std::countr_zero(g->minp);
    g->Wmax = (uint32_t)((g->chunk / g->minp + 63) / 64);
    g->gen_bits = 32 - g->chunk_bits < 24 ? 32 - g->chunk_bits : 24;
    g->gmask = g->gen_bits >= 32 ? 0xFFFFFFFFu : ((1u << g->gen_bits) - 1u);
    g->cmask = g->chunk_bits == 0 ? 0u : (g->chunk_bits >= 32 ? 0xFFFFFFFFu : ((1u << g->chunk_bits) - 1u));
    // limits of this build beyond validate(): <= 32 classes; virtual flavours
    // need a list header plus one slot per segment (chunk >= 32 B)
    if (g->K > OURO_MAX_CLASSES) return OURO_ERR_CONFIG;
    if (c->queue_flavor != OURO_FLAVOR_ARRAY && g->chunk < 32) return OURO_ERR_CONFIG;
    return OURO_OK;
}

}  // namespace ouro_host

extern "C" {

ouro_status ouro_config_default(ouro_config* cfg) {
    if (!cfg) return OURO_ERR_USAGE;
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->heap_bytes = 64ull << 20;
    cfg->chunk_bytes = 64ull << 10;
    cfg->min_page_bytes = 16;
    cfg->max_page_bytes = 8192;
    cfg->queue_flavor = OURO_FLAVOR_ARRAY;
    cfg->allocator_kind = OURO_KIND_PAGE;
    cfg->backoff = OURO_BACKOFF_FENCE;
    cfg->max_retries = 64;
    cfg->sleep_base_ns = 100;
    cfg->sleep_cap_ns = 100000;
    return OURO_OK;
}

ouro_status ouro_config_validate(const ouro_config* cfg, char* msg, size_t msg_len) {
    const char* why;
    const ouro_status s = check(cfg, &why);
    if (msg && msg_len) std::snprintf(msg, msg_len, "%s", why);
    return s;
}

ouro_status ouro_config_geometry(const ouro_config* cfg, ouro_geometry* out) {
    ouro_host::Geometry g;
    const ouro_status s = ouro_host::geometry(cfg, &g);
    if (s != OURO_OK) return s;
    out->num_chunks = g.N;
    out->max_pages_per_chunk = (uint32_t)(g.chunk / g.minp);
    out->num_classes = g.K;
    out->page_bits = g.page_bits;
    out->chunk_bits = g.chunk_bits;
    out->gen_bits = g.gen_bits;
    out->bitmap_words = g.Wmax;
    out->reserved0 = 0;
    return OURO_OK;
}

const char* ouro_variant_name(uint8_t kind, uint8_t flavor) {
    static const char* names[2][3] = {{"page", "va-page", "vl-page"}, {"chunk", "va-chunk", "vl-chunk"}};
    if (kind > 1 || flavor > 2) return "?";
    return names[kind][flavor];
}

int ouro_variant_from_name(const char* name, uint8_t* kind, uint8_t* flavor) {
    if (!name) return 0;
    // kAllVariants order (config.hpp:62-69): page, chunk, va-page, va-chunk, vl-page, vl-chunk
    for (uint8_t f = 0; f < 3; ++f)
        for (uint8_t k = 0; k < 2; ++k)
            if (std::strcmp(ouro_variant_name(k, f), name) == 0) {
                if (kind) *kind = k;
                if (flavor) *flavor = f;
                return 1;
            }
    return 0;
}

ouro_status ouro_size_class(const ouro_config* cfg, uint64_t bytes, uint32_t* cls) {
    ouro_host::Geometry g;
    if (ouro_host::geometry(cfg, &g) != OURO_OK) return OURO_ERR_CONFIG;
    if (bytes == 0 || bytes > g.maxp) return OURO_ERR_TOO_LARGE;
    const uint32_t lg = bytes <= 1 ? 0u : (uint32_t)std::bit_width(bytes - 1);
    *cls = lg > g.min_shift ? lg - g.min_shift : 0u;
    return OURO_OK;
}

ouro_status ouro_handle_encode(const ouro_config* cfg, uint32_t chunk, uint32_t page, uint32_t* h) {
    ouro_host::Geometry g;
    if (ouro_host::geometry(cfg, &g) != OURO_OK) return OURO_ERR_CONFIG;
    if (chunk >= g.N || (uint64_t)page >= g.chunk / g.minp) return OURO_ERR_RANGE;
    *h = (chunk << g.page_bits) | page;
    return OURO_OK;
}

ouro_status ouro_handle_decode(const ouro_config* cfg, uint32_t h, uint32_t* chunk, uint32_t* page) {
    ouro_host::Geometry g;
    if (ouro_host::geometry(cfg, &g) != OURO_OK) return OURO_ERR_CONFIG;
    const uint64_t c = (uint64_t)h >> g.page_bits;
    if (c >= g.N) return OURO_ERR_RANGE;
    *chunk = (uint32_t)c;
    *page = h & ((1u << g.page_bits) - 1u);
    return OURO_OK;
}

uint64_t ouro_backoff_ns(uint8_t policy, uint32_t attempt, uint32_t base_ns, uint32_t cap_ns) {
    if (policy != OURO_BACKOFF_SLEEP) return 0;
    if (attempt >= 40) return cap_ns;
    const uint64_t v = (uint64_t)base_ns << attempt;
    return v > cap_ns ? cap_ns : v;
}

ouro_status ouro_trial_means(const double* ms, uint32_t n, double* mean_all, double* mean_subsequent) {
    if (!ms || n < 2) return OURO_ERR_USAGE;
    double a = 0, s = 0;
    for (uint32_t i = 0; i < n; ++i) { a += ms[i]; if (i) s += ms[i]; }
    *mean_all = a / n;
    *mean_subsequent = s / (n - 1);
    return OURO_OK;
}

const char* ouro_status_name(ouro_status s) {
    switch (s) {
    case OURO_OK: return "Ok";
    case OURO_ERR_CONFIG: return "ConfigError";
    case OURO_ERR_INVALID_HANDLE: return "InvalidHandle";
    case OURO_ERR_DOUBLE_FREE: return "DoubleFree";
    case OURO_ERR_RANGE: return "RangeError";
    case OURO_ERR_TIMEOUT: return "Timeout";
    case OURO_ERR_CORRUPTION: return "Corruption";
    case OURO_ERR_OOM: return "OutOfMemory";
    case OURO_ERR_TOO_LARGE: return "TooLarge";
    case OURO_ERR_CUDA: return "CudaError";
    case OURO_ERR_FULL: return "Full";
    case OURO_ERR_EMPTY: return "Empty";
    case OURO_ERR_CHUNK_FULL: return "ChunkFull";
    case OURO_ERR_ALREADY_ASSIGNED: return "AlreadyAssigned";
    case OURO_ERR_VERIFICATION: return "VerificationFailed";
    case OURO_ERR_USAGE: return "UsageError";
    }
    return "?";
}

}  // extern "C"
