// runtime.cu -- status plumbing, format helpers, buffers, worker pool, slots.
#include <algorithm>
#include <cerrno>
#include <cstdlib>

#include "runtime.h"

namespace fb200 {

namespace {
thread_local std::string t_last_error;
}

falcon_status set_error(falcon_status s, const std::string& msg) {
    t_last_error = msg;
    return s;
}

const char* last_error_text() { return t_last_error.c_str(); }

// Texts of the reference's throw sites (chunk_codec.hpp:92-117, bitplane.hpp:165-177,
// container.cpp:114-128, pipeline.hpp:415, 461, numeric.hpp:154).
const char* device_error_text(uint32_t code) {
    switch (code) {
    case DEV_E_SCALE: return "decimal_round_scale: scaled value exceeds 63 bits";
    case DEV_E_CAPACITY: return "output capacity too small for the compressed archive";
    case DEV_E_HDR_TRUNC: return "chunk header truncated";
    case DEV_E_META: return "chunk meta bytes out of range";
    case DEV_E_W: return "plane count out of range";
    case DEV_E_FLAGS_TRUNC: return "plane flags truncated";
    case DEV_E_FLAG_PAD: return "nonzero flag padding bits";
    case DEV_E_ROW_TRUNC: return "row data truncated";
    case DEV_E_BITMAP_TRUNC: return "row bitmap truncated";
    case DEV_E_PAYLOAD_TRUNC: return "row payload truncated";
    case DEV_E_SIZE: return "chunk size mismatch";
    case DEV_E_BATCH_HDR_TRUNC: return "batch header truncated";
    case DEV_E_TABLE_TRUNC: return "batch size table truncated";
    case DEV_E_PAYLOAD_BATCH_TRUNC: return "batch payload truncated";
    case DEV_E_CHUNK_COUNT: return "chunk count mismatch";
    case DEV_E_TRAILING: return "trailing bytes after final batch";
    default: return "unknown device error";
    }
}

falcon_status device_error_status(uint32_t code) {
    if (code == DEV_E_CAPACITY) return FALCON_ERR_CAPACITY;
    if (code == DEV_E_SCALE) return FALCON_ERR_INVALID;
    return FALCON_ERR_CORRUPT;
}

// max_encoded_chunk_size (chunk_codec.hpp:36-41)
uint64_t max_chunk_bytes(int prec, uint32_t chunk_n) {
    const uint64_t width = prec == FALCON_F64 ? 64 : 32;
    return 3 + lane_bytes(prec) + (width + 7) / 8 + width * ((uint64_t)(chunk_n - 1) / 8);
}

uint64_t frame_bound(int prec, uint64_t count, uint32_t chunk_n) {
    const uint64_t chunks = (count + chunk_n - 1) / chunk_n;
    return 4 + 4 * chunks + chunks * max_chunk_bytes(prec, chunk_n);
}

// validate_pipeline_options (pipeline.hpp:136-143), same messages
falcon_status validate_options(uint32_t chunk_n, uint64_t batch_values) {
    if (chunk_n < 65 || (chunk_n - 1) % 64 != 0)
        return set_error(FALCON_ERR_INVALID, "chunk length must be a multiple of 64 plus one");
    if (batch_values == 0) return set_error(FALCON_ERR_INVALID, "batch size must be positive");
    if (chunk_n > 4097)
        return set_error(FALCON_ERR_UNSUPPORTED,
                         "chunk_n > 4097 is not supported by the sm_100a kernels of this build");
    return FALCON_OK;
}

falcon_status make_geometry(uint64_t n, uint32_t chunk_n, uint64_t bv, uint64_t header_bytes,
                            geometry& g) {
    g.header_bytes = header_bytes;
    g.n_values = n;
    g.batch_values = bv;
    g.chunk_n = chunk_n;
    const uint64_t cpb = (bv + chunk_n - 1) / chunk_n;
    g.n_batches = n ? (n + bv - 1) / bv : 0;
    g.cpb_magic = 0;
    if (g.n_batches == 0) {
        g.cpb = 1;
        g.last_cpb = 0;
        g.n_chunks = 0;
        return FALCON_OK;
    }
    const uint64_t last = n - (g.n_batches - 1) * bv;
    g.last_cpb = (uint32_t)((last + chunk_n - 1) / chunk_n);
    if (g.n_batches > 1 && cpb > 0xffffffffull)
        return set_error(FALCON_ERR_INVALID, "append_batch: too many chunks");  // container.cpp:90-91
    g.cpb = g.n_batches > 1 ? (uint32_t)cpb : g.last_cpb;
    g.n_chunks = (g.n_batches - 1) * (uint64_t)g.cpb + g.last_cpb;
    g.cpb_magic = g.cpb > 1 ? ~0ull / g.cpb + 1 : 0;
    if (g.n_chunks + 1 > 0x7fffffffull)
        return set_error(FALCON_ERR_UNSUPPORTED,
                         "more than 2^31-2 chunks in one device call; shard the input");
    return FALCON_OK;
}

static void put_le(uint64_t v, uint8_t* p, int bytes) {
    for (int i = 0; i < bytes; ++i) p[i] = (uint8_t)(v >> (8 * i));
}

// write_header (container.cpp:44-55)
archive_header_bytes header_bytes_of(int prec, uint32_t chunk_n, uint64_t bv, uint64_t total,
                                     uint64_t batches) {
    archive_header_bytes h{};
    static const uint8_t magic[8] = {'F', 'A', 'L', 'C', 'O', 'N', 'A', 0};
    std::memcpy(h.b, magic, 8);
    put_le(1, h.b + 8, 2);
    h.b[10] = (uint8_t)prec;
    put_le(chunk_n, h.b + 11, 4);
    put_le(bv, h.b + 15, 8);
    put_le(total, h.b + 23, 8);
    put_le(batches, h.b + 31, 8);
    put_le(0, h.b + 39, 8);
    return h;
}

// ---- buffers -----------------------------------------------------------------
falcon_status device_buffer::ensure(size_t bytes) {
    if (bytes <= cap && p) return FALCON_OK;
    release();
    const size_t want = bytes < 256 ? 256 : bytes;
    FB_CUDA(cudaMalloc(&p, want));
    cap = want;
    return FALCON_OK;
}
void device_buffer::release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
}

falcon_status pinned_buffer::ensure(size_t bytes) {
    if (bytes <= cap && p) return FALCON_OK;
    release();
    const size_t want = bytes < 256 ? 256 : bytes;
    FB_CUDA(cudaHostAlloc(&p, want, cudaHostAllocPortable));
    cap = want;
    return FALCON_OK;
}
void pinned_buffer::release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
}

bool is_pinned(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// ---- task pool ---------------------------------------------------------------------
worker_pool::worker_pool(unsigned workers) : ring_(1024) {
    const unsigned n = workers ? workers : default_workers();
    threads_.reserve(n);
    while (threads_.size() < n) threads_.emplace_back(&worker_pool::worker_main, this);
}

worker_pool::~worker_pool() {
    {
        std::unique_lock<std::mutex> g(lock_);
        closing_ = true;
    }
    has_job_.notify_all();
    has_room_.notify_all();
    for (std::thread& t : threads_) t.join();
}

void worker_pool::submit(std::function<void()> job) {
    std::unique_lock<std::mutex> g(lock_);
    has_room_.wait(g, [&] { return tail_ - head_ < ring_.size(); });
    ring_[tail_++ % ring_.size()] = std::move(job);
    g.unlock();
    has_job_.notify_one();
}

void worker_pool::worker_main() {
    std::unique_lock<std::mutex> g(lock_);
    for (;;) {
        has_job_.wait(g, [&] { return closing_ || head_ != tail_; });
        if (head_ == tail_) return;          // closing and drained
        std::function<void()> job = std::move(ring_[head_++ % ring_.size()]);
        g.unlock();
        has_room_.notify_one();
        job();
        g.lock();
    }
}

void worker_pool::fork_join(unsigned parts, const std::function<void(unsigned)>& fn) {
    if (parts <= 1 || threads_.empty()) {
        for (unsigned i = 0; i < parts; ++i) fn(i);
        return;
    }
    // parts are claimed from a shared counter by the helpers and the caller alike, so a
    // busy pool never stalls the caller
    struct join_state {
        std::atomic<unsigned> next{0}, left;
        std::mutex m;
        std::condition_variable cv;
        explicit join_state(unsigned n) : left(n) {}
    };
    auto st = std::make_shared<join_state>(parts);
    auto drain = [st, parts, &fn] {
        for (unsigned i; (i = st->next.fetch_add(1)) < parts;) {
            fn(i);
            if (st->left.fetch_sub(1) == 1) {
                std::lock_guard<std::mutex> g(st->m);
                st->cv.notify_all();
            }
        }
    };
    const unsigned helpers = std::min<unsigned>(parts - 1, (unsigned)threads_.size());
    for (unsigned h = 0; h < helpers; ++h) submit(drain);
    drain();
    std::unique_lock<std::mutex> g(st->m);
    st->cv.wait(g, [&] { return st->left.load() == 0; });
}

unsigned worker_pool::default_workers() {
    // FALCON_WORKERS: a positive decimal integer, anything else is ignored
    // (worker_pool.hpp:30-38 default)
    if (const char* env = std::getenv("FALCON_WORKERS")) {
        char* end = nullptr;
        errno = 0;
        const unsigned long v = std::strtoul(env, &end, 10);
        if (errno == 0 && end != env && *end == '\0' && v > 0 && v <= 4096 && env[0] != '-')
            return (unsigned)v;
    }
    const unsigned hw = std::thread::hardware_concurrency();
    return hw > 0 ? hw : 1;
}

// ---- slots ---------------------------------------------------------------------
falcon_status pipeline_slot::init() {
    if (stream) return FALCON_OK;
    FB_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    FB_CUDA(cudaEventCreateWithFlags(&ev_size, cudaEventDisableTiming));
    FB_CUDA(cudaEventCreateWithFlags(&ev_data, cudaEventDisableTiming));
    FB_CUDA(cudaHostAlloc((void**)&box, sizeof(slot_mailbox), cudaHostAllocPortable));
    FB_TRY(d_misc.ensure(64));
    done.fire();
    return FALCON_OK;
}
pipeline_slot::~pipeline_slot() {
    if (stream) cudaStreamSynchronize(stream);
    if (ev_size) cudaEventDestroy(ev_size);
    if (ev_data) cudaEventDestroy(ev_data);
    if (stream) cudaStreamDestroy(stream);
    if (box) cudaFreeHost(box);
}

}  // namespace fb200

fb200::worker_pool& falcon_ctx::get_pool(unsigned workers) {
    const unsigned want = workers ? workers : fb200::worker_pool::default_workers();
    if (!pool || pool_workers != want) {
        pool.reset();
        pool = std::make_unique<fb200::worker_pool>(want);
        pool_workers = want;
    }
    return *pool;
}
