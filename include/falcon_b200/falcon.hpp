// falcon.hpp -- C++ drop-in for the reference's public API, backed by the B200 library.
//
// Mirrors /root/reference/proj/include/falcon/{pipeline,chunk_codec,container,error}.hpp
// name for name inside namespace falcon_b200 (a user switches by changing the include
// and the namespace, e.g. `namespace falcon = falcon_b200;`):
//
//   value_source / value_sink / memory_source / memory_sink   pipeline.hpp:21-64
//   pipeline_options / pipeline_stats / stage_* ids           pipeline.hpp:66-85
//   compress_pipeline<T>                                      pipeline.hpp:156-159
//   decompress_pipeline<T>, decompress_to_vector<T>           pipeline.hpp:370-476
//   chunk_workspace<T>, compress_chunk<T>, decompress_chunk<T> chunk_codec.hpp:43-131
//   max_encoded_chunk_size<T>                                 chunk_codec.hpp:36-41
//   archive_header, write_header, read_header                 container.hpp:12-27, container.cpp:44-86
//   error / corrupt_error / io_error                          error.hpp:8-19
//
// Same exception types and messages (including the " (batch N)" suffix), same output
// bytes for any n_streams/workers, same threading contract: read() runs on the calling
// thread, put() may run concurrently from worker threads, stage_delay runs right before
// a stage's completion is signalled.  Everything computes on the GPU through the C ABI
// in falcon_b200.h; there is no CPU codec behind it.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <functional>
#include <memory>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "../falcon_b200.h"

namespace falcon_b200 {

struct error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct corrupt_error : error {
    using error::error;
};
struct io_error : error {
    using error::error;
};

namespace detail {
[[noreturn]] inline void throw_status(falcon_status s) {
    const std::string msg = falcon_last_error();
    switch (s) {
    case FALCON_ERR_CORRUPT: throw corrupt_error(msg);
    case FALCON_ERR_IO: throw io_error(msg);
    default: throw error(msg);
    }
}
inline void check(falcon_status s) {
    if (s != FALCON_OK) throw_status(s);
}

// One context per process on FALCON_DEVICE (default 0), created on first use.
inline falcon_ctx* context() {
    static std::once_flag once;
    static falcon_ctx* ctx = nullptr;
    static falcon_status st = FALCON_OK;
    std::call_once(once, [] {
        const char* d = std::getenv("FALCON_DEVICE");
        st = falcon_ctx_create(d ? std::atoi(d) : 0, &ctx);
    });
    if (st != FALCON_OK) throw_status(st);
    return ctx;
}

template <typename T> constexpr int prec = FALCON_F64;
template <> constexpr int prec<float> = FALCON_F32;

// first exception raised inside a callback wins; rethrown after the call drains
struct callback_errors {
    std::mutex m;
    std::exception_ptr first;
    void record(std::exception_ptr e) {
        std::lock_guard<std::mutex> l(m);
        if (!first) first = e;
    }
    void rethrow() {
        if (first) std::rethrow_exception(first);
    }
};
}  // namespace detail

template <typename T>
class value_source {
public:
    virtual ~value_source() = default;
    // Fill as much of dst as possible; 0 means end of stream.
    virtual std::size_t read(std::span<T> dst) = 0;
};

template <typename T>
class value_sink {
public:
    virtual ~value_sink() = default;
    // One call per batch, possibly out of order and from worker threads.
    virtual void put(std::uint64_t first_value_index, std::span<const T> values) = 0;
};

template <typename T>
class memory_source final : public value_source<T> {
public:
    explicit memory_source(std::span<const T> data) : data_(data) {}
    std::size_t read(std::span<T> dst) override {
        const std::size_t k = std::min(dst.size(), data_.size() - pos_);
        std::memcpy(dst.data(), data_.data() + pos_, k * sizeof(T));
        pos_ += k;
        return k;
    }
    std::span<const T> remaining() const { return data_.subspan(pos_); }
    void consume(std::size_t k) { pos_ += k; }

private:
    std::span<const T> data_;
    std::size_t pos_ = 0;
};

template <typename T>
class memory_sink final : public value_sink<T> {
public:
    explicit memory_sink(std::size_t total) : values(total) {}
    void put(std::uint64_t first, std::span<const T> v) override {
        std::memcpy(values.data() + first, v.data(), v.size() * sizeof(T));
    }
    std::vector<T> values;
};

inline constexpr int stage_compress = FALCON_STAGE_COMPRESS;
inline constexpr int stage_store = FALCON_STAGE_STORE;
inline constexpr int stage_decode = FALCON_STAGE_DECODE;

struct pipeline_options {
    std::uint32_t chunk_n = 1025;
    std::uint64_t batch_values = std::uint64_t{1025} * 1024 * 4;
    unsigned n_streams = 16;
    unsigned workers = 0;  // 0 = FALCON_WORKERS / hardware default
    std::function<void(int stage, unsigned slot, std::uint64_t seq)> stage_delay;
};

struct pipeline_stats {
    std::uint64_t batches = 0;
    std::uint64_t values = 0;
    std::uint64_t blocking_waits = 0;
};

enum class precision_tag : std::uint8_t { f64 = 0, f32 = 1 };
template <typename T> inline constexpr precision_tag precision_of = precision_tag::f64;
template <> inline constexpr precision_tag precision_of<float> = precision_tag::f32;

struct archive_header {
    precision_tag precision = precision_tag::f64;
    std::uint32_t chunk_n = 1025;
    std::uint64_t batch_values = 0;
    std::uint64_t total_values = 0;
    std::uint64_t batch_count = 0;
};
inline constexpr std::size_t archive_header_bytes = 47;

inline std::vector<std::uint8_t> write_header(const archive_header& h) {
    falcon_archive_info i{static_cast<std::uint8_t>(h.precision), h.chunk_n, h.batch_values,
                          h.total_values, h.batch_count};
    std::vector<std::uint8_t> out(archive_header_bytes);
    falcon_write_header(&i, out.data());
    return out;
}

inline archive_header read_header(std::span<const std::uint8_t> in) {
    falcon_archive_info i{};
    detail::check(falcon_read_header(in.data(), in.size(), &i));
    return {static_cast<precision_tag>(i.precision), i.chunk_n, i.batch_values, i.total_values,
            i.batch_count};
}

namespace detail {
inline falcon_pipeline_options to_c(const pipeline_options& o) {
    falcon_pipeline_options c{};
    c.chunk_n = o.chunk_n;
    c.batch_values = o.batch_values;
    c.n_streams = o.n_streams;
    c.workers = o.workers;
    if (o.stage_delay) {
        c.stage_delay = [](void* u, int stage, unsigned slot, std::uint64_t seq) {
            (*static_cast<const std::function<void(int, unsigned, std::uint64_t)>*>(u))(stage, slot, seq);
        };
        c.stage_delay_user = const_cast<void*>(static_cast<const void*>(&o.stage_delay));
    }
    return c;
}
}  // namespace detail

// compress_pipeline (pipeline.hpp:156-365): whole archive returned by value.
template <typename T>
std::vector<std::uint8_t> compress_pipeline(value_source<T>& in, const pipeline_options& opt,
                                            pipeline_stats* stats_out = nullptr) {
    struct state {
        value_source<T>* src;
        std::vector<std::uint8_t> archive;
        std::mutex m;
        detail::callback_errors errs;
    } st;
    st.src = &in;
    const falcon_pipeline_options copt = detail::to_c(opt);
    falcon_pipeline_stats cst{};
    auto rd = [](void* u, void* dst, std::uint64_t maxv) -> std::int64_t {
        auto* s = static_cast<state*>(u);
        try {
            return static_cast<std::int64_t>(s->src->read(std::span<T>(static_cast<T*>(dst), maxv)));
        } catch (...) {
            s->errs.record(std::current_exception());
            return -1;
        }
    };
    auto store = [](void* u, std::uint64_t off, const void* bytes, std::uint64_t len) -> int {
        auto* s = static_cast<state*>(u);
        try {  // run_store (pipeline.hpp:237-252)
            std::lock_guard<std::mutex> l(s->m);
            if (s->archive.size() < off + len) s->archive.resize(off + len);
            std::memcpy(s->archive.data() + off, bytes, len);
            return 0;
        } catch (...) {
            s->errs.record(std::current_exception());
            return 1;
        }
    };
    const falcon_status rc = falcon_compress_stream(detail::context(), detail::prec<T>, rd, &st, store,
                                                    &st, &copt, &cst);
    st.errs.rethrow();
    detail::check(rc);
    if (stats_out) *stats_out = {cst.batches, cst.values, cst.blocking_waits};
    return std::move(st.archive);
}

// decompress_pipeline (pipeline.hpp:370-467)
template <typename T>
pipeline_stats decompress_pipeline(std::span<const std::uint8_t> archive, value_sink<T>& sink,
                                   const pipeline_options& opt = {}) {
    struct state {
        value_sink<T>* sink;
        detail::callback_errors errs;
    } st;
    st.sink = &sink;
    const falcon_pipeline_options copt = detail::to_c(opt);
    falcon_pipeline_stats cst{};
    auto put = [](void* u, std::uint64_t first, const void* v, std::uint64_t count) -> int {
        auto* s = static_cast<state*>(u);
        try {
            s->sink->put(first, std::span<const T>(static_cast<const T*>(v), count));
            return 0;
        } catch (...) {
            s->errs.record(std::current_exception());
            return 1;
        }
    };
    const falcon_status rc = falcon_decompress_stream(detail::context(), detail::prec<T>, archive.data(),
                                                      archive.size(), put, &st, &copt, &cst);
    st.errs.rethrow();
    detail::check(rc);
    return {cst.batches, cst.values, cst.blocking_waits};
}

// decompress_to_vector (pipeline.hpp:469-476)
template <typename T>
std::vector<T> decompress_to_vector(std::span<const std::uint8_t> archive, const pipeline_options& opt = {}) {
    const archive_header h = read_header(archive);
    std::vector<T> out(h.total_values);
    const falcon_pipeline_options copt = detail::to_c(opt);
    std::uint64_t n = 0;
    detail::check(falcon_decompress_host(detail::context(), detail::prec<T>, archive.data(), archive.size(),
                                         out.data(), out.size(), &n, &copt, nullptr));
    return out;
}

template <typename T>
constexpr std::size_t max_encoded_chunk_size(std::size_t n) noexcept {
    return 3 + sizeof(T) + (sizeof(T) * 8 + 7) / 8 + sizeof(T) * 8 * ((n - 1) / 8);
}

// chunk_workspace (chunk_codec.hpp:43-48): the reference keeps its lane and plane scratch
// here so steady-state calls allocate nothing.  On the GPU the scratch (device input and
// output buffers) lives in the library context and is reused across calls; the workspace
// keeps a host staging vector for the encoded bytes.
template <typename T>
struct chunk_workspace {
    std::vector<std::uint8_t> enc;
};

// compress_chunk (chunk_codec.hpp:50-74): appends the encoded chunk to `out`
template <typename T>
void compress_chunk(std::span<const T> values, chunk_workspace<T>& ws, std::vector<std::uint8_t>& out) {
    ws.enc.resize(max_encoded_chunk_size<T>(values.size()));
    std::uint64_t len = 0;
    detail::check(falcon_compress_chunk(detail::context(), detail::prec<T>, values.data(),
                                        static_cast<std::uint32_t>(values.size()), ws.enc.data(), ws.enc.size(),
                                        &len));
    out.insert(out.end(), ws.enc.begin(), ws.enc.begin() + static_cast<std::ptrdiff_t>(len));
}

template <typename T>
std::vector<std::uint8_t> compress_chunk(std::span<const T> values) {
    chunk_workspace<T> ws;
    std::vector<std::uint8_t> out;
    compress_chunk<T>(values, ws, out);
    return out;
}

// decompress_chunk (chunk_codec.hpp:86-122): `in` spans exactly one encoded chunk; `out`
// is resized to `count` values (the padded tail of a final chunk is dropped)
template <typename T>
void decompress_chunk(std::span<const std::uint8_t> in, std::size_t n, std::size_t count, chunk_workspace<T>&,
                      std::vector<T>& out) {
    if (count > n) throw error("decompress_chunk: count exceeds chunk capacity");
    out.resize(count);
    detail::check(falcon_decompress_chunk(detail::context(), detail::prec<T>, in.data(), in.size(),
                                          static_cast<std::uint32_t>(n), static_cast<std::uint32_t>(count),
                                          out.data()));
}

template <typename T>
std::vector<T> decompress_chunk(std::span<const std::uint8_t> in, std::size_t n, std::size_t count) {
    chunk_workspace<T> ws;
    std::vector<T> out;
    decompress_chunk<T>(in, n, count, ws, out);
    return out;
}

}  // namespace falcon_b200
