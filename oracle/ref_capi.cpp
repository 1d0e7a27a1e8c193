// ref_capi.cpp -- C ABI over the UNMODIFIED reference library, so tests and the
// bench's CPU arm can drive it through ctypes.  TEST / BASELINE INFRASTRUCTURE ONLY.
//
// Built by oracle/Makefile against /root/reference/proj/include and
// /root/reference/proj/src/*.cpp (read in place, never copied) into
// oracle/_ref/libfalcon_ref.so.  Every call goes through the reference's own
// public entry points: compress_chunk / decompress_chunk (chunk_codec.hpp:50-131),
// compress_pipeline / decompress_pipeline (pipeline.hpp:156-467),
// dp_ds_calculate_counted (numeric.hpp:108-140), synth::generator (synthetic.hpp:36-115).
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "falcon/chunk_codec.hpp"
#include "falcon/container.hpp"
#include "falcon/pipeline.hpp"
#include "falcon/synthetic.hpp"

namespace {

// 0 ok, 1 falcon::error, 2 falcon::corrupt_error, 3 other exception
int classify(const std::exception& e, char* msg, std::size_t cap) {
    if (msg && cap) {
        std::strncpy(msg, e.what(), cap - 1);
        msg[cap - 1] = 0;
    }
    if (dynamic_cast<const falcon::corrupt_error*>(&e)) return 2;
    if (dynamic_cast<const falcon::error*>(&e)) return 1;
    return 3;
}

falcon::pipeline_options opts(std::uint32_t chunk_n, std::uint64_t bv, unsigned streams,
                              unsigned workers) {
    falcon::pipeline_options o;
    o.chunk_n = chunk_n;
    o.batch_values = bv;
    o.n_streams = streams;
    o.workers = workers;
    return o;
}

template<typename T>
int compress_pipe(const void* values, std::uint64_t count, std::uint32_t chunk_n,
                  std::uint64_t bv, unsigned streams, unsigned workers, std::uint8_t** out,
                  std::uint64_t* len, char* msg, std::size_t cap) {
    try {
        falcon::memory_source<T> src(std::span<const T>(static_cast<const T*>(values), count));
        auto a = falcon::compress_pipeline<T>(src, opts(chunk_n, bv, streams, workers));
        *out = static_cast<std::uint8_t*>(std::malloc(a.size() ? a.size() : 1));
        std::memcpy(*out, a.data(), a.size());
        *len = a.size();
        return 0;
    } catch (const std::exception& e) {
        return classify(e, msg, cap);
    }
}

struct ptr_sink_base {};

template<typename T>
struct ptr_sink final : falcon::value_sink<T> {
    T* dst;
    std::uint64_t cap;
    void put(std::uint64_t first, std::span<const T> v) override {
        if (first + v.size() <= cap)
            std::memcpy(dst + first, v.data(), v.size() * sizeof(T));
    }
};

template<typename T>
int decompress_pipe(const std::uint8_t* in, std::uint64_t len, void* values, std::uint64_t cap,
                    std::uint64_t* n_values, unsigned streams, unsigned workers, char* msg,
                    std::size_t mcap) {
    try {
        ptr_sink<T> sink;
        sink.dst = static_cast<T*>(values);
        sink.cap = cap;
        falcon::pipeline_options o;
        o.n_streams = streams;
        o.workers = workers;
        auto st = falcon::decompress_pipeline<T>(std::span<const std::uint8_t>(in, len), sink, o);
        *n_values = st.values;
        return 0;
    } catch (const std::exception& e) {
        return classify(e, msg, mcap);
    }
}

} // namespace

extern "C" {

unsigned ref_hardware_threads() {
    const unsigned hw = std::thread::hardware_concurrency();
    return hw ? hw : 1;
}

void ref_free(void* p) { std::free(p); }

int ref_dp_ds(int prec, double v, std::uint8_t* alpha, std::uint8_t* beta, int* iters) {
    if (prec == 0) {
        auto r = falcon::detail::dp_ds_calculate_counted<double>(v);
        *alpha = r.meta.alpha; *beta = r.meta.beta; *iters = r.iterations;
    } else {
        auto r = falcon::detail::dp_ds_calculate_counted<float>(static_cast<float>(v));
        *alpha = r.meta.alpha; *beta = r.meta.beta; *iters = r.iterations;
    }
    return 0;
}

int ref_floor_log10(int prec, double v) {
    return prec == 0 ? falcon::floor_log10<double>(v) : falcon::floor_log10<float>(static_cast<float>(v));
}

// Returns the encoded size, or 0 with msg set on error (never happens for valid n).
std::uint64_t ref_compress_chunk(int prec, const void* values, std::uint64_t n,
                                 std::uint8_t* out, std::uint64_t cap) {
    std::vector<std::uint8_t> enc;
    if (prec == 0)
        enc = falcon::compress_chunk<double>(std::span<const double>(static_cast<const double*>(values), n));
    else
        enc = falcon::compress_chunk<float>(std::span<const float>(static_cast<const float*>(values), n));
    if (enc.size() > cap) return 0;
    std::memcpy(out, enc.data(), enc.size());
    return enc.size();
}

int ref_decompress_chunk(int prec, const std::uint8_t* in, std::uint64_t len, std::uint64_t n,
                         std::uint64_t count, void* out, char* msg, std::size_t mcap) {
    try {
        if (prec == 0) {
            auto v = falcon::decompress_chunk<double>(std::span<const std::uint8_t>(in, len), n, count);
            std::memcpy(out, v.data(), v.size() * sizeof(double));
        } else {
            auto v = falcon::decompress_chunk<float>(std::span<const std::uint8_t>(in, len), n, count);
            std::memcpy(out, v.data(), v.size() * sizeof(float));
        }
        return 0;
    } catch (const std::exception& e) {
        return classify(e, msg, mcap);
    }
}

int ref_compress_pipeline(int prec, const void* values, std::uint64_t count, std::uint32_t chunk_n,
                          std::uint64_t bv, unsigned streams, unsigned workers, std::uint8_t** out,
                          std::uint64_t* len, char* msg, std::size_t mcap) {
    return prec == 0 ? compress_pipe<double>(values, count, chunk_n, bv, streams, workers, out, len, msg, mcap)
                     : compress_pipe<float>(values, count, chunk_n, bv, streams, workers, out, len, msg, mcap);
}

int ref_decompress_pipeline(int prec, const std::uint8_t* in, std::uint64_t len, void* values,
                            std::uint64_t cap, std::uint64_t* n_values, unsigned streams,
                            unsigned workers, char* msg, std::size_t mcap) {
    return prec == 0 ? decompress_pipe<double>(in, len, values, cap, n_values, streams, workers, msg, mcap)
                     : decompress_pipe<float>(in, len, values, cap, n_values, streams, workers, msg, mcap);
}

// Reference generators; kind is synth::kind's ordinal (synthetic.hpp:14-20).
int ref_synth_fill(int prec, int kind, int dp, std::uint64_t seed, int step,
                   std::uint64_t period, std::int64_t units, void* out, std::uint64_t count) {
    try {
        falcon::synth::spec s;
        s.kind = static_cast<falcon::synth::kind>(kind);
        s.decimal_places = dp;
        s.seed = seed;
        s.max_step_units = step;
        s.outlier_period = period;
        s.outlier_units = units;
        if (prec == 0) {
            falcon::synth::generator<double> g(s);
            g.fill(std::span<double>(static_cast<double*>(out), count));
        } else {
            falcon::synth::generator<float> g(s);
            g.fill(std::span<float>(static_cast<float*>(out), count));
        }
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

} // extern "C"
