// Conformance of the C++ drop-in (include/falcon_b200/falcon.hpp) with the reference's
// own pipeline tests (proj/tests/test_pipeline.cpp:85-353, test_chunk_codec.cpp:32-70):
// same bytes as the sequential reference archive for any stream/worker count, same
// exceptions and messages, sink coverage, jitter, the blocking-wait safeguard.
#include <atomic>
#include <chrono>
#include <cstdio>
#include <mutex>
#include <random>
#include <thread>

#include "falcon_b200/falcon.hpp"
#include "falcon_oracle.h"

namespace fb = falcon_b200;

static int g_failures = 0, g_checks = 0;
#define CHECK(cond)                                                               \
    do {                                                                          \
        ++g_checks;                                                               \
        if (!(cond)) {                                                            \
            ++g_failures;                                                         \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);           \
        }                                                                         \
    } while (0)
#define CHECK_THROWS_WITH(expr, type, msg)                                        \
    do {                                                                          \
        ++g_checks;                                                               \
        bool ok_ = false;                                                         \
        try {                                                                     \
            (void)(expr);                                                         \
        } catch (const type& e_) {                                                \
            ok_ = std::string(e_.what()) == (msg);                                \
            if (!ok_) std::printf("  got message: %s\n", e_.what());              \
        } catch (...) {                                                           \
        }                                                                         \
        if (!ok_) {                                                               \
            ++g_failures;                                                         \
            std::printf("FAIL %s:%d: %s did not throw %s(\"%s\")\n", __FILE__, __LINE__, #expr, #type, msg); \
        }                                                                         \
    } while (0)

template <typename T>
static std::vector<std::uint8_t> reference_archive(const std::vector<T>& v, std::uint32_t n, std::uint64_t bv) {
    const int prec = sizeof(T) == 8 ? 0 : 1;
    std::vector<std::uint8_t> out(or_compress_bound(prec, v.size(), n, bv));
    std::uint64_t len = 0;
    if (or_compress_archive(prec, v.data(), v.size(), n, bv, out.data(), out.size(), &len)) std::abort();
    out.resize(len);
    return out;
}

static std::vector<double> mixed_values(std::size_t total, std::uint64_t seed) {
    std::vector<double> v(total);
    const int kinds[] = {OR_KIND_WALK, OR_KIND_DECIMAL, OR_KIND_BITS, OR_KIND_SIGNFLIP, OR_KIND_OUTLIER};
    const std::size_t slice = total / 5 + 1;
    std::size_t at = 0;
    for (int k : kinds) {
        const std::size_t m = std::min(slice, total - at);
        or_spec s{k, 2, seed + (std::uint64_t)k, 127, 1025, 3575, 1025};
        if (m) or_synth_fill(0, &s, v.data() + at, m);
        at += m;
    }
    return v;
}

template <typename T>
static bool same_bits(const std::vector<T>& a, const std::vector<T>& b) {
    return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(T)) == 0;
}

struct recording_sink final : fb::value_sink<double> {
    void put(std::uint64_t first, std::span<const double> v) override {
        std::lock_guard<std::mutex> l(m);
        calls.emplace_back(first, v.size());
    }
    std::mutex m;
    std::vector<std::pair<std::uint64_t, std::size_t>> calls;
};

int main() {
    // option validation (test_pipeline.cpp:95-107)
    {
        std::vector<double> vals(10, 1.0);
        fb::pipeline_options opt;
        opt.chunk_n = 64;
        fb::memory_source<double> s1(vals);
        CHECK_THROWS_WITH(fb::compress_pipeline<double>(s1, opt), fb::error, "chunk length must be a multiple of 64 plus one");
        opt.chunk_n = 1025;
        opt.batch_values = 0;
        fb::memory_source<double> s2(vals);
        CHECK_THROWS_WITH(fb::compress_pipeline<double>(s2, opt), fb::error, "batch size must be positive");
        opt.batch_values = 1025;
        opt.n_streams = 0;
        fb::memory_source<double> s3(vals);
        CHECK_THROWS_WITH(fb::compress_pipeline<double>(s3, opt), fb::error, "stream count must be positive");
    }
    // empty input yields a bare header (109-122)
    {
        std::vector<double> vals;
        fb::memory_source<double> src(vals);
        fb::pipeline_stats st;
        const auto a = fb::compress_pipeline<double>(src, fb::pipeline_options{}, &st);
        CHECK(a.size() == fb::archive_header_bytes);
        CHECK(st.batches == 0 && st.values == 0);
        CHECK(fb::read_header(a).total_values == 0);
        CHECK(fb::decompress_to_vector<double>(a).empty());
    }
    // single stream reproduces the sequential reference bytes (124-138)
    {
        const auto vals = mixed_values(5 * 1025 + 400, 17);
        const auto expect = reference_archive(vals, 1025, 2 * 1025);
        fb::memory_source<double> src(vals);
        fb::pipeline_options opt;
        opt.batch_values = 2 * 1025;
        opt.n_streams = 1;
        opt.workers = 1;
        fb::pipeline_stats st;
        CHECK(fb::compress_pipeline<double>(src, opt, &st) == expect);
        CHECK(st.batches == 3 && st.values == vals.size());
    }
    // stream and worker counts never change the bytes (140-154)
    {
        const auto vals = mixed_values(37 * 1025 + 11, 23);
        const auto expect = reference_archive(vals, 1025, 3 * 1025);
        for (unsigned streams : {1u, 2u, 5u, 16u})
            for (unsigned workers : {1u, 3u, 8u}) {
                fb::memory_source<double> src(vals);
                fb::pipeline_options opt;
                opt.batch_values = 3 * 1025;
                opt.n_streams = streams;
                opt.workers = workers;
                CHECK(fb::compress_pipeline<double>(src, opt) == expect);
            }
    }
    // round trip with specials (156-173)
    {
        std::vector<double> vals = {0.0, -0.0, 1.0 / 0.0, -1.0 / 0.0, 5e-324, 1.7976931348623157e308, 1.0, -1.0};
        const auto tail = mixed_values(9000, 5);
        vals.insert(vals.end(), tail.begin(), tail.end());
        double nan = 0;
        const std::uint64_t nb = 0x7ff8000000000123ull;
        std::memcpy(&nan, &nb, 8);
        vals.push_back(nan);
        fb::memory_source<double> src(vals);
        fb::pipeline_options opt;
        opt.batch_values = 2000;
        const auto a = fb::compress_pipeline<double>(src, opt);
        CHECK(a == reference_archive(vals, 1025, 2000));
        CHECK(same_bits(fb::decompress_to_vector<double>(a, opt), vals));
    }
    // sink coverage: every batch exactly once (175-192)
    {
        const auto vals = mixed_values(10 * 1025 + 3, 7);
        fb::memory_source<double> src(vals);
        fb::pipeline_options opt;
        opt.batch_values = 1025;
        const auto a = fb::compress_pipeline<double>(src, opt);
        recording_sink sink;
        const auto st = fb::decompress_pipeline<double>(a, sink, opt);
        CHECK(st.batches == 11);
        std::sort(sink.calls.begin(), sink.calls.end());
        CHECK(sink.calls.size() == 11);
        std::uint64_t next = 0;
        for (auto& [f, n] : sink.calls) {
            CHECK(f == next);
            next += n;
        }
        CHECK(next == vals.size());
    }
    // scheduling jitter never changes the bytes (194-216)
    {
        const auto vals = mixed_values(12 * 1025, 31);
        const auto expect = reference_archive(vals, 1025, 1025);
        std::mt19937_64 rng(99);
        std::mutex rm;
        for (int trial = 0; trial < 12; ++trial) {
            fb::pipeline_options opt;
            opt.batch_values = 1025;
            opt.n_streams = 4;
            opt.stage_delay = [&](int, unsigned, std::uint64_t) {
                unsigned us;
                {
                    std::lock_guard<std::mutex> l(rm);
                    us = (unsigned)(rng() % 300);
                }
                std::this_thread::sleep_for(std::chrono::microseconds(us));
            };
            fb::memory_source<double> src(vals);
            CHECK(fb::compress_pipeline<double>(src, opt) == expect);
            fb::memory_sink<double> sink(vals.size());
            fb::decompress_pipeline<double>(expect, sink, opt);
            CHECK(same_bits(sink.values, vals));
        }
    }
    // a starved oldest slot engages the blocking-wait safeguard (236-252)
    {
        const auto vals = mixed_values(8 * 1025, 3);
        fb::pipeline_options opt;
        opt.batch_values = 1025;
        opt.n_streams = 4;
        opt.stage_delay = [](int stage, unsigned, std::uint64_t seq) {
            if (stage == fb::stage_compress && seq == 0) std::this_thread::sleep_for(std::chrono::milliseconds(50));
        };
        fb::memory_source<double> src(vals);
        fb::pipeline_stats st;
        CHECK(fb::compress_pipeline<double>(src, opt, &st) == reference_archive(vals, 1025, 1025));
        CHECK(st.blocking_waits > 0);
    }
    // precision mismatch (278-289)
    {
        const auto vals = mixed_values(3000, 1);
        fb::memory_source<double> src(vals);
        const auto a = fb::compress_pipeline<double>(src, fb::pipeline_options{});
        fb::memory_sink<float> sink(vals.size());
        CHECK_THROWS_WITH(fb::decompress_pipeline<float>(a, sink), fb::error,
                          "archive precision does not match the requested value type");
    }
    // corruption messages carry the batch index (291-334)
    {
        const auto vals = mixed_values(4 * 1025, 2);
        fb::pipeline_options opt;
        opt.batch_values = 1025;
        fb::memory_source<double> src(vals);
        auto a = fb::compress_pipeline<double>(src, opt);
        auto longer = a;
        longer.push_back(0);
        CHECK_THROWS_WITH(fb::decompress_to_vector<double>(longer, opt), fb::corrupt_error, "trailing bytes after final batch");
        auto cut = a;
        cut.resize(cut.size() - 3);
        CHECK_THROWS_WITH(fb::decompress_to_vector<double>(cut, opt), fb::corrupt_error, "batch payload truncated (batch 3)");
        auto badcount = a;
        badcount[47] = 2;  // batch 0 claims two chunks
        ++g_checks;
        try {
            (void)fb::decompress_to_vector<double>(badcount, opt);
            ++g_failures;
            std::printf("FAIL: corrupted chunk count accepted\n");
        } catch (const fb::corrupt_error& e) {
            if (std::string(e.what()).find("(batch ") == std::string::npos) {
                ++g_failures;
                std::printf("FAIL: no batch suffix: %s\n", e.what());
            }
        }
    }
    // f32 pipeline (336-353)
    {
        std::vector<float> vals(20000);
        or_spec s{OR_KIND_WALK, 1, 9, 127, 1025, 3575, 1025};
        or_synth_fill(1, &s, vals.data(), vals.size());
        fb::memory_source<float> src(vals);
        fb::pipeline_options opt;
        opt.batch_values = 4100;
        const auto a = fb::compress_pipeline<float>(src, opt);
        CHECK(a == reference_archive(vals, 1025, 4100));
        CHECK(same_bits(fb::decompress_to_vector<float>(a, opt), vals));
    }
    // chunk golden vectors (test_chunk_codec.cpp:32-70)
    {
        std::vector<double> z(1025, 0.0), c(1025, 2.5), sp(65, 0.0);
        sp[0] = 2.5;
        CHECK(fb::compress_chunk<double>(z) == std::vector<std::uint8_t>(11, 0));
        const auto e = fb::compress_chunk<double>(c);
        CHECK(e.size() == 11 && e[0] == 1 && e[1] == 2 && e[2] == 25);
        const std::vector<std::uint8_t> golden{0x01, 0x02, 25, 0, 0, 0, 0, 0, 0, 0, 0x06, 0x00,
                                               0x80, 0x80, 0x80, 0x80, 0x00, 0x00, 0x00, 0x80, 0x80};
        CHECK(fb::compress_chunk<double>(sp) == golden);
        CHECK(same_bits(fb::decompress_chunk<double>(golden, 65, 65), sp));
        CHECK_THROWS_WITH(fb::decompress_chunk<double>(golden, 65, 66), fb::error,
                          "decompress_chunk: count exceeds chunk capacity");
        auto bad = golden;
        bad[11] |= 0x40;
        CHECK_THROWS_WITH(fb::decompress_chunk<double>(bad, 65, 65), fb::corrupt_error, "nonzero flag padding bits");
        // workspace forms (chunk_codec.hpp:50-131): compress appends, decompress resizes,
        // one workspace reused across chunks of both kinds
        fb::chunk_workspace<double> ws;
        std::vector<std::uint8_t> stream{0xAB};
        fb::compress_chunk<double>(std::span<const double>(sp), ws, stream);
        fb::compress_chunk<double>(std::span<const double>(z), ws, stream);
        CHECK(stream.size() == 1 + golden.size() + 11 && stream[0] == 0xAB);
        CHECK(std::equal(golden.begin(), golden.end(), stream.begin() + 1));
        std::vector<double> back(7, -1.0);
        fb::decompress_chunk<double>(std::span<const std::uint8_t>(stream.data() + 1, golden.size()), 65, 40, ws,
                                     back);
        CHECK(back.size() == 40 && same_bits(back, std::vector<double>(sp.begin(), sp.begin() + 40)));
    }
    std::printf("%d checks, %d failures\n", g_checks, g_failures);
    return g_failures ? 1 : 0;
}
