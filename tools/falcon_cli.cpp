// falcon -- the reference CLI's front end (proj/tools/falcon_cli.cpp) on the B200 library.
//
//   falcon compress   data.raw data.fln --precision 64
//   falcon decompress data.fln data.raw
//   falcon verify     data.raw data.fln
//   falcon inspect    data.fln
//   falcon gen        data.raw --kind walk --count 1000000
//   falcon bench      --kind walk --count 10000000 [--device]
//
// Same subcommands, flags and key=value report as the reference (falcon_cli.cpp:251-512);
// archives are byte-identical, so files move freely between the two tools.  The codec
// calls go through the drop-in header include/falcon_b200/falcon.hpp (compress/decompress)
// and the C ABI (synthetic data, device-resident bench).  CLI11 is not vendored in the
// reference snapshot, so a small flag parser stands in for it.
#include <cuda_runtime.h>

#include <algorithm>
#include <charconv>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "falcon_b200/falcon.hpp"

using namespace falcon_b200;

namespace {

double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

std::vector<std::uint8_t> slurp(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw io_error("cannot open " + path);
    return std::vector<std::uint8_t>((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
}

void spill(const std::string& path, std::span<const std::uint8_t> bytes) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw io_error("cannot open " + path);
    out.write(reinterpret_cast<const char*>(bytes.data()), static_cast<std::streamsize>(bytes.size()));
    if (!out) throw io_error("write failed on " + path);
}

template <typename T>
class raw_file_source final : public value_source<T> {
public:
    explicit raw_file_source(const std::string& path) : in_(path, std::ios::binary) {
        if (!in_) throw io_error("cannot open " + path);
    }
    std::size_t read(std::span<T> dst) override {
        in_.read(reinterpret_cast<char*>(dst.data()), static_cast<std::streamsize>(dst.size() * sizeof(T)));
        const auto got = static_cast<std::size_t>(in_.gcount());
        if (got % sizeof(T) != 0) throw io_error("input ends inside a value");
        return got / sizeof(T);
    }

private:
    std::ifstream in_;
};

// out-of-order batches land at their value offset (falcon_cli.cpp:75-101)
template <typename T>
class raw_file_sink final : public value_sink<T> {
public:
    explicit raw_file_sink(const std::string& path) {
        std::ofstream(path, std::ios::binary | std::ios::trunc);
        out_.open(path, std::ios::binary | std::ios::in | std::ios::out);
        if (!out_) throw io_error("cannot open " + path);
    }
    void put(std::uint64_t first, std::span<const T> v) override {
        std::lock_guard lock(m_);
        out_.seekp(static_cast<std::streamoff>(first * sizeof(T)));
        out_.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(T)));
        if (!out_) throw io_error("write failed");
    }

private:
    std::mutex m_;
    std::fstream out_;
};

template <typename T>
std::uint64_t bits(T v) {
    if constexpr (sizeof(T) == 8) {
        std::uint64_t b;
        std::memcpy(&b, &v, 8);
        return b;
    } else {
        std::uint32_t b;
        std::memcpy(&b, &v, 4);
        return b;
    }
}

// compares decompressed batches against the original raw file (falcon_cli.cpp:103-132)
template <typename T>
class compare_sink final : public value_sink<T> {
public:
    explicit compare_sink(const std::string& path) : in_(path, std::ios::binary) {
        if (!in_) throw io_error("cannot open " + path);
    }
    void put(std::uint64_t first, std::span<const T> v) override {
        std::vector<T> expect(v.size());
        {
            std::lock_guard lock(m_);
            in_.clear();
            in_.seekg(static_cast<std::streamoff>(first * sizeof(T)));
            in_.read(reinterpret_cast<char*>(expect.data()), static_cast<std::streamsize>(expect.size() * sizeof(T)));
            if (static_cast<std::size_t>(in_.gcount()) != expect.size() * sizeof(T))
                throw error("original file is shorter than the archive claims");
        }
        for (std::size_t i = 0; i < v.size(); ++i)
            if (bits(v[i]) != bits(expect[i])) throw error("value mismatch at index " + std::to_string(first + i));
    }

private:
    std::mutex m_;
    std::ifstream in_;
};

template <typename T>
std::vector<T> load_csv(const std::string& path, unsigned column) {
    std::ifstream in(path);
    if (!in) throw io_error("cannot open " + path);
    std::vector<T> values;
    std::string line;
    bool first_line = true;
    while (std::getline(in, line)) {
        if (!line.empty() && line.back() == '\r') line.pop_back();
        if (line.empty()) continue;
        std::size_t begin = 0;
        for (unsigned c = 0; c < column; ++c) {
            const auto comma = line.find(',', begin);
            if (comma == std::string::npos) throw io_error("row has no column " + std::to_string(column));
            begin = comma + 1;
        }
        auto end = line.find(',', begin);
        if (end == std::string::npos) end = line.size();
        T v{};
        const auto r = std::from_chars(line.data() + begin, line.data() + end, v);
        if (r.ec != std::errc{} || r.ptr != line.data() + end) {
            if (first_line) {  // a header row is fine, anything later is not
                first_line = false;
                continue;
            }
            throw io_error("cannot parse value: " + line.substr(begin, end - begin));
        }
        first_line = false;
        values.push_back(v);
    }
    return values;
}

template <typename T>
void save_csv(const std::string& path, std::span<const T> values) {
    std::ofstream out(path, std::ios::trunc);
    if (!out) throw io_error("cannot open " + path);
    char buf[64];
    for (const T v : values) {
        const auto r = std::to_chars(buf, buf + sizeof buf, v);
        *r.ptr = '\n';
        out.write(buf, r.ptr + 1 - buf);
    }
    if (!out) throw io_error("write failed on " + path);
}

void report(const char* key, const std::string& value) { std::cout << key << "=" << value << "\n"; }
void report(const char* key, double value) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.6g", value);
    report(key, std::string(buf));
}
void report(const char* key, std::uint64_t value) { report(key, std::to_string(value)); }

// ---- flags ----
struct args {
    std::vector<std::string> pos;
    std::map<std::string, std::string> opt;
    bool has(const std::string& k) const { return opt.count(k) != 0; }
    std::string str(const std::string& k, const std::string& d) const { return has(k) ? opt.at(k) : d; }
    std::uint64_t u64(const std::string& k, std::uint64_t d) const { return has(k) ? std::stoull(opt.at(k)) : d; }
    std::int64_t i64(const std::string& k, std::int64_t d) const { return has(k) ? std::stoll(opt.at(k)) : d; }
};

args parse(int argc, char** argv, int from) {
    args a;
    for (int i = from; i < argc; ++i) {
        std::string s = argv[i];
        if (s.rfind("--", 0) == 0) {
            const auto eq = s.find('=');
            if (eq != std::string::npos) {
                a.opt[s.substr(2, eq - 2)] = s.substr(eq + 1);
            } else if (s == "--device") {
                a.opt["device"] = "1";
            } else {
                if (i + 1 >= argc) throw error("flag " + s + " needs a value");
                a.opt[s.substr(2)] = argv[++i];
            }
        } else {
            a.pos.push_back(s);
        }
    }
    return a;
}

pipeline_options codec_options(const args& a) {
    pipeline_options o;
    o.chunk_n = static_cast<std::uint32_t>(a.u64("chunk-n", 1025));
    o.batch_values = a.u64("batch-values", std::uint64_t{1025} * 1024 * 4);
    o.n_streams = static_cast<unsigned>(a.u64("streams", 16));
    o.workers = static_cast<unsigned>(a.u64("workers", 0));
    return o;
}

falcon_synth_spec spec_from(const args& a) {
    static const std::map<std::string, int> kinds = {
        {"walk", FALCON_KIND_WALK},         {"random_walk", FALCON_KIND_WALK},
        {"decimal", FALCON_KIND_DECIMAL},   {"fixed_decimal", FALCON_KIND_DECIMAL},
        {"signflip", FALCON_KIND_SIGNFLIP}, {"sign_flip", FALCON_KIND_SIGNFLIP},
        {"outlier", FALCON_KIND_OUTLIER},   {"outlier_injected", FALCON_KIND_OUTLIER},
        {"bits", FALCON_KIND_BITS},         {"uniform_bits", FALCON_KIND_BITS},
        {"mixed", FALCON_KIND_MIXED_BLOCKS}};
    const std::string k = a.str("kind", "walk");
    if (!kinds.count(k)) throw error("unknown kind: " + k);
    falcon_synth_spec sp{};
    sp.kind = kinds.at(k);
    sp.seed = a.u64("seed", 1);
    sp.decimal_places = static_cast<int>(a.i64("dp", 2));
    sp.max_step_units = static_cast<int>(a.i64("step", 127));
    sp.outlier_period = a.u64("period", 1025);
    sp.outlier_units = a.i64("spike", 3575);
    sp.block = static_cast<std::uint32_t>(a.u64("chunk-n", 1025));
    return sp;
}

template <typename T>
std::vector<T> synth_values(const falcon_synth_spec& sp, std::uint64_t count) {
    std::vector<T> v(count);
    detail::check(falcon_synth_fill(detail::prec<T>, &sp, v.data(), count));
    return v;
}

template <typename T>
int run_compress(const args& a) {
    const auto t0 = std::chrono::steady_clock::now();
    pipeline_stats stats;
    std::vector<std::uint8_t> archive;
    if (a.str("format", "raw") == "csv") {
        const auto values = load_csv<T>(a.pos.at(0), static_cast<unsigned>(a.u64("column", 0)));
        memory_source<T> src(values);
        archive = compress_pipeline<T>(src, codec_options(a), &stats);
    } else {
        raw_file_source<T> src(a.pos.at(0));
        archive = compress_pipeline<T>(src, codec_options(a), &stats);
    }
    const double dt = seconds_since(t0);
    spill(a.pos.at(1), archive);
    const std::uint64_t raw_bytes = stats.values * sizeof(T);
    report("values", stats.values);
    report("batches", stats.batches);
    report("raw_bytes", raw_bytes);
    report("archive_bytes", static_cast<std::uint64_t>(archive.size()));
    report("ratio", raw_bytes ? static_cast<double>(archive.size()) / raw_bytes : 0.0);
    report("seconds", dt);
    report("mb_per_s", dt > 0 ? raw_bytes / dt / 1e6 : 0.0);
    return 0;
}

template <typename T>
int run_decompress(const args& a, const std::vector<std::uint8_t>& archive) {
    const auto t0 = std::chrono::steady_clock::now();
    pipeline_stats stats;
    if (a.str("format", "raw") == "csv") {
        const auto values = decompress_to_vector<T>(archive, codec_options(a));
        stats.values = values.size();
        save_csv<T>(a.pos.at(1), std::span<const T>(values));
    } else {
        raw_file_sink<T> sink(a.pos.at(1));
        stats = decompress_pipeline<T>(archive, sink, codec_options(a));
    }
    const double dt = seconds_since(t0);
    report("values", stats.values);
    report("seconds", dt);
    report("mb_per_s", dt > 0 ? stats.values * sizeof(T) / dt / 1e6 : 0.0);
    return 0;
}

template <typename T>
int run_verify(const args& a, const std::vector<std::uint8_t>& archive) {
    try {
        if (a.str("format", "raw") == "csv") {
            const auto values = decompress_to_vector<T>(archive, codec_options(a));
            const auto expect = load_csv<T>(a.pos.at(0), static_cast<unsigned>(a.u64("column", 0)));
            if (values.size() != expect.size())
                throw error("value count mismatch: " + std::to_string(expect.size()) + " in the original, " +
                            std::to_string(values.size()) + " in the archive");
            for (std::size_t i = 0; i < values.size(); ++i)
                if (bits(values[i]) != bits(expect[i])) throw error("value mismatch at index " + std::to_string(i));
        } else {
            compare_sink<T> sink(a.pos.at(0));
            decompress_pipeline<T>(archive, sink, codec_options(a));
        }
    } catch (const std::exception& e) {
        report("verify", std::string("mismatch"));
        report("detail", std::string(e.what()));
        return 1;
    }
    report("verify", std::string("ok"));
    return 0;
}

std::uint32_t le32(const std::uint8_t* p) {
    return std::uint32_t(p[0]) | std::uint32_t(p[1]) << 8 | std::uint32_t(p[2]) << 16 | std::uint32_t(p[3]) << 24;
}

// header + frame walk (falcon_cli.cpp:327-361; read_batch, container.cpp:113-132)
int run_inspect(const args& a) {
    const auto archive = slurp(a.pos.at(0));
    const archive_header h = read_header(archive);
    report("precision", std::string(h.precision == precision_tag::f64 ? "64" : "32"));
    report("chunk_n", static_cast<std::uint64_t>(h.chunk_n));
    report("batch_values", h.batch_values);
    report("total_values", h.total_values);
    report("batch_count", h.batch_count);
    report("archive_bytes", static_cast<std::uint64_t>(archive.size()));
    const std::size_t width = h.precision == precision_tag::f64 ? 8 : 4;
    report("ratio", h.total_values ? static_cast<double>(archive.size()) / (h.total_values * width) : 0.0);
    std::size_t cursor = archive_header_bytes;
    std::uint64_t chunks = 0;
    std::uint32_t min_chunk = ~std::uint32_t{0}, max_chunk = 0;
    for (std::uint64_t b = 0; b < h.batch_count; ++b) {
        const std::size_t left = archive.size() - cursor;
        if (left < 4) throw corrupt_error("truncated batch header");
        const std::uint32_t count = le32(archive.data() + cursor);
        if (left < 4 + 4 * std::uint64_t{count}) throw corrupt_error("truncated chunk size table");
        std::uint64_t payload = 0;
        for (std::uint32_t i = 0; i < count; ++i) {
            const std::uint32_t s = le32(archive.data() + cursor + 4 + 4 * std::uint64_t{i});
            payload += s;
            min_chunk = std::min(min_chunk, s);
            max_chunk = std::max(max_chunk, s);
        }
        if (left - 4 - 4 * std::uint64_t{count} < payload) throw corrupt_error("truncated batch payload");
        cursor += 4 + 4 * std::size_t{count} + payload;
        chunks += count;
    }
    if (cursor != archive.size()) throw corrupt_error("trailing bytes after final batch");
    report("chunks", chunks);
    if (chunks) {
        report("min_chunk_bytes", static_cast<std::uint64_t>(min_chunk));
        report("max_chunk_bytes", static_cast<std::uint64_t>(max_chunk));
    }
    return 0;
}

template <typename T>
int run_gen(const args& a) {
    const std::uint64_t count = a.u64("count", 1000000);
    const auto sp = spec_from(a);
    const auto values = synth_values<T>(sp, count);
    if (a.str("format", "raw") == "csv") {
        save_csv<T>(a.pos.at(0), std::span<const T>(values));
    } else {
        spill(a.pos.at(0), std::span<const std::uint8_t>(reinterpret_cast<const std::uint8_t*>(values.data()),
                                                          values.size() * sizeof(T)));
    }
    report("values", count);
    report("kind", a.str("kind", "walk"));
    return 0;
}

#define CUDA_OK(x)                                                                        \
    do {                                                                                  \
        cudaError_t e_ = (x);                                                             \
        if (e_ != cudaSuccess) throw error(std::string("CUDA: ") + cudaGetErrorString(e_)); \
    } while (0)

// host pipeline (as the reference's bench, falcon_cli.cpp:391-422), or with --device the
// HBM-resident kernels timed with CUDA events (median of --reps)
template <typename T>
int run_bench(const args& a) {
    const std::uint64_t count = a.u64("count", 1000000);
    const auto sp = spec_from(a);
    const auto values = synth_values<T>(sp, count);
    const auto opt = codec_options(a);
    const std::uint64_t raw_bytes = count * sizeof(T);
    double enc_dt, dec_dt;
    std::uint64_t archive_bytes, waits = 0;
    if (a.has("device")) {
        falcon_ctx* ctx = detail::context();
        T *d_in = nullptr, *d_out = nullptr;
        std::uint8_t* d_arc = nullptr;
        const std::uint64_t cap = falcon_compress_bound(detail::prec<T>, count, opt.chunk_n, opt.batch_values);
        CUDA_OK(cudaMalloc(&d_in, raw_bytes ? raw_bytes : 1));
        CUDA_OK(cudaMalloc(&d_out, raw_bytes ? raw_bytes : 1));
        CUDA_OK(cudaMalloc(&d_arc, cap));
        CUDA_OK(cudaMemcpy(d_in, values.data(), raw_bytes, cudaMemcpyHostToDevice));
        cudaEvent_t e0, e1, e2;
        CUDA_OK(cudaEventCreate(&e0));
        CUDA_OK(cudaEventCreate(&e1));
        CUDA_OK(cudaEventCreate(&e2));
        const int reps = static_cast<int>(a.u64("reps", 10));
        std::vector<float> te, td;
        std::uint64_t nb = 0;
        for (int r = 0; r < reps + 2; ++r) {
            CUDA_OK(cudaEventRecord(e0, nullptr));
            detail::check(falcon_compress_device(ctx, detail::prec<T>, d_in, count, opt.chunk_n, opt.batch_values, d_arc, cap,
                                                 &nb, nullptr));
            CUDA_OK(cudaEventRecord(e1, nullptr));
            std::uint64_t nv = 0;
            detail::check(falcon_decompress_device(ctx, detail::prec<T>, d_arc, nb, d_out, count, &nv, nullptr));
            CUDA_OK(cudaEventRecord(e2, nullptr));
            CUDA_OK(cudaEventSynchronize(e2));
            float a1, a2;
            CUDA_OK(cudaEventElapsedTime(&a1, e0, e1));
            CUDA_OK(cudaEventElapsedTime(&a2, e1, e2));
            if (r >= 2) {
                te.push_back(a1);
                td.push_back(a2);
            }
        }
        std::vector<T> back(count);
        CUDA_OK(cudaMemcpy(back.data(), d_out, raw_bytes, cudaMemcpyDeviceToHost));
        if (std::memcmp(back.data(), values.data(), raw_bytes) != 0) throw error("device round trip mismatch");
        std::sort(te.begin(), te.end());
        std::sort(td.begin(), td.end());
        enc_dt = te[te.size() / 2] / 1e3;
        dec_dt = td[td.size() / 2] / 1e3;
        archive_bytes = nb;
        cudaFree(d_in);
        cudaFree(d_out);
        cudaFree(d_arc);
    } else {
        memory_source<T> src(values);
        pipeline_stats stats;
        const auto t0 = std::chrono::steady_clock::now();
        const auto archive = compress_pipeline<T>(src, opt, &stats);
        enc_dt = seconds_since(t0);
        struct null_sink final : value_sink<T> {
            void put(std::uint64_t, std::span<const T>) override {}
        } sink;
        const auto t1 = std::chrono::steady_clock::now();
        decompress_pipeline<T>(archive, sink, opt);
        dec_dt = seconds_since(t1);
        archive_bytes = archive.size();
        waits = stats.blocking_waits;
    }
    report("kind", a.str("kind", "walk"));
    report("values", count);
    report("raw_bytes", raw_bytes);
    report("archive_bytes", archive_bytes);
    report("ratio", raw_bytes ? static_cast<double>(archive_bytes) / raw_bytes : 0.0);
    report("compress_seconds", enc_dt);
    report("compress_mb_per_s", raw_bytes / enc_dt / 1e6);
    report("decompress_seconds", dec_dt);
    report("decompress_mb_per_s", raw_bytes / dec_dt / 1e6);
    report("blocking_waits", waits);
    report("mode", std::string(a.has("device") ? "device" : "host-pipeline"));
    return 0;
}

int usage() {
    std::cerr << "usage: falcon {compress IN OUT | decompress IN OUT | verify ORIGINAL ARCHIVE | inspect ARCHIVE |\n"
                 "               gen OUT | bench} [--precision 32|64] [--format raw|csv] [--column N]\n"
                 "               [--chunk-n N] [--batch-values N] [--streams N] [--workers N]\n"
                 "               [--kind K] [--count N] [--seed S] [--dp D] [--step S] [--period P] [--spike S]\n"
                 "               [--device] [--reps R]\n";
    return 2;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage();
    const std::string cmd = argv[1];
    try {
        const args a = parse(argc, argv, 2);
        const bool f64 = a.u64("precision", 64) == 64;
        if (a.has("precision") && !(a.u64("precision", 64) == 64 || a.u64("precision", 64) == 32))
            throw error("--precision must be 32 or 64");
        auto need = [&](std::size_t k) {
            if (a.pos.size() != k) throw error(cmd + " takes " + std::to_string(k) + " file argument(s)");
        };
        if (cmd == "compress") {
            need(2);
            return f64 ? run_compress<double>(a) : run_compress<float>(a);
        }
        if (cmd == "decompress" || cmd == "verify") {
            need(2);
            const auto archive = slurp(cmd == "verify" ? a.pos[1] : a.pos[0]);
            const bool archive_f64 = read_header(archive).precision == precision_tag::f64;
            if (cmd == "decompress") return archive_f64 ? run_decompress<double>(a, archive) : run_decompress<float>(a, archive);
            return archive_f64 ? run_verify<double>(a, archive) : run_verify<float>(a, archive);
        }
        if (cmd == "inspect") {
            need(1);
            return run_inspect(a);
        }
        if (cmd == "gen") {
            need(1);
            return f64 ? run_gen<double>(a) : run_gen<float>(a);
        }
        if (cmd == "bench") return f64 ? run_bench<double>(a) : run_bench<float>(a);
        return usage();
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
