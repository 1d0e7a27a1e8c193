// falcon -- command-line front end of the B200 codec.
//
// Subcommands, flags and the key=value report follow the reference tool
// (proj/tools/falcon_cli.cpp:251-512; FORMAT.md), so scripts and archives move freely
// between the two:
//
//   falcon compress   IN OUT   [--precision 64|32] [--format raw|csv] [--column N]
//   falcon decompress IN OUT   [--format raw|csv]
//   falcon verify     ORIGINAL ARCHIVE
//   falcon inspect    ARCHIVE
//   falcon gen        OUT      [--kind K] [--count N] [--seed S] [--dp D] ...
//   falcon bench               [--kind K] [--count N] [--device] [--reps R]
//   (+ --chunk-n --batch-values --streams --workers everywhere)
//
// Files are memory-mapped (raw inputs feed the pipeline without a copy); decompressed
// batches are written with pwrite at their value offset, so out-of-order sink calls from
// the pipeline's worker threads need no lock.  The codec goes through the drop-in header
// include/falcon_b200/falcon.hpp; synthetic data and the device bench through the C ABI.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <charconv>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "falcon_b200/falcon.hpp"

namespace fb = falcon_b200;

namespace {

// ---------------------------------------------------------------- report ----
// key=value lines in insertion order (the reference's report format)
class kv_report {
public:
    void add(const char* k, std::string v) { rows_.emplace_back(k, std::move(v)); }
    void add(const char* k, std::uint64_t v) { add(k, std::to_string(v)); }
    void add(const char* k, double v) {
        char b[48];
        std::snprintf(b, sizeof b, "%.6g", v);
        add(k, std::string(b));
    }
    void print() const {
        std::string out;
        for (const auto& [k, v] : rows_) out.append(k).append("=").append(v).append("\n");
        std::fwrite(out.data(), 1, out.size(), stdout);
    }

private:
    std::vector<std::pair<std::string, std::string>> rows_;
};

// ------------------------------------------------------------------ files ----
class mapped_file {
public:
    explicit mapped_file(const std::string& path) {
        fd_ = ::open(path.c_str(), O_RDONLY);
        if (fd_ < 0) throw fb::io_error("cannot open " + path);
        struct stat st {};
        if (::fstat(fd_, &st) != 0) throw fb::io_error("cannot stat " + path);
        size_ = static_cast<std::size_t>(st.st_size);
        if (size_) {
            void* p = ::mmap(nullptr, size_, PROT_READ, MAP_PRIVATE, fd_, 0);
            if (p == MAP_FAILED) throw fb::io_error("cannot map " + path);
            base_ = static_cast<const std::uint8_t*>(p);
            ::madvise(p, size_, MADV_SEQUENTIAL);
        }
    }
    ~mapped_file() {
        if (base_) ::munmap(const_cast<std::uint8_t*>(base_), size_);
        if (fd_ >= 0) ::close(fd_);
    }
    mapped_file(const mapped_file&) = delete;
    mapped_file& operator=(const mapped_file&) = delete;
    std::span<const std::uint8_t> bytes() const { return {base_ ? base_ : empty_, size_}; }

private:
    int fd_ = -1;
    const std::uint8_t* base_ = nullptr;
    std::size_t size_ = 0;
    static constexpr std::uint8_t empty_[1] = {0};
};

class out_file {
public:
    explicit out_file(const std::string& path) : path_(path) {
        fd_ = ::open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
        if (fd_ < 0) throw fb::io_error("cannot open " + path);
    }
    ~out_file() {
        if (fd_ >= 0) ::close(fd_);
    }
    out_file(const out_file&) = delete;
    out_file& operator=(const out_file&) = delete;
    // positional write: safe from several threads for disjoint ranges
    void write_at(std::uint64_t off, const void* p, std::size_t n) const {
        const auto* c = static_cast<const char*>(p);
        while (n) {
            const ssize_t w = ::pwrite(fd_, c, n, static_cast<off_t>(off));
            if (w <= 0) throw fb::io_error("write failed on " + path_);
            c += w;
            off += static_cast<std::uint64_t>(w);
            n -= static_cast<std::size_t>(w);
        }
    }

private:
    int fd_ = -1;
    std::string path_;
};

template <typename T>
std::span<const T> as_values(std::span<const std::uint8_t> b) {
    if (b.size() % sizeof(T) != 0) throw fb::io_error("input ends inside a value");
    return {reinterpret_cast<const T*>(b.data()), b.size() / sizeof(T)};
}

template <typename T>
struct pwrite_sink final : fb::value_sink<T> {
    const out_file& f;
    explicit pwrite_sink(const out_file& o) : f(o) {}
    void put(std::uint64_t first, std::span<const T> v) override {
        f.write_at(first * sizeof(T), v.data(), v.size_bytes());
    }
};

// compares each decoded batch with the mapped original (first mismatch wins)
template <typename T>
struct check_sink final : fb::value_sink<T> {
    std::span<const T> want;
    explicit check_sink(std::span<const T> w) : want(w) {}
    void put(std::uint64_t first, std::span<const T> v) override {
        if (first + v.size() > want.size()) throw fb::error("original file is shorter than the archive claims");
        if (std::memcmp(v.data(), want.data() + first, v.size_bytes()) == 0) return;
        for (std::size_t i = 0; i < v.size(); ++i)
            if (std::memcmp(&v[i], &want[first + i], sizeof(T)) != 0)
                throw fb::error("value mismatch at index " + std::to_string(first + i));
    }
};

// ------------------------------------------------------------------- csv ----
// One value per row from column `col` (comma separated); a first row that does not parse
// is a header and skipped, any later one is an error.
template <typename T>
std::vector<T> parse_csv(std::span<const std::uint8_t> text, unsigned col) {
    std::vector<T> out;
    const char* p = reinterpret_cast<const char*>(text.data());
    const char* const end = p + text.size();
    bool first_row = true;
    while (p < end) {
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<std::size_t>(end - p)));
        const char* row_end = nl ? nl : end;
        std::string_view row(p, static_cast<std::size_t>(row_end - p));
        p = nl ? nl + 1 : end;
        if (!row.empty() && row.back() == '\r') row.remove_suffix(1);
        if (row.empty()) continue;
        std::string_view cell = row;
        for (unsigned c = 0; c < col; ++c) {
            const auto k = cell.find(',');
            if (k == std::string_view::npos) throw fb::io_error("row has no column " + std::to_string(col));
            cell.remove_prefix(k + 1);
        }
        cell = cell.substr(0, cell.find(','));
        T v{};
        const auto r = std::from_chars(cell.data(), cell.data() + cell.size(), v);
        const bool ok = r.ec == std::errc{} && r.ptr == cell.data() + cell.size();
        if (!ok && !first_row) throw fb::io_error("cannot parse value: " + std::string(cell));
        if (ok) out.push_back(v);
        first_row = false;
    }
    return out;
}

// shortest round-trip text, one value per line
template <typename T>
void write_csv(const std::string& path, std::span<const T> values) {
    std::string buf;
    buf.reserve(values.size() * 12);
    char tmp[40];
    for (const T v : values) {
        const auto r = std::to_chars(tmp, tmp + sizeof tmp, v);
        buf.append(tmp, r.ptr).push_back('\n');
    }
    out_file(path).write_at(0, buf.data(), buf.size());
}

// ----------------------------------------------------------------- flags ----
struct cli_args {
    std::vector<std::string> files;
    std::map<std::string, std::string> flags;

    bool has(const char* k) const { return flags.count(k) != 0; }
    std::string text(const char* k, const char* dflt) const {
        const auto it = flags.find(k);
        return it == flags.end() ? dflt : it->second;
    }
    template <typename I>
    I number(const char* k, I dflt) const {
        const auto it = flags.find(k);
        if (it == flags.end()) return dflt;
        I v{};
        const auto& s = it->second;
        const auto r = std::from_chars(s.data(), s.data() + s.size(), v);
        if (r.ec != std::errc{} || r.ptr != s.data() + s.size())
            throw fb::error("--" + std::string(k) + ": not a number: " + s);
        return v;
    }
};

// flags that take a value; --device is the one switch
const char* const kValueFlags[] = {"precision", "format", "column", "chunk-n", "batch-values", "streams",
                                   "workers", "kind", "count", "seed", "dp", "step", "period", "spike", "reps"};

cli_args parse_args(int argc, char** argv) {
    cli_args a;
    for (int i = 2; i < argc; ++i) {
        std::string_view s = argv[i];
        if (s.substr(0, 2) != "--") {
            a.files.emplace_back(s);
            continue;
        }
        s.remove_prefix(2);
        std::string key(s.substr(0, s.find('=')));
        if (key == "device") {
            a.flags[key] = "1";
            continue;
        }
        if (std::none_of(std::begin(kValueFlags), std::end(kValueFlags), [&](const char* f) { return key == f; }))
            throw fb::error("unknown flag --" + key);
        if (s.find('=') != std::string_view::npos) {
            a.flags[key] = std::string(s.substr(s.find('=') + 1));
        } else {
            if (i + 1 >= argc) throw fb::error("flag --" + key + " needs a value");
            a.flags[key] = argv[++i];
        }
    }
    return a;
}

fb::pipeline_options pipeline_opts(const cli_args& a) {
    fb::pipeline_options o;
    o.chunk_n = a.number<std::uint32_t>("chunk-n", 1025);
    o.batch_values = a.number<std::uint64_t>("batch-values", 1025ull * 1024 * 4);
    o.n_streams = a.number<unsigned>("streams", 16);
    o.workers = a.number<unsigned>("workers", 0);
    return o;
}

bool wants_f64(const cli_args& a) {
    const unsigned bits = a.number<unsigned>("precision", 64);
    if (bits != 64 && bits != 32) throw fb::error("--precision must be 32 or 64");
    return bits == 64;
}

bool csv_format(const cli_args& a) {
    const std::string f = a.text("format", "raw");
    if (f != "raw" && f != "csv") throw fb::error("--format must be raw or csv");
    return f == "csv";
}

// synth::kind names (synthetic.hpp:14-20) plus this build's pinned kinds
falcon_synth_spec synth_spec(const cli_args& a) {
    static const std::pair<const char*, int> names[] = {
        {"random_walk", FALCON_KIND_WALK},      {"walk", FALCON_KIND_WALK},
        {"fixed_decimal", FALCON_KIND_DECIMAL}, {"decimal", FALCON_KIND_DECIMAL},
        {"sign_flip", FALCON_KIND_SIGNFLIP},    {"signflip", FALCON_KIND_SIGNFLIP},
        {"outlier_injected", FALCON_KIND_OUTLIER}, {"outlier", FALCON_KIND_OUTLIER},
        {"uniform_bits", FALCON_KIND_BITS},     {"bits", FALCON_KIND_BITS},
        {"mixed", FALCON_KIND_MIXED_BLOCKS},    {"field", FALCON_KIND_FIELD}};
    const std::string k = a.text("kind", "walk");
    const auto* hit = std::find_if(std::begin(names), std::end(names), [&](const auto& n) { return k == n.first; });
    if (hit == std::end(names)) throw fb::error("unknown kind: " + k);
    falcon_synth_spec sp{};
    sp.kind = hit->second;
    sp.decimal_places = a.number<int>("dp", 2);
    sp.seed = a.number<std::uint64_t>("seed", 1);
    sp.max_step_units = a.number<int>("step", 127);
    sp.outlier_period = a.number<std::uint64_t>("period", 1025);
    sp.outlier_units = a.number<std::int64_t>("spike", 3575);
    sp.block = a.number<std::uint32_t>("chunk-n", 1025);
    return sp;
}

template <typename T>
std::vector<T> synthesize(const falcon_synth_spec& sp, std::uint64_t n) {
    std::vector<T> v(n);
    fb::detail::check(falcon_synth_fill(fb::detail::prec<T>, &sp, v.data(), n));
    return v;
}

double since(std::chrono::steady_clock::time_point t) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t).count();
}

// -------------------------------------------------------------- commands ----
template <typename T>
int cmd_compress(const cli_args& a) {
    mapped_file in(a.files.at(0));
    std::vector<T> parsed;
    std::span<const T> values;
    if (csv_format(a)) {
        parsed = parse_csv<T>(in.bytes(), a.number<unsigned>("column", 0));
        values = parsed;
    } else {
        values = as_values<T>(in.bytes());
    }
    const auto t0 = std::chrono::steady_clock::now();
    fb::memory_source<T> src(values);
    fb::pipeline_stats st;
    const std::vector<std::uint8_t> arc = fb::compress_pipeline<T>(src, pipeline_opts(a), &st);
    const double dt = since(t0);
    out_file(a.files.at(1)).write_at(0, arc.data(), arc.size());
    const std::uint64_t raw = st.values * sizeof(T);
    kv_report r;
    r.add("values", st.values);
    r.add("batches", st.batches);
    r.add("raw_bytes", raw);
    r.add("archive_bytes", static_cast<std::uint64_t>(arc.size()));
    r.add("ratio", raw ? static_cast<double>(arc.size()) / static_cast<double>(raw) : 0.0);
    r.add("seconds", dt);
    r.add("mb_per_s", dt > 0 ? static_cast<double>(raw) / dt / 1e6 : 0.0);
    r.print();
    return 0;
}

template <typename T>
int cmd_decompress(const cli_args& a, std::span<const std::uint8_t> arc) {
    const auto t0 = std::chrono::steady_clock::now();
    std::uint64_t n = 0;
    if (csv_format(a)) {
        const std::vector<T> v = fb::decompress_to_vector<T>(arc, pipeline_opts(a));
        n = v.size();
        write_csv<T>(a.files.at(1), std::span<const T>(v));
    } else {
        out_file out(a.files.at(1));
        pwrite_sink<T> sink(out);
        n = fb::decompress_pipeline<T>(arc, sink, pipeline_opts(a)).values;
    }
    const double dt = since(t0);
    kv_report r;
    r.add("values", n);
    r.add("seconds", dt);
    r.add("mb_per_s", dt > 0 ? static_cast<double>(n * sizeof(T)) / dt / 1e6 : 0.0);
    r.print();
    return 0;
}

template <typename T>
int cmd_verify(const cli_args& a, std::span<const std::uint8_t> arc) {
    kv_report r;
    try {
        mapped_file orig(a.files.at(0));
        std::vector<T> parsed;
        std::span<const T> want;
        if (csv_format(a)) {
            parsed = parse_csv<T>(orig.bytes(), a.number<unsigned>("column", 0));
            want = parsed;
        } else {
            want = as_values<T>(orig.bytes());
        }
        check_sink<T> sink(want);
        const std::uint64_t n = fb::decompress_pipeline<T>(arc, sink, pipeline_opts(a)).values;
        // the count is checked for csv input only, as the reference tool does (a raw
        // original may run past the archive)
        if (!parsed.empty() && n != want.size())
            throw fb::error("value count mismatch: " + std::to_string(want.size()) + " in the original, " +
                            std::to_string(n) + " in the archive");
    } catch (const std::exception& e) {
        r.add("verify", std::string("mismatch"));
        r.add("detail", std::string(e.what()));
        r.print();
        return 1;
    }
    r.add("verify", std::string("ok"));
    r.print();
    return 0;
}

// header plus a frame walk (read_batch, container.cpp:113-132)
int cmd_inspect(const cli_args& a) {
    mapped_file f(a.files.at(0));
    const auto arc = f.bytes();
    const fb::archive_header h = fb::read_header(arc);
    const bool f64 = h.precision == fb::precision_tag::f64;
    auto le32 = [&](std::uint64_t at) {
        std::uint32_t v;
        std::memcpy(&v, arc.data() + at, 4);
        return v;
    };
    std::uint64_t pos = fb::archive_header_bytes, chunks = 0;
    std::uint32_t lo = UINT32_MAX, hi = 0;
    for (std::uint64_t b = 0; b < h.batch_count; ++b) {
        const std::uint64_t room = arc.size() - pos;
        if (room < 4) throw fb::corrupt_error("truncated batch header");
        const std::uint64_t cnt = le32(pos), table = 4 + 4 * cnt;
        if (room < table) throw fb::corrupt_error("truncated chunk size table");
        std::uint64_t payload = 0;
        for (std::uint64_t i = 0; i < cnt; ++i) {
            const std::uint32_t s = le32(pos + 4 + 4 * i);
            payload += s;
            lo = std::min(lo, s);
            hi = std::max(hi, s);
        }
        if (room - table < payload) throw fb::corrupt_error("truncated batch payload");
        pos += table + payload;
        chunks += cnt;
    }
    if (pos != arc.size()) throw fb::corrupt_error("trailing bytes after final batch");
    kv_report r;
    r.add("precision", std::string(f64 ? "64" : "32"));
    r.add("chunk_n", static_cast<std::uint64_t>(h.chunk_n));
    r.add("batch_values", h.batch_values);
    r.add("total_values", h.total_values);
    r.add("batch_count", h.batch_count);
    r.add("archive_bytes", static_cast<std::uint64_t>(arc.size()));
    const double raw = static_cast<double>(h.total_values) * (f64 ? 8.0 : 4.0);
    r.add("ratio", raw > 0 ? static_cast<double>(arc.size()) / raw : 0.0);
    r.add("chunks", chunks);
    if (chunks) {
        r.add("min_chunk_bytes", static_cast<std::uint64_t>(lo));
        r.add("max_chunk_bytes", static_cast<std::uint64_t>(hi));
    }
    r.print();
    return 0;
}

template <typename T>
int cmd_gen(const cli_args& a) {
    const std::uint64_t n = a.number<std::uint64_t>("count", 1000000);
    const std::vector<T> v = synthesize<T>(synth_spec(a), n);
    if (csv_format(a)) write_csv<T>(a.files.at(0), std::span<const T>(v));
    else out_file(a.files.at(0)).write_at(0, v.data(), v.size() * sizeof(T));
    kv_report r;
    r.add("values", n);
    r.add("kind", a.text("kind", "walk"));
    r.print();
    return 0;
}

void cuda_ok(cudaError_t e) {
    if (e != cudaSuccess) throw fb::error(std::string("CUDA: ") + cudaGetErrorString(e));
}

// median of the per-rep times of the HBM-resident kernels (CUDA events)
template <typename T>
std::pair<double, double> device_round_trips(const std::vector<T>& host, const fb::pipeline_options& o, int reps,
                                             std::uint64_t& archive_bytes) {
    const std::uint64_t n = host.size(), raw = n * sizeof(T);
    const std::uint64_t cap = falcon_compress_bound(fb::detail::prec<T>, n, o.chunk_n, o.batch_values);
    void *d_in = nullptr, *d_back = nullptr, *d_arc = nullptr;
    cuda_ok(cudaMalloc(&d_in, raw ? raw : 1));
    cuda_ok(cudaMalloc(&d_back, raw ? raw : 1));
    cuda_ok(cudaMalloc(&d_arc, cap));
    cuda_ok(cudaMemcpy(d_in, host.data(), raw, cudaMemcpyHostToDevice));
    cudaEvent_t ev[3];
    for (auto& e : ev) cuda_ok(cudaEventCreate(&e));
    std::vector<float> tc, td;
    falcon_ctx* ctx = fb::detail::context();
    for (int r = -2; r < reps; ++r) {
        std::uint64_t nv = 0;
        cuda_ok(cudaEventRecord(ev[0], nullptr));
        fb::detail::check(falcon_compress_device(ctx, fb::detail::prec<T>, d_in, n, o.chunk_n, o.batch_values,
                                                 d_arc, cap, &archive_bytes, nullptr));
        cuda_ok(cudaEventRecord(ev[1], nullptr));
        fb::detail::check(falcon_decompress_device(ctx, fb::detail::prec<T>, d_arc, archive_bytes, d_back, n, &nv,
                                                   nullptr));
        cuda_ok(cudaEventRecord(ev[2], nullptr));
        cuda_ok(cudaEventSynchronize(ev[2]));
        float a = 0, b = 0;
        cuda_ok(cudaEventElapsedTime(&a, ev[0], ev[1]));
        cuda_ok(cudaEventElapsedTime(&b, ev[1], ev[2]));
        if (r >= 0) {
            tc.push_back(a);
            td.push_back(b);
        }
    }
    std::vector<T> back(n);
    cuda_ok(cudaMemcpy(back.data(), d_back, raw, cudaMemcpyDeviceToHost));
    const bool same = std::memcmp(back.data(), host.data(), raw) == 0;
    for (auto& e : ev) cudaEventDestroy(e);
    cudaFree(d_in);
    cudaFree(d_back);
    cudaFree(d_arc);
    if (!same) throw fb::error("device round trip mismatch");
    std::nth_element(tc.begin(), tc.begin() + tc.size() / 2, tc.end());
    std::nth_element(td.begin(), td.begin() + td.size() / 2, td.end());
    return {tc[tc.size() / 2] / 1e3, td[td.size() / 2] / 1e3};
}

template <typename T>
int cmd_bench(const cli_args& a) {
    const std::uint64_t n = a.number<std::uint64_t>("count", 1000000);
    const std::vector<T> values = synthesize<T>(synth_spec(a), n);
    const fb::pipeline_options o = pipeline_opts(a);
    const bool device = a.has("device");
    double tc = 0, td = 0;
    std::uint64_t arc_bytes = 0, waits = 0;
    if (device) {
        const auto [c, d] = device_round_trips<T>(values, o, a.number<int>("reps", 10), arc_bytes);
        tc = c;
        td = d;
    } else {
        fb::memory_source<T> src(values);
        fb::pipeline_stats st;
        auto t = std::chrono::steady_clock::now();
        const auto arc = fb::compress_pipeline<T>(src, o, &st);
        tc = since(t);
        struct discard final : fb::value_sink<T> {
            void put(std::uint64_t, std::span<const T>) override {}
        } sink;
        t = std::chrono::steady_clock::now();
        fb::decompress_pipeline<T>(arc, sink, o);
        td = since(t);
        arc_bytes = arc.size();
        waits = st.blocking_waits;
    }
    const double raw = static_cast<double>(n * sizeof(T));
    kv_report r;
    r.add("kind", a.text("kind", "walk"));
    r.add("values", n);
    r.add("raw_bytes", n * sizeof(T));
    r.add("archive_bytes", arc_bytes);
    r.add("ratio", raw > 0 ? static_cast<double>(arc_bytes) / raw : 0.0);
    r.add("compress_seconds", tc);
    r.add("compress_mb_per_s", raw / tc / 1e6);
    r.add("decompress_seconds", td);
    r.add("decompress_mb_per_s", raw / td / 1e6);
    r.add("blocking_waits", waits);
    r.add("mode", std::string(device ? "device" : "host-pipeline"));
    r.print();
    return 0;
}

int usage() {
    std::fputs(
        "usage: falcon compress IN OUT | decompress IN OUT | verify ORIGINAL ARCHIVE |\n"
        "              inspect ARCHIVE | gen OUT | bench\n"
        "  --precision 32|64  --format raw|csv  --column N\n"
        "  --chunk-n N  --batch-values N  --streams N  --workers N\n"
        "  --kind K  --count N  --seed S  --dp D  --step S  --period P  --spike S\n"
        "  --device  --reps R   (bench: HBM-resident kernels timed with CUDA events)\n",
        stderr);
    return 2;
}

struct command {
    const char* name;
    std::size_t files;
    std::function<int(const cli_args&)> run;
};

// decompress / verify take their value type from the archive header
template <template <typename> class Fn>
int by_archive_precision(const cli_args& a, const std::string& archive_path) {
    mapped_file f(archive_path);
    const bool f64 = fb::read_header(f.bytes()).precision == fb::precision_tag::f64;
    return f64 ? Fn<double>::run(a, f.bytes()) : Fn<float>::run(a, f.bytes());
}
template <typename T> struct decompress_fn {
    static int run(const cli_args& a, std::span<const std::uint8_t> b) { return cmd_decompress<T>(a, b); }
};
template <typename T> struct verify_fn {
    static int run(const cli_args& a, std::span<const std::uint8_t> b) { return cmd_verify<T>(a, b); }
};

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage();
    const std::vector<command> commands = {
        {"compress", 2, [](const cli_args& a) { return wants_f64(a) ? cmd_compress<double>(a) : cmd_compress<float>(a); }},
        {"decompress", 2, [](const cli_args& a) { return by_archive_precision<decompress_fn>(a, a.files[0]); }},
        {"verify", 2, [](const cli_args& a) { return by_archive_precision<verify_fn>(a, a.files[1]); }},
        {"inspect", 1, [](const cli_args& a) { return cmd_inspect(a); }},
        {"gen", 1, [](const cli_args& a) { return wants_f64(a) ? cmd_gen<double>(a) : cmd_gen<float>(a); }},
        {"bench", 0, [](const cli_args& a) { return wants_f64(a) ? cmd_bench<double>(a) : cmd_bench<float>(a); }},
    };
    const std::string name = argv[1];
    const auto it = std::find_if(commands.begin(), commands.end(), [&](const command& c) { return name == c.name; });
    if (it == commands.end()) return usage();
    try {
        const cli_args a = parse_args(argc, argv);
        if (a.files.size() != it->files)
            throw fb::error(name + " takes " + std::to_string(it->files) + " file argument(s)");
        return it->run(a);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
