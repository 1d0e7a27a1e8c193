// capi.cu -- C ABI: library/context, format helpers, device-resident compress and
// decompress, per-chunk operators, synthetic inputs.  The host-resident multi-stream
// pipeline lives in pipeline.cu.
#include <mutex>
#include <random>

#include "field.cuh"
#include "runtime.h"

namespace fb200 {
const char* last_error_text();
}

using namespace fb200;

namespace {

struct device_guard {
    int prev = -1;
    explicit device_guard(int d) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != d) cudaSetDevice(d);
    }
    ~device_guard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

std::once_flag g_table_once[64];
cudaError_t g_table_err[64];

// misc scratch layout (ctx->misc, device)
constexpr size_t kEncTicket = 0, kEncError = 8, kEncTotal = 16, kDecTicket = 24, kDecAbort = 32,
                 kDecError = 40, kMiscBytes = 64;

uint8_t* misc_at(falcon_ctx* ctx, size_t off) { return ctx->misc.as<uint8_t>() + off; }

// A synchronous call reads its device error word and leaves it cleared, so a later
// falcon_ctx_sync on the context does not report the same error again.
falcon_status take_error(falcon_ctx* ctx, size_t off, cudaStream_t st, unsigned long long* err) {
    uint8_t* hb = ctx->host_box.as<uint8_t>();
    FB_CUDA(cudaMemcpyAsync(hb, misc_at(ctx, off), 8, cudaMemcpyDeviceToHost, st));
    FB_CUDA(cudaMemsetAsync(misc_at(ctx, off), 0xff, 8, st));
    FB_CUDA(cudaStreamSynchronize(st));
    std::memcpy(err, hb, 8);
    return FALCON_OK;
}

falcon_status error_from_device(unsigned long long word, uint64_t cpb, bool batch_suffix,
                                uint64_t first_batch = 0) {
    if (word == ~0ull) return FALCON_OK;
    const uint32_t code = (uint32_t)(word & 0xff);
    const uint64_t key = word >> 8;
    std::string msg = device_error_text(code);
    if (batch_suffix && code != DEV_E_TRAILING && code != DEV_E_CAPACITY && code != DEV_E_SCALE)
        msg += " (batch " + std::to_string(first_batch + key / cpb) + ")";
    return set_error(device_error_status(code), msg);
}

decode_ws ctx_decode_ws(falcon_ctx* ctx) {
    decode_ws ws;
    ws.ticket = reinterpret_cast<uint32_t*>(misc_at(ctx, kDecTicket));
    ws.ready = ctx->dec_ready.as<uint32_t>();
    ws.abort_at = reinterpret_cast<unsigned long long*>(misc_at(ctx, kDecAbort));
    ws.chunk_off = ctx->dec_off.as<uint64_t>();
    ws.chunk_size = ctx->dec_size.as<uint32_t>();
    ws.error = reinterpret_cast<unsigned long long*>(misc_at(ctx, kDecError));
    return ws;
}

falcon_status enqueue_compress(falcon_ctx* ctx, int prec, const void* d_values, uint64_t n,
                               uint32_t chunk_n, uint64_t bv, void* d_out, uint64_t cap,
                               uint64_t* d_total, cudaStream_t st, geometry& g, uint64_t header_bytes = 47) {
    FB_TRY(validate_options(chunk_n, bv));
    FB_TRY(make_geometry(n, chunk_n, bv, header_bytes, g));
    const size_t scratch = prec == FALCON_F64 ? encode_scratch_bytes<double>(g) : encode_scratch_bytes<float>(g);
    FB_TRY(ctx->enc_status.ensure(scratch));
    const archive_header_bytes hdr = header_bytes_of(prec, chunk_n, bv, n, g.n_batches);
    if (cap < header_bytes) return set_error(FALCON_ERR_CAPACITY, "output capacity too small for the header");
    uint32_t* ticket = reinterpret_cast<uint32_t*>(misc_at(ctx, kEncTicket));
    auto* err = reinterpret_cast<unsigned long long*>(misc_at(ctx, kEncError));
    uint64_t* total = d_total ? d_total : reinterpret_cast<uint64_t*>(misc_at(ctx, kEncTotal));
    const encode_ws ws = prec == FALCON_F64 ? carve_encode_ws<double>(ctx->enc_status.p, g, ticket, err, total)
                                            : carve_encode_ws<float>(ctx->enc_status.p, g, ticket, err, total);
    cudaError_t e = prec == FALCON_F64
                        ? launch_encode<double>(static_cast<const double*>(d_values), g,
                                                static_cast<uint8_t*>(d_out), cap, ws, hdr, st,
                                                ctx->prof_ev[0], ctx->prof_ev[1])
                        : launch_encode<float>(static_cast<const float*>(d_values), g,
                                               static_cast<uint8_t*>(d_out), cap, ws, hdr, st,
                                               ctx->prof_ev[0], ctx->prof_ev[1]);
    if (e != cudaSuccess) return set_error(FALCON_ERR_CUDA, std::string("encode launch: ") + cudaGetErrorString(e));
    return FALCON_OK;
}

falcon_status parse_header(const uint8_t* in, uint64_t len, falcon_archive_info* h) {
    // read_header (container.cpp:57-86)
    static const uint8_t magic[8] = {'F', 'A', 'L', 'C', 'O', 'N', 'A', 0};
    auto get = [&](int off, int bytes) {
        uint64_t v = 0;
        for (int i = 0; i < bytes; ++i) v |= (uint64_t)in[off + i] << (8 * i);
        return v;
    };
    if (len < 47) return set_error(FALCON_ERR_CORRUPT, "archive header truncated");
    if (std::memcmp(in, magic, 8) != 0) return set_error(FALCON_ERR_CORRUPT, "bad archive magic");
    if (get(8, 2) != 1) return set_error(FALCON_ERR_CORRUPT, "unsupported archive version");
    if (in[10] > 1) return set_error(FALCON_ERR_CORRUPT, "unknown precision tag");
    h->precision = in[10];
    h->chunk_n = (uint32_t)get(11, 4);
    if (h->chunk_n < 65 || (h->chunk_n - 1) % 64 != 0)
        return set_error(FALCON_ERR_CORRUPT, "invalid chunk length");
    h->batch_values = get(15, 8);
    h->total_values = get(23, 8);
    h->batch_count = get(31, 8);
    if (h->batch_values == 0 && h->total_values != 0)
        return set_error(FALCON_ERR_CORRUPT, "zero batch size with nonzero value count");
    if (h->batch_values != 0) {
        const uint64_t expect = (h->total_values + h->batch_values - 1) / h->batch_values;
        if (expect != h->batch_count)
            return set_error(FALCON_ERR_CORRUPT, "batch count disagrees with value count");
    } else if (h->batch_count != 0) {
        return set_error(FALCON_ERR_CORRUPT, "batch count disagrees with value count");
    }
    return FALCON_OK;
}

falcon_status enqueue_decompress(falcon_ctx* ctx, int prec, const void* d_archive, uint64_t bytes,
                                 const falcon_archive_info* info, void* d_values, uint64_t cap,
                                 cudaStream_t st, geometry& g, const uint64_t* d_bytes = nullptr) {
    if (info->precision != prec)
        return set_error(FALCON_ERR_INVALID, "archive precision does not match the requested value type");
    if (info->total_values > cap)
        return set_error(FALCON_ERR_CAPACITY, "value capacity too small for the archive");
    if (info->chunk_n > 4097)
        return set_error(FALCON_ERR_UNSUPPORTED,
                         "chunk_n > 4097 is not supported by the sm_100a kernels of this build");
    FB_TRY(make_geometry(info->total_values, info->chunk_n, info->batch_values ? info->batch_values : 1,
                         47, g));
    if (g.n_chunks == 0) {  // (a chained call cannot check the length of an empty archive)
        if (!d_bytes && bytes != 47) return set_error(FALCON_ERR_CORRUPT, "trailing bytes after final batch");
        return FALCON_OK;
    }
    FB_TRY(ctx->dec_off.ensure(g.n_chunks * sizeof(uint64_t)));
    FB_TRY(ctx->dec_size.ensure(g.n_chunks * sizeof(uint32_t)));
    FB_TRY(ctx->dec_ready.ensure(g.n_batches * sizeof(uint32_t)));
    ctx->dec_err_cpb = g.cpb;   // falcon_ctx_sync maps an async error's chunk to its batch
    ctx->dec_err_first = 0;
    const decode_ws ws = ctx_decode_ws(ctx);
    cudaError_t e = prec == FALCON_F64
                        ? launch_decode<double>(static_cast<const uint8_t*>(d_archive), bytes, g,
                                                static_cast<double*>(d_values), ws, st,
                                                ctx->prof_ev[2], ctx->prof_ev[3], d_bytes)
                        : launch_decode<float>(static_cast<const uint8_t*>(d_archive), bytes, g,
                                               static_cast<float*>(d_values), ws, st,
                                               ctx->prof_ev[2], ctx->prof_ev[3], d_bytes);
    if (e != cudaSuccess) return set_error(FALCON_ERR_CUDA, std::string("decode launch: ") + cudaGetErrorString(e));
    return FALCON_OK;
}

}  // namespace

// ============================================================================
extern "C" {

int falcon_abi_version(void) { return FALCON_B200_ABI_VERSION; }

const char* falcon_last_error(void) { return fb200::last_error_text(); }

void falcon_default_options(falcon_pipeline_options* opt) {
    // pipeline_options defaults (pipeline.hpp:70-79)
    opt->chunk_n = 1025;
    opt->batch_values = 1025ull * 1024 * 4;
    opt->n_streams = 16;
    opt->workers = 0;
    opt->stage_delay = nullptr;
    opt->stage_delay_user = nullptr;
}

falcon_status falcon_ctx_create(int device, falcon_ctx** out) {
    *out = nullptr;
    int count = 0;
    FB_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count || device >= 64)
        return set_error(FALCON_ERR_INVALID, "invalid CUDA device index");
    device_guard dg(device);
    std::call_once(g_table_once[device], [device] { g_table_err[device] = upload_tables(); });
    if (g_table_err[device] != cudaSuccess)
        return set_error(FALCON_ERR_CUDA, std::string("table upload: ") + cudaGetErrorString(g_table_err[device]));
    auto ctx = std::make_unique<falcon_ctx>();
    ctx->device = device;
    FB_TRY(ctx->misc.ensure(kMiscBytes));
    FB_CUDA(cudaMemset(ctx->misc.p, 0xff, kMiscBytes));
    FB_TRY(ctx->host_box.ensure(sizeof(slot_mailbox) * 4));
    *out = ctx.release();
    return FALCON_OK;
}

void falcon_ctx_destroy(falcon_ctx* ctx) {
    if (!ctx) return;
    device_guard dg(ctx->device);
    cudaDeviceSynchronize();
    delete ctx;
}

uint64_t falcon_max_encoded_chunk_size(int precision, uint32_t chunk_n) {
    return max_chunk_bytes(precision, chunk_n);
}

uint64_t falcon_compress_bound(int precision, uint64_t n_values, uint32_t chunk_n,
                               uint64_t batch_values) {
    if (chunk_n < 65 || batch_values == 0) return 0;
    uint64_t total = 47;
    const uint64_t batches = (n_values + batch_values - 1) / batch_values;
    if (batches == 0) return total;
    total += (batches - 1) * frame_bound(precision, batch_values, chunk_n);
    total += frame_bound(precision, n_values - (batches - 1) * batch_values, chunk_n);
    return total;
}

void falcon_write_header(const falcon_archive_info* info, uint8_t out[47]) {
    const archive_header_bytes h = header_bytes_of(info->precision, info->chunk_n, info->batch_values,
                                                   info->total_values, info->batch_count);
    std::memcpy(out, h.b, 47);
}

falcon_status falcon_read_header(const uint8_t* bytes, uint64_t len, falcon_archive_info* out) {
    return parse_header(bytes, len, out);
}

// ---- device-resident ----------------------------------------------------------
falcon_status falcon_compress_device_async(falcon_ctx* ctx, int precision, const void* d_values,
                                           uint64_t n_values, uint32_t chunk_n,
                                           uint64_t batch_values, void* d_out, uint64_t out_cap,
                                           uint64_t* d_out_bytes, void* stream) {
    FB_NVTX("falcon_compress_device_async");
    if (!ctx) return set_error(FALCON_ERR_INVALID, "null context");
    std::lock_guard<std::mutex> lock(ctx->api_mutex);
    device_guard dg(ctx->device);
    geometry g;
    return enqueue_compress(ctx, precision, d_values, n_values, chunk_n, batch_values, d_out, out_cap,
                            d_out_bytes, static_cast<cudaStream_t>(stream), g);
}

falcon_status falcon_compress_device_frames(falcon_ctx* ctx, int precision, const void* d_values,
                                            uint64_t n_values, uint32_t chunk_n, uint64_t batch_values,
                                            void* d_out, uint64_t out_cap, uint64_t* d_out_bytes, void* stream) {
    FB_NVTX("falcon_compress_device_frames");
    if (!ctx || !d_out_bytes) return set_error(FALCON_ERR_INVALID, "null argument");
    std::lock_guard<std::mutex> lock(ctx->api_mutex);
    device_guard dg(ctx->device);
    geometry g;
    return enqueue_compress(ctx, precision, d_values, n_values, chunk_n, batch_values, d_out, out_cap,
                            d_out_bytes, static_cast<cudaStream_t>(stream), g, 0);
}

falcon_status falcon_compress_device(falcon_ctx* ctx, int precision, const void* d_values,
                                     uint64_t n_values, uint32_t chunk_n, uint64_t batch_values,
                                     void* d_out, uint64_t out_cap, uint64_t* out_bytes,
                                     void* stream) {
    FB_NVTX("falcon_compress_device");
    if (!ctx) return set_error(FALCON_ERR_INVALID, "null context");
    std::lock_guard<std::mutex> lock(ctx->api_mutex);
    device_guard dg(ctx->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    FB_CUDA(cudaMemsetAsync(misc_at(ctx, kEncError), 0xff, 8, st));
    geometry g;
    FB_TRY(enqueue_compress(ctx, precision, d_values, n_values, chunk_n, batch_values, d_out, out_cap,
                            nullptr, st, g));
    slot_mailbox* box = ctx->host_box.as<slot_mailbox>();
    FB_CUDA(cudaMemcpyAsync(&box->total, misc_at(ctx, kEncTotal), 8, cudaMemcpyDeviceToHost, st));
    FB_CUDA(cudaMemcpyAsync(&box->error, misc_at(ctx, kEncError), 8, cudaMemcpyDeviceToHost, st));
    FB_CUDA(cudaMemsetAsync(misc_at(ctx, kEncError), 0xff, 8, st));
    FB_CUDA(cudaStreamSynchronize(st));
    FB_TRY(error_from_device(box->error, g.cpb, false));
    if (box->total > out_cap)
        return set_error(FALCON_ERR_CAPACITY, "output capacity too small for the compressed archive");
    if (out_bytes) *out_bytes = box->total;
    return FALCON_OK;
}

falcon_status falcon_decompress_device_async(falcon_ctx* ctx, int precision,
                                             const void* d_archive, uint64_t archive_bytes,
                                             const falcon_archive_info* info, void* d_values,
                                             uint64_t cap_values, void* stream) {
    FB_NVTX("falcon_decompress_device_async");
    if (!ctx || !info) return set_error(FALCON_ERR_INVALID, "null argument");
    std::lock_guard<std::mutex> lock(ctx->api_mutex);
    device_guard dg(ctx->device);
    geometry g;
    return enqueue_decompress(ctx, precision, d_archive, archive_bytes, info, d_values, cap_values,
                              static_cast<cudaStream_t>(stream), g);
}

falcon_status falcon_decompress_device_chained(falcon_ctx* ctx, int precision, const void* d_archive,
                                               const uint64_t* d_archive_bytes,
                                               const falcon_archive_info* info, void* d_values,
                                               uint64_t cap_values, void* stream) {
    FB_NVTX("falcon_decompress_device_chained");
    if (!ctx || !info || !d_archive_bytes) return set_error(FALCON_ERR_INVALID, "null argument");
    std::lock_guard<std::mutex> lock(ctx->api_mutex);
    device_guard dg(ctx->device);
    geometry g;
    return enqueue_decompress(ctx, precision, d_archive, 0, info, d_values, cap_values,
                              static_cast<cudaStream_t>(stream), g, d_archive_bytes);
}

falcon_status falcon_decompress_device(falcon_ctx* ctx, int precision, const void* d_archive,
                                       uint64_t archive_bytes, void* d_values,
                                       uint64_t cap_values, uint64_t* n_values, void* stream) {
    FB_NVTX("falcon_decompress_device");
    if (!ctx) return set_error(FALCON_ERR_INVALID, "null context");
    std::lock_guard<std::mutex> lock(ctx->api_mutex);
    device_guard dg(ctx->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint8_t* hb = ctx->host_box.as<uint8_t>();   // reuse pinned mailbox for the header
    FB_TRY(ctx->host_box.ensure(64));
    hb = ctx->host_box.as<uint8_t>();
    const uint64_t hl = archive_bytes < 47 ? archive_bytes : 47;
    if (hl) FB_CUDA(cudaMemcpyAsync(hb, d_archive, hl, cudaMemcpyDeviceToHost, st));
    FB_CUDA(cudaStreamSynchronize(st));
    uint8_t header[47];
    std::memcpy(header, hb, hl);
    falcon_archive_info info;
    FB_TRY(parse_header(header, archive_bytes, &info));
    FB_CUDA(cudaMemsetAsync(misc_at(ctx, kDecError), 0xff, 8, st));
    geometry g;
    FB_TRY(enqueue_decompress(ctx, precision, d_archive, archive_bytes, &info, d_values, cap_values, st, g));
    unsigned long long err = ~0ull;
    FB_TRY(take_error(ctx, kDecError, st, &err));
    FB_TRY(error_from_device(err, g.cpb, true));
    if (n_values) *n_values = info.total_values;
    return FALCON_OK;
}

falcon_status falcon_archive_index(falcon_ctx* ctx, const void* d_archive, uint64_t archive_bytes,
                                   const falcon_archive_info* info, uint64_t* d_index, void* stream) {
    FB_NVTX("falcon_archive_index");
    if (!ctx || !info || !d_index) return set_error(FALCON_ERR_INVALID, "null argument");
    std::lock_guard<std::mutex> lock(ctx->api_mutex);
    device_guard dg(ctx->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    FB_CUDA(cudaMemsetAsync(misc_at(ctx, kDecError), 0xff, 8, st));
    FB_CUDA(launch_index(static_cast<const uint8_t*>(d_archive), archive_bytes, 47, info->batch_count, d_index,
                         reinterpret_cast<unsigned long long*>(misc_at(ctx, kDecError)), st));
    unsigned long long err;
    FB_TRY(take_error(ctx, kDecError, st, &err));
    return error_from_device(err, 1, true);  // keys are batch numbers
}

falcon_status falcon_decompress_device_range(falcon_ctx* ctx, int precision, const void* d_archive,
                                             const falcon_archive_info* info, const uint64_t* index,
                                             uint64_t first_batch, uint64_t n_batches, void* d_values,
                                             uint64_t cap_values, uint64_t* n_values, void* stream) {
    FB_NVTX("falcon_decompress_device_range");
    if (!ctx || !info || !index) return set_error(FALCON_ERR_INVALID, "null argument");
    if (first_batch > info->batch_count || n_batches > info->batch_count - first_batch)
        return set_error(FALCON_ERR_INVALID, "batch range outside the archive");
    if (info->precision != precision)
        return set_error(FALCON_ERR_INVALID, "archive precision does not match the requested value type");
    std::lock_guard<std::mutex> lock(ctx->api_mutex);
    device_guard dg(ctx->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint64_t bv = info->batch_values;
    const uint64_t v0 = first_batch * bv;
    const uint64_t v1 = (first_batch + n_batches) * bv < info->total_values ? (first_batch + n_batches) * bv
                                                                           : info->total_values;
    const uint64_t count = n_batches ? v1 - v0 : 0;
    if (count > cap_values) return set_error(FALCON_ERR_CAPACITY, "value capacity too small for the batch range");
    if (n_values) *n_values = count;
    if (count == 0) return FALCON_OK;
    // the range's frames form a frames-only archive (no header) of `count` values
    const uint64_t start = index[first_batch], end = index[first_batch + n_batches];
    if (end < start) return set_error(FALCON_ERR_CORRUPT, "batch index is not increasing");
    geometry g;
    FB_TRY(make_geometry(count, info->chunk_n, bv, 0, g));
    FB_TRY(ctx->dec_off.ensure(g.n_chunks * sizeof(uint64_t)));
    FB_TRY(ctx->dec_size.ensure(g.n_chunks * sizeof(uint32_t)));
    FB_TRY(ctx->dec_ready.ensure(g.n_batches * sizeof(uint32_t)));
    FB_CUDA(cudaMemsetAsync(misc_at(ctx, kDecError), 0xff, 8, st));
    const decode_ws ws = ctx_decode_ws(ctx);
    const uint8_t* arc = static_cast<const uint8_t*>(d_archive) + start;
    cudaError_t e = precision == FALCON_F64
                        ? launch_decode<double>(arc, end - start, g, static_cast<double*>(d_values), ws, st)
                        : launch_decode<float>(arc, end - start, g, static_cast<float*>(d_values), ws, st);
    if (e != cudaSuccess) return set_error(FALCON_ERR_CUDA, std::string("decode launch: ") + cudaGetErrorString(e));
    unsigned long long err;
    FB_TRY(take_error(ctx, kDecError, st, &err));
    return error_from_device(err, g.cpb, true, first_batch);
}

falcon_status falcon_ctx_set_kernel_events(falcon_ctx* ctx, void* enc_start, void* enc_stop,
                                           void* dec_start, void* dec_stop) {
    if (!ctx) return set_error(FALCON_ERR_INVALID, "null context");
    std::lock_guard<std::mutex> lock(ctx->api_mutex);
    ctx->prof_ev[0] = static_cast<cudaEvent_t>(enc_start);
    ctx->prof_ev[1] = static_cast<cudaEvent_t>(enc_stop);
    ctx->prof_ev[2] = static_cast<cudaEvent_t>(dec_start);
    ctx->prof_ev[3] = static_cast<cudaEvent_t>(dec_stop);
    return FALCON_OK;
}

falcon_status falcon_ctx_sync(falcon_ctx* ctx, void* stream) {
    FB_NVTX("falcon_ctx_sync");
    if (!ctx) return set_error(FALCON_ERR_INVALID, "null context");
    std::lock_guard<std::mutex> lock(ctx->api_mutex);
    device_guard dg(ctx->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    unsigned long long errs[2];
    uint8_t* hb = ctx->host_box.as<uint8_t>();
    FB_CUDA(cudaMemcpyAsync(hb, misc_at(ctx, kEncError), 8, cudaMemcpyDeviceToHost, st));
    FB_CUDA(cudaMemcpyAsync(hb + 8, misc_at(ctx, kDecError), 8, cudaMemcpyDeviceToHost, st));
    FB_CUDA(cudaStreamSynchronize(st));
    std::memcpy(errs, hb, 16);
    FB_CUDA(cudaMemsetAsync(misc_at(ctx, kEncError), 0xff, 8, st));
    FB_CUDA(cudaMemsetAsync(misc_at(ctx, kDecError), 0xff, 8, st));
    FB_CUDA(cudaStreamSynchronize(st));
    // decode errors carry the reference's " (batch N)" suffix (pipeline.hpp:404-405,
    // 415-416), mapped through the geometry of the most recent async decode on ctx
    FB_TRY(error_from_device(errs[0], 1, false));
    FB_TRY(error_from_device(errs[1], ctx->dec_err_cpb, true, ctx->dec_err_first));
    return FALCON_OK;
}

falcon_status falcon_selftest_dp(falcon_ctx* ctx, int precision, const void* d_values, uint64_t n,
                                 int candidate_alpha, int8_t* d_full, int8_t* d_literal,
                                 int8_t* d_cert, int64_t* d_g, void* stream) {
    if (!ctx) return set_error(FALCON_ERR_INVALID, "null context");
    device_guard dg(ctx->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    FB_CUDA(launch_selftest_dp(precision, d_values, n, candidate_alpha, d_full, d_literal, d_cert, d_g, st));
    FB_CUDA(cudaStreamSynchronize(st));
    return FALCON_OK;
}

falcon_status falcon_selftest_div(falcon_ctx* ctx, int precision, const int64_t* d_g, uint64_t n, int alpha,
                                  void* d_out, void* stream) {
    if (!ctx) return set_error(FALCON_ERR_INVALID, "null context");
    if (alpha < 0 || alpha > (precision == 0 ? 21 : 9)) return set_error(FALCON_ERR_INVALID, "alpha out of range");
    device_guard dg(ctx->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    FB_CUDA(launch_selftest_div(precision, d_g, n, alpha, d_out, st));
    FB_CUDA(cudaStreamSynchronize(st));
    return FALCON_OK;
}

// ---- per-chunk operators ---------------------------------------------------------
falcon_status falcon_compress_chunk(falcon_ctx* ctx, int precision, const void* values,
                                    uint32_t chunk_n, uint8_t* out, uint64_t out_cap,
                                    uint64_t* out_len) {
    FB_NVTX("falcon_compress_chunk");
    if (!ctx) return set_error(FALCON_ERR_INVALID, "null context");
    FB_TRY(validate_options(chunk_n, chunk_n));
    const size_t esz = lane_bytes(precision);
    const uint64_t bound = falcon_compress_bound(precision, chunk_n, chunk_n, chunk_n);
    // device scratch reused across calls (chunk_workspace, chunk_codec.hpp:43-48)
    std::lock_guard<std::mutex> chunk_lock(ctx->chunk_mutex);
    device_buffer& din = ctx->chunk_a;
    device_buffer& dout = ctx->chunk_b;
    FB_TRY(din.ensure(chunk_n * esz));
    FB_TRY(dout.ensure(bound));
    {
        device_guard dg(ctx->device);
        FB_CUDA(cudaMemcpy(din.p, values, chunk_n * esz, cudaMemcpyHostToDevice));
    }
    uint64_t bytes = 0;
    FB_TRY(falcon_compress_device(ctx, precision, din.p, chunk_n, chunk_n, chunk_n, dout.p, bound,
                                  &bytes, nullptr));
    // archive = 47 header + [u32 1][u32 size] + chunk
    const uint64_t len = bytes - 47 - 8;
    if (len > out_cap) return set_error(FALCON_ERR_CAPACITY, "chunk output capacity too small");
    {
        device_guard dg(ctx->device);
        FB_CUDA(cudaMemcpy(out, dout.as<uint8_t>() + 47 + 8, len, cudaMemcpyDeviceToHost));
    }
    *out_len = len;
    return FALCON_OK;
}

falcon_status falcon_decompress_chunk(falcon_ctx* ctx, int precision, const uint8_t* in,
                                      uint64_t len, uint32_t chunk_n, uint32_t count, void* values) {
    FB_NVTX("falcon_decompress_chunk");
    if (!ctx) return set_error(FALCON_ERR_INVALID, "null context");
    if (count > chunk_n)  // chunk_codec.hpp:92-93
        return set_error(FALCON_ERR_INVALID, "decompress_chunk: count exceeds chunk capacity");
    if (len > 0xffffffffull) return set_error(FALCON_ERR_CORRUPT, "chunk size mismatch");
    // wrap the chunk in a one-chunk archive: the device decoder runs the exact
    // decompress_chunk validation; decode all chunk_n lanes, keep `count`
    std::vector<uint8_t> arc(47 + 8 + len);
    const archive_header_bytes h = header_bytes_of(precision, chunk_n, chunk_n, chunk_n, 1);
    std::memcpy(arc.data(), h.b, 47);
    const uint32_t one = 1, sz = (uint32_t)len;
    std::memcpy(arc.data() + 47, &one, 4);
    std::memcpy(arc.data() + 51, &sz, 4);
    if (len) std::memcpy(arc.data() + 55, in, len);
    const size_t esz = lane_bytes(precision);
    std::lock_guard<std::mutex> chunk_lock(ctx->chunk_mutex);
    device_buffer& darc = ctx->chunk_a;
    device_buffer& dval = ctx->chunk_b;
    FB_TRY(darc.ensure(arc.size()));
    FB_TRY(dval.ensure(chunk_n * esz));
    {
        device_guard dg(ctx->device);
        FB_CUDA(cudaMemcpy(darc.p, arc.data(), arc.size(), cudaMemcpyHostToDevice));
    }
    uint64_t nv = 0;
    falcon_status s = falcon_decompress_device(ctx, precision, darc.p, arc.size(), dval.p, chunk_n, &nv,
                                               nullptr);
    if (s != FALCON_OK) {
        // strip the synthetic " (batch 0)" suffix: chunk-level calls carry no batch index
        std::string m = falcon_last_error();
        const std::string suf = " (batch 0)";
        if (m.size() > suf.size() && m.compare(m.size() - suf.size(), suf.size(), suf) == 0)
            m.resize(m.size() - suf.size());
        return set_error(s, m);
    }
    {
        device_guard dg(ctx->device);
        if (count) FB_CUDA(cudaMemcpy(values, dval.p, count * esz, cudaMemcpyDeviceToHost));
    }
    return FALCON_OK;
}

// ---- synthetic generators (synthetic.hpp:36-115) ------------------------------------
falcon_status falcon_synth_fill_at(int precision, const falcon_synth_spec* s, uint64_t first, void* out,
                                   uint64_t count) {
    if (s->kind != FALCON_KIND_FIELD) {
        if (first != 0)
            return set_error(FALCON_ERR_INVALID, "only counter-based generator kinds start at an offset");
        return falcon_synth_fill(precision, s, out, count);
    }
    if (s->decimal_places < 0 || s->decimal_places > (precision == FALCON_F64 ? 22 : 10))
        return set_error(FALCON_ERR_INVALID, "decimal_places out of range for this precision");
    double p64 = 1;
    float p32 = 1;
    for (int i = 0; i < s->decimal_places; ++i) {
        p64 *= 10;
        p32 *= 10;
    }
    for (uint64_t i = 0; i < count; ++i) {
        const int64_t u = field_units(s->seed, first + i);
        if (precision == FALCON_F64) static_cast<double*>(out)[i] = (double)u / p64;
        else static_cast<float*>(out)[i] = (float)u / p32;
    }
    return FALCON_OK;
}

falcon_status falcon_synth_device(falcon_ctx* ctx, int precision, const falcon_synth_spec* s, uint64_t first,
                                  void* d_out, uint64_t count, void* stream) {
    FB_NVTX("falcon_synth_device");
    if (!ctx || !s) return set_error(FALCON_ERR_INVALID, "null argument");
    if (s->kind != FALCON_KIND_FIELD)
        return set_error(FALCON_ERR_UNSUPPORTED, "the device generator supports counter-based kinds only");
    if (s->decimal_places < 0 || s->decimal_places > (precision == FALCON_F64 ? 22 : 10))
        return set_error(FALCON_ERR_INVALID, "decimal_places out of range for this precision");
    device_guard dg(ctx->device);
    FB_CUDA(launch_field(precision, d_out, first, count, s->seed, s->decimal_places,
                         static_cast<cudaStream_t>(stream)));
    return FALCON_OK;
}

falcon_status falcon_synth_fill(int precision, const falcon_synth_spec* s, void* out, uint64_t count) {
    if (s->kind == FALCON_KIND_FIELD) return falcon_synth_fill_at(precision, s, 0, out, count);
    const int max_alpha = precision == FALCON_F64 ? 22 : 10;
    const int max_beta = precision == FALCON_F64 ? 15 : 6;
    if (s->decimal_places < 0 || s->decimal_places > max_alpha)
        return set_error(FALCON_ERR_INVALID, "decimal_places out of range for this precision");
    if (s->max_step_units < 1) return set_error(FALCON_ERR_INVALID, "max_step_units must be positive");
    std::mt19937_64 rng(s->seed);
    int64_t acc = (int64_t)(rng() % 20001) - 10000;
    uint64_t next_outlier = 0;
    if (s->kind == FALCON_KIND_OUTLIER) {
        if (s->outlier_period == 0) return set_error(FALCON_ERR_INVALID, "outlier_period must be positive");
        next_outlier = rng() % s->outlier_period;
    }
    if (s->kind == FALCON_KIND_MIXED_BLOCKS && s->block == 0)
        return set_error(FALCON_ERR_INVALID, "mixed-blocks generator needs a block length");
    double p64[23];
    float p32[11];
    {
        double d = 1;
        for (int i = 0; i < 23; ++i, d *= 10) p64[i] = d;
        float f = 1;
        for (int i = 0; i < 11; ++i, f *= 10) p32[i] = f;
    }
    auto emit = [&](uint64_t i, int64_t units, int dp) {
        if (precision == FALCON_F64) static_cast<double*>(out)[i] = (double)units / p64[dp];
        else static_cast<float*>(out)[i] = (float)units / p32[dp];
    };
    int dp_block = s->decimal_places;
    for (uint64_t i = 0; i < count; ++i) {
        switch (s->kind) {
        case FALCON_KIND_WALK:
        case FALCON_KIND_OUTLIER: {
            const int64_t span = 2 * (int64_t)s->max_step_units + 1;
            acc += (int64_t)(rng() % (uint64_t)span) - s->max_step_units;
            int64_t units = acc;
            if (s->kind == FALCON_KIND_OUTLIER && i == next_outlier) {
                units += s->outlier_units;
                next_outlier += s->outlier_period;
            }
            emit(i, units, s->decimal_places);
            break;
        }
        case FALCON_KIND_DECIMAL: {
            const int digits = 1 + (int)(rng() % (uint64_t)max_beta);
            int64_t lo = 1, hi = 10;
            for (int k = 1; k < digits; ++k) {
                lo *= 10;
                hi *= 10;
            }
            int64_t d = lo + (int64_t)(rng() % (uint64_t)(hi - lo));
            if (d % 10 == 0) ++d;
            if (rng() & 1) d = -d;
            emit(i, d, s->decimal_places);
            break;
        }
        case FALCON_KIND_SIGNFLIP: {
            const uint64_t r = rng();
            if (precision == FALCON_F64) {
                uint64_t b = (r & ((1ull << 52) - 1)) | (1023ull << 52) | ((i & 1) << 63);
                std::memcpy(static_cast<double*>(out) + i, &b, 8);
            } else {
                uint32_t b = ((uint32_t)r & ((1u << 23) - 1)) | (127u << 23) | ((uint32_t)(i & 1) << 31);
                std::memcpy(static_cast<float*>(out) + i, &b, 4);
            }
            break;
        }
        case FALCON_KIND_BITS: {
            const uint64_t r = rng();
            if (precision == FALCON_F64) std::memcpy(static_cast<double*>(out) + i, &r, 8);
            else {
                const uint32_t b = (uint32_t)r;
                std::memcpy(static_cast<float*>(out) + i, &b, 4);
            }
            break;
        }
        case FALCON_KIND_MIXED_BLOCKS: {
            // pinned cfg3 generator: reflecting walk in +/-999999 units,
            // decimal place redrawn from [1,6] every `block` values
            if (i % s->block == 0) dp_block = 1 + (int)(rng() % 6);
            const int64_t span = 2 * (int64_t)s->max_step_units + 1;
            acc += (int64_t)(rng() % (uint64_t)span) - s->max_step_units;
            if (acc > 999999) acc = 2 * 999999 - acc;
            if (acc < -999999) acc = -2 * 999999 - acc;
            emit(i, acc, dp_block);
            break;
        }
        default:
            return set_error(FALCON_ERR_INVALID, "unknown generator kind");
        }
    }
    return FALCON_OK;
}

}  // extern "C"
