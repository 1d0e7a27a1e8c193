/*
 * falcon_b200.h -- C ABI of the B200-native Falcon codec (libfalcon_b200.so).
 *
 * Plain pointers and sizes only; no torch or C++ types cross this boundary.  Every
 * entry point replaces one reference interface (paths under /root/reference/proj):
 *
 *   falcon_compress_stream    <- falcon::compress_pipeline<T>(value_source<T>&,
 *                                   const pipeline_options&, pipeline_stats*)
 *                                   include/falcon/pipeline.hpp:156-159
 *   falcon_decompress_stream  <- falcon::decompress_pipeline<T>(span<const u8>,
 *                                   value_sink<T>&, const pipeline_options&)
 *                                   include/falcon/pipeline.hpp:370-373
 *   falcon_decompress_host    <- falcon::decompress_to_vector<T> (pipeline.hpp:469-476)
 *   falcon_compress_host      <- compress_pipeline over a memory_source (pipeline.hpp:37-52)
 *   falcon_compress_device    <- (new) device-resident form of compress_pipeline
 *   falcon_decompress_device  <- (new) device-resident form of decompress_pipeline
 *   falcon_compress_chunk     <- falcon::compress_chunk<T>   chunk_codec.hpp:50-82
 *   falcon_decompress_chunk   <- falcon::decompress_chunk<T> chunk_codec.hpp:86-131
 *   falcon_max_encoded_chunk_size <- max_encoded_chunk_size<T> chunk_codec.hpp:36-41
 *   falcon_write_header / falcon_read_header <- write_header / read_header
 *                                   src/container.cpp:44-86
 *   falcon_synth_fill         <- synth::generator<T>::fill   include/falcon/synthetic.hpp:36-115
 *
 * Errors: every call returns a falcon_status; the message of the last failure on the
 * calling thread is falcon_last_error().  The status maps onto the reference's
 * exception types (error.hpp:8-19): FALCON_ERR_INVALID -> falcon::error,
 * FALCON_ERR_CORRUPT -> falcon::corrupt_error, FALCON_ERR_IO -> falcon::io_error.
 * Messages are the reference's own texts, including the " (batch N)" suffix.
 *
 * Output bytes never depend on n_streams, workers or the GPU count (FORMAT.md:3-6).
 */
#ifndef FALCON_B200_H
#define FALCON_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FALCON_B200_ABI_VERSION 1

typedef enum {
    FALCON_OK = 0,
    FALCON_ERR_INVALID = 1,     /* falcon::error: bad options, precision mismatch, ... */
    FALCON_ERR_CORRUPT = 2,     /* falcon::corrupt_error: malformed archive bytes */
    FALCON_ERR_IO = 3,          /* falcon::io_error */
    FALCON_ERR_CUDA = 4,        /* CUDA runtime failure (message has the CUDA error) */
    FALCON_ERR_CALLBACK = 5,    /* a source/sink callback reported failure */
    FALCON_ERR_CAPACITY = 6,    /* caller-provided output buffer too small */
    FALCON_ERR_UNSUPPORTED = 7  /* valid but not supported by this build (chunk_n > 4097) */
} falcon_status;

typedef enum { FALCON_F64 = 0, FALCON_F32 = 1 } falcon_precision;  /* container.hpp:15 tag */

/* Pipeline stage ids for the stage_delay test hook (pipeline.hpp:66-68). */
#define FALCON_STAGE_COMPRESS 0
#define FALCON_STAGE_STORE 1
#define FALCON_STAGE_DECODE 2

/* pipeline_options (pipeline.hpp:70-79). */
typedef struct {
    uint32_t chunk_n;        /* values per chunk, 64k+1 (default 1025) */
    uint64_t batch_values;   /* values per batch (default 1025*1024*4) */
    uint32_t n_streams;      /* batches in flight (default 16) */
    uint32_t workers;        /* host threads for source/sink work (0 = FALCON_WORKERS / hw) */
    /* optional: runs right before a stage's completion is signalled (test hook) */
    void (*stage_delay)(void* user, int stage, unsigned slot, uint64_t seq);
    void* stage_delay_user;
} falcon_pipeline_options;

/* pipeline_stats (pipeline.hpp:81-85). */
typedef struct {
    uint64_t batches;
    uint64_t values;
    uint64_t blocking_waits;
} falcon_pipeline_stats;

/* archive_header (container.hpp:12-27). */
typedef struct {
    uint8_t precision;
    uint32_t chunk_n;
    uint64_t batch_values;
    uint64_t total_values;
    uint64_t batch_count;
} falcon_archive_info;

typedef struct falcon_ctx falcon_ctx;

/* value_source<T>::read (pipeline.hpp:21-27): fill up to max_values values at dst and
 * return how many were written; 0 = end of stream; < 0 = failure (the call then fails
 * with FALCON_ERR_CALLBACK after in-flight work drains). */
typedef int64_t (*falcon_read_fn)(void* user, void* dst, uint64_t max_values);
/* Archive writer used by falcon_compress_stream: called once per batch frame, in launch
 * order, with the frame's final archive offset; plus once with offset 0 for the 47-byte
 * header at the end.  Nonzero return = failure. */
typedef int (*falcon_store_fn)(void* user, uint64_t offset, const void* bytes, uint64_t len);
/* value_sink<T>::put (pipeline.hpp:29-35): one call per batch, possibly out of order and
 * from several host threads; the span is only valid during the call.  Nonzero = failure. */
typedef int (*falcon_put_fn)(void* user, uint64_t first_value, const void* values, uint64_t count);

/* ---- library / context ---- */
int falcon_abi_version(void);
const char* falcon_last_error(void);
void falcon_default_options(falcon_pipeline_options* opt);
falcon_status falcon_ctx_create(int device, falcon_ctx** out);
void falcon_ctx_destroy(falcon_ctx* ctx);

/* ---- format helpers (host only, no GPU) ---- */
uint64_t falcon_max_encoded_chunk_size(int precision, uint32_t chunk_n);
/* Worst-case archive size: 47 + sum_b (4 + 4*C_b + C_b * max_encoded_chunk_size). */
uint64_t falcon_compress_bound(int precision, uint64_t n_values, uint32_t chunk_n,
                               uint64_t batch_values);
void falcon_write_header(const falcon_archive_info* info, uint8_t out[47]);
falcon_status falcon_read_header(const uint8_t* bytes, uint64_t len, falcon_archive_info* out);

/* ---- device-resident (all pointers are device pointers on ctx's GPU) ---- */
/* Compress n_values values at d_values into d_out (capacity out_cap >= bound).  The
 * archive length is returned in *out_bytes (host); the call synchronises `stream`. */
falcon_status falcon_compress_device(falcon_ctx* ctx, int precision, const void* d_values,
                                     uint64_t n_values, uint32_t chunk_n, uint64_t batch_values,
                                     void* d_out, uint64_t out_cap, uint64_t* out_bytes,
                                     void* stream);
/* Asynchronous form: enqueues the work on `stream` and returns.  The archive length is
 * written to d_out_bytes (device u64).  Errors surface in falcon_ctx_sync(). */
falcon_status falcon_compress_device_async(falcon_ctx* ctx, int precision, const void* d_values,
                                           uint64_t n_values, uint32_t chunk_n,
                                           uint64_t batch_values, void* d_out, uint64_t out_cap,
                                           uint64_t* d_out_bytes, void* stream);
/* Frames only: the batch frames of n_values values with no 47-byte header -- one shard of
 * a larger archive (frames are context-free, container.cpp:88-111).  Asynchronous like
 * falcon_compress_device_async; the byte total goes to d_out_bytes (device u64). */
falcon_status falcon_compress_device_frames(falcon_ctx* ctx, int precision, const void* d_values,
                                            uint64_t n_values, uint32_t chunk_n,
                                            uint64_t batch_values, void* d_out, uint64_t out_cap,
                                            uint64_t* d_out_bytes, void* stream);
/* Decompress the archive at d_archive (archive_bytes long) into d_values (cap_values).
 * Reads the header back to the host first; synchronises `stream`. */
falcon_status falcon_decompress_device(falcon_ctx* ctx, int precision, const void* d_archive,
                                       uint64_t archive_bytes, void* d_values,
                                       uint64_t cap_values, uint64_t* n_values, void* stream);
/* Asynchronous form for a caller that already holds the parsed header. */
falcon_status falcon_decompress_device_async(falcon_ctx* ctx, int precision,
                                             const void* d_archive, uint64_t archive_bytes,
                                             const falcon_archive_info* info, void* d_values,
                                             uint64_t cap_values, void* stream);
/* Chained form: the archive length is read on the device from d_archive_bytes (e.g. the
 * d_out_bytes of falcon_compress_device_async on the same stream), so a compress ->
 * decompress chain runs without a host round trip (device-resident form of
 * decompress_pipeline, pipeline.hpp:370-373).  Errors surface in falcon_ctx_sync(). */
falcon_status falcon_decompress_device_chained(falcon_ctx* ctx, int precision, const void* d_archive,
                                               const uint64_t* d_archive_bytes,
                                               const falcon_archive_info* info, void* d_values,
                                               uint64_t cap_values, void* stream);
/* ---- batch index and random-access decode (the format itself has no batch
 * index, FORMAT.md:10-14, so frames are otherwise located by a sequential walk) ---- */
/* d_index (device, batch_count + 1 u64): index[b] = archive offset of batch b's frame
 * (read_batch, container.cpp:113-132), index[batch_count] = end of the last frame.
 * Synchronises `stream`; a malformed frame fails with the walker's message. */
falcon_status falcon_archive_index(falcon_ctx* ctx, const void* d_archive, uint64_t archive_bytes,
                                   const falcon_archive_info* info, uint64_t* d_index, void* stream);
/* Decode batches [first_batch, first_batch + n_batches) only, given a HOST copy of the
 * index: values first_batch * batch_values ... land at d_values[0 ...]; *n_values gets the
 * count.  Same validation and messages as falcon_decompress_device (batch numbers absolute). */
falcon_status falcon_decompress_device_range(falcon_ctx* ctx, int precision, const void* d_archive,
                                             const falcon_archive_info* info, const uint64_t* index,
                                             uint64_t first_batch, uint64_t n_batches, void* d_values,
                                             uint64_t cap_values, uint64_t* n_values, void* stream);
/* Profiling hook: when set (non-null), device-resident calls on ctx record enc_start /
 * enc_stop right before / after the encode kernel and dec_start / dec_stop around the
 * decode kernel, on the call's stream.  Pass nulls to clear. */
falcon_status falcon_ctx_set_kernel_events(falcon_ctx* ctx, void* enc_start, void* enc_stop,
                                           void* dec_start, void* dec_stop);
/* Wait for `stream` and report the first error raised by async calls on ctx.  Decode
 * errors carry the reference's " (batch N)" suffix, numbered in the most recent async
 * decode's archive.
 * Async calls on one context share its device scratch (sizes, offsets, error words):
 * enqueue them all on ONE stream (they then run in order); use one context per stream
 * for concurrent work. */
falcon_status falcon_ctx_sync(falcon_ctx* ctx, void* stream);

/* ---- host-resident: multi-stream pinned H2D / kernel / D2H pipeline ---- */
falcon_status falcon_compress_stream(falcon_ctx* ctx, int precision, falcon_read_fn read,
                                     void* read_user, falcon_store_fn store, void* store_user,
                                     const falcon_pipeline_options* opt,
                                     falcon_pipeline_stats* stats);
falcon_status falcon_decompress_stream(falcon_ctx* ctx, int precision, const uint8_t* archive,
                                       uint64_t archive_bytes, falcon_put_fn put, void* put_user,
                                       const falcon_pipeline_options* opt,
                                       falcon_pipeline_stats* stats);
/* Convenience: host buffers in, host buffers out. */
falcon_status falcon_compress_host(falcon_ctx* ctx, int precision, const void* values,
                                   uint64_t n_values, const falcon_pipeline_options* opt,
                                   uint8_t* out, uint64_t out_cap, uint64_t* out_bytes,
                                   falcon_pipeline_stats* stats);
falcon_status falcon_decompress_host(falcon_ctx* ctx, int precision, const uint8_t* archive,
                                     uint64_t archive_bytes, void* values, uint64_t cap_values,
                                     uint64_t* n_values, const falcon_pipeline_options* opt,
                                     falcon_pipeline_stats* stats);

/* ---- host-resident across several GPUs ("a device list") ----
 * ctxs[0..n_ctx): one context per GPU.  Batches are split into contiguous ranges, one per
 * context (batch frames are context-free, container.cpp:88-111); each GPU runs its own
 * multi-stream pipeline concurrently (one host thread per context) and the frames are
 * concatenated in batch order after the one 47-byte header.  The archive bytes equal
 * falcon_compress_host's for any n_ctx.  Decompress locates the frames once on the host
 * (size tables only), then every GPU decodes its batch range into its value range.
 * Errors: the lowest-numbered failing context's status and message. */
falcon_status falcon_compress_host_multi(falcon_ctx* const* ctxs, unsigned n_ctx, int precision,
                                         const void* values, uint64_t n_values,
                                         const falcon_pipeline_options* opt, uint8_t* out,
                                         uint64_t out_cap, uint64_t* out_bytes,
                                         falcon_pipeline_stats* stats);
falcon_status falcon_decompress_host_multi(falcon_ctx* const* ctxs, unsigned n_ctx, int precision,
                                           const uint8_t* archive, uint64_t archive_bytes,
                                           void* values, uint64_t cap_values, uint64_t* n_values,
                                           const falcon_pipeline_options* opt,
                                           falcon_pipeline_stats* stats);

/* ---- files through GPU-direct storage ----
 * Raw value files are read into device memory through a pinned double buffer (pread +
 * async H2D), or with cuFile (GPUDirect Storage, or cuFile's compat path) when the
 * environment sets FALCON_CUFILE=1 and libcufile loads -- opt-in because cuFileDriverOpen()
 * hung on hosts without nvidia-fs.  *io_path (optional) gets 1 for cuFile, 0 for the
 * bounce path.  Compress runs the
 * device codec over windows of whole batches and writes frames, then the header: the
 * archive equals falcon_compress_host's.  Decompress reads the archive into HBM, indexes
 * its frames on the device and decodes batch windows into the raw file. */
falcon_status falcon_compress_file(falcon_ctx* ctx, int precision, const char* raw_path,
                                   const char* archive_path, const falcon_pipeline_options* opt,
                                   uint64_t* archive_bytes, int* io_path);
falcon_status falcon_decompress_file(falcon_ctx* ctx, int precision, const char* archive_path,
                                     const char* raw_path, const falcon_pipeline_options* opt,
                                     uint64_t* n_values, int* io_path);

/* ---- per-chunk operators (GPU-backed; host buffers) ---- */
/* Encodes exactly chunk_n values; returns the encoded length in *out_len. */
falcon_status falcon_compress_chunk(falcon_ctx* ctx, int precision, const void* values,
                                    uint32_t chunk_n, uint8_t* out, uint64_t out_cap,
                                    uint64_t* out_len);
/* Decodes one encoded chunk of `len` bytes; emits `count` (<= chunk_n) values. */
falcon_status falcon_decompress_chunk(falcon_ctx* ctx, int precision, const uint8_t* in,
                                      uint64_t len, uint32_t chunk_n, uint32_t count,
                                      void* values);

/* ---- self-test (device pointers): the per-value decimal analysis used by the encoder.
 * d_full[i] = alpha of v[i] by the exact fast loop (-1 = exception), d_literal[i] = the
 * literal reference loop (std::round + IEEE division), d_cert[i] = certification of v[i]
 * against candidate_alpha (0 undecided, 1 certified, 2 certified exception) and d_g[i]
 * the certified lane integer.  Used by tests/test_gpu_dpds.py against the CPU oracle. */
falcon_status falcon_selftest_dp(falcon_ctx* ctx, int precision, const void* d_values, uint64_t n,
                                 int candidate_alpha, int8_t* d_full, int8_t* d_literal,
                                 int8_t* d_cert, int64_t* d_g, void* stream);

/* d_out[i] (double or float per precision) = the decoder's division-free inverse scale
 * RN((T)d_g[i] / 10^alpha) (numeric.hpp:159-162), for alpha <= 21 (f64) / 9 (f32).
 * Checked against IEEE division by tests/test_gpu_dpds.py. */
falcon_status falcon_selftest_div(falcon_ctx* ctx, int precision, const int64_t* d_g, uint64_t n,
                                  int alpha, void* d_out, void* stream);

/* ---- synthetic inputs (synthetic.hpp:14-32 kinds; kind 5 = the pinned cfg3 kind) ---- */
#define FALCON_KIND_WALK 0
#define FALCON_KIND_DECIMAL 1
#define FALCON_KIND_SIGNFLIP 2
#define FALCON_KIND_OUTLIER 3
#define FALCON_KIND_BITS 4
#define FALCON_KIND_MIXED_BLOCKS 5
/* Counter-based "HPC field" for the sharded configs (not a reference kind; pinned in
 * csrc/field.cuh and restated in oracle/): value i depends on (seed, i) only, so any
 * range is produced directly, on the host or on the device. */
#define FALCON_KIND_FIELD 6
typedef struct {
    int kind;
    int decimal_places;
    uint64_t seed;
    int max_step_units;
    uint64_t outlier_period;
    int64_t outlier_units;
    uint32_t block;     /* MIXED_BLOCKS: values per decimal-place block (chunk_n) */
} falcon_synth_spec;
falcon_status falcon_synth_fill(int precision, const falcon_synth_spec* spec, void* out,
                                uint64_t count);
/* Values [first, first + count) of the stream.  first > 0 needs a counter-based kind
 * (FALCON_KIND_FIELD); the reference's kinds are sequential (synthetic.hpp:111). */
falcon_status falcon_synth_fill_at(int precision, const falcon_synth_spec* spec, uint64_t first,
                                   void* out, uint64_t count);
/* Device twin of falcon_synth_fill_at for counter-based kinds: writes d_out (device) on
 * `stream` (asynchronous).  Other kinds: FALCON_ERR_UNSUPPORTED. */
falcon_status falcon_synth_device(falcon_ctx* ctx, int precision, const falcon_synth_spec* spec,
                                  uint64_t first, void* d_out, uint64_t count, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FALCON_B200_H */
