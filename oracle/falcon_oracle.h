/*
 * falcon_oracle.h -- CPU restatement of the Falcon (arXiv 2511.04140) hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the B200 product in
 * paper_2511_04140_b200/.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product never links it.
 *
 * Parity status: PINNED.  The restatement is checked against
 *   (1) the golden vectors / known answers of the reference's own tests
 *       (proj/tests/test_chunk_codec.cpp:32-70,216-227, test_numeric.cpp:98-122,
 *        test_container.cpp:29-60,115-127, FORMAT.md:106-123), and
 *   (2) the reference library itself compiled from /root/reference/proj/src by
 *       oracle/Makefile into oracle/_ref/libfalcon_ref.so (tests/test_oracle_*.py).
 *
 * Every function cites the reference file:line it restates.  Plain C11, compiled
 * with -ffp-contract=off so that no multiply/add is fused (the reference builds
 * with default g++ flags and no -march, i.e. SSE2 scalar IEEE arithmetic).
 */
#ifndef FALCON_ORACLE_H
#define FALCON_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes.  Messages are identical to the reference's exception texts. */
enum {
    OR_OK = 0,
    /* falcon::error */
    OR_E_COUNT = 1,          /* chunk_codec.hpp:92-93 */
    OR_E_SCALE_RANGE = 2,    /* numeric.hpp:153-154 */
    OR_E_PRECISION = 3,      /* pipeline.hpp:375-376 */
    OR_E_CAPACITY = 4,       /* oracle-only: output buffer too small */
    /* falcon::corrupt_error, chunk level (chunk_codec.hpp:94-117, bitplane.hpp:165-177) */
    OR_E_HDR_TRUNC = 10,
    OR_E_META = 11,
    OR_E_W = 12,
    OR_E_FLAGS_TRUNC = 13,
    OR_E_FLAG_PAD = 14,
    OR_E_ROW_TRUNC = 15,
    OR_E_BITMAP_TRUNC = 16,
    OR_E_PAYLOAD_TRUNC = 17,
    OR_E_SIZE = 18,
    /* archive level (container.cpp:58-83, 114-128; pipeline.hpp:412-416, 460-461) */
    OR_E_ARCH_TRUNC = 20,
    OR_E_MAGIC = 21,
    OR_E_VERSION = 22,
    OR_E_PREC_TAG = 23,
    OR_E_CHUNK_N = 24,
    OR_E_ZERO_BATCH = 25,
    OR_E_BATCH_COUNT = 26,
    OR_E_BATCH_HDR_TRUNC = 27,
    OR_E_TABLE_TRUNC = 28,
    OR_E_PAYLOAD_BATCH_TRUNC = 29,
    OR_E_CHUNK_COUNT = 30,
    OR_E_TRAILING = 31,
};

const char* or_error_message(int code);
/* 1 if the code maps to falcon::corrupt_error, else 0 (falcon::error). */
int or_error_is_corrupt(int code);

/* ---- numeric.hpp ---- */
int or_floor_log10_f64(double v);
int or_floor_log10_f32(float v);
/* dp_ds_calculate_counted (numeric.hpp:108-140): returns iterations. */
int or_dp_ds_f64(double v, uint8_t* alpha, uint8_t* beta);
int or_dp_ds_f32(float v, uint8_t* alpha, uint8_t* beta);
/* Batch form: alpha of each value, -1 for the exception path (numeric.hpp:88-94). */
void or_dp_alpha_batch(int prec, const void* values, uint64_t n, int8_t* alpha_out);
/* decimal_round_scale (numeric.hpp:150-156); returns OR_E_SCALE_RANGE on overflow. */
int or_round_scale_f64(double v, int alpha, int64_t* out);
int or_round_scale_f32(float v, int alpha, int64_t* out);
double or_inverse_scale_f64(int64_t g, int alpha);
float or_inverse_scale_f32(int64_t g, int alpha);

/* ---- transform.hpp:47-68 ---- */
void or_analyze_chunk_f64(const double* v, size_t n, uint8_t* alpha_max, uint8_t* beta_hat);
void or_analyze_chunk_f32(const float* v, size_t n, uint8_t* alpha_max, uint8_t* beta_hat);

/* ---- chunk_codec.hpp ---- */
size_t or_max_encoded_chunk_size(int prec, size_t n);
/* compress_chunk (chunk_codec.hpp:50-74): writes the encoded chunk, returns its length. */
size_t or_compress_chunk_f64(const double* v, size_t n, uint8_t* out);
size_t or_compress_chunk_f32(const float* v, size_t n, uint8_t* out);
/* decompress_chunk (chunk_codec.hpp:86-122): emits `count` values. */
int or_decompress_chunk_f64(const uint8_t* in, size_t len, size_t n, size_t count, double* out);
int or_decompress_chunk_f32(const uint8_t* in, size_t len, size_t n, size_t count, float* out);

/* ---- container + sequential archive (container.cpp, pipeline.hpp semantics) ---- */
typedef struct {
    uint8_t precision;      /* 0 = f64, 1 = f32 */
    uint32_t chunk_n;
    uint64_t batch_values;
    uint64_t total_values;
    uint64_t batch_count;
} or_header;

void or_write_header(const or_header* h, uint8_t out[47]);
int or_read_header(const uint8_t* in, size_t len, or_header* h);
uint64_t or_compress_bound(int prec, uint64_t count, uint32_t chunk_n, uint64_t batch_values);
/* Sequential restatement of compress_pipeline's output (test_pipeline.cpp:19-47). */
int or_compress_archive(int prec, const void* values, uint64_t count, uint32_t chunk_n,
                        uint64_t batch_values, uint8_t* out, uint64_t cap, uint64_t* out_len);
/* Sequential restatement of decompress_pipeline (pipeline.hpp:370-467).  On a corrupt
 * batch, *bad_batch receives the batch index ((uint64_t)-1 if not batch-scoped). */
int or_decompress_archive(int prec, const uint8_t* in, uint64_t len, void* values, uint64_t cap,
                          uint64_t* n_values, uint64_t* bad_batch);

/* ---- synthetic.hpp generators (synthetic.hpp:36-115) + the pinned cfg3 kind ---- */
enum { OR_KIND_WALK = 0, OR_KIND_DECIMAL = 1, OR_KIND_SIGNFLIP = 2, OR_KIND_OUTLIER = 3,
       OR_KIND_BITS = 4, OR_KIND_MIXED_BLOCKS = 5, OR_KIND_FIELD = 6 };
typedef struct {
    int kind;
    int decimal_places;
    uint64_t seed;
    int max_step_units;
    uint64_t outlier_period;
    int64_t outlier_units;
    uint32_t block;         /* MIXED_BLOCKS only: values per decimal-place block */
} or_spec;
int or_synth_fill(int prec, const or_spec* s, void* out, uint64_t count);
/* Counter-based kinds (OR_KIND_FIELD) from any absolute value index `first`. */
int or_synth_fill_at(int prec, const or_spec* s, uint64_t first, void* out, uint64_t count);

#ifdef __cplusplus
}
#endif
#endif
