/*
 * falcon_oracle.c -- CPU restatement of the Falcon chunk codec, container and
 * synthetic generators.  TEST INFRASTRUCTURE ONLY (see falcon_oracle.h).
 *
 * Written independently of the reference's code structure: bit planes are built
 * and read back one bit at a time (no 64x64 block transpose), the row codec walks
 * bytes directly, and the archive is produced by a single sequential loop.  The
 * arithmetic that decides bytes (dp_ds, scaling, zigzag, thresholds) follows the
 * cited reference lines exactly, because that is what parity means.
 */
#include "falcon_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* messages (error.hpp:8-19 types; texts from the throw sites cited in .h)    */
/* ------------------------------------------------------------------------- */
const char* or_error_message(int code) {
    switch (code) {
    case OR_OK: return "ok";
    case OR_E_COUNT: return "decompress_chunk: count exceeds chunk capacity";
    case OR_E_SCALE_RANGE: return "decimal_round_scale: scaled value exceeds 63 bits";
    case OR_E_PRECISION: return "archive precision does not match the requested value type";
    case OR_E_CAPACITY: return "output capacity too small";
    case OR_E_HDR_TRUNC: return "chunk header truncated";
    case OR_E_META: return "chunk meta bytes out of range";
    case OR_E_W: return "plane count out of range";
    case OR_E_FLAGS_TRUNC: return "plane flags truncated";
    case OR_E_FLAG_PAD: return "nonzero flag padding bits";
    case OR_E_ROW_TRUNC: return "row data truncated";
    case OR_E_BITMAP_TRUNC: return "row bitmap truncated";
    case OR_E_PAYLOAD_TRUNC: return "row payload truncated";
    case OR_E_SIZE: return "chunk size mismatch";
    case OR_E_ARCH_TRUNC: return "archive header truncated";
    case OR_E_MAGIC: return "bad archive magic";
    case OR_E_VERSION: return "unsupported archive version";
    case OR_E_PREC_TAG: return "unknown precision tag";
    case OR_E_CHUNK_N: return "invalid chunk length";
    case OR_E_ZERO_BATCH: return "zero batch size with nonzero value count";
    case OR_E_BATCH_COUNT: return "batch count disagrees with value count";
    case OR_E_BATCH_HDR_TRUNC: return "batch header truncated";
    case OR_E_TABLE_TRUNC: return "batch size table truncated";
    case OR_E_PAYLOAD_BATCH_TRUNC: return "batch payload truncated";
    case OR_E_CHUNK_COUNT: return "chunk count mismatch";
    case OR_E_TRAILING: return "trailing bytes after final batch";
    default: return "unknown error";
    }
}

int or_error_is_corrupt(int code) { return code >= 10; }

/* ------------------------------------------------------------------------- */
/* decade tables: correctly rounded 10^k (numeric.cpp:10-39).  glibc strtod /  */
/* strtof are correctly rounded, as is std::from_chars, so the tables agree.  */
/* ------------------------------------------------------------------------- */
static double g_dec64[617];
static float g_dec32[77];
static int g_dec_ready = 0;

static void dec_init(void) {
    if (g_dec_ready) return;
    char buf[16];
    for (int k = -308; k <= 308; ++k) {
        snprintf(buf, sizeof buf, "1e%d", k);
        g_dec64[k + 308] = strtod(buf, NULL);
    }
    for (int k = -38; k <= 38; ++k) {
        snprintf(buf, sizeof buf, "1e%d", k);
        g_dec32[k + 38] = strtof(buf, NULL);
    }
    g_dec_ready = 1;
}

/* exact powers 10^0..10^22 / 10^0..10^10 by repeated *10 (numeric.hpp:17-41) */
static double p64(int a) {
    double p = 1.0;
    for (int i = 0; i < a; ++i) p *= 10.0;
    return p;
}
static float p32(int a) {
    float p = 1.0f;
    for (int i = 0; i < a; ++i) p *= 10.0f;
    return p;
}

static uint64_t bits64(double v) { uint64_t b; memcpy(&b, &v, 8); return b; }
static double val64(uint64_t b) { double v; memcpy(&v, &b, 8); return v; }
static uint32_t bits32(float v) { uint32_t b; memcpy(&b, &v, 4); return b; }
static float val32(uint32_t b) { float v; memcpy(&v, &b, 4); return v; }

/* ------------------------------------------------------------------------- */
/* Type-generic section, stamped out for f64 and f32.                         */
/* ------------------------------------------------------------------------- */
#define OR_DEFINE(SUF, T, B, S, WIDTH, MANT, BIAS, EMASK, MAXA, MAXB, EXA, EXB, EPS, \
                  MIND, MAXD, DEC, POW, BITS, VAL, FABS, ROUND, LLROUND)               \
                                                                                     \
    /* floor_log2 from the exponent field (numeric.hpp:44-48) */                     \
    static int flog2_##SUF(T v) {                                                    \
        return (int)((BITS(v) >> MANT) & EMASK) - BIAS;                              \
    }                                                                                \
                                                                                     \
    /* floor_log10 via the decade table (numeric.hpp:54-66) */                       \
    int or_floor_log10_##SUF(T v) {                                                  \
        dec_init();                                                                  \
        const T a = FABS(v);                                                         \
        int k = (int)(((long long)flog2_##SUF(v) * 78913) >> 18);                    \
        if (k < MIND) k = MIND;                                                      \
        if (k > MAXD) k = MAXD;                                                      \
        while (k > MIND && a < DEC[k - MIND]) --k;                                   \
        while (k < MAXD && a >= DEC[k + 1 - MIND]) ++k;                              \
        return k;                                                                    \
    }                                                                                \
                                                                                     \
    /* dp_ds_calculate_counted (numeric.hpp:108-140) */                              \
    int or_dp_ds_##SUF(T v, uint8_t* alpha_o, uint8_t* beta_o) {                     \
        *alpha_o = EXA; *beta_o = EXB;                                               \
        if (v == (T)0) {                                                             \
            if (signbit(v)) return 0;                                                \
            *alpha_o = 0; *beta_o = 0;                                               \
            return 0;                                                                \
        }                                                                            \
        if (fpclassify(v) != FP_NORMAL) return 0;                                    \
        const int mag = or_floor_log10_##SUF(v);                                     \
        int alpha = mag < 0 ? -mag : 0;                                              \
        int beta = alpha + mag + 1;                                                  \
        int it = 0;                                                                  \
        while (beta <= MAXB && alpha <= MAXA) {                                      \
            ++it;                                                                    \
            const T scaled = v * POW(alpha);                                         \
            const T nearest = ROUND(scaled);                                         \
            const T gap = FABS(scaled - nearest);                                    \
            if (gap <= FABS(scaled) * EPS) {                                         \
                if (nearest / POW(alpha) != v) return it;                            \
                *alpha_o = (uint8_t)alpha; *beta_o = (uint8_t)beta;                  \
                return it;                                                           \
            }                                                                        \
            ++alpha; ++beta;                                                         \
        }                                                                            \
        return it;                                                                   \
    }                                                                                \
                                                                                     \
    /* decimal_round_scale (numeric.hpp:150-156) */                                  \
    int or_round_scale_##SUF(T v, int alpha, int64_t* out) {                         \
        const T scaled = v * POW(alpha);                                             \
        if (!(FABS(scaled) < (T)0x1p62)) return OR_E_SCALE_RANGE;                    \
        *out = (int64_t)LLROUND(scaled);                                             \
        return OR_OK;                                                                \
    }                                                                                \
                                                                                     \
    /* inverse_scale (numeric.hpp:159-162) */                                        \
    T or_inverse_scale_##SUF(int64_t g, int alpha) { return (T)g / POW(alpha); }     \
                                                                                     \
    /* analyze_chunk (transform.hpp:47-68) */                                        \
    void or_analyze_chunk_##SUF(const T* v, size_t n, uint8_t* am, uint8_t* bh) {    \
        int alpha_max = 0;                                                           \
        T vmax = 0;                                                                  \
        for (size_t i = 0; i < n; ++i) {                                             \
            uint8_t a, b;                                                            \
            or_dp_ds_##SUF(v[i], &a, &b);                                            \
            if (a > MAXA || b > MAXB) { *am = EXA; *bh = EXB; return; }              \
            if (a > alpha_max) alpha_max = a;                                        \
            const T x = FABS(v[i]);                                                  \
            if (x > vmax) vmax = x;                                                  \
        }                                                                            \
        const int bhat = vmax == (T)0 ? 0 : alpha_max + or_floor_log10_##SUF(vmax) + 1; \
        if (alpha_max > MAXA || bhat > MAXB) { *am = EXA; *bh = EXB; return; }       \
        *am = (uint8_t)alpha_max; *bh = (uint8_t)bhat;                               \
    }                                                                                \
                                                                                     \
    static B zz_##SUF(S x) { return ((B)x << 1) ^ (B)(x >> (WIDTH - 1)); }           \
    static S unzz_##SUF(B z) { return (S)((z >> 1) ^ ((B)0 - (z & 1))); }            \
                                                                                     \
    /* compress_chunk (chunk_codec.hpp:50-74) with forward_transform               \
       (transform.hpp:72-89) and a bit-at-a-time restatement of build_planes +      \
       encode_rows (bitplane.hpp:64-90, 113-148). */                                 \
    size_t or_compress_chunk_##SUF(const T* v, size_t n, uint8_t* out) {             \
        uint8_t am, bh;                                                              \
        or_analyze_chunk_##SUF(v, n, &am, &bh);                                      \
        const int case2 = am > MAXA || bh > MAXB;                                    \
        B* z = (B*)malloc(n * sizeof(B));                                            \
        for (size_t i = 0; i < n; ++i) {                                             \
            if (case2) {                                                             \
                z[i] = zz_##SUF((S)BITS(v[i]));                                      \
            } else {                                                                 \
                int64_t g = 0;                                                       \
                or_round_scale_##SUF(v[i], am, &g);                                  \
                z[i] = (B)(S)g;                                                      \
            }                                                                        \
        }                                                                            \
        for (size_t i = n; i-- > 1;) z[i] = zz_##SUF((S)(B)(z[i] - z[i - 1]));        \
        B all = 0;                                                                   \
        for (size_t i = 1; i < n; ++i) all |= z[i];                                  \
        int w = 0;                                                                   \
        while (w < WIDTH && (all >> w) != 0) ++w;                                    \
        size_t pos = 0;                                                              \
        out[pos++] = am;                                                             \
        out[pos++] = bh;                                                             \
        for (size_t i = 0; i < sizeof(B); ++i) out[pos++] = (uint8_t)(z[0] >> (8 * i)); \
        out[pos++] = (uint8_t)w;                                                     \
        if (w == 0) { free(z); return pos; }                                         \
        const size_t lanes = n - 1, row_bytes = lanes / 8, bm_bytes = lanes / 64;    \
        const size_t fb = (size_t)(w + 7) / 8;                                       \
        const size_t flags_at = pos;                                                 \
        memset(out + pos, 0, fb);                                                    \
        pos += fb;                                                                   \
        uint8_t* row = (uint8_t*)malloc(row_bytes);                                  \
        for (int r = 0; r < w; ++r) {                                                \
            const int bit = w - 1 - r;                                               \
            memset(row, 0, row_bytes);                                               \
            size_t zeros = 0;                                                        \
            for (size_t j = 0; j < lanes; ++j)                                       \
                if ((z[1 + j] >> bit) & 1) row[j / 8] |= (uint8_t)(0x80u >> (j % 8)); \
            for (size_t j = 0; j < row_bytes; ++j) zeros += row[j] == 0;             \
            if (zeros <= bm_bytes) {                                                 \
                /* dense: flag bit (w-1-r) of the big-endian flag string */          \
                out[flags_at + fb - 1 - (size_t)bit / 8] |= (uint8_t)(1u << (bit % 8)); \
                memcpy(out + pos, row, row_bytes);                                   \
                pos += row_bytes;                                                    \
            } else {                                                                 \
                uint8_t* bm = out + pos;                                             \
                memset(bm, 0, bm_bytes);                                             \
                pos += bm_bytes;                                                     \
                for (size_t j = 0; j < row_bytes; ++j)                               \
                    if (row[j]) {                                                    \
                        bm[j / 8] |= (uint8_t)(0x80u >> (j % 8));                    \
                        out[pos++] = row[j];                                         \
                    }                                                                \
            }                                                                        \
        }                                                                            \
        free(row);                                                                   \
        free(z);                                                                     \
        return pos;                                                                  \
    }                                                                                \
                                                                                     \
    /* decompress_chunk (chunk_codec.hpp:86-122), decode_rows (bitplane.hpp:152-186), \
       inverse_transform (transform.hpp:91-106); same check order. */                \
    int or_decompress_chunk_##SUF(const uint8_t* in, size_t len, size_t n,           \
                                  size_t count, T* out) {                            \
        const size_t hdr = 3 + sizeof(B);                                            \
        if (count > n) return OR_E_COUNT;                                            \
        if (len < hdr) return OR_E_HDR_TRUNC;                                        \
        const int am = in[0], bh = in[1];                                            \
        const int case2 = am > MAXA || bh > MAXB;                                    \
        if (case2 && !(am == EXA && bh == EXB)) return OR_E_META;                    \
        B z1 = 0;                                                                    \
        for (size_t i = 0; i < sizeof(B); ++i) z1 |= (B)in[2 + i] << (8 * i);        \
        const int w = in[2 + sizeof(B)];                                             \
        if (w > WIDTH) return OR_E_W;                                                \
        size_t pos = hdr;                                                            \
        uint64_t flags = 0;                                                          \
        if (w > 0) {                                                                 \
            const size_t fb = (size_t)(w + 7) / 8;                                   \
            if (len - pos < fb) return OR_E_FLAGS_TRUNC;                             \
            for (size_t i = 0; i < fb; ++i) flags = flags << 8 | in[pos + i];        \
            if (fb * 8 > (size_t)w && (flags >> w) != 0) return OR_E_FLAG_PAD;      \
            pos += fb;                                                               \
        }                                                                            \
        const size_t lanes = n - 1, row_bytes = lanes / 8, bm_bytes = lanes / 64;    \
        B* z = (B*)calloc(n, sizeof(B));                                             \
        uint8_t* row = (uint8_t*)malloc(row_bytes ? row_bytes : 1);                  \
        for (int r = 0; r < w; ++r) {                                                \
            const int bit = w - 1 - r;                                               \
            if ((flags >> bit) & 1) {                                                \
                if (len - pos < row_bytes) { free(z); free(row); return OR_E_ROW_TRUNC; } \
                memcpy(row, in + pos, row_bytes);                                    \
                pos += row_bytes;                                                    \
            } else {                                                                 \
                if (len - pos < bm_bytes) { free(z); free(row); return OR_E_BITMAP_TRUNC; } \
                const uint8_t* bm = in + pos;                                        \
                pos += bm_bytes;                                                     \
                for (size_t j = 0; j < row_bytes; ++j) {                             \
                    row[j] = 0;                                                      \
                    if ((bm[j / 8] >> (7 - j % 8)) & 1) {                            \
                        if (pos >= len) { free(z); free(row); return OR_E_PAYLOAD_TRUNC; } \
                        row[j] = in[pos++];                                          \
                    }                                                                \
                }                                                                    \
            }                                                                        \
            for (size_t j = 0; j < lanes; ++j)                                       \
                if ((row[j / 8] >> (7 - j % 8)) & 1) z[1 + j] |= (B)1 << bit;        \
        }                                                                            \
        free(row);                                                                   \
        if (pos != len) { free(z); return OR_E_SIZE; }                               \
        z[0] = z1;                                                                   \
        B g = 0;                                                                     \
        for (size_t i = 0; i < count; ++i) {                                         \
            g = i == 0 ? z[0] : (B)(g + (B)unzz_##SUF(z[i]));                        \
            if (case2) out[i] = VAL((B)unzz_##SUF(g));                               \
            else out[i] = or_inverse_scale_##SUF((int64_t)(S)g, am);                 \
        }                                                                            \
        free(z);                                                                     \
        return OR_OK;                                                                \
    }

OR_DEFINE(f64, double, uint64_t, int64_t, 64, 52, 1023, 0x7ffu, 22, 15, 23, 16, 0x1p-52,
          -308, 308, g_dec64, p64, bits64, val64, fabs, round, llround)
OR_DEFINE(f32, float, uint32_t, int32_t, 32, 23, 127, 0xffu, 10, 6, 11, 7, 0x1p-23f,
          -38, 38, g_dec32, p32, bits32, val32, fabsf, roundf, llroundf)

void or_dp_alpha_batch(int prec, const void* values, uint64_t n, int8_t* alpha_out) {
    for (uint64_t i = 0; i < n; ++i) {
        uint8_t a, b;
        if (prec == 0) {
            or_dp_ds_f64(((const double*)values)[i], &a, &b);
            alpha_out[i] = (a > 22 || b > 15) ? -1 : (int8_t)a;
        } else {
            or_dp_ds_f32(((const float*)values)[i], &a, &b);
            alpha_out[i] = (a > 10 || b > 6) ? -1 : (int8_t)a;
        }
    }
}

/* max_encoded_chunk_size (chunk_codec.hpp:36-41) */
size_t or_max_encoded_chunk_size(int prec, size_t n) {
    const size_t lane = prec == 0 ? 8 : 4, width = prec == 0 ? 64 : 32;
    return 3 + lane + (width + 7) / 8 + width * ((n - 1) / 8);
}

/* ------------------------------------------------------------------------- */
/* container (container.cpp:44-132)                                          */
/* ------------------------------------------------------------------------- */
static void put_le(uint64_t v, uint8_t* p, int bytes) {
    for (int i = 0; i < bytes; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
static uint64_t get_le(const uint8_t* p, int bytes) {
    uint64_t v = 0;
    for (int i = 0; i < bytes; ++i) v |= (uint64_t)p[i] << (8 * i);
    return v;
}

void or_write_header(const or_header* h, uint8_t out[47]) {
    static const uint8_t magic[8] = {'F', 'A', 'L', 'C', 'O', 'N', 'A', 0};
    memcpy(out, magic, 8);
    put_le(1, out + 8, 2);
    out[10] = h->precision;
    put_le(h->chunk_n, out + 11, 4);
    put_le(h->batch_values, out + 15, 8);
    put_le(h->total_values, out + 23, 8);
    put_le(h->batch_count, out + 31, 8);
    put_le(0, out + 39, 8);
}

int or_read_header(const uint8_t* in, size_t len, or_header* h) {
    static const uint8_t magic[8] = {'F', 'A', 'L', 'C', 'O', 'N', 'A', 0};
    if (len < 47) return OR_E_ARCH_TRUNC;
    if (memcmp(in, magic, 8) != 0) return OR_E_MAGIC;
    if (get_le(in + 8, 2) != 1) return OR_E_VERSION;
    if (in[10] > 1) return OR_E_PREC_TAG;
    h->precision = in[10];
    h->chunk_n = (uint32_t)get_le(in + 11, 4);
    if (h->chunk_n < 65 || (h->chunk_n - 1) % 64 != 0) return OR_E_CHUNK_N;
    h->batch_values = get_le(in + 15, 8);
    h->total_values = get_le(in + 23, 8);
    h->batch_count = get_le(in + 31, 8);
    if (h->batch_values == 0 && h->total_values != 0) return OR_E_ZERO_BATCH;
    if (h->batch_values != 0) {
        const uint64_t expect = (h->total_values + h->batch_values - 1) / h->batch_values;
        if (expect != h->batch_count) return OR_E_BATCH_COUNT;
    } else if (h->batch_count != 0) {
        return OR_E_BATCH_COUNT;
    }
    return OR_OK;
}

uint64_t or_compress_bound(int prec, uint64_t count, uint32_t n, uint64_t bv) {
    uint64_t total = 47;
    const uint64_t mx = or_max_encoded_chunk_size(prec, n);
    for (uint64_t first = 0; first < count; first += bv) {
        const uint64_t c = count - first < bv ? count - first : bv;
        const uint64_t chunks = (c + n - 1) / n;
        total += 4 + 4 * chunks + chunks * mx;
    }
    return total;
}

/* Sequential archive: header, then per batch [u32 C][u32 size*C][chunks], the short
 * final chunk padded with +0.0 (pipeline.hpp:205-215; container.cpp:88-111). */
int or_compress_archive(int prec, const void* values, uint64_t count, uint32_t n, uint64_t bv,
                        uint8_t* out, uint64_t cap, uint64_t* out_len) {
    const size_t esz = prec == 0 ? 8 : 4;
    const size_t mx = or_max_encoded_chunk_size(prec, n);
    if (cap < 47) return OR_E_CAPACITY;
    uint64_t pos = 47, batches = 0;
    uint8_t* tmp = (uint8_t*)malloc(mx);
    void* pad = malloc((size_t)n * esz);
    for (uint64_t first = 0; first < count; first += bv) {
        const uint64_t c = count - first < bv ? count - first : bv;
        const uint64_t chunks = (c + n - 1) / n;
        if (pos + 4 + 4 * chunks > cap) { free(tmp); free(pad); return OR_E_CAPACITY; }
        const uint64_t table = pos + 4;
        put_le(chunks, out + pos, 4);
        pos += 4 + 4 * chunks;
        for (uint64_t ci = 0; ci < chunks; ++ci) {
            const uint64_t v0 = first + ci * n;
            const uint64_t len = c - ci * n < n ? c - ci * n : n;
            memset(pad, 0, (size_t)n * esz);
            memcpy(pad, (const uint8_t*)values + v0 * esz, (size_t)len * esz);
            const size_t sz = prec == 0 ? or_compress_chunk_f64((const double*)pad, n, tmp)
                                        : or_compress_chunk_f32((const float*)pad, n, tmp);
            if (pos + sz > cap) { free(tmp); free(pad); return OR_E_CAPACITY; }
            memcpy(out + pos, tmp, sz);
            put_le(sz, out + table + 4 * ci, 4);
            pos += sz;
        }
        ++batches;
    }
    free(tmp);
    free(pad);
    or_header h = {(uint8_t)prec, n, bv, count, batches};
    or_write_header(&h, out);
    *out_len = pos;
    return OR_OK;
}

/* decompress_pipeline (pipeline.hpp:370-467) run sequentially: frame walk via
 * read_batch (container.cpp:113-132), chunk-count check, per-chunk decode, and the
 * trailing-bytes check last. */
int or_decompress_archive(int prec, const uint8_t* in, uint64_t len, void* values, uint64_t cap,
                          uint64_t* n_values, uint64_t* bad_batch) {
    or_header h;
    *bad_batch = (uint64_t)-1;
    int rc = or_read_header(in, len, &h);
    if (rc) return rc;
    if (h.precision != prec) return OR_E_PRECISION;
    if (h.total_values > cap) return OR_E_CAPACITY;
    const size_t esz = prec == 0 ? 8 : 4;
    const uint64_t n = h.chunk_n;
    uint64_t cursor = 47;
    for (uint64_t b = 0; b < h.batch_count; ++b) {
        *bad_batch = b;
        const uint64_t rem = len - cursor;
        if (rem < 4) return OR_E_BATCH_HDR_TRUNC;
        const uint64_t cnt = get_le(in + cursor, 4);
        const uint64_t table_end = 4 + 4 * cnt;
        if (rem < table_end) return OR_E_TABLE_TRUNC;
        uint64_t payload = 0;
        for (uint64_t i = 0; i < cnt; ++i) payload += get_le(in + cursor + 4 + 4 * i, 4);
        if (rem - table_end < payload) return OR_E_PAYLOAD_BATCH_TRUNC;
        const uint64_t first = b * h.batch_values;
        const uint64_t count = h.total_values - first < h.batch_values ? h.total_values - first
                                                                        : h.batch_values;
        const uint64_t chunks = (count + n - 1) / n;
        if (cnt != chunks) return OR_E_CHUNK_COUNT;
        uint64_t off = cursor + table_end;
        for (uint64_t c = 0; c < cnt; ++c) {
            const uint64_t sz = get_le(in + cursor + 4 + 4 * c, 4);
            const uint64_t k = count - c * n < n ? count - c * n : n;
            uint8_t* dst = (uint8_t*)values + (first + c * n) * esz;
            rc = prec == 0 ? or_decompress_chunk_f64(in + off, sz, n, k, (double*)dst)
                           : or_decompress_chunk_f32(in + off, sz, n, k, (float*)dst);
            if (rc) return rc;
            off += sz;
        }
        cursor += table_end + payload;
    }
    *bad_batch = (uint64_t)-1;
    if (cursor != len) return OR_E_TRAILING;
    *n_values = h.total_values;
    return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* std::mt19937_64 (its output sequence is fixed by the C++ standard) and the  */
/* synthetic generators (synthetic.hpp:36-115).                               */
/* ------------------------------------------------------------------------- */
typedef struct { uint64_t mt[312]; int idx; } mt64;

static void mt64_seed(mt64* m, uint64_t seed) {
    m->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        m->mt[i] = 6364136223846793005ULL * (m->mt[i - 1] ^ (m->mt[i - 1] >> 62)) + (uint64_t)i;
    m->idx = 312;
}

static uint64_t mt64_next(mt64* m) {
    if (m->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (m->mt[i] & 0xFFFFFFFF80000000ULL) |
                               (m->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
            m->mt[i] = m->mt[(i + 156) % 312] ^ xa;
        }
        m->idx = 0;
    }
    uint64_t y = m->mt[m->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

/* Counter-based "HPC field" of the sharded configs.  Not a reference kind: pinned by the
 * product's csrc/field.cuh (restated here independently, bit for bit): two integer
 * triangle waves plus splitmix64 noise, quantised to decimal_places. */
static uint64_t or_field_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static int64_t or_tri(uint64_t x, uint64_t period, int64_t amp) {
    const uint64_t half = period / 2, r = x % period;
    return amp * (int64_t)(r < half ? r : period - r) / (int64_t)half;
}
int or_synth_fill_at(int prec, const or_spec* s, uint64_t first, void* out, uint64_t count) {
    if (s->kind != OR_KIND_FIELD) return first == 0 ? or_synth_fill(prec, s, out, count) : -1;
    if (s->decimal_places < 0 || s->decimal_places > (prec == 0 ? 22 : 10)) return -1;
    for (uint64_t i = 0; i < count; ++i) {
        const uint64_t x = first + i;
        const uint64_t h = or_field_mix(x + (s->seed + 1) * 0x9E3779B97F4A7C15ULL);
        const int64_t units = or_tri(x, 65536, 50000) + or_tri(x, 1048573, 400000) - 225000 +
                              ((int64_t)(h % 127) - 63);
        if (prec == 0) ((double*)out)[i] = or_inverse_scale_f64(units, s->decimal_places);
        else ((float*)out)[i] = or_inverse_scale_f32(units, s->decimal_places);
    }
    return 0;
}

int or_synth_fill(int prec, const or_spec* s, void* out, uint64_t count) {
    if (s->kind == OR_KIND_FIELD) return or_synth_fill_at(prec, s, 0, out, count);
    const int max_alpha = prec == 0 ? 22 : 10, max_beta = prec == 0 ? 15 : 6;
    if (s->decimal_places < 0 || s->decimal_places > max_alpha) return -1;
    if (s->max_step_units < 1) return -1;
    mt64 rng;
    mt64_seed(&rng, s->seed);
    int64_t acc = (int64_t)(mt64_next(&rng) % 20001) - 10000;
    uint64_t next_outlier = 0;
    if (s->kind == OR_KIND_OUTLIER) {
        if (s->outlier_period == 0) return -1;
        next_outlier = mt64_next(&rng) % s->outlier_period;
    }
    int dp_block = s->decimal_places;
    for (uint64_t i = 0; i < count; ++i) {
        double d = 0;
        float f = 0;
        switch (s->kind) {
        case OR_KIND_WALK:
        case OR_KIND_OUTLIER: {
            const int64_t span = 2 * (int64_t)s->max_step_units + 1;
            acc += (int64_t)(mt64_next(&rng) % (uint64_t)span) - s->max_step_units;
            int64_t units = acc;
            if (s->kind == OR_KIND_OUTLIER && i == next_outlier) {
                units += s->outlier_units;
                next_outlier += s->outlier_period;
            }
            d = or_inverse_scale_f64(units, s->decimal_places);
            f = or_inverse_scale_f32(units, s->decimal_places);
            break;
        }
        case OR_KIND_DECIMAL: {
            const int digits = 1 + (int)(mt64_next(&rng) % (uint64_t)max_beta);
            int64_t lo = 1, hi = 10;
            for (int k = 1; k < digits; ++k) { lo *= 10; hi *= 10; }
            if (digits == 1) lo = 1;
            int64_t dd = lo + (int64_t)(mt64_next(&rng) % (uint64_t)(hi - lo));
            if (dd % 10 == 0) ++dd;
            if (mt64_next(&rng) & 1) dd = -dd;
            d = or_inverse_scale_f64(dd, s->decimal_places);
            f = or_inverse_scale_f32(dd, s->decimal_places);
            break;
        }
        case OR_KIND_SIGNFLIP: {
            const uint64_t r = mt64_next(&rng);
            uint64_t b = r & ((1ULL << 52) - 1);
            b |= (uint64_t)1023 << 52;
            b |= (uint64_t)(i & 1) << 63;
            d = val64(b);
            uint32_t b32 = (uint32_t)r & ((1u << 23) - 1);
            b32 |= (uint32_t)127 << 23;
            b32 |= (uint32_t)(i & 1) << 31;
            f = val32(b32);
            break;
        }
        case OR_KIND_BITS: {
            const uint64_t r = mt64_next(&rng);
            d = val64(r);
            f = val32((uint32_t)r);
            break;
        }
        case OR_KIND_MIXED_BLOCKS: {
            /* Pinned cfg3 generator (not in the reference; DESIGN.md "Synthetic
             * inputs"): a reflecting random walk in +/-999999 units whose decimal
             * place is redrawn from [1,6] at the start of every `block` values. */
            if (s->block == 0) return -1;
            if (i % s->block == 0) dp_block = 1 + (int)(mt64_next(&rng) % 6);
            const int64_t span = 2 * (int64_t)s->max_step_units + 1;
            acc += (int64_t)(mt64_next(&rng) % (uint64_t)span) - s->max_step_units;
            if (acc > 999999) acc = 2 * 999999 - acc;
            if (acc < -999999) acc = -2 * 999999 - acc;
            d = or_inverse_scale_f64(acc, dp_block);
            f = or_inverse_scale_f32(acc, dp_block);
            break;
        }
        default:
            return -1;
        }
        if (prec == 0) ((double*)out)[i] = d;
        else ((float*)out)[i] = f;
    }
    return 0;
}
