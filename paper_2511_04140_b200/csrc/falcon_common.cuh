// falcon_common.cuh -- shared device-side definitions for the B200 Falcon codec.
//
// Lane traits mirror fp_traits<T> (reference proj/include/falcon/fp_bits.hpp:14-62);
// the arithmetic helpers restate numeric.hpp:44-162 and transform.hpp:13-22 with
// explicitly rounded intrinsics (__dmul_rn, __ddiv_rn, ...) so that ptxas can never
// contract a multiply/add into an FMA: every byte must equal the CPU reference's.
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace fb200 {

template <typename T> struct lane_traits;

template <> struct lane_traits<double> {
    using B = uint64_t;
    using S = int64_t;
    static constexpr int width = 64;
    static constexpr int mant = 52;
    static constexpr int bias = 1023;
    static constexpr unsigned emask = 0x7ffu;
    static constexpr int max_alpha = 22;
    static constexpr int max_beta = 15;
    static constexpr int exc_alpha = 23;
    static constexpr int exc_beta = 16;
    static constexpr int min_decade = -308;
    static constexpr int max_decade = 308;
    static constexpr int header = 11;  // chunk_header_bytes<double> (chunk_codec.hpp:33-34)
    static constexpr int prec_tag = 0;
};

template <> struct lane_traits<float> {
    using B = uint32_t;
    using S = int32_t;
    static constexpr int width = 32;
    static constexpr int mant = 23;
    static constexpr int bias = 127;
    static constexpr unsigned emask = 0xffu;
    static constexpr int max_alpha = 10;
    static constexpr int max_beta = 6;
    static constexpr int exc_alpha = 11;
    static constexpr int exc_beta = 7;
    static constexpr int min_decade = -38;
    static constexpr int max_decade = 38;
    static constexpr int header = 7;
    static constexpr int prec_tag = 1;
};

// Device tables, filled once per process by fb200::upload_tables() (capi.cu):
//   pow10: exact 10^0..10^22 / 10^0..10^10 (numeric.hpp:17-41)
//   decade bits: correctly rounded 10^k as IEEE bit patterns (numeric.cpp:10-39),
//   compared as unsigned integers (valid for the positive normal operands used).
// They are defined (and every device helper below compiled) only in the single
// kernel translation unit kernels_all.cu, which defines FB200_KERNEL_TU.
#ifdef FB200_KERNEL_TU
// In the constant bank (5.4 KB): the encoder's sampling chain (mag_of -> pow10 -> the
// certification parameters) reads them back to back, and constant-cache hits keep that
// dependent chain off the L1/L2 path the streaming value loads thrash.
#ifdef FB_TABLES_GLOBAL
#define FB_TABLE_SPACE __device__
#else
#define FB_TABLE_SPACE __constant__
#endif
FB_TABLE_SPACE double g_pow10_f64[23];
FB_TABLE_SPACE float g_pow10_f32[11];
FB_TABLE_SPACE double g_rpow10_f64[23];      // RN(1 / 10^a)
FB_TABLE_SPACE float g_rpow10_f32[11];
FB_TABLE_SPACE uint64_t g_decade_f64[618];  // + guard entry (+inf) for exponent 0x7ff
FB_TABLE_SPACE uint32_t g_decade_f32[78];   // + guard entry (+inf) for exponent 0xff
#endif

// The encoder's chunk-uniform certification parameters per candidate scale A (dpds.cuh
// cert_params, built on the host from the tables above by upload_tables): one uniform
// constant-bank read instead of a dependent table chain after the chunk's A0 is known.
struct cert_row64 {
    double p;          // 10^A
    uint32_t lo1;      // hi(dec(-A)) + 1
    uint32_t span;     // hi(dec(15 - A)) - hi(dec(-A)) - 1 (0 if negative)
    uint32_t hk;       // hi(p) - (1076 << 20)
    uint32_t plo;      // lo(p)
    uint32_t lim;      // 32-bit delta bound: |v| high word below it -> |v * 10^A| < 2^30
    uint32_t pad;
};
struct cert_row32 {
    float p;
    uint32_t lo;       // bits(dec(-A))
    uint32_t span;     // bits(dec(6 - A)) - bits(dec(-A))
    uint32_t hk;       // bits(p) - (151 << 23)
};
#ifdef FB200_KERNEL_TU
FB_TABLE_SPACE cert_row64 g_cert_f64[23];
FB_TABLE_SPACE cert_row32 g_cert_f32[11];
#endif

// Device error word: ((key) << 8) | code, lowest key wins (atomicMin).
enum : uint32_t {
    DEV_OK = 0,
    DEV_E_SCALE = 2,
    DEV_E_CAPACITY = 4,
    DEV_E_HDR_TRUNC = 10,
    DEV_E_META = 11,
    DEV_E_W = 12,
    DEV_E_FLAGS_TRUNC = 13,
    DEV_E_FLAG_PAD = 14,
    DEV_E_ROW_TRUNC = 15,
    DEV_E_BITMAP_TRUNC = 16,
    DEV_E_PAYLOAD_TRUNC = 17,
    DEV_E_SIZE = 18,
    DEV_E_BATCH_HDR_TRUNC = 27,
    DEV_E_TABLE_TRUNC = 28,
    DEV_E_PAYLOAD_BATCH_TRUNC = 29,
    DEV_E_CHUNK_COUNT = 30,
    DEV_E_TRAILING = 31,
};

#ifdef FB200_KERNEL_TU
__device__ __forceinline__ uint64_t bits_of(double v) { return (uint64_t)__double_as_longlong(v); }
__device__ __forceinline__ uint32_t bits_of(float v) { return (uint32_t)__float_as_uint(v); }
__device__ __forceinline__ double value_of(uint64_t b) { return __longlong_as_double((long long)b); }
__device__ __forceinline__ float value_of(uint32_t b) { return __uint_as_float(b); }

__device__ __forceinline__ double pow10_of(double, int a) { return g_pow10_f64[a]; }
__device__ __forceinline__ float pow10_of(float, int a) { return g_pow10_f32[a]; }
__device__ __forceinline__ double rpow10_of(double, int a) { return g_rpow10_f64[a]; }
__device__ __forceinline__ float rpow10_of(float, int a) { return g_rpow10_f32[a]; }

__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
// std::round: half away from zero (numeric.hpp:127)
__device__ __forceinline__ double round_away(double x) { return round(x); }
__device__ __forceinline__ float round_away(float x) { return roundf(x); }
__device__ __forceinline__ long long llround_away(double x) { return llround(x); }
__device__ __forceinline__ long long llround_away(float x) { return llroundf(x); }
// (T)g for int64 g, round to nearest (numeric.hpp:161)
__device__ __forceinline__ double from_i64(double, long long g) { return __ll2double_rn(g); }
__device__ __forceinline__ float from_i64(float, long long g) { return __ll2float_rn(g); }

template <typename T> __device__ __forceinline__ T rel_eps();
template <> __device__ __forceinline__ double rel_eps<double>() { return 0x1p-52; }
template <> __device__ __forceinline__ float rel_eps<float>() { return 0x1p-23f; }

// floor_log10 of a positive normal value given its bit pattern (numeric.hpp:54-66).
__device__ __forceinline__ int floor_log10_bits(uint64_t a) {
    using tr = lane_traits<double>;
    const int e = (int)((a >> tr::mant) & tr::emask) - tr::bias;
    int k = (int)(((long long)e * 78913) >> 18);
    k = k < tr::min_decade ? tr::min_decade : (k > tr::max_decade ? tr::max_decade : k);
    while (k > tr::min_decade && a < g_decade_f64[k - tr::min_decade]) --k;
    while (k < tr::max_decade && a >= g_decade_f64[k + 1 - tr::min_decade]) ++k;
    return k;
}
__device__ __forceinline__ int floor_log10_bits(uint32_t a) {
    using tr = lane_traits<float>;
    const int e = (int)((a >> tr::mant) & tr::emask) - tr::bias;
    int k = (int)(((long long)e * 78913) >> 18);
    k = k < tr::min_decade ? tr::min_decade : (k > tr::max_decade ? tr::max_decade : k);
    while (k > tr::min_decade && a < g_decade_f32[k - tr::min_decade]) --k;
    while (k < tr::max_decade && a >= g_decade_f32[k + 1 - tr::min_decade]) ++k;
    return k;
}

// Per-value decimal place (dp_ds_calculate, numeric.hpp:108-140).  Returns alpha in
// [0, max_alpha], or -1 when the value takes the exception path (the chunk then goes
// to Case 2: transform.hpp:54-55).  Only alpha is needed by analyze_chunk; beta's bound
// is enforced inside the loop exactly as the reference does.
template <typename T>
__device__ __forceinline__ int dp_alpha(T v) {
    using tr = lane_traits<T>;
    using B = typename tr::B;
    const B b = bits_of(v);
    const B mag_bits = b & ~((B)1 << (tr::width - 1));
    if (mag_bits == 0) return (b >> (tr::width - 1)) ? -1 : 0;  // +0 -> (0,0); -0 -> exc
    const unsigned e = (unsigned)(b >> tr::mant) & tr::emask;
    if (e == 0 || e == tr::emask) return -1;                     // subnormal / inf / nan
    const int mag = floor_log10_bits(mag_bits);
    int alpha = mag < 0 ? -mag : 0;
    int beta = alpha + mag + 1;
    while (beta <= tr::max_beta && alpha <= tr::max_alpha) {
        const T p = pow10_of(T{}, alpha);
        const T scaled = mul_rn(v, p);
        const T nearest = round_away(scaled);
        const T gap = fabs(sub_rn(scaled, nearest));
        if (gap <= mul_rn(fabs(scaled), rel_eps<T>())) {
            if (div_rn(nearest, p) != v) return -1;
            return alpha;
        }
        ++alpha;
        ++beta;
    }
    return -1;
}

template <typename B>
__device__ __forceinline__ B zigzag(B x_as_unsigned) {
    using S = typename std::conditional<sizeof(B) == 8, int64_t, int32_t>::type;
    const S x = (S)x_as_unsigned;
    return ((B)x << 1) ^ (B)(x >> (sizeof(B) * 8 - 1));
}
template <typename B>
__device__ __forceinline__ B unzigzag(B z) {
    return (z >> 1) ^ ((B)0 - (z & 1));
}

// 8x8 bit-matrix transpose within a 64-bit word: bit (8r + c) <-> bit (8c + r).
// Self-inverse.  Used by both encode (lanes -> plane bytes) and decode.
__host__ __device__ __forceinline__ uint64_t transpose8x8(uint64_t x) {
    uint64_t t;
    t = (x ^ (x >> 7)) & 0x00AA00AA00AA00AAull;
    x ^= t ^ (t << 7);
    t = (x ^ (x >> 14)) & 0x0000CCCC0000CCCCull;
    x ^= t ^ (t << 14);
    t = (x ^ (x >> 28)) & 0x00000000F0F0F0F0ull;
    x ^= t ^ (t << 28);
    return x;
}

// relaxed GPU-scope 64-bit load/store for the decoupled look-back status words
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// relaxed 32-bit load/store without a compiler memory clobber (self-contained words: the
// encoder's look-ahead sample verdicts, see encode.cu)
__device__ __forceinline__ uint32_t ld_relaxed32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void st_relaxed32(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v));
}
__device__ __forceinline__ uint32_t ld_acquire32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release32(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void record_error(unsigned long long* err, uint64_t key, uint32_t code) {
    atomicMin(err, (unsigned long long)((key << 8) | code));
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    return v;
}

#endif  // FB200_KERNEL_TU

// Geometry shared by encode and decode: the archive places batch b's frame after
// 47 header bytes, all earlier frames' (4 + 4*C) table bytes and all earlier chunks'
// payload bytes (FORMAT.md:33-45; container.cpp:88-111).  Every batch but the last
// holds exactly `cpb` chunks (batch_values is fixed per archive).
struct geometry {
    uint64_t header_bytes;   // 47 for a whole archive, 0 for a frames-only shard / batch
    uint64_t n_values;       // total values
    uint64_t batch_values;
    uint32_t chunk_n;
    uint32_t cpb;            // chunks per full batch = ceil(batch_values / chunk_n)
    uint64_t n_batches;
    uint64_t n_chunks;       // total chunks over all batches
    uint32_t last_cpb;       // chunks in the final batch
    uint64_t cpb_magic;      // ceil(2^64 / cpb) (0 when cpb == 1), make_geometry

    // c / cpb; on the device one 64-bit multiply-high (exact for c < 2^32 chunks: the error
    // of ceil(2^64/cpb) moves c/cpb by less than 2^-32 < 1/cpb)
    __host__ __device__ uint64_t batch_of(uint64_t c) const {
#ifdef __CUDA_ARCH__
        return cpb_magic ? __umul64hi(c, cpb_magic) : c;
#else
        return c / cpb;
#endif
    }
    __host__ __device__ uint32_t chunks_in(uint64_t b) const {
        return b + 1 == n_batches ? last_cpb : cpb;
    }
    __host__ __device__ uint64_t values_in(uint64_t b) const {
        const uint64_t first = b * batch_values;
        const uint64_t rest = n_values - first;
        return rest < batch_values ? rest : batch_values;
    }
    // archive offset of batch b's frame minus the payload of all earlier chunks
    __host__ __device__ uint64_t frame_base(uint64_t b) const {
        return header_bytes + b * (4 + 4 * (uint64_t)cpb);
    }
    // archive offset of chunk c's payload minus the payload of all earlier chunks
    __host__ __device__ uint64_t chunk_base(uint64_t c) const {
        const uint64_t b = batch_of(c);
        return frame_base(b) + 4 + 4 * (uint64_t)chunks_in(b);
    }
};

}  // namespace fb200
