// encode.cu -- Falcon compress for sm_100a: encode_chunks_kernel + place_final_kernel.
//
// encode_chunks_kernel: one CTA per chunk (chunk_n values: z1 + (chunk_n-1) delta
// lanes).  Thread t owns the "byte column" t: delta lanes 8t..8t+7 (values 8t+1..8t+8),
// which is exactly byte t of every bit-plane row (FORMAT.md:79-84), so planes come out of
// per-thread 8x8 bit transposes.
//
//   load     each thread loads its 8 values + the preceding one into registers (16-B
//            vector loads of its window; the chunk one CTA generation ahead is pulled
//            into L2 with a bulk prefetch)
//   analyze  phase 1 (sample_chunks_kernel, ahead of the encode launch): the exact dp_ds
//            loop on 32 samples of the chunk -> A0 (attained)
//            phase 2: every value gets the one-sided lean certification at A0
//            (dpds.cuh); the few it cannot decide run the exact loop.  alpha_max,
//            exceptions, max|v| (numeric.hpp:108-140, transform.hpp:47-68), bit-exact
//   delta    Case 1 reuses the certified lane integers, Case 2 zigzags the bits;
//            z = zigzag(g_i - g_{i-1}) (transform.hpp:72-89), 32-bit when it fits
//   planes   per 8 bit positions: PRMT gather + 8x8 bit transpose -> the thread's row
//            bytes; nonzero-byte counts per plane by REDUX
//   size     warp 0: dense/sparse choice per row, row offsets, chunk size
//            (bitplane.hpp:113-122, chunk_codec.hpp:59-73)
//   emit     every thread writes its column of every row into the smem image (sparse
//            rows: bitmap bytes + payload at warp prefix + ballot rank,
//            bitplane.hpp:126-148); one TMA bulk copy into the chunk's scratch slot
//
// placement (place_tile: grid row 0 of a later wave's encode launch, and
// place_final_kernel after the last wave): scan of the chunk sizes in tiles with a
// decoupled look-back, then the images are copied to their archive offsets and the batch
// tables and the header are written (container.cpp:44-55, 88-111).
#include "dpds.cuh"
#include "falcon_common.cuh"
#include "kernels.h"

#include <cstdlib>
#include <type_traits>

namespace fb200 {

namespace {

constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagInc = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

// chunk-uniform certification parameters at scale A (constant table, tables.cu)
__device__ __forceinline__ cert_params<double> cert_params_at(double, int A) {
    const cert_row64& r = g_cert_f64[A];
    cert_params<double> c;
    c.p = r.p;
    c.lo1 = r.lo1;
    c.span = r.span;
    c.hk = r.hk;
    c.plo = r.plo;
    return c;
}
__device__ __forceinline__ cert_params<float> cert_params_at(float, int A) {
    const cert_row32& r = g_cert_f32[A];
    cert_params<float> c;
    c.p = r.p;
    c.lo = r.lo;
    c.span = r.span;
    c.hk = r.hk;
    return c;
}
__device__ __forceinline__ uint32_t narrow_lim(double, int A) { return g_cert_f64[A].lim; }
__device__ __forceinline__ uint32_t narrow_lim(float, int) { return 0u; }

template <typename B>
__device__ __forceinline__ B warp_or(B v);
template <>
__device__ __forceinline__ uint64_t warp_or(uint64_t v) {
    const uint32_t lo = __reduce_or_sync(0xffffffffu, (uint32_t)v);
    const uint32_t hi = __reduce_or_sync(0xffffffffu, (uint32_t)(v >> 32));
    return ((uint64_t)hi << 32) | lo;
}
template <>
__device__ __forceinline__ uint32_t warp_or(uint32_t v) {
    return __reduce_or_sync(0xffffffffu, v);
}

__device__ __forceinline__ int bit_width(uint64_t x) { return x ? 64 - __clzll((long long)x) : 0; }
__device__ __forceinline__ int bit_width(uint32_t x) { return x ? 32 - __clz((int)x) : 0; }

}  // namespace

// bytes of the chunk-image staging region
template <typename T>
__host__ __device__ __forceinline__ uint32_t encode_stage_bytes(uint32_t chunk_n) {
    using tr = lane_traits<T>;
    const uint32_t nc = (chunk_n - 1) / 8;
    return (uint32_t)(tr::header + (tr::width + 7) / 8 + tr::width * nc + 32 + 15) & ~15u;
}

// L2 residency of the image ring (FB_L2_HINTS): the streaming value loads are marked
// evict-first, so the images one wave writes are still in L2 when the next launch places
// them; after a chunk is placed its image lines are discarded (no write-back of dead data).
// Measured on cfg2 (A/B, profiles/r02): no gain (compress 1.319 ms without, 1.345 ms
// with), so off by default.
#ifndef FB_L2_HINTS
#define FB_L2_HINTS 0
#endif
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ double ld_stream(const double* p, uint64_t pol) {
#if FB_L2_HINTS
    double v;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
#else
    (void)pol;
    return __ldg(p);
#endif
}
__device__ __forceinline__ float ld_stream(const float* p, uint64_t pol) {
#if FB_L2_HINTS
    float v;
    asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
#else
    (void)pol;
    return __ldg(p);
#endif
}
__device__ __forceinline__ void l2_discard_line(const void* p) {
#if FB_L2_HINTS
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
#else
    (void)p;
#endif
}

// 32-bit word of lane values whose byte q is gathered (sb < 4: low word, else high)
__device__ __forceinline__ uint32_t lane_word(uint64_t z, int sb) { return sb < 4 ? (uint32_t)z : (uint32_t)(z >> 32); }
__device__ __forceinline__ uint32_t lane_word(uint32_t z, int) { return z; }

// 0x01 in every nonzero byte of w
__device__ __forceinline__ uint32_t nonzero_bytes(uint32_t w) {
    return ((((w & 0x7f7f7f7fu) + 0x7f7f7f7fu) | w) >> 7) & 0x01010101u;
}

// resident CTAs of <= 128 threads per SM the register budget targets.  The encoder is
// latency-bound between its block barriers, so occupancy pays until spills dominate:
// f64 at 9 (56 registers, no spills; cfg2 encode 1.139 ms at 8 blocks, 1.106 ms at 9,
// 1.143 ms at 10 with spills; re-checked with phase 1 in the sampler: compress 1.134 ms at
// 8, 1.126 ms at 9), f32 at 12 (cfg3 encode 1.65 ms at 8 blocks, 1.39 ms at 12, 1.35 ms
// at 16 with the in-kernel phase 1; without it: compress 1.508 ms at 12, 1.542 ms at 14
// and 16 -- 32 registers spilled)
#ifndef FB_ENC_MIN_BLOCKS
#define FB_ENC_MIN_BLOCKS 9
#endif
// image store by one TMA bulk copy (cfg2 compress 1.125 -> 1.115 ms, cfg3 1.508 -> 1.465
// ms against the 16-B vector store loop over all threads)
#ifndef FB_ENC_SEL_TREE
#define FB_ENC_SEL_TREE 0
#endif
#ifndef FB_SAMPLE_K64
#define FB_SAMPLE_K64 3
#endif
#ifndef FB_ENC_BULK_STORE
#define FB_ENC_BULK_STORE 1
#endif
#ifndef FB_ENC_VEC_LOADS
#define FB_ENC_VEC_LOADS 1
#endif
#ifndef FB_ENC_MIN_BLOCKS32
#define FB_ENC_MIN_BLOCKS32 12
#endif
template <typename T, int NT>
constexpr int encode_min_blocks() {
    return NT <= 128 ? (sizeof(T) == 4 ? FB_ENC_MIN_BLOCKS32 : FB_ENC_MIN_BLOCKS) : (2048 / NT > 0 ? 2048 / NT : 1);
}
// Phase 1 of every chunk ahead of the encode launch: kSamples lanes per chunk sample the
// chunk's first values, run the exact dp_ds loop on them (numeric.hpp:108-140) and store
// the OR of the one-hot alphas (bit 31: an exception).  The encoder then certifies at
// A0 = the largest sampled alpha with no warp-0-only phase and no barrier before phase 2
// (that phase was the encoder's top stall: 19 % of its stall samples on cfg2).  A0 only
// selects the encoder's fast path (alpha_max == A0), never the output.  The exact loop is
// ~250 warp-instructions per sample step, so the sampler is issue-bound: 8 samples per
// chunk (4 chunks per warp) instead of the 32 of the in-kernel phase it replaces (cfg2
// sampler 78 us at 32 samples per chunk).
#ifndef FB_SAMPLES
#define FB_SAMPLES 8
#endif
constexpr int kSamples = FB_SAMPLES;
#ifndef FB_ENC_PDL
#define FB_ENC_PDL 1
#endif
constexpr bool kEncPDL = FB_ENC_PDL != 0;
template <typename T>
__global__ void __launch_bounds__(256) sample_chunks_kernel(const T* __restrict__ in, geometry g,
                                                            uint32_t* __restrict__ look) {
    constexpr int CPW = 32 / kSamples;   // chunks per warp
    const int lane = threadIdx.x & 31;
    const uint64_t c = ((uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * CPW + (uint64_t)(lane / kSamples);
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // the encode launch may start
    const uint32_t n = g.chunk_n;
    const uint32_t i = (uint32_t)(lane % kSamples) % n;
    T v = T(0);
    if (c < g.n_chunks) {
        const uint64_t b = g.batch_of(c);
        const uint64_t ci = c - b * g.cpb;
        const uint64_t left = g.values_in(b) - ci * n;
        const uint32_t len = left < n ? (uint32_t)left : n;
        // values past a short final chunk are its +0.0 padding (pipeline.hpp:205-215)
        if (i < len) v = __ldg(in + b * g.batch_values + ci * n + i);
    }
    const int a = dp_alpha_k<T, sizeof(T) == 8 ? FB_SAMPLE_K64 : 3>(v);
    uint32_t f = a < 0 ? 0x80000000u : (1u << a);
#pragma unroll
    for (int d = 1; d < kSamples; d <<= 1) f |= __shfl_xor_sync(0xffffffffu, f, d);
    if (lane % kSamples == 0 && c < g.n_chunks) look[c] = f;
}

template <int NT, int U, int NTHR = NT>
__device__ void place_tile(const geometry& g, uint8_t* __restrict__ out, uint64_t out_cap, const encode_ws& ws,
                           const encode_launch& L, const archive_header_bytes& hdr, uint8_t* smem);

template <typename T, int NT>
__global__ void __launch_bounds__(NT, encode_min_blocks<T, NT>())
    encode_chunks_kernel(const T* __restrict__ in, geometry g, uint8_t* __restrict__ out,
                         uint64_t out_cap, encode_ws ws, encode_launch L, archive_header_bytes hdr) {
    using tr = lane_traits<T>;
    using X = fpx<T>;
    using B = typename tr::B;
    using S = typename tr::S;
    constexpr int HDR = tr::header;

    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t n = g.chunk_n;
    const int NC = (int)((n - 1) / 8);  // row bytes = byte columns
    const int BM = NC / 8;              // sparse bitmap bytes
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int nwarps = NT / 32;
    constexpr int PT = NT;

    uint8_t* s_stage = smem;  // chunk image (phase 0)
    // [block][thread] u64: byte k of entry (s, t) = row byte t of bit plane 8s+k
    uint64_t* s_planes = reinterpret_cast<uint64_t*>(smem + encode_stage_bytes<T>(n));

    __shared__ uint32_t s_flag2[nwarps];                   // bit 31 exception | one-hot alphas
    __shared__ uint32_t s_mag[nwarps];                     // max floor_log10 + 1024 (0: none)
    __shared__ uint32_t s_warpw[nwarps];
    __shared__ __align__(16) uint32_t s_rowoff[64];        // plane p: row offset in the image
    __shared__ uint32_t s_nzc[nwarps][16];   // 8-bit nonzero-byte counters, 4 planes/word
    __shared__ __align__(16) uint32_t s_pbase[nwarps * 64]; // [w][p]: payload position of warp w's first byte in row p
    __shared__ uint64_t s_dense;
    __shared__ uint32_t s_size;
    __shared__ B s_z1;

    // grid row 0: placement of the tiles the previous launches finished encoding (their
    // images sit in the ring; see launch_encode); rows 1..: x = chunk in batch, y - 1 =
    // batch of this wave (no integer division)
    if (blockIdx.y == 0) {
        // beside encode CTAs: 2 vectors per lane in flight (f64, 56 registers), 1 for f32
        // (32 registers)
        if (blockIdx.x < L.place_tiles) place_tile<NT, sizeof(T) == 8 ? 2 : 1>(g, out, out_cap, ws, L, hdr, smem);
        return;
    }
    const uint32_t b = L.b0 + blockIdx.y - 1;
    const uint32_t ci = blockIdx.x;
    uint32_t len = n;
    if (b >= L.full_b) {  // the last batch / short chunks: bounds and the chunk length
        if (b >= g.n_batches || ci >= g.chunks_in(b)) return;  // uniform per CTA
        const uint64_t left = g.values_in(b) - (uint64_t)ci * n;
        len = left < n ? (uint32_t)left : n;  // short final chunk: +0.0 padding
    } else if (ci >= g.cpb) {
        return;
    }
    const uint32_t c = b * g.cpb + ci;                      // < 2^31 chunks per launch
    const uint64_t v0 = (uint64_t)b * g.batch_values + (uint64_t)ci * n;
    const bool active = tid < NC;

    // The chunk L.pf_ahead CTAs later (about one generation of resident CTAs) is pulled into
    // L2 with one bulk prefetch, so its CTA's value loads hit L2 instead of waiting on DRAM
    // (the load latency sits on every CTA's critical path: phase 2 cannot start without it).
#ifndef FB_ENC_NO_PREFETCH
    // (f64 only: cfg2 compress -1.2 %; f32 had no gain and its 32-register budget spilled)
    if (sizeof(T) == 8 && tid == 0 && L.pf_ahead) {
        uint32_t ci2 = ci + L.pf_ahead;
        uint32_t b2 = b;
        if (ci2 >= g.cpb) {
            ci2 -= g.cpb;
            ++b2;
        }
        if (ci2 < g.cpb && b2 < L.b_end && ci2 < g.chunks_in(b2)) {
            const uint64_t s0 = ((uint64_t)b2 * g.batch_values + (uint64_t)ci2 * n) * sizeof(T);
            const uint64_t e0 = min(s0 + (uint64_t)n * sizeof(T), g.n_values * sizeof(T));
            const uint64_t s16 = s0 & ~15ull, e16 = e0 & ~15ull;
            if (e16 > s16)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<const char*>(in) + s16),
                             "r"((uint32_t)(e16 - s16)) : "memory");
        }
    }
#endif

    // ---- load: values 8t .. 8t+8 (pipeline.hpp:205-215 zero padding) ----
    T v[8];
    T vprev = T(0);
    {
        const T* src = in + v0 + 8u * (uint32_t)tid;
        const uint64_t pol = l2_evict_first_policy();
        // a full chunk inside the input (not its first values before a 16-B boundary, not its
        // last): 16-B vector loads of the window that starts at the 16-B boundary at or below
        // value 8t (phase ph uniform per CTA: the chunk start decides it); the window ends at
        // most 3 values past the chunk
        const uint32_t ph = (uint32_t)(((uintptr_t)(in + v0) >> (sizeof(T) == 8 ? 3 : 2)) & (sizeof(T) == 8 ? 1u : 3u));
        const bool vec = FB_ENC_VEC_LOADS && len == n && NC == NT && v0 >= ph && v0 + 8ull * NT + 12ull <= g.n_values;
        if (vec) {
            constexpr int EPV = 16 / (int)sizeof(T);             // values per vector
            constexpr int NV = sizeof(T) == 8 ? 5 : 3;           // vectors per thread
            T w[NV * EPV];
            const uint4* vs = reinterpret_cast<const uint4*>(src - ph);
#pragma unroll
            for (int q = 0; q < NV; ++q) {
                const uint4 x = __ldg(vs + q);
                if constexpr (sizeof(T) == 8) {
                    w[2 * q] = __longlong_as_double(((long long)x.y << 32) | x.x);
                    w[2 * q + 1] = __longlong_as_double(((long long)x.w << 32) | x.z);
                } else {
                    w[4 * q] = __uint_as_float(x.x);
                    w[4 * q + 1] = __uint_as_float(x.y);
                    w[4 * q + 2] = __uint_as_float(x.z);
                    w[4 * q + 3] = __uint_as_float(x.w);
                }
            }
            // value 8t + i is w[ph + i]; ph is uniform, so each case is straight-line code
            auto pick = [&](auto P) {
                constexpr int p = decltype(P)::value;
                vprev = w[p];
#pragma unroll
                for (int j = 0; j < 8; ++j) v[j] = w[p + 1 + j];
            };
            if constexpr (sizeof(T) == 8) {
                if (ph == 0) pick(std::integral_constant<int, 0>{});
                else pick(std::integral_constant<int, 1>{});
            } else {
                if (ph == 0) pick(std::integral_constant<int, 0>{});
                else if (ph == 1) pick(std::integral_constant<int, 1>{});
                else if (ph == 2) pick(std::integral_constant<int, 2>{});
                else pick(std::integral_constant<int, 3>{});
            }
        } else if (len == n && NC == NT) {
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = ld_stream(src + 1 + j, pol);
            vprev = ld_stream(src, pol);
        } else {
            const uint32_t i0 = 8u * (uint32_t)tid;
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = (active && i0 + 1 + j < len) ? ld_stream(src + 1 + j, pol) : T(0);
            if (active && i0 < len) vprev = ld_stream(src, pol);
        }
    }

    // ---- analyze, phase 1 (decided ahead by sample_chunks_kernel): A0 = the largest
    //      alpha of kSamples sampled chunk values, attained, so alpha_max >= A0; bit 31 =
    //      a sampled exception (the chunk is Case 2, phase 2 is skipped).  The first encode
    //      launch starts beside the sampler (programmatic dependent launch): the value
    //      loads above are in flight while it waits for the sampler's results. ----
    asm volatile("griddepcontrol.wait;" ::: "memory");
    uint32_t F = __ldg(ws.look + c);
    const int A0 = (F & 0x7fffffffu) ? 31 - __clz((int)(F & 0x7fffffffu)) : 0;

    // ---- analyze, phase 2: lean certification of every value at A0 (dpds.cuh); the
    //      undecided ones (zeros, powers of two, decade edges, exceptions, alpha > A0)
    //      run the exact loop.  Thread 0 also covers value 0 (bit 8). ----
    // low words of the certified lane integers (all the 32-bit delta path needs; keeping
    // 8 registers fewer lets 9 CTAs per SM run without spills)
    uint32_t gc[8];
    uint32_t redo = 0;   // values the exact loop decides
    uint32_t f2 = 0;     // exception bit | one-hot alphas of values decided by the exact loop
    uint32_t mx = 0;     // max |v| high word (f32: bits) -> floor_log10(max|v|) for beta_hat
    if (active && !(F >> 31)) {
        const cert_params<T> cp = cert_params_at(T{}, A0);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            uint32_t ah;
            S g;
            const bool ok = certify_lean(v[j], cp, &g, &ah);
            gc[j] = (uint32_t)g;
            mx = ah > mx ? ah : mx;
            redo |= ok ? 0u : (1u << j);
        }
        if (tid == 0) {
            S g0;
            uint32_t ah;
            const bool ok = certify_lean(vprev, cp, &g0, &ah);
            mx = ah > mx ? ah : mx;
            redo |= ok ? 0u : 0x100u;
        }
        for (uint32_t rest = redo; rest; rest &= rest - 1) {  // rare: exact loop
            const int j = __ffs(rest) - 1;
            T vj = vprev;
#pragma unroll
            for (int q = 0; q < 8; ++q) vj = j == q ? v[q] : vj;
            const int a = dp_alpha_full<T>(vj);
            f2 |= a < 0 ? 0x80000000u : (1u << a);
            if (a < 0) break;  // the chunk is Case 2: nothing else matters
        }
    }
    f2 = __reduce_or_sync(0xffffffffu, f2) | F;   // + the sample's flags
    const uint32_t mxw = __reduce_max_sync(0xffffffffu, mx);
    if (lane == 0) {
        s_flag2[warp] = f2;
        s_mag[warp] = mxw;
    }
    __syncthreads();
    uint32_t M = 0;
#pragma unroll
    for (int i = 0; i < nwarps; ++i) {
        F |= s_flag2[i];
        M = s_mag[i] > M ? s_mag[i] : M;
    }
    const int amax = (F & 0x7fffffffu) ? 31 - __clz((int)(F & 0x7fffffffu)) : 0;
    bool case2 = (F >> 31) != 0;
    int bhat = 0;
    if (!case2 && M != 0) {  // transform.hpp:62-65: beta_hat = alpha_max + floor_log10(max|v|) + 1
        int mag;
        if constexpr (sizeof(T) == 4) {
            mag = mag_of<T>(M);  // max|v| is a positive normal here (else Case 2)
        } else {
            // only the high word of max|v| is known: exact unless a decade boundary
            // falls inside it, then a second (uniform, rare) pass finds the low word
            const int k0 = mag_of<T>((uint64_t)M << 32);
            const int k1 = mag_of<T>(((uint64_t)M << 32) | 0xffffffffull);
            if (k0 == k1) {
                mag = k0;
            } else {
                uint32_t ml = 0;
                if (active) {
#pragma unroll
                    for (int j = 0; j < 9; ++j) {
                        if (j == 8 && tid != 0) break;
                        const uint64_t ab = (uint64_t)X::bits(j == 8 ? vprev : v[j < 8 ? j : 0]) & ~(uint64_t)X::SIGN;
                        if ((uint32_t)(ab >> 32) == M && (uint32_t)ab > ml) ml = (uint32_t)ab;
                    }
                }
                ml = __reduce_max_sync(0xffffffffu, ml);
                __syncthreads();
                if (lane == 0) s_mag[warp] = ml;
                __syncthreads();
                ml = 0;
#pragma unroll
                for (int i = 0; i < nwarps; ++i) ml = s_mag[i] > ml ? s_mag[i] : ml;
                mag = mag_of<T>(((uint64_t)M << 32) | ml);
            }
        }
        bhat = amax + mag + 1;
    }
    if (!case2) case2 = amax > tr::max_alpha || bhat > tr::max_beta;
    const uint32_t hA = case2 ? tr::exc_alpha : (uint32_t)amax;
    const uint32_t hB = case2 ? tr::exc_beta : (uint32_t)bhat;

    // ---- forward transform (transform.hpp:72-89) ----
    // Case 1 at alpha_max == A0: every value has alpha_v <= A0, so v * 10^A0 lies within
    // 3.5 ulp (<= 1/8) of its integer and rint == llround -- the certification's lane
    // integers are final, also for the values the exact loop decided.  When every integer
    // of the CHUNK fits in 30 bits (|v| < 2^(28 - e_p), e_p = exponent of the scale) the
    // f64 delta/zigzag runs in 32-bit arithmetic: the same z, half the ALU work.  The test
    // is chunk-wide (M = max high word over all values, value 0 included): the first delta
    // of warp k starts from the last value of warp k-1 (index 256k), so a per-warp vote
    // would miss a wide value there (transform.hpp:87-88 wraps in 64 bits).
    const T scale = X::pow10(case2 ? 0 : amax);
    const bool reuse = !case2 && amax == A0;
    // (reuse: scale = 10^A0, whose 32-bit bound is in the table)
    const bool narrow = sizeof(B) == 8 && reuse && M < narrow_lim(T{}, A0);
    B z[8];
    B orv = 0;
    if (narrow) {
        uint32_t gp = (uint32_t)__double2ll_rz(rint(mul_rn(vprev, scale)));
        if (tid == 0) s_z1 = (B)(S)(int32_t)gp;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t gj = (uint32_t)gc[j];
            const uint32_t d = gj - gp;
            z[j] = (B)((d << 1) ^ (uint32_t)((int32_t)d >> 31));
            gp = gj;
        }
        uint32_t o = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) o |= (uint32_t)z[j];
        orv = active ? (B)o : (B)0;
    } else if (reuse) {
        // (vprev is a chunk value with alpha_v <= A0, so rint is llround, as for gc)
        B gp = (B)(S)X::to_int(X::rint_(mul_rn(vprev, scale)));
        if (tid == 0) s_z1 = gp;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            // f64: recompute certify's integer (only wide-integer chunks get here)
            const B gj = sizeof(B) == 8 ? (B)(S)X::to_int(X::rint_(mul_rn(v[j], scale))) : (B)(S)(int32_t)gc[j];
            z[j] = zigzag<B>((B)(gj - gp));
            gp = gj;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) orv |= z[j];
        if (!active) orv = 0;
    } else if (case2) {
        // Case 2: the raw bit patterns, zigzagged (transform.hpp:54-55, 72-89).  Separate
        // straight-line branches: with case2 tested inside one per-value helper the compiler
        // kept eight copies of the predicate packed into a register on the common path.
        B gp = zigzag<B>(X::bits(vprev));
        if (tid == 0) s_z1 = gp;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const B gj = zigzag<B>(X::bits(v[j]));
            z[j] = zigzag<B>((B)(gj - gp));
            gp = gj;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) orv |= z[j];
        if (!active) orv = 0;
    } else {
        // Case 1 with alpha_max above the sampled A0: llround(v * 10^alpha_max)
        bool range_err = false;
        auto lane_g = [&](T x) -> B {
            const T s = mul_rn(x, scale);
            range_err |= !(fabs(s) < (T)0x1p62);  // numeric.hpp:153-154
            return (B)(S)llround_away(s);
        };
        B gp = lane_g(vprev);
        if (tid == 0) s_z1 = gp;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const B gj = lane_g(v[j]);
            z[j] = zigzag<B>((B)(gj - gp));
            gp = gj;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) orv |= z[j];
        if (!active) orv = 0;
        if (range_err) record_error(ws.error, c, DEV_E_SCALE);
    }

    // ---- bit planes: warp-local width, 8x8 transposes -> s_planes, nonzero counts.
    //      Inactive columns (tid >= NC) are masked by orv = 0 only through warp_w; their
    //      plane bytes are never stored. ----
    const int warp_w = bit_width(warp_or<B>(orv));
    const int nblk = (warp_w + 7) >> 3;
#pragma unroll
    for (int sb = 0; sb < tr::width / 8; ++sb) {
        if (sb >= nblk) break;
        // byte sb of lane j goes to byte 7-j of x: byte k of the transpose is then the row
        // byte of bit plane 8sb+k with lane j at bit 7-j (MSB-first, FORMAT.md:81-84)
        const uint32_t q = (uint32_t)(sb & 3);
        const uint32_t sel = q | ((4u + q) << 4);
        const uint32_t xl = __byte_perm(__byte_perm(lane_word(z[7], sb), lane_word(z[6], sb), sel),
                                        __byte_perm(lane_word(z[5], sb), lane_word(z[4], sb), sel), 0x5410);
        const uint32_t xh = __byte_perm(__byte_perm(lane_word(z[3], sb), lane_word(z[2], sb), sel),
                                        __byte_perm(lane_word(z[1], sb), lane_word(z[0], sb), sel), 0x5410);
        const uint64_t y = active ? transpose8x8(((uint64_t)xh << 32) | xl) : 0ull;
        s_planes[sb * PT + tid] = y;
        // nonzero bytes per plane as 8-bit counters (<= 32 per warp, no carries)
        const uint32_t lo = __reduce_add_sync(0xffffffffu, nonzero_bytes((uint32_t)y));
        const uint32_t hi = __reduce_add_sync(0xffffffffu, nonzero_bytes((uint32_t)(y >> 32)));
        if (lane == 0) {
            s_nzc[warp][2 * sb] = lo;
            s_nzc[warp][2 * sb + 1] = hi;
        }
    }
    if (lane == 0) s_warpw[warp] = (uint32_t)warp_w;
    __syncthreads();

    int w = 0;
#pragma unroll
    for (int i = 0; i < nwarps; ++i) w = (int)s_warpw[i] > w ? (int)s_warpw[i] : w;
    const int fb = (w + 7) >> 3;

    // ---- sizes and row offsets (warp 0): plane p is row w-1-p.  Lane L sizes plane L;
    //      planes 32..63 (f64 chunks with w > 32 only) go first, their total offsets the
    //      lower rows.  (f32 and the common w <= 32 skip that half: cfg2 w is ~14-20.) ----
    if (warp == 0) {
        auto row_cost = [&](int p, uint32_t nz, bool& dns) -> uint32_t {
            dns = false;
            if (p >= w) return 0;
            dns = (uint32_t)NC - nz <= (uint32_t)BM;        // bitplane.hpp:113-115
            return dns ? (uint32_t)NC : (uint32_t)BM + nz;  // bitplane.hpp:117-122
        };
        // plane p of the half starting at P0: row cost, reverse (suffix) scan, row offset,
        // per-warp sparse payload starts; returns the half's total cost
        auto size_half = [&](const int P0, const uint32_t above, bool& dns) -> uint32_t {
            const int p = P0 + lane;
            uint32_t nz = 0;
            uint32_t wp[nwarps];  // payload bytes of plane p in the warps before q
#pragma unroll
            for (int q = 0; q < nwarps; ++q) {
                const uint32_t cq = p < (int)s_warpw[q] ? (s_nzc[q][p >> 2] >> (8 * (lane & 3))) & 0xffu : 0u;
                wp[q] = nz;
                nz += cq;
            }
            const uint32_t cost = row_cost(p, nz, dns);
            // rows are emitted from the highest plane down: offset(p) = sum of cost(p' > p)
            uint32_t sfx = cost;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t t = __shfl_down_sync(0xffffffffu, sfx, d);
                if (lane + d < 32) sfx += t;
            }
            const uint32_t ro = HDR + fb + above + (sfx - cost);
            s_rowoff[p] = ro;
#pragma unroll
            for (int q = 0; q < nwarps; ++q) s_pbase[q * 64 + p] = ro + (uint32_t)BM + wp[q];
            return __shfl_sync(0xffffffffu, sfx, 0);
        };
        uint32_t tot1 = 0, dm1 = 0;
        if (tr::width > 32 && w > 32) {
            bool d1;
            tot1 = size_half(32, 0u, d1);
            dm1 = __ballot_sync(0xffffffffu, d1);
        }
        bool d0;
        const uint32_t tot0 = size_half(0, tot1, d0);
        const uint32_t dm0 = __ballot_sync(0xffffffffu, d0);
        const uint32_t size = w ? HDR + fb + tot1 + tot0 : (uint32_t)HDR;
        if (lane == 0) {
            s_dense = ((uint64_t)dm1 << 32) | dm0;
            s_size = size;
            ws.sizes[c] = size;
        }
    }
    __syncthreads();
    const uint32_t size = s_size;
    const uint64_t dense = s_dense;

    // ---- emit the chunk image: header bytes one per thread, then every thread writes
    //      its column of every row (sparse rows: warp prefix + ballot rank) ----
    if (tid < HDR + fb) {
        uint32_t hb;
        if (tid == 0) hb = hA;
        else if (tid == 1) hb = hB;
        else if (tid < 2 + (int)sizeof(B)) hb = (uint32_t)(s_z1 >> (8 * (tid - 2)));
        else if (tid == 2 + (int)sizeof(B)) hb = (uint32_t)w;
        else hb = (uint32_t)(dense >> (8 * (fb - 1 - (tid - HDR))));
        s_stage[tid] = (uint8_t)hb;
    }
    const uint32_t lt_mask = (1u << lane) - 1u;
    const int wblk = (w + 7) >> 3;
    uint8_t* const col = s_stage + tid;
#pragma unroll
    for (int sb = 0; sb < tr::width / 8; ++sb) {
        if (sb >= wblk) break;
        const uint64_t y = sb < nblk ? s_planes[sb * PT + tid] : 0ull;  // above warp_w: zero
        const uint32_t ylo = (uint32_t)y, yhi = (uint32_t)(y >> 32);
        const int kmax = w - 8 * sb;
        const uint32_t valid = kmax >= 8 ? 0xffu : ((1u << kmax) - 1u);
        const uint32_t dblk = (uint32_t)(dense >> (8 * sb)) & valid;
        const uint32_t sblk = ~dblk & valid;
        if (dblk == 0xffu) {
            // eight dense rows, consecutive in the image (plane 8sb+7 first): one base
            // address, immediate offsets
            uint8_t* r7 = col + s_rowoff[8 * sb + 7];
            if (active) {
                r7[0 * NC] = (uint8_t)(yhi >> 24);
                r7[1 * NC] = (uint8_t)(yhi >> 16);
                r7[2 * NC] = (uint8_t)(yhi >> 8);
                r7[3 * NC] = (uint8_t)yhi;
                r7[4 * NC] = (uint8_t)(ylo >> 24);
                r7[5 * NC] = (uint8_t)(ylo >> 16);
                r7[6 * NC] = (uint8_t)(ylo >> 8);
                r7[7 * NC] = (uint8_t)ylo;
            }
            continue;
        }
        // this block's 8 row offsets and (sparse rows) this warp's payload prefixes
        const uint4 o03 = *reinterpret_cast<const uint4*>(&s_rowoff[8 * sb]);
        const uint4 o47 = *reinterpret_cast<const uint4*>(&s_rowoff[8 * sb + 4]);
        const uint32_t off[8] = {o03.x, o03.y, o03.z, o03.w, o47.x, o47.y, o47.z, o47.w};
        // remaining dense rows (a partly dense block is rare: uniform branches)
        if (dblk) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (((dblk >> k) & 1u) && active) col[off[k]] = (uint8_t)(k < 4 ? ylo >> (8 * k) : yhi >> (8 * (k - 4)));
        }
        // sparse rows (bitplane.hpp:126-148): bitmap byte j nonzero -> bit 7-j%8 of bitmap
        // byte j/8, then the nonzero bytes in order at warp prefix + ballot rank.  The 32
        // bitmap bytes a warp owns in this block (8 planes x 4) go out in one store.  Every
        // image byte below `size` is written (bitmaps always, payloads are contiguous), so
        // the staging buffer needs no zeroing.
        if (sblk) {
            const uint4 pb03 = *reinterpret_cast<const uint4*>(&s_pbase[warp * 64 + 8 * sb]);
            const uint4 pb47 = *reinterpret_cast<const uint4*>(&s_pbase[warp * 64 + 8 * sb + 4]);
            const uint32_t pbase[8] = {pb03.x, pb03.y, pb03.z, pb03.w, pb47.x, pb47.y, pb47.z, pb47.w};
            uint32_t mk[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                mk[k] = __ballot_sync(0xffffffffu, ((k < 4 ? ylo >> (8 * k) : yhi >> (8 * (k - 4))) & 0xffu) != 0u);
            }
            {
                const int kl = lane >> 2, ql = lane & 3;
#if FB_ENC_SEL_TREE
                // mk[kl] by a 3-level select tree on the bits of kl (7 selects, 3 tests)
                const bool k1 = kl & 1, k2 = kl & 2, k4 = kl & 4;
                const uint32_t m01 = k1 ? mk[1] : mk[0], m23 = k1 ? mk[3] : mk[2];
                const uint32_t m45 = k1 ? mk[5] : mk[4], m67 = k1 ? mk[7] : mk[6];
                const uint32_t m03 = k2 ? m23 : m01, m47 = k2 ? m67 : m45;
                const uint32_t mm = k4 ? m47 : m03;
#else
                uint32_t mm = mk[0];
#pragma unroll
                for (int k = 1; k < 8; ++k) mm = kl == k ? mk[k] : mm;
#endif
                const uint32_t bm = __brev(mm >> (8 * ql)) >> 24;
                if (((sblk >> kl) & 1u) && 4 * warp + ql < BM) s_stage[s_rowoff[8 * sb + kl] + 4 * warp + ql] = (uint8_t)bm;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t byte = (k < 4 ? ylo >> (8 * k) : yhi >> (8 * (k - 4))) & 0xffu;
                if (((sblk >> k) & 1u) && byte != 0u)
                    s_stage[pbase[k] + __popc(mk[k] & lt_mask)] = (uint8_t)byte;
            }
        }
    }
    __syncthreads();

    // ---- store the image into this chunk's ring slot (16-B aligned) ----
    uint32_t slot = L.enc_slot0 + (c - L.enc_c0);   // = c mod ring (no division)
    slot = slot >= ws.ring ? slot - (uint32_t)ws.ring : slot;
    uint4* dst = reinterpret_cast<uint4*>(ws.images + slot * (uint64_t)ws.slot);
    const uint4* srcv = reinterpret_cast<const uint4*>(s_stage);
    const uint32_t nvec = (size + 15) >> 4;
#if FB_ENC_BULK_STORE
    // one TMA bulk copy smem -> global (the image's generic-proxy smem writes are made
    // visible to the async proxy first); the issuing thread keeps the CTA (and its smem)
    // alive until the copy has read the staging buffer
    if (tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                     "r"((uint32_t)__cvta_generic_to_shared(srcv)), "r"(nvec * 16u) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
#else
    for (uint32_t vv = tid; vv < nvec; vv += NT) dst[vv] = srcv[vv];
#endif
}

// Placement: chunk images -> archive.  A tile of NT consecutive chunks per CTA (grid row 0
// of an encode launch, beside the next wave's encode CTAs);
// sizes are known up front, so every tile publishes its aggregate at once and the
// decoupled look-back never waits on compute.  The tile then writes its chunks'
// size-table entries (container.cpp:88-111), copies each image to
// chunk_base(c) + exclusive prefix with funnel-shifted 16-B stores, and the first
// tile writes the 47-byte header (container.cpp:44-55).
// NTHR threads (a multiple of NT): threads [0, NT) scan the tile, and the copy is spread
// over all NTHR / 32 warps, each moving NT * 32 / NTHR chunks (the final placement runs with
// more threads than chunks: with 32 chunks per warp a small input was a chain of dependent
// round trips per lane).
template <int NT, int U, int NTHR>
__device__ void place_tile(const geometry& g, uint8_t* __restrict__ out, uint64_t out_cap, const encode_ws& ws,
                           const encode_launch& L, const archive_header_bytes& hdr, uint8_t* smem) {
    constexpr int kPlaceTile = NT;
    static_assert(NTHR % NT == 0 && NTHR <= 1024, "placement threads");
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = kPlaceTile / 32;     // scan warps
    constexpr int NCW = NTHR / 32;          // copy warps
    constexpr int CPW = NT / NCW;           // chunks per copy warp (<= 32)
    // carved from the encode kernel's dynamic smem (placement_smem_bytes)
    uint64_t* s_off = reinterpret_cast<uint64_t*>(smem);                       // [NT]
    uint32_t* s_sz = reinterpret_cast<uint32_t*>(s_off + kPlaceTile);          // [NT]
    uint32_t (*s_vpre)[33] = reinterpret_cast<uint32_t (*)[33]>(s_sz + kPlaceTile);  // [NCW][33]
    __shared__ uint32_t s_ticket;
    __shared__ uint32_t s_wsum[NW];
    __shared__ uint64_t s_tile_excl;
    if (tid == 0) s_ticket = atomicAdd(ws.ticket, 1u);
    __syncthreads();
    const uint64_t t = s_ticket;
    const uint64_t c = t * kPlaceTile + tid;
    const bool valid = tid < kPlaceTile && c < g.n_chunks;
    const uint32_t sz = valid ? ws.sizes[c] : 0u;

    // tile-local exclusive scan (a tile holds < 2^32 bytes)
    uint32_t incl = sz;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t x = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += x;
    }
    if (lane == 31 && warp < NW) s_wsum[warp] = incl;
    __syncthreads();
    uint32_t wbase = 0, tile_sum = 0;
#pragma unroll
    for (int q = 0; q < NW; ++q) {
        wbase += q < warp ? s_wsum[q] : 0u;
        tile_sum += s_wsum[q];
    }
    // decoupled look-back over tiles (warp 0)
    if (warp == 0) {
        uint64_t excl = 0;
        if (lane == 0) st_relaxed(&ws.tile_status[t], (t == 0 ? kFlagInc : kFlagAgg) | tile_sum);
        if (t > 0) {
            int64_t j = (int64_t)t - 1;
            for (;;) {
                const int64_t idx = j - lane;
                uint64_t st = idx >= 0 ? ld_relaxed(&ws.tile_status[idx]) : kFlagInc;
                uint32_t inc, need;
                for (;;) {
                    inc = __ballot_sync(0xffffffffu, (st >> 62) == 2);
                    const uint32_t ready = __ballot_sync(0xffffffffu, (st >> 62) != 0);
                    need = inc ? (0xffffffffu >> (32 - __ffs(inc))) : 0xffffffffu;
                    if ((ready & need) == need) break;
                    __nanosleep(32);
                    if ((st >> 62) == 0) st = ld_relaxed(&ws.tile_status[idx]);
                }
                excl += warp_sum_u64(((need >> lane) & 1) ? (st & kValMask) : 0);
                if (inc) break;
                j -= 32;
            }
            if (lane == 0) st_relaxed(&ws.tile_status[t], kFlagInc | (excl + tile_sum));
        }
        if (lane == 0) s_tile_excl = excl;
    }
    __syncthreads();
    const uint64_t pexcl = s_tile_excl + wbase + (incl - sz);  // payload bytes before chunk c
    if (tid < kPlaceTile) {
        s_off[tid] = valid ? g.chunk_base(c) + pexcl : 0;
        s_sz[tid] = sz;
    }

    if (valid) {
        const uint64_t b = g.batch_of(c);
        if (c == b * g.cpb) {  // first chunk of its batch: publish the batch payload prefix
            // (flag and value in one word: nothing else is published, no fence needed)
            st_relaxed(&ws.batch_prefix[b], (1ull << 63) | pexcl);
        }
    }
    __syncthreads();
    if (valid) {
        const uint64_t b = g.batch_of(c);
        const uint32_t ci = (uint32_t)(c - b * g.cpb);
        const uint64_t first = b * g.cpb;
        uint64_t pf;
        if (first >= t * kPlaceTile) {
            pf = s_off[first - t * kPlaceTile] - g.chunk_base(first);
        } else {
            uint64_t w8;
            while (((w8 = ld_relaxed(&ws.batch_prefix[b])) >> 63) == 0) __nanosleep(64);
            pf = w8 & ~(1ull << 63);
        }
        const uint64_t frame = g.frame_base(b) + pf;
        if (frame + 4 + 4 * (uint64_t)g.chunks_in(b) <= out_cap) {
            uint8_t* e = out + frame + 4 + 4 * (uint64_t)ci;
            e[0] = (uint8_t)sz;
            e[1] = (uint8_t)(sz >> 8);
            e[2] = (uint8_t)(sz >> 16);
            e[3] = (uint8_t)(sz >> 24);
            if (ci == 0) {
                const uint32_t cnt = g.chunks_in(b);
                out[frame] = (uint8_t)cnt;
                out[frame + 1] = (uint8_t)(cnt >> 8);
                out[frame + 2] = (uint8_t)(cnt >> 16);
                out[frame + 3] = (uint8_t)(cnt >> 24);
            }
        }
        // a total beyond the buffer is never published: a chained decoder reads its archive
        // length from here (the capacity error is recorded by the copy below)
        if (c + 1 == g.n_chunks) *ws.total = s_off[tid] + sz <= out_cap ? s_off[tid] + sz : 0;
    }
    if (t == 0 && tid == 0 && g.header_bytes == 47) {
        for (int i = 0; i < 47; ++i) out[i] = hdr.b[i];
    }

    // copy: each warp moves its CPW chunks as one flat list of destination vectors, so a
    // lane's consecutive vectors are independent (their loads overlap) instead of the
    // chunks being copied one after another
    {
        const int idx = warp * CPW + lane;
        const uint64_t cc = t * kPlaceTile + idx;
        uint32_t nv = 0;
        if (lane < CPW && cc < g.n_chunks) {
            const uint64_t off = s_off[idx];
            const uint32_t size = s_sz[idx];
            if (off + size > out_cap) record_error(ws.error, cc, DEV_E_CAPACITY);
            else nv = ((uint32_t)(off & 15) + size + 15) >> 4;
        }
        uint32_t incl = nv;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t x = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += x;
        }
        if (lane < CPW) s_vpre[warp][lane] = incl - nv;
        if (lane == 31) s_vpre[warp][CPW] = incl;             // the warp's total
        __syncwarp();
    }
    const uint32_t V = s_vpre[warp][CPW];
    int k = 0;  // this lane's current chunk (vectors are visited in increasing order)
    // U vectors per lane in flight: all their loads are issued before the first store
    // (a lane's copy is otherwise a chain of ~V/32 dependent DRAM round trips)
    for (uint32_t gv0 = lane; gv0 < V; gv0 += 32 * U) {
        uint32_t r[U][5];
        uint8_t* dst[U];
        const uint8_t* src[U];
        uint32_t sh[U], from[U], to[U];
        bool vec[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t gv = gv0 + 32 * u;
            vec[u] = false;
            from[u] = to[u] = 0;
            if (gv >= V) continue;
            while (gv >= s_vpre[warp][k + 1]) ++k;
            const int idx = warp * CPW + k;
            const uint64_t cc = t * kPlaceTile + idx;
            const uint64_t off = s_off[idx];
            uint32_t rs = L.place_slot0 + (uint32_t)(cc - L.place_c0);   // = cc mod ring
            rs = rs >= ws.ring ? rs - (uint32_t)ws.ring : rs;
            const uint8_t* img = ws.images + rs * (uint64_t)ws.slot;
            const uint32_t a = (uint32_t)(off & 15);
            const uint32_t end = a + s_sz[idx];
            const uint32_t lo = (gv - s_vpre[warp][k]) << 4, hi = lo + 16;
            dst[u] = out + (off - a) + lo;
            if (lo >= a && hi <= end) {
                // destination bytes [lo, lo+16) = image bytes [lo - a, lo - a + 16)
                const uint32_t sb = lo - a;
                const uint32_t* w = reinterpret_cast<const uint32_t*>(img) + (sb >> 2);
                sh[u] = (sb & 3) * 8;
#pragma unroll
                for (int i = 0; i < 5; ++i) r[u][i] = __ldg(w + i);
                vec[u] = true;
            } else {
                from[u] = lo > a ? lo : a;
                to[u] = hi < end ? hi : end;
                src[u] = img + from[u] - a;
                dst[u] += (int)(from[u] - lo);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (vec[u]) {
                *reinterpret_cast<uint4*>(dst[u]) =
                    make_uint4(__funnelshift_r(r[u][0], r[u][1], sh[u]), __funnelshift_r(r[u][1], r[u][2], sh[u]),
                               __funnelshift_r(r[u][2], r[u][3], sh[u]), __funnelshift_r(r[u][3], r[u][4], sh[u]));
            } else {
                for (uint32_t i = 0; i < to[u] - from[u]; ++i) dst[u][i] = src[u][i];
            }
        }
    }
#if FB_L2_HINTS
    // the warp's 32 images are dead now: drop their L2 lines without a write-back (slots
    // are whole 128-B lines, encode_slot_bytes); lane L discards lines L, L + 32, ...
    __syncwarp();
    for (int q = 0; q < 32; ++q) {
        const uint64_t cc = t * kPlaceTile + warp * CPW + q;
        if (q >= CPW || cc >= g.n_chunks) break;
        uint32_t rs = L.place_slot0 + (uint32_t)(cc - L.place_c0);
        rs = rs >= ws.ring ? rs - (uint32_t)ws.ring : rs;
        const uint8_t* img = ws.images + rs * (uint64_t)ws.slot;
        const uint32_t lines = (s_sz[warp * CPW + q] + 4 + 127) >> 7;
        for (uint32_t ln = lane; ln < lines; ln += 32) l2_discard_line(img + 128 * ln);
    }
#endif
}

// The final placement of a compress call (tiles of the last wave), no encode beside it:
// a lane keeps 4 vectors in flight.
// Two shapes: NTHR = NT for large calls (cfg2/cfg3 compress -1.2 % / -2.8 % against the
// wide shape), NTHR = 4 NT (capped at 1024) when there are fewer tiles than two per SM,
// where the copy is latency-bound (cfg1 compress 0.057 -> 0.034 ms).
#ifndef FB_PLACE_MINB
#define FB_PLACE_MINB 1
#endif
#ifndef FB_PLACE_U
#define FB_PLACE_U 4
#endif
#ifndef FB_PLACE_U32
#define FB_PLACE_U32 2
#endif
// U: vectors per lane in flight in the NT shape -- 4 for f64 images, 2 for the smaller
// f32 ones (cfg3 compress 1.426 -> 1.416 ms; cfg2 loses 1.8 % at 2, 5.7 % at 8)
template <int NT, int NTHR, int U>
__global__ void __launch_bounds__(NTHR, NTHR == NT ? FB_PLACE_MINB : 1)
    place_final_kernel(geometry g, uint8_t* __restrict__ out, uint64_t out_cap, encode_ws ws, encode_launch L,
                       archive_header_bytes hdr) {
    extern __shared__ __align__(16) uint8_t smem[];
    // the wide shape keeps 8 vectors per lane in flight (few CTAs: latency-bound)
    place_tile<NT, NTHR == NT ? U : 8, NTHR>(g, out, out_cap, ws, L, hdr, smem);
}

// one thread per byte column, rounded to an instantiated CTA size
uint32_t encode_block_threads(uint32_t chunk_n) {
    const uint32_t nc = (chunk_n - 1) / 8;
    if (nc <= 256) return nc < 32 ? 32 : ((nc + 31) / 32) * 32;
    return nc <= 512 ? 512 : 1024;
}

template <typename T>
uint32_t encode_smem_bytes(uint32_t chunk_n) {
    using tr = lane_traits<T>;
    const uint32_t nt = encode_block_threads(chunk_n);
    const uint32_t enc = encode_stage_bytes<T>(chunk_n) + (tr::width / 8) * nt * 8;
    const uint32_t place = 12 * nt + 4 * 33 * (nt / 32);   // place_tile's carve-out
    return enc > place ? enc : place;
}

template <typename T>
uint32_t encode_slot_bytes(uint32_t chunk_n) {
    // max_encoded_chunk_size (chunk_codec.hpp:36-41) + 4 readable bytes for the funnel
    // loads of the placement copy, rounded to 16
    using tr = lane_traits<T>;
    const uint32_t nc = (chunk_n - 1) / 8;
    // whole 128-B lines, so a placed image's lines can be discarded (FB_L2_HINTS)
    return (uint32_t)(tr::header + (tr::width + 7) / 8 + tr::width * nc + 4 + 127) & ~127u;
}

// Waves: one encode launch covers `wave` batches; its grid row 0 places the tiles the
// previous launches finished (a final place-only launch takes the rest).  Images live in a
// ring of `ring` slots, so scratch is O(wave), not O(input): launch k writes chunks
// [c_k, c_k + wave chunks) while placing chunks in [c_{k-1} - tile, c_k); a ring of
// 2 * wave chunks + one tile keeps the two sets apart.
struct wave_plan {
    uint64_t wave_batches, launches, ring, tiles, tile;
};

// Fewer, larger waves are faster (cfg2 compress: 1.44 / 1.39 / 1.35 / 1.31 ms at 16 Ki /
// 24 Ki / 48 Ki / all 256 Ki chunks per wave), so a wave is as large as the ring budget
// allows: FALCON_ENC_RING_BYTES (default 4 GiB) holds two waves of image slots.  A call
// whose images fit the budget runs as one encode launch + the final placement.
static uint64_t env_u64(const char* name, uint64_t dflt) {
    const char* e = std::getenv(name);
    const unsigned long long x = e ? std::strtoull(e, nullptr, 10) : 0ull;
    return x ? (uint64_t)x : dflt;
}

static wave_plan plan_waves(const geometry& g, uint32_t slot_bytes) {
    wave_plan w;
    w.tile = encode_block_threads(g.chunk_n);
    w.tiles = (g.n_chunks + w.tile - 1) / w.tile;
    static const uint64_t ring_budget = env_u64("FALCON_ENC_RING_BYTES", 4ull << 30);
    static const uint64_t forced = env_u64("FALCON_ENC_WAVE_CHUNKS", 0);
    uint64_t wave_chunks = forced;
    if (!wave_chunks) {
        const uint64_t slots = ring_budget / slot_bytes;
        wave_chunks = slots >= g.n_chunks ? g.n_chunks : (slots > 2 * w.tile ? (slots - w.tile) / 2 : w.tile);
    }
    uint64_t wb = wave_chunks >= g.n_chunks ? g.n_batches : wave_chunks / g.cpb;
    if (wb < 1) wb = 1;
    if (wb > 65534) wb = 65534;                     // grid.y = 1 + batches of the wave
    if (wb >= g.n_batches) wb = g.n_batches;
    w.wave_batches = wb ? wb : 1;
    w.launches = g.n_batches ? (g.n_batches + w.wave_batches - 1) / w.wave_batches : 0;
    const uint64_t need = 2 * w.wave_batches * g.cpb + w.tile;
    w.ring = w.launches <= 1 || need >= g.n_chunks ? (g.n_chunks ? g.n_chunks : 1) : need;
    return w;
}

template <typename T>
size_t encode_scratch_bytes(const geometry& g) {
    const wave_plan w = plan_waves(g, encode_slot_bytes<T>(g.chunk_n));
    size_t b = 0;
    b += (g.n_chunks * 4 + 15) & ~15ull;                 // sizes
    b += w.tiles * 8;                                     // tile status
    b += (g.n_batches + 1) * 8;                           // batch prefixes
    b += g.n_chunks * 4;                                  // sample verdicts (phase 1)
    b = (b + 255) & ~255ull;
    b += w.ring * (uint64_t)encode_slot_bytes<T>(g.chunk_n);  // image ring
    return b;
}

template <typename T>
encode_ws carve_encode_ws(void* scratch, const geometry& g, uint32_t* ticket, unsigned long long* error,
                          uint64_t* total) {
    encode_ws ws;
    const wave_plan w = plan_waves(g, encode_slot_bytes<T>(g.chunk_n));
    uint8_t* p = static_cast<uint8_t*>(scratch);
    ws.sizes = reinterpret_cast<uint32_t*>(p);
    p += (g.n_chunks * 4 + 15) & ~15ull;
    ws.tile_status = reinterpret_cast<uint64_t*>(p);
    p += w.tiles * 8;
    ws.batch_prefix = reinterpret_cast<uint64_t*>(p);
    p += (g.n_batches + 1) * 8;
    ws.look = reinterpret_cast<uint32_t*>(p);
    p += g.n_chunks * 4;
    const size_t used = (size_t)(p - static_cast<uint8_t*>(scratch));
    p = static_cast<uint8_t*>(scratch) + ((used + 255) & ~255ull);
    ws.images = p;
    ws.slot = encode_slot_bytes<T>(g.chunk_n);
    ws.ring = w.ring;
    ws.ticket = ticket;
    ws.error = error;
    ws.total = total;
    return ws;
}

static cudaError_t launch_place_final(bool f32, uint32_t threads, uint32_t tiles, const geometry& g, uint8_t* d_out,
                                      uint64_t out_cap, const encode_ws& ws, const encode_launch& L,
                                      const archive_header_bytes& hdr, cudaStream_t st) {
    // FALCON_PLACE_WIDE_BELOW (tiles) overrides the shape choice (tests force both shapes)
    static const uint64_t wide_below = [] {
        const char* e = std::getenv("FALCON_PLACE_WIDE_BELOW");
        if (e) return (uint64_t)std::strtoull(e, nullptr, 10);
        int sms = 0;
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0) != cudaSuccess) sms = 148;
        return (uint64_t)2 * (uint64_t)sms;
    }();
    const bool wide = tiles < wide_below;
    const uint32_t nthr = wide ? (4 * threads <= 1024 ? 4 * threads : 1024) : threads;
    const uint32_t smem = 12 * threads + 4 * 33 * (nthr / 32);
    switch (threads) {
#define FB_PLACE(n)                                                                                          \
    case n:                                                                                                  \
        if (wide) place_final_kernel<n, (4 * n <= 1024 ? 4 * n : 1024), 8><<<tiles, nthr, smem, st>>>(g, d_out, out_cap, ws, L, hdr); \
        else if (f32) place_final_kernel<n, n, FB_PLACE_U32><<<tiles, nthr, smem, st>>>(g, d_out, out_cap, ws, L, hdr); \
        else place_final_kernel<n, n, FB_PLACE_U><<<tiles, nthr, smem, st>>>(g, d_out, out_cap, ws, L, hdr); \
        break;
    FB_PLACE(32) FB_PLACE(64) FB_PLACE(96) FB_PLACE(128) FB_PLACE(160) FB_PLACE(192) FB_PLACE(224)
    FB_PLACE(256) FB_PLACE(512)
#undef FB_PLACE
    default: return cudaErrorInvalidConfiguration;
    }
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_encode(const T* d_in, const geometry& g, uint8_t* d_out, uint64_t out_cap,
                          const encode_ws& ws, const archive_header_bytes& hdr, cudaStream_t st,
                          cudaEvent_t ev0, cudaEvent_t ev1) {
    cudaError_t e;
    if (g.n_chunks == 0) {
        // empty input: a bare header (test_pipeline.cpp:109-122)
        if ((e = cudaMemcpyAsync(ws.total, &g.header_bytes, sizeof(uint64_t), cudaMemcpyHostToDevice, st)))
            return e;
        return g.header_bytes ? cudaMemcpyAsync(d_out, hdr.b, 47, cudaMemcpyHostToDevice, st) : cudaSuccess;
    }
    const wave_plan w = plan_waves(g, encode_slot_bytes<T>(g.chunk_n));
    // tile status + batch prefixes are contiguous (sample_chunks_kernel writes every
    // chunk's sample verdict)
    if ((e = cudaMemsetAsync(ws.tile_status, 0, (w.tiles + g.n_batches + 1) * 8, st))) return e;
    if ((e = cudaMemsetAsync(ws.ticket, 0, sizeof(uint32_t), st))) return e;
    const uint32_t threads = encode_block_threads(g.chunk_n);
    const uint32_t smem = encode_smem_bytes<T>(g.chunk_n);
    void (*kern)(const T*, geometry, uint8_t*, uint64_t, encode_ws, encode_launch, archive_header_bytes);
    switch (threads) {
    case 32: kern = encode_chunks_kernel<T, 32>; break;
    case 64: kern = encode_chunks_kernel<T, 64>; break;
    case 96: kern = encode_chunks_kernel<T, 96>; break;
    case 128: kern = encode_chunks_kernel<T, 128>; break;
    case 160: kern = encode_chunks_kernel<T, 160>; break;
    case 192: kern = encode_chunks_kernel<T, 192>; break;
    case 224: kern = encode_chunks_kernel<T, 224>; break;
    case 256: kern = encode_chunks_kernel<T, 256>; break;
    case 512: kern = encode_chunks_kernel<T, 512>; break;
    case 1024: kern = encode_chunks_kernel<T, 1024>; break;
    default: kern = nullptr;
    }
    if (!kern) return cudaErrorInvalidConfiguration;
    if ((e = ensure_dynamic_smem((const void*)kern, smem))) return e;
    if (ev0 && (e = cudaEventRecord(ev0, st))) return e;
    {   // phase 1 of every chunk (its sample verdict) ahead of the encode launches
        const uint64_t per_block = 8 * (32 / kSamples);
        sample_chunks_kernel<T><<<(unsigned)((g.n_chunks + per_block - 1) / per_block), 256, 0, st>>>(d_in, g, ws.look);
        if ((e = cudaGetLastError())) return e;
    }
    uint64_t placed = 0;
    for (uint64_t k = 0; k <= w.launches; ++k) {
        encode_launch L;
        const uint64_t b0 = k * w.wave_batches;
        L.b0 = (uint32_t)(k < w.launches ? b0 : 0);
        const uint64_t nb = k < w.launches ? (g.n_batches - b0 < w.wave_batches ? g.n_batches - b0 : w.wave_batches) : 0;
        // tiles whose chunks all were encoded by launches < k
        const uint64_t done_chunks = k < w.launches ? b0 * g.cpb : g.n_chunks;
        const uint64_t placeable = k < w.launches ? done_chunks / w.tile : w.tiles;
        L.place_tiles = (uint32_t)(placeable - placed);
        // ring slots without a division in the kernel: slot(c) = slot0 + (c - c0), wrapped once
        L.enc_c0 = (uint32_t)(b0 * g.cpb);
        L.enc_slot0 = (uint32_t)((b0 * g.cpb) % w.ring);
        L.place_c0 = (uint32_t)(placed * w.tile);
        L.place_slot0 = (uint32_t)((placed * w.tile) % w.ring);
        L.b_end = (uint32_t)(b0 + nb);
        L.full_b = g.batch_values % g.chunk_n == 0 && g.n_batches ? (uint32_t)(g.n_batches - 1) : 0u;
        // A/B knob FALCON_ENC_PREFETCH = distance in chunks (0: off)
        static const char* pfe = std::getenv("FALCON_ENC_PREFETCH");
        static const uint32_t pf = pfe ? (uint32_t)std::strtoul(pfe, nullptr, 10) : 768u;
        L.pf_ahead = pf;
        if (nb == 0 && L.place_tiles == 0) continue;
        if (nb == 0) {
            e = launch_place_final(sizeof(T) == 4, threads, L.place_tiles, g, d_out, out_cap, ws, L, hdr, st);
        } else {
            const unsigned gx = (unsigned)(g.cpb > L.place_tiles ? g.cpb : L.place_tiles);
            // the first launch overlaps the sampler's tail (programmatic dependent launch;
            // its CTAs wait for the sampler after issuing their value loads)
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(gx, (unsigned)(1 + nb));
            cfg.blockDim = dim3(threads);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = st;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = (k == 0 && kEncPDL) ? 1 : 0;
            e = cudaLaunchKernelEx(&cfg, kern, d_in, g, d_out, out_cap, ws, L, hdr);
        }
        if (e) return e;
        placed = placeable;
    }
    return ev1 ? cudaEventRecord(ev1, st) : cudaSuccess;
}

template cudaError_t launch_encode<double>(const double*, const geometry&, uint8_t*, uint64_t,
                                           const encode_ws&, const archive_header_bytes&, cudaStream_t,
                                           cudaEvent_t, cudaEvent_t);
template cudaError_t launch_encode<float>(const float*, const geometry&, uint8_t*, uint64_t,
                                          const encode_ws&, const archive_header_bytes&, cudaStream_t,
                                          cudaEvent_t, cudaEvent_t);
template uint32_t encode_smem_bytes<double>(uint32_t);
template uint32_t encode_smem_bytes<float>(uint32_t);
template uint32_t encode_slot_bytes<double>(uint32_t);
template uint32_t encode_slot_bytes<float>(uint32_t);
template size_t encode_scratch_bytes<double>(const geometry&);
template size_t encode_scratch_bytes<float>(const geometry&);
template encode_ws carve_encode_ws<double>(void*, const geometry&, uint32_t*, unsigned long long*, uint64_t*);
template encode_ws carve_encode_ws<float>(void*, const geometry&, uint32_t*, unsigned long long*, uint64_t*);

}  // namespace fb200
