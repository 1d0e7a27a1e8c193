// encode.cu -- fused single-pass Falcon compress for sm_100a.
//
// One CTA encodes one chunk (chunk_n values: z1 + (chunk_n-1) delta lanes) and
// writes it straight into its final archive position:
//
//   load    chunk values -> padded smem                       (coalesced 8/4-B loads)
//   analyze dp_ds per value -> alpha_max, any-exception, max|v| (warp redux + smem)
//           (numeric.hpp:108-140, transform.hpp:47-68)
//   delta   g_i = llround(v*10^a) | zigzag(bits); z_i = zigzag(g_i - g_{i-1})
//           (transform.hpp:72-89), thread t owns lanes 8t..8t+7 ("byte column" t)
//   planes  per 8 bit-planes: pack one byte of each of the 8 lanes, 8x8 bit transpose
//           -> the thread's byte of each plane row (bitplane.hpp:64-90 semantics)
//   size    per-row zero-byte count via ballot, dense/sparse choice, row offsets
//           (bitplane.hpp:113-122, chunk_codec.hpp:59-73)
//   place   decoupled look-back over chunk sizes in ticket order -> archive offset;
//           the batch frame's table bytes are added analytically (container.cpp:88-111)
//   emit    chunk image built in smem at the destination's 16-B phase, then stored
//           with 16-B vector stores (sparse rows compacted with ballot prefix counts)
//
// A second, tiny kernel (frame_tables) writes the per-batch [u32 count][u32 size..]
// tables and the 47-byte header once every chunk's prefix is known.
#include "falcon_common.cuh"
#include "kernels.h"

namespace fb200 {

namespace {

constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagInc = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;


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

template <typename B>
__device__ __forceinline__ B warp_max(B v);
template <>
__device__ __forceinline__ uint64_t warp_max(uint64_t v) {
    const uint32_t hi = __reduce_max_sync(0xffffffffu, (uint32_t)(v >> 32));
    const uint32_t lo = __reduce_max_sync(0xffffffffu, (uint32_t)(v >> 32) == hi ? (uint32_t)v : 0u);
    return ((uint64_t)hi << 32) | lo;
}
template <>
__device__ __forceinline__ uint32_t warp_max(uint32_t v) {
    return __reduce_max_sync(0xffffffffu, v);
}

__device__ __forceinline__ int bit_width(uint64_t x) { return x ? 64 - __clzll((long long)x) : 0; }
__device__ __forceinline__ int bit_width(uint32_t x) { return x ? 32 - __clz((int)x) : 0; }

// byte s of lane value x (s < sizeof(B))
__device__ __forceinline__ uint32_t byte_of(uint64_t x, int s) {
    return (uint32_t)(x >> (8 * s)) & 0xffu;
}
__device__ __forceinline__ uint32_t byte_of(uint32_t x, int s) { return (x >> (8 * s)) & 0xffu; }

}  // namespace

// bytes of the values region, which is reused as the chunk-image staging buffer
template <typename T>
__host__ __device__ __forceinline__ uint32_t encode_region_bytes(uint32_t chunk_n) {
    using tr = lane_traits<T>;
    const uint32_t nc = (chunk_n - 1) / 8;
    const uint32_t vals = (uint32_t)((pidx(chunk_n) + 1) * sizeof(T) + 15) & ~15u;
    const uint32_t stage = (uint32_t)(tr::header + (tr::width + 7) / 8 + tr::width * nc + 16 + 15) & ~15u;
    return vals > stage ? vals : stage;
}

template <typename T, int MAXT>
__global__ void __launch_bounds__(MAXT, MAXT <= 256 ? 1024 / MAXT : 1) encode_chunks_kernel(const T* __restrict__ in, geometry g,
                                                             uint8_t* __restrict__ out,
                                                             uint64_t out_cap, encode_ws ws) {
    using tr = lane_traits<T>;
    using B = typename tr::B;
    using S = typename tr::S;
    constexpr int W = tr::width;
    constexpr int HDR = tr::header;

    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t n = g.chunk_n;
    const int NC = (int)((n - 1) / 8);  // row bytes = byte columns
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = blockDim.x >> 5;

    // smem carve-up (sizes must match encode_smem_bytes())
    const uint32_t vals_region = encode_region_bytes<T>(n);
    T* s_v = reinterpret_cast<T*>(smem);
    uint8_t* s_stage = smem;                                    // aliases s_v after transform
    uint8_t* s_rows = smem + vals_region;                       // [W][NC]
    uint16_t* s_nzw = reinterpret_cast<uint16_t*>(s_rows + ((W * NC + 15) & ~15));  // [W][nwarps]

    __shared__ uint32_t s_ticket;
    __shared__ uint32_t s_amax[32], s_exc[32], s_warpw[32];
    __shared__ B s_vmax[32];
    __shared__ uint32_t s_nz[64];
    __shared__ uint32_t s_rowoff[64];
    __shared__ uint64_t s_dense, s_off;
    __shared__ uint32_t s_size;
    __shared__ B s_z1;

    if (tid == 0) s_ticket = atomicAdd(ws.ticket, 1u);
    for (int i = tid; i < 64; i += blockDim.x) s_nz[i] = 0;
    __syncthreads();
    const uint64_t c = s_ticket;
    const uint64_t b = g.batch_of(c);
    const uint32_t ci = (uint32_t)(c - b * g.cpb);
    const uint64_t bcount = g.values_in(b);
    const uint64_t v0 = b * g.batch_values + (uint64_t)ci * n;
    const uint64_t left = bcount - (uint64_t)ci * n;
    const uint32_t len = left < n ? (uint32_t)left : n;   // short final chunk: +0.0 padding

    // ---- load (pipeline.hpp:205-215 padding) ----
    for (uint32_t i = tid; i < n; i += blockDim.x) s_v[pidx(i)] = i < len ? in[v0 + i] : T(0);
    __syncthreads();

    // ---- analyze (transform.hpp:47-68) ----
    int amax = 0;
    bool exc = false;
    B vmax = 0;
    for (uint32_t i = tid; i < n; i += blockDim.x) {
        const T v = s_v[pidx(i)];
        const int a = dp_alpha<T>(v);
        exc |= a < 0;
        amax = a > amax ? a : amax;
        const B m = bits_of(v) & ~((B)1 << (W - 1));
        vmax = m > vmax ? m : vmax;
    }
    {
        const uint32_t wa = __reduce_max_sync(0xffffffffu, (uint32_t)amax);
        const bool we = __any_sync(0xffffffffu, exc);
        const B wv = warp_max<B>(vmax);
        if (lane == 0) {
            s_amax[warp] = wa;
            s_exc[warp] = we;
            s_vmax[warp] = wv;
        }
    }
    __syncthreads();
    amax = 0;
    exc = false;
    vmax = 0;
    for (int w = 0; w < nwarps; ++w) {
        amax = (int)s_amax[w] > amax ? (int)s_amax[w] : amax;
        exc |= s_exc[w] != 0;
        vmax = s_vmax[w] > vmax ? s_vmax[w] : vmax;
    }
    bool case2 = exc;
    int bhat = 0;
    if (!case2) {
        bhat = vmax == 0 ? 0 : amax + floor_log10_bits(vmax) + 1;
        case2 = amax > tr::max_alpha || bhat > tr::max_beta;
    }
    const uint32_t hA = case2 ? tr::exc_alpha : (uint32_t)amax;
    const uint32_t hB = case2 ? tr::exc_beta : (uint32_t)bhat;

    // ---- forward transform in byte-column layout (transform.hpp:72-89) ----
    const T scale = pow10_of(T{}, case2 ? 0 : amax);
    bool range_err = false;
    auto lane_g = [&](T v) -> B {
        if (case2) return zigzag<B>(bits_of(v));
        const T s = mul_rn(v, scale);
        range_err |= !(fabs(s) < (T)0x1p62);                  // numeric.hpp:153-154
        return (B)(S)llround_away(s);
    };
    B z[8];
    B orv = 0;
    if (tid < NC) {
        B gp = lane_g(s_v[pidx(8 * tid)]);
        if (tid == 0) s_z1 = gp;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const B gj = lane_g(s_v[pidx(8 * tid + 1 + j)]);
            z[j] = zigzag<B>((B)(gj - gp));
            gp = gj;
            orv |= z[j];
        }
    } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) z[j] = 0;
    }
    if (range_err) record_error(ws.error, c, DEV_E_SCALE);

    // ---- bit planes: warp-local width, 8x8 transposes, zero-byte counts ----
    const int warp_w = bit_width(warp_or<B>(orv));
    const int nblk = (warp_w + 7) >> 3;
    for (int s = 0; s < nblk; ++s) {
        // lane j's byte s at byte (7-j): the transpose then yields, in byte k, the
        // row byte of bit plane 8s+k with lane j at bit 7-j (MSB-first, FORMAT.md:81-84)
        uint64_t x = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) x |= (uint64_t)byte_of(z[j], s) << (8 * (7 - j));
        const uint64_t y = transpose8x8(x);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int p = 8 * s + k;
            if (p < warp_w) {
                const uint32_t byte = (uint32_t)(y >> (8 * k)) & 0xffu;
                if (tid < NC) s_rows[p * NC + tid] = (uint8_t)byte;
                const uint32_t nzm = __ballot_sync(0xffffffffu, byte != 0);
                if (lane == 0) {
                    s_nzw[p * nwarps + warp] = (uint16_t)__popc(nzm);
                    atomicAdd(&s_nz[p], (uint32_t)__popc(nzm));
                }
            }
        }
    }
    if (lane == 0) s_warpw[warp] = (uint32_t)warp_w;
    __syncthreads();

    int w = 0;
    for (int i = 0; i < nwarps; ++i) w = (int)s_warpw[i] > w ? (int)s_warpw[i] : w;
    const int fb = (w + 7) >> 3;

    // ---- sizes, row offsets, look-back (warp 0) ----
    if (warp == 0) {
        auto row_cost = [&](int p, bool& dense) -> uint32_t {
            dense = false;
            if (p >= w) return 0;
            const uint32_t nz = s_nz[p];
            const uint32_t zeros = (uint32_t)NC - nz;
            dense = zeros <= (uint32_t)(NC / 8);                   // bitplane.hpp:113-115
            return dense ? (uint32_t)NC : (uint32_t)(NC / 8) + nz;  // bitplane.hpp:117-122
        };
        bool d0, d1;
        const uint32_t c0 = row_cost(lane, d0);
        const uint32_t c1 = row_cost(lane + 32, d1);
        // rows are emitted from the highest plane down: offset(p) = sum of cost(p' > p)
        uint32_t s1 = c1, s0 = c0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t t1 = __shfl_down_sync(0xffffffffu, s1, d);
            const uint32_t t0 = __shfl_down_sync(0xffffffffu, s0, d);
            if (lane + d < 32) {
                s1 += t1;
                s0 += t0;
            }
        }
        const uint32_t tot1 = __shfl_sync(0xffffffffu, s1, 0);
        const uint32_t tot0 = __shfl_sync(0xffffffffu, s0, 0);
        const uint32_t base = HDR + fb;
        s_rowoff[lane + 32] = base + (s1 - c1);
        s_rowoff[lane] = base + tot1 + (s0 - c0);
        const uint32_t dm0 = __ballot_sync(0xffffffffu, d0);
        const uint32_t dm1 = __ballot_sync(0xffffffffu, d1);
        const uint32_t size = w ? base + tot1 + tot0 : (uint32_t)HDR;

        // decoupled look-back over chunk sizes, in ticket (= chunk) order
        uint64_t excl = 0;
        if (lane == 0) st_relaxed(&ws.status[c], (c == 0 ? kFlagInc : kFlagAgg) | size);
        if (c > 0) {
            int64_t j = (int64_t)c - 1;
            for (;;) {
                const int64_t idx = j - lane;
                uint64_t st = idx >= 0 ? ld_relaxed(&ws.status[idx]) : kFlagInc;
                while (__ballot_sync(0xffffffffu, (st >> 62) == 0) != 0) {
                    __nanosleep(64);
                    if ((st >> 62) == 0) st = ld_relaxed(&ws.status[idx]);
                }
                const uint32_t inc = __ballot_sync(0xffffffffu, (st >> 62) == 2);
                uint64_t val = st & kValMask;
                if (inc) {
                    const int first = __ffs(inc) - 1;
                    excl += warp_sum_u64(lane <= first ? val : 0);
                    break;
                }
                excl += warp_sum_u64(val);
                j -= 32;
            }
            if (lane == 0) st_relaxed(&ws.status[c], kFlagInc | (excl + size));
        }
        if (lane == 0) {
            s_dense = ((uint64_t)dm1 << 32) | dm0;
            s_size = size;
            s_off = g.chunk_base(c) + excl;
        }
    }
    __syncthreads();

    const uint32_t size = s_size;
    const uint64_t off = s_off;
    if (off + size > out_cap) {
        if (tid == 0) record_error(ws.error, c, DEV_E_CAPACITY);
        return;
    }
    const uint32_t a = (uint32_t)(off & 15);
    const uint64_t dense = s_dense;

    // ---- emit the chunk image into staging at the destination's 16-B phase ----
    if (tid == 0) {
        uint8_t* h = s_stage + a;
        h[0] = (uint8_t)hA;
        h[1] = (uint8_t)hB;
        const B z1 = s_z1;
#pragma unroll
        for (int i = 0; i < (int)sizeof(B); ++i) h[2 + i] = (uint8_t)(z1 >> (8 * i));
        h[2 + sizeof(B)] = (uint8_t)w;
        for (int i = 0; i < fb; ++i) h[HDR + i] = (uint8_t)(dense >> (8 * (fb - 1 - i)));
    }
    const uint32_t lt_mask = (1u << lane) - 1u;
    for (int p = 0; p < w; ++p) {
        const bool mine = tid < NC && p < (int)s_warpw[warp];
        const uint32_t byte = mine ? s_rows[p * NC + tid] : 0u;
        uint8_t* row = s_stage + a + s_rowoff[p];
        if ((dense >> p) & 1) {
            if (tid < NC) row[tid] = (uint8_t)byte;
        } else {
            const uint32_t nzm = __ballot_sync(0xffffffffu, byte != 0);
            if (tid < NC && (lane & 7) == 0) row[tid >> 3] = (uint8_t)(__brev(nzm >> lane) >> 24);
            if (byte != 0) {
                uint32_t before = 0;
                for (int q = 0; q < warp; ++q)
                    before += p < (int)s_warpw[q] ? s_nzw[p * nwarps + q] : 0u;
                row[NC / 8 + before + __popc(nzm & lt_mask)] = (uint8_t)byte;
            }
        }
    }
    __syncthreads();

    // ---- store: 16-B vectors for whole segments, bytes at the two ragged ends ----
    uint8_t* dst = out + (off - a);
    const uint32_t end = a + size;
    const uint32_t nvec = (end + 15) >> 4;
    for (uint32_t v = tid; v < nvec; v += blockDim.x) {
        const uint32_t lo = v << 4, hi = lo + 16;
        if (lo >= a && hi <= end) {
            *reinterpret_cast<uint4*>(dst + lo) = *reinterpret_cast<const uint4*>(s_stage + lo);
        } else {
            const uint32_t from = lo > a ? lo : a, to = hi < end ? hi : end;
            for (uint32_t i = from; i < to; ++i) dst[i] = s_stage[i];
        }
    }
}

// Batch tables + header (container.cpp:44-55, 88-111).  Every chunk's inclusive
// prefix is final once encode_chunks_kernel has returned.
__global__ void frame_tables_kernel(geometry g, uint8_t* __restrict__ out, uint64_t out_cap,
                                    encode_ws ws, archive_header_bytes hdr) {
    const uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c == 0 && g.header_bytes == 47) {
        for (int i = 0; i < 47; ++i) out[i] = hdr.b[i];
    }
    if (c >= g.n_chunks) return;
    const uint64_t inc = ws.status[c] & kValMask;
    const uint64_t prev = c ? (ws.status[c - 1] & kValMask) : 0;
    const uint64_t b = g.batch_of(c);
    const uint32_t ci = (uint32_t)(c - b * g.cpb);
    const uint64_t first = b * g.cpb;
    const uint64_t pfirst = first ? (ws.status[first - 1] & kValMask) : 0;
    const uint64_t frame = g.frame_base(b) + pfirst;
    const uint32_t size = (uint32_t)(inc - prev);
    if (frame + 4 + 4 * (uint64_t)g.chunks_in(b) > out_cap) return;  // capacity error already raised
    uint8_t* e = out + frame + 4 + 4 * (uint64_t)ci;
    e[0] = (uint8_t)size;
    e[1] = (uint8_t)(size >> 8);
    e[2] = (uint8_t)(size >> 16);
    e[3] = (uint8_t)(size >> 24);
    if (ci == 0) {
        const uint32_t cnt = g.chunks_in(b);
        out[frame] = (uint8_t)cnt;
        out[frame + 1] = (uint8_t)(cnt >> 8);
        out[frame + 2] = (uint8_t)(cnt >> 16);
        out[frame + 3] = (uint8_t)(cnt >> 24);
    }
    if (c + 1 == g.n_chunks) *ws.total = g.chunk_base(c) + inc;
}

uint32_t encode_block_threads(uint32_t chunk_n) {
    const uint32_t nc = (chunk_n - 1) / 8;
    return nc < 32 ? 32 : ((nc + 31) / 32) * 32;
}

template <typename T>
uint32_t encode_smem_bytes(uint32_t chunk_n) {
    using tr = lane_traits<T>;
    const uint32_t nc = (chunk_n - 1) / 8;
    // staging for the largest chunk image plus its 16-B phase shares the values region
    const uint32_t vals = encode_region_bytes<T>(chunk_n);
    const uint32_t rows = (tr::width * nc + 15) & ~15u;
    const uint32_t nzw = tr::width * (encode_block_threads(chunk_n) / 32) * 2;
    return vals + rows + nzw;
}

template <typename T>
cudaError_t launch_encode(const T* d_in, const geometry& g, uint8_t* d_out, uint64_t out_cap,
                          const encode_ws& ws, const archive_header_bytes& hdr, cudaStream_t st) {
    cudaError_t e;
    if ((e = cudaMemsetAsync(ws.status, 0, g.n_chunks * sizeof(uint64_t), st))) return e;
    if ((e = cudaMemsetAsync(ws.ticket, 0, sizeof(uint32_t), st))) return e;
    if (g.n_chunks == 0) {
        // empty input: a bare header (test_pipeline.cpp:109-122)
        if ((e = cudaMemcpyAsync(ws.total, &g.header_bytes, sizeof(uint64_t), cudaMemcpyHostToDevice, st)))
            return e;
        return g.header_bytes ? cudaMemcpyAsync(d_out, hdr.b, 47, cudaMemcpyHostToDevice, st) : cudaSuccess;
    }
    const uint32_t threads = encode_block_threads(g.chunk_n);
    const uint32_t smem = encode_smem_bytes<T>(g.chunk_n);
    auto kern = threads <= 256 ? encode_chunks_kernel<T, 256> : encode_chunks_kernel<T, 1024>;
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return e;
    kern<<<(unsigned)g.n_chunks, threads, smem, st>>>(d_in, g, d_out, out_cap, ws);
    if ((e = cudaGetLastError())) return e;
    const unsigned tb = 256;
    frame_tables_kernel<<<(unsigned)((g.n_chunks + tb - 1) / tb), tb, 0, st>>>(g, d_out, out_cap, ws, hdr);
    return cudaGetLastError();
}

template cudaError_t launch_encode<double>(const double*, const geometry&, uint8_t*, uint64_t,
                                           const encode_ws&, const archive_header_bytes&, cudaStream_t);
template cudaError_t launch_encode<float>(const float*, const geometry&, uint8_t*, uint64_t,
                                          const encode_ws&, const archive_header_bytes&, cudaStream_t);
template uint32_t encode_smem_bytes<double>(uint32_t);
template uint32_t encode_smem_bytes<float>(uint32_t);

}  // namespace fb200
