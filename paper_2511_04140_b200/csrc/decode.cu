// decode.cu -- single-launch Falcon decompress for sm_100a.
//
// The archive has no batch index (FORMAT.md:10-14): batch b+1's frame starts where
// batch b's payload ends, so frames must be located sequentially.  Ticket 0 of the
// launch is a *frame walker* CTA that runs the read_batch chain (container.cpp:113-132,
// pipeline.hpp:394-417): it validates each frame, scans its u32 size table into
// per-chunk offsets and publishes the batch.  Every other ticket decodes one chunk as
// soon as its batch is published, so the walk overlaps the decode of earlier batches.
//
// Per chunk (decompress_chunk, chunk_codec.hpp:86-122):
//   stage   chunk bytes -> smem with 16-B vector loads at the source's 16-B phase
//   parse   header + flag + row-walk validation in reference check order (warp 0)
//   rows    dense rows copied, sparse rows expanded with ballot ranks (one warp/row)
//   planes  thread t owns byte column t: 8x8 transposes rebuild lanes 8t..8t+7
//   scan    block-wide wrapping inclusive scan of unzigzagged deltas (transform.hpp:91-106)
//   values  Case 1: (T)g / 10^alpha (IEEE division), Case 2: raw bits; coalesced stores
#include "falcon_common.cuh"
#include "kernels.h"

namespace fb200 {

namespace {


__device__ __forceinline__ uint32_t ld_u32_le(const uint8_t* p) {
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

// Frame walker: validates frames in archive order and publishes per-chunk offsets.
__device__ void walk_frames(const uint8_t* __restrict__ arc, uint64_t len, const geometry& g,
                            const decode_ws& ws) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nthreads = blockDim.x, nwarps = nthreads >> 5;
    __shared__ uint32_t s_cnt, s_code;
    __shared__ uint64_t s_wsum[32];
    __shared__ uint64_t s_payload;
    uint64_t cursor = g.header_bytes;
    for (uint64_t b = 0; b < g.n_batches; ++b) {
        const uint64_t first = b * g.cpb;
        if (tid == 0) {
            s_code = 0;
            if (len - cursor < 4) {
                s_code = DEV_E_BATCH_HDR_TRUNC;                        // container.cpp:114-115
            } else {
                s_cnt = ld_u32_le(arc + cursor);
                if (len - cursor < 4 + 4 * (uint64_t)s_cnt) s_code = DEV_E_TABLE_TRUNC;  // :118-119
            }
        }
        __syncthreads();
        uint32_t code = s_code;
        const uint32_t cnt = code ? 0 : s_cnt;
        const uint64_t table = cursor + 4;
        // thread-contiguous ranges of the size table, block exclusive scan of their sums
        const uint32_t per = (cnt + nthreads - 1) / nthreads;
        const uint32_t i0 = min(cnt, (uint32_t)tid * per), i1 = min(cnt, i0 + per);
        uint64_t mine = 0;
        for (uint32_t i = i0; i < i1; ++i) mine += ld_u32_le(arc + table + 4 * (uint64_t)i);
        uint64_t incl = mine;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint64_t t = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += t;
        }
        if (lane == 31) s_wsum[warp] = incl;
        __syncthreads();
        uint64_t before = 0, payload = 0;
        for (int w = 0; w < nwarps; ++w) {
            if (w < warp) before += s_wsum[w];
            payload += s_wsum[w];
        }
        if (tid == 0) {
            if (!code && len - table - 4 * (uint64_t)cnt < payload) code = DEV_E_PAYLOAD_BATCH_TRUNC;  // :127-128
            if (!code && cnt != g.chunks_in(b)) code = DEV_E_CHUNK_COUNT;  // pipeline.hpp:411-416
            s_code = code;
            s_payload = payload;
        }
        __syncthreads();
        code = s_code;
        if (code) {
            if (tid == 0) {
                record_error(ws.error, first, code);
                atomicMin(ws.abort_at, (unsigned long long)b);
            }
            return;
        }
        uint64_t off = table + 4 * (uint64_t)cnt + before + (incl - mine);
        for (uint32_t i = i0; i < i1; ++i) {
            const uint32_t sz = ld_u32_le(arc + table + 4 * (uint64_t)i);
            ws.chunk_off[first + i] = off;
            ws.chunk_size[first + i] = sz;
            off += sz;
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) st_release32(&ws.ready[b], 1u);
        cursor = table + 4 * (uint64_t)cnt + s_payload;
        __syncthreads();
    }
    if (tid == 0 && cursor != len) record_error(ws.error, g.n_chunks, DEV_E_TRAILING);  // pipeline.hpp:460-461
}

}  // namespace

template <typename T, int MAXT>
__global__ void __launch_bounds__(MAXT, MAXT <= 256 ? 1024 / MAXT : 1) decode_chunks_kernel(const uint8_t* __restrict__ arc,
                                                             uint64_t len, geometry g,
                                                             T* __restrict__ out, decode_ws ws) {
    using tr = lane_traits<T>;
    using B = typename tr::B;
    using S = typename tr::S;
    constexpr int W = tr::width;
    constexpr int HDR = tr::header;

    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t n = g.chunk_n;
    const int NC = (int)((n - 1) / 8);
    const int BM = NC / 8;  // sparse bitmap bytes (bitplane.hpp:113-122)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = blockDim.x >> 5;

    const uint32_t pn = pidx(n) + 1;
    uint32_t region = (uint32_t)(pn * sizeof(T) + 15) & ~15u;
    const uint32_t stage_need = (uint32_t)(HDR + (W + 7) / 8 + W * NC + 16 + 15) & ~15u;
    region = stage_need > region ? stage_need : region;
    uint8_t* s_stage = smem;                       // chunk bytes, then output values
    T* s_out = reinterpret_cast<T*>(smem);
    uint8_t* s_rows = smem + region;               // [W][NC]

    __shared__ uint32_t s_ticket, s_abort, s_code, s_w, s_hA;
    __shared__ uint64_t s_off;
    __shared__ uint32_t s_size;
    __shared__ uint64_t s_dense;
    __shared__ B s_z1;
    __shared__ uint32_t s_rowoff[64];
    __shared__ B s_wtot[32];

    if (tid == 0) s_ticket = atomicAdd(ws.ticket, 1u);
    __syncthreads();
    if (s_ticket == 0) {
        walk_frames(arc, len, g, ws);
        return;
    }
    const uint64_t c = s_ticket - 1;
    const uint64_t b = g.batch_of(c);
    const uint32_t ci = (uint32_t)(c - b * g.cpb);
    const uint64_t bcount = g.values_in(b);
    const uint64_t v0 = b * g.batch_values + (uint64_t)ci * n;
    const uint64_t left = bcount - (uint64_t)ci * n;
    const uint32_t count = left < n ? (uint32_t)left : n;

    // ---- wait for the walker to publish this batch ----
    if (tid == 0) {
        s_abort = 0;
        while (ld_acquire32(&ws.ready[b]) == 0) {
            if (*(volatile unsigned long long*)ws.abort_at <= b) {
                s_abort = 1;
                break;
            }
            __nanosleep(128);
        }
        if (!s_abort) {
            s_off = ws.chunk_off[c];
            s_size = ws.chunk_size[c];
        }
    }
    __syncthreads();
    if (s_abort) return;
    const uint64_t off = s_off;
    const uint32_t size = s_size;

    // ---- stage the chunk bytes at the source's 16-B phase ----
    const uint32_t a = (uint32_t)(off & 15);
    const uint8_t* src = arc + (off - a);
    const uint32_t end = a + size;
    const bool src_aligned = ((uintptr_t)arc & 15) == 0;
    if (end <= region) {
        const uint32_t nvec = (end + 15) >> 4;
        for (uint32_t v = tid; v < nvec; v += blockDim.x) {
            const uint32_t lo = v << 4;
            if (src_aligned && (off - a) + lo + 16 <= len) {
                *reinterpret_cast<uint4*>(s_stage + lo) = __ldg(reinterpret_cast<const uint4*>(src + lo));
            } else {
                const uint32_t from = lo > a ? lo : a, to = lo + 16 < end ? lo + 16 : end;
                for (uint32_t i = from; i < to; ++i) s_stage[i] = src[i];
            }
        }
    }
    __syncthreads();

    // ---- parse + validate in the reference's order (chunk_codec.hpp:92-117,
    //      bitplane.hpp:160-186); warp 0 walks the rows, popcounts in parallel ----
    if (warp == 0) {
        const uint8_t* p = s_stage + a;
        uint32_t code = 0, w = 0, hA = 0;
        uint64_t flags = 0;
        B z1 = 0;
        if (end > region || size < (uint32_t)HDR) {
            code = DEV_E_HDR_TRUNC;
            if (end > region) {
                // longer than any valid chunk: the row walk must end in a size mismatch or
                // truncation; decide it from the header alone is not possible, so report
                // the first check that such a chunk fails below after reading the header
                code = 0;
            }
        }
        // an oversized chunk cannot be staged; read its header straight from global
        const uint8_t* hp = end > region ? arc + off : p;
        if (!code) {
            hA = hp[0];
            const uint32_t hB = hp[1];
            const bool case2 = hA > (uint32_t)tr::max_alpha || hB > (uint32_t)tr::max_beta;
            if (case2 && !(hA == (uint32_t)tr::exc_alpha && hB == (uint32_t)tr::exc_beta)) code = DEV_E_META;
            if (!code) {
#pragma unroll
                for (int i = 0; i < (int)sizeof(B); ++i) z1 |= (B)hp[2 + i] << (8 * i);
                w = hp[2 + sizeof(B)];
                if (w > (uint32_t)W) code = DEV_E_W;
            }
            uint32_t pos = HDR;
            if (!code && w > 0) {
                const uint32_t fb = (w + 7) / 8;
                if (size - pos < fb) {
                    code = DEV_E_FLAGS_TRUNC;
                } else {
                    for (uint32_t i = 0; i < fb; ++i) flags = flags << 8 | hp[pos + i];
                    if (fb * 8 > w && (flags >> w) != 0) code = DEV_E_FLAG_PAD;
                    pos += fb;
                }
            }
            if (!code && end > region) {
                code = DEV_E_SIZE;  // no valid chunk of this geometry is that long
            }
            if (!code) {
                for (int r = 0; r < (int)w; ++r) {
                    const int pb = (int)w - 1 - r;
                    if ((flags >> pb) & 1) {
                        if (size - pos < (uint32_t)NC) { code = DEV_E_ROW_TRUNC; break; }
                        if (lane == 0) s_rowoff[pb] = pos;
                        pos += NC;
                    } else {
                        if (size - pos < (uint32_t)BM) { code = DEV_E_BITMAP_TRUNC; break; }
                        if (lane == 0) s_rowoff[pb] = pos;
                        uint32_t cntp = 0;
                        for (int k = lane; k < BM; k += 32) cntp += __popc(p[pos + k]);
                        cntp = __reduce_add_sync(0xffffffffu, cntp);
                        pos += BM;
                        if (size - pos < cntp) { code = DEV_E_PAYLOAD_TRUNC; break; }
                        pos += cntp;
                    }
                }
                if (!code && pos != size) code = DEV_E_SIZE;
            }
        }
        if (lane == 0) {
            s_code = code;
            s_w = w;
            s_hA = hA;
            s_dense = flags;
            s_z1 = z1;
        }
    }
    __syncthreads();
    if (s_code) {
        if (tid == 0) record_error(ws.error, c, s_code);
        return;
    }
    const int w = (int)s_w;
    const uint64_t dense = s_dense;
    const uint32_t hA = s_hA;
    const bool case2 = hA > (uint32_t)tr::max_alpha;

    // ---- rows -> dense plane bytes, one warp per row ----
    const uint32_t lt_mask = (1u << lane) - 1u;
    for (int p = warp; p < w; p += nwarps) {
        const uint8_t* rs = s_stage + a + s_rowoff[p];
        uint8_t* rd = s_rows + p * NC;
        if ((dense >> p) & 1) {
            for (int col = lane; col < NC; col += 32) rd[col] = rs[col];
        } else {
            const uint8_t* payload = rs + BM;
            uint32_t running = 0;
            for (int base = 0; base < NC; base += 32) {
                const int col = base + lane;
                const uint32_t bit = col < NC ? (rs[col >> 3] >> (7 - (col & 7))) & 1u : 0u;
                const uint32_t m = __ballot_sync(0xffffffffu, bit);
                if (col < NC) rd[col] = bit ? payload[running + __popc(m & lt_mask)] : (uint8_t)0;
                running += __popc(m);
            }
        }
    }
    __syncthreads();

    // ---- untranspose: byte column t -> lanes 8t..8t+7 ----
    B z[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) z[j] = 0;
    if (tid < NC) {
        const int nblk = (w + 7) >> 3;
        for (int s = 0; s < nblk; ++s) {
            uint64_t x = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int p = 8 * s + k;
                if (p < w) x |= (uint64_t)s_rows[p * NC + tid] << (8 * k);
            }
            const uint64_t y = transpose8x8(x);
#pragma unroll
            for (int j = 0; j < 8; ++j) z[j] |= (B)((y >> (8 * (7 - j))) & 0xffu) << (8 * s);
        }
    }

    // ---- inverse transform: wrapping inclusive scan (transform.hpp:97-100) ----
    B d[8];
    B tsum = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        tsum += unzigzag<B>(z[j]);
        d[j] = tsum;  // thread-local inclusive prefix
    }
    B incl = tsum;
#pragma unroll
    for (int k = 1; k < 32; k <<= 1) {
        const B t = __shfl_up_sync(0xffffffffu, incl, k);
        if (lane >= k) incl += t;
    }
    if (lane == 31) s_wtot[warp] = incl;
    __syncthreads();
    B before = s_z1;
    for (int q = 0; q < warp; ++q) before += s_wtot[q];
    before += incl - tsum;  // exclusive prefix of this thread
    const T scale = pow10_of(T{}, case2 ? 0 : (int)hA);
    auto to_value = [&](B gv) -> T {
        if (case2) return value_of(unzigzag<B>(gv));
        return div_rn(from_i64(T{}, (long long)(S)gv), scale);   // numeric.hpp:159-162
    };
    if (tid < NC) {
#pragma unroll
        for (int j = 0; j < 8; ++j) s_out[pidx(8 * tid + 1 + j)] = to_value((B)(before + d[j]));
    }
    if (tid == 0) s_out[pidx(0)] = to_value(s_z1);
    __syncthreads();
    T* dst = out + v0;
    for (uint32_t i = tid; i < count; i += blockDim.x) dst[i] = s_out[pidx(i)];
}

template <typename T>
uint32_t decode_smem_bytes(uint32_t chunk_n) {
    using tr = lane_traits<T>;
    const uint32_t nc = (chunk_n - 1) / 8;
    const uint32_t pn = chunk_n + (chunk_n >> 3) + 1;
    uint32_t region = (uint32_t)(pn * sizeof(T) + 15) & ~15u;
    const uint32_t stage = (uint32_t)(tr::header + (tr::width + 7) / 8 + tr::width * nc + 16 + 15) & ~15u;
    if (stage > region) region = stage;
    return region + tr::width * nc;
}

template <typename T>
cudaError_t launch_decode(const uint8_t* d_archive, uint64_t len, const geometry& g, T* d_out,
                          const decode_ws& ws, cudaStream_t st, cudaEvent_t ev0, cudaEvent_t ev1) {
    cudaError_t e;
    if (g.n_chunks == 0) return cudaSuccess;
    if ((e = cudaMemsetAsync(ws.ticket, 0, sizeof(uint32_t), st))) return e;
    if ((e = cudaMemsetAsync(ws.ready, 0, g.n_batches * sizeof(uint32_t), st))) return e;
    if ((e = cudaMemsetAsync(ws.abort_at, 0xff, sizeof(unsigned long long), st))) return e;
    const uint32_t threads = encode_block_threads(g.chunk_n);
    const uint32_t smem = decode_smem_bytes<T>(g.chunk_n);
    auto kern = threads <= 256 ? decode_chunks_kernel<T, 256> : decode_chunks_kernel<T, 1024>;
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return e;
    if (ev0 && (e = cudaEventRecord(ev0, st))) return e;
    kern<<<(unsigned)(g.n_chunks + 1), threads, smem, st>>>(d_archive, len, g, d_out, ws);
    if ((e = cudaGetLastError())) return e;
    return ev1 ? cudaEventRecord(ev1, st) : cudaSuccess;
}

template cudaError_t launch_decode<double>(const uint8_t*, uint64_t, const geometry&, double*,
                                           const decode_ws&, cudaStream_t, cudaEvent_t, cudaEvent_t);
template cudaError_t launch_decode<float>(const uint8_t*, uint64_t, const geometry&, float*,
                                          const decode_ws&, cudaStream_t, cudaEvent_t, cudaEvent_t);
template uint32_t decode_smem_bytes<double>(uint32_t);
template uint32_t decode_smem_bytes<float>(uint32_t);

}  // namespace fb200
