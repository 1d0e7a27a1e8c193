// decode.cu -- Falcon decompress for sm_100a: frame walker + persistent, warp-specialised
// decoder, launched back to back with programmatic dependent launch.
//
// The archive has no batch index (FORMAT.md:10-14): batch b+1's frame starts where
// batch b's payload ends, so frames must be located sequentially.  walker_kernel (one
// block) is the *frame walker* (read_batch chain, container.cpp:113-132,
// pipeline.hpp:394-417): per batch its chain warps load the count + size table with 16-B
// vector loads and sum it, its writer warps validate the entries, scan them into per-chunk
// offsets and publish the batch (walk_frames_split).  In every decoder block:
//   producers (2 warps)  take chunk tickets, wait for the chunk's batch, stage the chunk
//                        bytes into a smem slot ring (cp.async at the 16-B phase), and
//                        parse + validate it in the reference's check order
//                        (chunk_codec.hpp:86-122, bitplane.hpp:152-186): row offsets,
//                        dense mask, per-warp sparse payload prefixes, scale constants
//   consumers (NT thr.)  thread t owns byte column t: gathers byte t of every row (dense
//                        rows verbatim; sparse rows: bitmap bit + ballot rank), 8x8 bit
//                        transposes + PRMT byte transposes rebuild lanes 8t..8t+7, a
//                        block-wide wrapping scan of unzigzagged deltas
//                        (transform.hpp:91-106), RN(g / 10^alpha) without a division
//                        (dpds.cuh) or the raw bits, and lane-contiguous value stores
//                        through the slot
#include "dpds.cuh"
#include "falcon_common.cuh"
#include "kernels.h"

#include <cstdlib>

namespace fb200 {

namespace {


__device__ __forceinline__ uint32_t ld_u32_le(const uint8_t* p) {
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

// Frame walker: validates frames in archive order and publishes per-chunk offsets.
// Per batch the size table is read with lane-contiguous loads into smem (segments of
// `cap` entries), scanned block-wide, and the chunk offsets/sizes are written back with
// lane-contiguous stores, so one batch costs about one DRAM round trip plus the fence.
__device__ void walk_frames(const uint8_t* __restrict__ arc, uint64_t len, const geometry& g,
                            const decode_ws& ws, uint4* s_raw, uint32_t* s_pref, uint32_t cap,
                            uint64_t b0, uint64_t cursor0) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nthreads = blockDim.x, nwarps = nthreads >> 5;
    __shared__ uint32_t s_cnt, s_code, s_stop;
    __shared__ uint64_t s_wsum[32];
    uint64_t cursor = cursor0;
    for (uint64_t b = b0; b < g.n_batches; ++b) {
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
        __syncthreads();
        const uint64_t table = cursor + 4;
        const uint64_t pay0 = table + 4 * (uint64_t)cnt;   // first chunk's payload
        // the offsets are written only for a frame with the expected chunk count; the
        // payload-truncation check (container.cpp:127-128) needs the full sum first
        const bool write = cnt == g.chunks_in(b);
        uint64_t carry = 0;
        for (uint32_t seg = 0; seg < cnt; seg += cap) {
            const uint32_t m = cnt - seg < cap ? cnt - seg : cap;
            // the segment's table bytes: 16-B vectors (all loads in flight at once), then
            // entries from smem.  s_raw holds the span from the vector below the table.
            const uint64_t tb = table + 4 * (uint64_t)seg;
            const uint64_t v0 = tb & ~15ull;
            const uint32_t ph = (uint32_t)(tb - v0);
            const uint32_t nvec = (ph + 4 * m + 15) >> 4;
            const bool vec_ok = (((uintptr_t)arc) & 15) == 0;
#pragma unroll 4
            for (uint32_t v = tid; v < nvec; v += nthreads) {
                const uint64_t at = v0 + 16ull * v;
                uint4 x;
                if (vec_ok && at + 16 <= len) {
                    x = __ldg(reinterpret_cast<const uint4*>(arc + at));
                } else {  // unaligned archive or its last bytes
                    uint32_t wv[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        wv[q] = 0;
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const uint64_t a = at + 4 * q + k;
                            if (a < len) wv[q] |= (uint32_t)arc[a] << (8 * k);
                        }
                    }
                    x = make_uint4(wv[0], wv[1], wv[2], wv[3]);
                }
                s_raw[v] = x;
            }
            __syncthreads();
            const uint8_t* rb = reinterpret_cast<const uint8_t*>(s_raw) + ph;
            auto entry = [&](uint32_t i) -> uint32_t { return ld_u32_le(rb + 4 * i); };
            // thread-contiguous ranges: local sums, block exclusive scan, local prefixes
            const uint32_t per = (m + nthreads - 1) / nthreads;
            const uint32_t i0 = min(m, (uint32_t)tid * per), i1 = min(m, i0 + per);
            // sums in u64 like read_batch (container.cpp:124-128): a crafted table must not
            // wrap past the payload-truncation check.  s_pref keeps the segment-relative
            // prefix in u32, exact up to the first entry above any valid chunk size; the
            // chunks after such an entry fail their producer's bounds check, after the
            // oversize chunk itself (lower index, so its error wins).
            uint64_t mine = 0;
            for (uint32_t i = i0; i < i1; ++i) mine += entry(i);
            uint64_t incl = mine;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint64_t t = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += t;
            }
            if (lane == 31) s_wsum[warp] = incl;
            __syncthreads();
            uint64_t run = incl - mine, segsum = 0;
            for (int w = 0; w < nwarps; ++w) {
                if (w < warp) run += s_wsum[w];
                segsum += s_wsum[w];
            }
            for (uint32_t i = i0; i < i1; ++i) {
                s_pref[i] = (uint32_t)run;
                run += entry(i);
            }
            __syncthreads();
            if (write) {
                for (uint32_t i = tid; i < m; i += nthreads) {
                    ws.chunk_off[first + seg + i] = pay0 + carry + s_pref[i];
                    ws.chunk_size[first + seg + i] = entry(i);
                }
            }
            carry += segsum;
            __syncthreads();
        }
        if (tid == 0) {
            if (!code && len - pay0 < carry) code = DEV_E_PAYLOAD_BATCH_TRUNC;  // container.cpp:127-128
            if (!code && !write) code = DEV_E_CHUNK_COUNT;                    // pipeline.hpp:411-416
            if (code) {
                record_error(ws.error, first, code);
                atomicMin(ws.abort_at, (unsigned long long)b);
            } else {
                // the block's offset stores are ordered before this point by the barrier
                // after the write loop; one gpu-scope release store publishes them (barrier,
                // then release: cumulative over what the barrier made this thread observe --
                // CUTLASS's semaphore release).  A __threadfence() here added MEMBAR.SC +
                // an L1 invalidate per batch.
                st_release32(&ws.ready[b], 1u);
            }
            s_stop = code;
        }
        __syncthreads();
        // (a separate word: s_code is rewritten at the top of the next batch while slower
        // threads may still read this verdict -- racecheck)
        if (s_stop) return;
        cursor = pay0 + carry;
    }
    if (tid == 0 && cursor != len) record_error(ws.error, g.n_chunks, DEV_E_TRAILING);  // pipeline.hpp:460-461
}


// Fast path of the frame walk for the common case (16-B aligned archive, every table fits
// the smem buffer): the next batch's count + size table are loaded into registers while
// the current batch's offsets are written, so a batch costs about one DRAM round trip
// less.  It stops, before writing anything for the batch, at the first frame that is not
// exactly as expected (wrong count, truncation); the general walker then resumes there
// and reports the reference's error.  Returns the first batch not published.
template <int PF>
__device__ uint64_t walk_frames_fast(const uint8_t* __restrict__ arc, uint64_t len, const geometry& g,
                                     const decode_ws& ws, uint4* s_raw, uint32_t* s_pref, uint32_t cap,
                                     uint32_t emax, uint64_t* cursor_out) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nthreads = blockDim.x, nwarps = nthreads >> 5;
    __shared__ uint32_t s_wsum[32];
    uint64_t cursor = g.header_bytes;
    *cursor_out = cursor;
    if ((((uintptr_t)arc) & 15) != 0 || (uint64_t)g.cpb + 8 > cap) return 0;
    auto nvec_of = [&](uint64_t cur, uint32_t cnt) -> uint32_t {
        return (uint32_t)(((cur & 15) + 4 + 4 * (uint64_t)cnt + 15) >> 4);
    };
    uint4 pf[PF];
    auto issue = [&](uint64_t cur, uint32_t cnt) {
        const uint64_t v0 = cur & ~15ull;
        const uint32_t nvec = nvec_of(cur, cnt);
#pragma unroll
        for (int k = 0; k < PF; ++k) {
            const uint32_t v = (uint32_t)tid + (uint32_t)k * nthreads;
            pf[k] = make_uint4(0u, 0u, 0u, 0u);
            if (v < nvec) {
                const uint64_t at = v0 + 16ull * v;
                if (at + 16 <= len) {
                    pf[k] = __ldg(reinterpret_cast<const uint4*>(arc + at));
                } else {
                    uint32_t wv[4] = {0u, 0u, 0u, 0u};
                    for (int q = 0; q < 16; ++q)
                        if (at + q < len) wv[q >> 2] |= (uint32_t)arc[at + q] << (8 * (q & 3));
                    pf[k] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
                }
            }
        }
    };
    if (g.n_batches == 0) return 0;
    if (nvec_of(cursor, g.chunks_in(0)) > (uint32_t)PF * nthreads) return 0;
    issue(cursor, g.chunks_in(0));
    uint64_t b = 0;
    for (; b < g.n_batches; ++b) {
        const uint32_t exp = g.chunks_in(b);
        const uint32_t nvec = nvec_of(cursor, exp);
#pragma unroll
        for (int k = 0; k < PF; ++k) {
            const uint32_t v = (uint32_t)tid + (uint32_t)k * nthreads;
            if (v < nvec) s_raw[v] = pf[k];
        }
        __syncthreads();
        const uint8_t* rb = reinterpret_cast<const uint8_t*>(s_raw) + (cursor & 15);
        // stop (uniformly) at anything unusual: the general walker takes over
        if (len - cursor < 4 + 4 * (uint64_t)exp || ld_u32_le(rb) != exp) break;
        const uint8_t* tb = rb + 4;
        auto entry = [&](uint32_t i) -> uint32_t { return ld_u32_le(tb + 4 * i); };
        const uint32_t per = (exp + nthreads - 1) / nthreads;
        const uint32_t i0 = min(exp, (uint32_t)tid * per), i1 = min(exp, i0 + per);
        // every entry <= emax (the largest valid chunk) keeps the u32 sums exact (a table
        // holds < 2^16 entries here); anything larger goes to the general walker
        uint32_t mine = 0;
        bool big = false;
        for (uint32_t i = i0; i < i1; ++i) {
            const uint32_t e = entry(i);
            big |= e > emax;
            mine += e;
        }
        if (__syncthreads_or(big)) break;
        uint32_t incl = mine;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += t;
        }
        if (lane == 31) s_wsum[warp] = incl;
        __syncthreads();
        uint32_t run = incl - mine, payload = 0;
        for (int w = 0; w < nwarps; ++w) {
            if (w < warp) run += s_wsum[w];
            payload += s_wsum[w];
        }
        for (uint32_t i = i0; i < i1; ++i) {
            s_pref[i] = run;
            run += entry(i);
        }
        const uint64_t pay0 = cursor + 4 + 4 * (uint64_t)exp;
        if (len - pay0 < payload) break;  // truncated payload: the general walker reports it
        const uint64_t next = pay0 + payload;
        const bool more = b + 1 < g.n_batches && nvec_of(next, g.chunks_in(b + 1)) <= (uint32_t)PF * nthreads;
        if (more) issue(next, g.chunks_in(b + 1));  // in flight while this batch is written
        __syncthreads();
        const uint64_t first = b * g.cpb;
        for (uint32_t i = tid; i < exp; i += nthreads) {
            ws.chunk_off[first + i] = pay0 + s_pref[i];
            ws.chunk_size[first + i] = entry(i);
        }
        __syncthreads();
        if (tid == 0) st_release32(&ws.ready[b], 1u);  // barrier, release (see walk_frames)
        cursor = next;
        *cursor_out = cursor;
        if (!more) {
            ++b;
            break;
        }
    }
    __syncthreads();
    return b;
}

// Two-role fast walk (the common case: 16-B aligned archive, every frame as expected).
// The serial chain of the walk is only "frame b's payload total -> frame b+1's position",
// so the block splits:
//   chain  (warps 0..7)   loads frame b's count + size table straight into registers
//                         (16-B vectors), sums the table as rotated 32-bit words (the sum
//                         of little-endian u32 entries at byte phase s is the sum of the
//                         covering aligned words rotated right by 8s, edge words masked),
//                         parks the vectors in one of two smem slots and moves on to frame
//                         b+1 at once;
//   writer (warps 8..15)  validates the entries, scans them into chunk offsets, stores
//                         offsets/sizes and publishes the batch (barrier, fence, flag) off the
//                         chain's critical path.
// Slots hand over through mbarriers (FULL: chain -> writers, EMPTY: writers -> chain).
// Either role stops at the first frame that is not exactly as expected (chain: count /
// truncation; writer: an entry above the largest valid chunk); the general walker then
// resumes at the first batch not published and reports the reference's error.
constexpr int kChainThreads = 256;
constexpr int kWalkPF = 5;  // vectors per chain thread: tables of up to 5108 entries
constexpr uint32_t kWalkSlotBytes = kWalkPF * kChainThreads * 16 + 16;
struct walk_slot_meta {
    uint64_t cursor;  // frame position
    uint64_t b;       // batch
    uint32_t stop;    // 1: not a frame as expected, the walk ends at (b, cursor)
};
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void wmbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void wmbar_arrive(uint64_t* bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void wmbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done) : "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(parity) : "memory");
    }
}

// u32 at byte offset o (0..15) of the 32-byte window lo:hi (little endian)
__device__ __forceinline__ uint32_t window_u32(const uint4& lo, const uint4& hi, uint32_t o) {
    const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    const uint32_t q = o >> 2, sh = (o & 3) * 8;
    uint32_t a = w[0], b = w[1];
#pragma unroll
    for (int i = 1; i < 4; ++i) {
        a = q == (uint32_t)i ? w[i] : a;
        b = q == (uint32_t)i ? w[i + 1] : b;
    }
    return __funnelshift_r(a, b, sh);
}

// Returns the first batch not published; *cursor_out = its frame position.  Needs 512
// threads and walk_split_smem() bytes of dynamic smem.
__host__ __device__ constexpr uint32_t walk_split_smem(uint32_t cpb) { return 2 * kWalkSlotBytes + 4 * cpb; }
__device__ uint64_t walk_frames_split(const uint8_t* __restrict__ arc, uint64_t len, const geometry& g,
                                      const decode_ws& ws, uint8_t* smem, uint32_t emax,
                                      uint64_t* cursor_out) {
    const int tid = threadIdx.x, lane = tid & 31;
    __shared__ walk_slot_meta s_meta[2];
    __shared__ __align__(8) uint64_t s_full[2], s_empty[2];
    __shared__ uint64_t s_csum[kChainThreads / 32];
    __shared__ uint32_t s_wsum[kChainThreads / 32], s_wbig[kChainThreads / 32];
    __shared__ uint64_t s_res_b, s_res_cursor;
    __shared__ uint32_t s_wstop;  // the writer stopped (its resume point stands)
    __shared__ uint32_t s_cok;
    uint4* slots = reinterpret_cast<uint4*>(smem);
    uint32_t* s_pref = reinterpret_cast<uint32_t*>(smem + 2 * kWalkSlotBytes);
    if (tid == 0) {
        s_wstop = 0;
        s_res_b = g.n_batches;
        s_res_cursor = 0;
        for (int i = 0; i < 2; ++i) {
            wmbar_init(&s_full[i], 1);
            wmbar_init(&s_empty[i], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid < kChainThreads) {
        // ============================ chain ============================
        const int warp = tid >> 5;
        uint64_t cursor = g.header_bytes;
        for (uint64_t b = 0;; ++b) {
            const int sl = (int)(b & 1);
            // the slot's previous batch (b - 2) is done; a writer stop ends the chain
            if (b >= 2) {
                wmbar_wait(&s_empty[sl], (uint32_t)(((b - 2) >> 1) & 1));
                if (atomicOr(&s_wstop, 0u)) break;
            }
            bool stop = b >= g.n_batches;
            uint64_t next = 0;
            if (!stop) {
                const uint32_t exp = g.chunks_in(b);
                const uint64_t v0 = cursor & ~15ull;
                const uint32_t nvec = (uint32_t)(((cursor & 15) + 4 + 4 * (uint64_t)exp + 15) >> 4);
                stop = len - cursor < 4 + 4 * (uint64_t)exp || len - v0 < 16ull * nvec;  // uniform
                if (!stop) {
                    const uint64_t tb = cursor + 4, te = tb + 4 * (uint64_t)exp;
                    const uint32_t rs = (uint32_t)(tb & 3) * 8;
                    uint4 pf[kWalkPF];
#pragma unroll
                    for (int k = 0; k < kWalkPF; ++k) {
                        const uint32_t v = (uint32_t)tid + (uint32_t)k * kChainThreads;
                        pf[k] = v < nvec ? __ldg(reinterpret_cast<const uint4*>(arc + v0 + 16ull * v)) : make_uint4(0, 0, 0, 0);
                    }
                    uint64_t sum = 0;
#pragma unroll
                    for (int k = 0; k < kWalkPF; ++k) {
                        const uint64_t a = v0 + 16ull * ((uint32_t)tid + (uint32_t)k * kChainThreads);
                        const uint32_t w4[4] = {pf[k].x, pf[k].y, pf[k].z, pf[k].w};
                        if (a >= tb && a + 16 <= te) {
#pragma unroll
                            for (int q = 0; q < 4; ++q) sum += __funnelshift_r(w4[q], w4[q], rs);
                        } else if (a + 16 > tb && a < te) {  // edge vectors: mask bytes outside the table
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                const uint64_t wa = a + 4 * q;
                                const uint32_t lo = wa >= tb ? 0u : (uint32_t)min(tb - wa, (uint64_t)4);
                                const uint32_t hi = wa >= te ? 0u : (uint32_t)min(te - wa, (uint64_t)4);
                                const uint32_t m = hi > lo ? (uint32_t)(((1ull << (8 * hi)) - 1) & ~((1ull << (8 * lo)) - 1)) : 0u;
                                sum += __funnelshift_r(w4[q] & m, w4[q] & m, rs);
                            }
                        }
                    }
                    sum = warp_sum_u64(sum);
                    // the count word (bytes [cursor, cursor + 4)) lies in vectors 0 and 1
                    const uint4 v1 = make_uint4(__shfl_sync(0xffffffffu, pf[0].x, 1), __shfl_sync(0xffffffffu, pf[0].y, 1),
                                                __shfl_sync(0xffffffffu, pf[0].z, 1), __shfl_sync(0xffffffffu, pf[0].w, 1));
                    if (lane == 0) s_csum[warp] = sum;
                    uint4* dst = slots + (size_t)sl * (kWalkSlotBytes / 16);
#pragma unroll
                    for (int k = 0; k < kWalkPF; ++k) {
                        const uint32_t v = (uint32_t)tid + (uint32_t)k * kChainThreads;
                        if (v < nvec) dst[v] = pf[k];
                    }
                    named_sync(1, kChainThreads);
                    uint64_t payload = 0;
#pragma unroll
                    for (int q = 0; q < kChainThreads / 32; ++q) payload += s_csum[q];
                    // count (container.cpp:116) and payload truncation (:127-128)
                    if (tid == 0) s_cok = window_u32(pf[0], v1, (uint32_t)(cursor & 15)) == exp && !(len - te < payload);
                    named_sync(1, kChainThreads);
                    stop = s_cok == 0;
                    next = te + payload;
                }
            }
            if (tid == 0) {
                s_meta[sl].cursor = cursor;
                s_meta[sl].b = b;
                s_meta[sl].stop = stop ? 1u : 0u;
                wmbar_arrive(&s_full[sl]);
            }
            if (stop) break;
            cursor = next;
        }
    } else {
        // ============================ writer ============================
        const int wt = tid - kChainThreads, wwarp = wt >> 5;
        for (uint64_t b = 0;; ++b) {
            const int sl = (int)(b & 1);
            wmbar_wait(&s_full[sl], (uint32_t)((b >> 1) & 1));
            const walk_slot_meta m = s_meta[sl];
            if (m.stop) {
                // (a writer that stopped by itself left the loop before any stop marker; no
                // read of s_res here: the other writers would race with this write)
                if (wt == 0) {
                    s_res_b = m.b;
                    s_res_cursor = m.cursor;
                }
                break;
            }
            const uint32_t exp = g.chunks_in(b);
            const uint32_t* W = reinterpret_cast<const uint32_t*>(slots + (size_t)sl * (kWalkSlotBytes / 16));
            const uint32_t tbr = (uint32_t)(m.cursor & 15) + 4;  // table start in the slot
            const uint32_t w0 = tbr >> 2, sh = (tbr & 3) * 8;
            auto entry = [&](uint32_t i) -> uint32_t { return __funnelshift_r(W[w0 + i], W[w0 + i + 1], sh); };
            // Warp w scans entries [wb, we) (a multiple of 32 per warp) in rounds of 32
            // consecutive entries, lane l taking entry l of the round: every smem access of the
            // table and of s_pref is lane-contiguous.  (Thread-contiguous ranges of 16 entries
            // put the lanes 64 B apart: 16-way bank conflicts on every read and write, which made
            // the writer, not the chain, the walk's bound at ~6 us per batch.)
            const uint32_t seg = ((exp + kChainThreads - 1) / kChainThreads) * 32;
            const uint32_t wb = min(exp, (uint32_t)wwarp * seg), we = min(exp, wb + seg);
            uint32_t wsum = 0, big = 0;
            for (uint32_t i = wb + lane; i < we; i += 32) {
                const uint32_t e = entry(i);
                big |= e > emax;
                wsum += e;
            }
            wsum = __reduce_add_sync(0xffffffffu, wsum);
            big = __reduce_or_sync(0xffffffffu, big);
            if (lane == 0) {
                s_wsum[wwarp] = wsum;
                s_wbig[wwarp] = big;
            }
            named_sync(2, kChainThreads);
            uint32_t run = 0, anybig = 0;
#pragma unroll
            for (int q = 0; q < kChainThreads / 32; ++q) {
                run += q < wwarp ? s_wsum[q] : 0u;
                anybig |= s_wbig[q];
            }
            if (anybig) {  // every entry <= emax keeps the u32 prefixes exact
                if (wt == 0) {
                    atomicOr(&s_wstop, 1u);
                    s_res_b = b;
                    s_res_cursor = m.cursor;
                    wmbar_arrive(&s_empty[sl]);  // releases a chain waiting on this slot
                }
                break;
            }
            for (uint32_t r0 = wb; r0 < we; r0 += 32) {
                const uint32_t i = r0 + lane;
                const uint32_t e = i < we ? entry(i) : 0u;
                uint32_t incl = e;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, d);
                    if (lane >= d) incl += t;
                }
                if (i < we) s_pref[i] = run + incl - e;
                run += __shfl_sync(0xffffffffu, incl, 31);
            }
            named_sync(2, kChainThreads);
            const uint64_t pay0 = m.cursor + 4 + 4 * (uint64_t)exp;
            const uint64_t first = b * g.cpb;
            for (uint32_t i = wt; i < exp; i += kChainThreads) {
                ws.chunk_off[first + i] = pay0 + s_pref[i];
                ws.chunk_size[first + i] = entry(i);
            }
            named_sync(2, kChainThreads);
            if (wt == 0) {  // barrier, release (see walk_frames); then the slot is free
                st_release32(&ws.ready[b], 1u);
                wmbar_arrive(&s_empty[sl]);
            }
        }
    }
    __syncthreads();
    *cursor_out = s_res_cursor;
    return s_res_b;
}

}  // namespace

// RN(g / p) for the Case-1 inverse scale (numeric.hpp:159-162) at alpha = 22 (beyond
// the division-free range of dpds.cuh): one Markstein correction step from the rounded
// reciprocal, accepted only when the exact residual test of dpds.cuh (2) proves it is
// the correctly rounded quotient; otherwise IEEE division.  f32 (alpha 10) divides.
__device__ __noinline__ double ddiv_fallback(double a, double b) { return __ddiv_rn(a, b); }

__device__ __forceinline__ double inverse_scale_rn(double gd, double p, double rp) {
    const double q0 = __dmul_rn(gd, rp);
    const double r = __fma_rn(-q0, p, gd);
    const double q = __fma_rn(r, rp, q0);
    // q == RN(gd / p) iff |gd - q*p| < p * ulp(q) / 2 (halved below a power of two when
    // the quotient lies below q); the residual is exact (dpds.cuh (2)).  Ties and
    // anything not proven take the IEEE division.
    const double e = __fma_rn(-q, p, gd);
    const int qhi = __double2hiint(q);
    const uint32_t qe = ((uint32_t)qhi >> 20) & 0x7ffu;
    const bool pow2 = (qhi & 0x000fffff) == 0 && __double2loint(q) == 0;
    const bool toward0 = (__double2hiint(e) ^ qhi) < 0;
    const double H = __dmul_rn(p, __hiloint2double((int)((qe - 53u - ((pow2 && toward0) ? 1u : 0u)) << 20), 0));
    if (fabs(e) < H && qe > 53u) return q;
    return ddiv_fallback(gd, p);
}
__device__ __forceinline__ float inverse_scale_rn(float gf, float p, float) { return __fdiv_rn(gf, p); }

// ---- mbarrier / cp.async helpers (producer -> consumer ring) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar)) : "memory");
}
// blocking wait: try_wait with a suspend-time hint parks the warp in hardware until the
// phase completes (or the hint expires), so waiting warps take no issue slots
__device__ __forceinline__ bool mbar_try_suspend(uint64_t* bar, uint32_t parity) {
    uint32_t done;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u) : "memory");
    return done != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_suspend(bar, parity)) {
    }
}
#ifndef FB_DEC_CONS_SLEEP
#define FB_DEC_CONS_SLEEP 0
#endif
// consumer-side wait: a failed try_wait backs off for FB_DEC_CONS_SLEEP ns (A/B knob)
__device__ __forceinline__ void mbar_wait_cons(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_suspend(bar, parity)) {
        if (FB_DEC_CONS_SLEEP) __nanosleep(FB_DEC_CONS_SLEEP);
    }
}
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
// shared loads at explicit 32-bit shared-window addresses: with smem[] indexing the
// compiler rebuilt the window base ((CgaCtaId << 24) + offset) for every load (2 extra
// ops per load in the gather).  The addresses depend on slot data read after the slot's
// mbarrier wait, so the loads cannot be hoisted above it.
// a value the compiler must keep in a register instead of rematerializing it
__device__ __forceinline__ uint32_t opaque_u32(uint32_t x) {
    asm volatile("" : "+r"(x));
    return x;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
    uint32_t v;
    asm("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds_u8_if(bool p, uint32_t a) {
    uint32_t v = 0;
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.shared.u8 %0, [%1];\n\t}"
        : "+r"(v) : "r"(a), "r"((uint32_t)p));
    return v;
}
template <int NT>
__device__ __forceinline__ void consumer_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
}

// Producer warps and smem ring depth per value type (A/B-measured on cfg2 / cfg3: 2 x 4
// for both; 1 x 3, 2 x 6, 3 x 6, 3 x 9, 4 x 8 are slower or unstable).  The ring depth is a
// multiple of the producer count: each slot is refilled by one producer only.
template <typename T> struct decode_cfg { static constexpr int producers = 2, slots = 4; };
// f32 at the default chunk size: 6 resident blocks of 192 threads (56 registers; A/B: vs no
// bound -0.3 %, vs a 1-block bound (62 registers, 5 blocks) -3 %, vs 7 / 8 blocks, which
// spill, -2 % / -1 %).  f64 (0 = no bound) allocates 56 registers or fewer by itself; the
// slot ring allows 6 f64 blocks per SM anyway.
template <typename T, int NT>
constexpr int decode_min_blocks() { return sizeof(T) == 4 && NT <= 128 ? 6 : 0; }
static_assert(decode_cfg<double>::slots % decode_cfg<double>::producers == 0, "slot reuse");
static_assert(decode_cfg<float>::slots % decode_cfg<float>::producers == 0, "slot reuse");
enum : uint32_t { SLOT_CHUNK = 0, SLOT_SKIP = 1, SLOT_EXIT = 2, SLOT_BOUNDS = 3 };

// value staging for coalesced stores: [8][NT + 2] values (+ value 0), reusing the slot
__host__ __device__ __forceinline__ uint32_t decode_stage_stride(uint32_t nt) { return nt + 2; }

template <typename T>
__host__ __device__ __forceinline__ uint32_t decode_region_bytes(uint32_t chunk_n) {
    using tr = lane_traits<T>;
    const uint32_t nc = (chunk_n - 1) / 8;
    const uint32_t nt = nc <= 256 ? (nc < 32 ? 32 : (nc + 31) / 32 * 32) : (nc <= 512 ? 512 : 1024);
    const uint32_t raw = (uint32_t)(tr::header + (tr::width + 7) / 8 + tr::width * nc + 16 + 15) & ~15u;
    const uint32_t vals = (uint32_t)((8 * decode_stage_stride(nt) + 1) * sizeof(T) + 15) & ~15u;
    return raw > vals ? raw : vals;
}

// Everything the consumers need about one staged chunk, written by the producer warp.
template <typename T, typename B, int NW>
struct __align__(16) slot_info {
    uint32_t rowoff[64];      // plane p: row offset from the chunk's first byte
    uint16_t wpre[NW * 64];   // [warp][plane]: sparse payload bytes of the warps before
    uint64_t dmask;           // bit p: plane p is dense
    uint64_t off;             // archive offset of the chunk
    uint64_t v0;              // index of the chunk's first value
    T scale, rscale;          // 10^alpha and RN(1 / 10^alpha)
    B z1;
    B wtot[NW];               // consumer scan scratch
    uint32_t chunk, size, kind, code, w, hA, count;
};

// Parse + validate one staged chunk in the reference's order (chunk_codec.hpp:92-117,
// bitplane.hpp:160-186), one warp.  Row offsets follow from the dense/sparse flags
// and the sparse rows' bitmap popcounts (a chain over sparse rows only); for each
// sparse row the consumer warps' payload prefixes are stored too.
template <typename T, int NW, typename SI>
__device__ __forceinline__ void parse_chunk(uint32_t ps, const uint8_t* hp, uint32_t size, bool oversize,
                                            int NC, int BM, SI& si, int lane) {
    using tr = lane_traits<T>;
    using B = typename tr::B;
    constexpr int W = tr::width;
    constexpr int HDR = tr::header;
    uint32_t code = 0, w = 0, hA = 0;
    uint64_t flags = 0, dmask = 0;
    B z1 = 0;
    if (size < (uint32_t)HDR) {
        code = DEV_E_HDR_TRUNC;
    } else {
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
        if (!code && oversize) code = DEV_E_SIZE;  // no valid chunk of this geometry is that long
        if (!code && w > 0) {
            // Row walk (bitplane.hpp:160-186).  Row r (plane w-1-r) sits at
            //   pos0 + NC * #dense rows before r + sum over sparse rows before r of (BM + popcount)
            // Lane L owns rows L and L+32; only the sparse rows' popcounts are sequential.
            const uint32_t pos0 = pos;
            const int r0 = lane, r1 = lane + 32;
            const bool v0r = r0 < (int)w, v1r = r1 < (int)w;
            const bool d0 = v0r && ((flags >> (w - 1 - r0)) & 1);
            const bool d1 = v1r && ((flags >> (w - 1 - r1)) & 1);
            const uint32_t dm0 = __ballot_sync(0xffffffffu, d0), dm1 = __ballot_sync(0xffffffffu, d1);
            const uint32_t sm0 = __ballot_sync(0xffffffffu, v0r && !d0), sm1 = __ballot_sync(0xffffffffu, v1r && !d1);
            const uint32_t lt = (1u << lane) - 1u;
            const uint32_t nd0 = __popc(dm0 & lt), nd1 = __popc(dm0) + __popc(dm1 & lt);
            uint32_t acc0 = 0, acc1 = 0;  // sparse bytes before rows r0 / r1
            uint32_t acc = 0;             // sparse bytes so far
            int bad = 64;                 // first row failing a truncation check
            uint32_t bad_code = 0;
            uint64_t sparse = ((uint64_t)sm1 << 32) | sm0;
            while (sparse) {
                const int r = __ffsll((long long)sparse) - 1;
                sparse &= sparse - 1;
                const uint32_t nd = r < 32 ? __popc(dm0 & ((1u << r) - 1u))
                                           : __popc(dm0) + __popc(dm1 & ((1u << (r - 32)) - 1u));
                const uint32_t rp = pos0 + nd * (uint32_t)NC + acc;
                if (size < rp + (uint32_t)BM) { bad = r; bad_code = DEV_E_BITMAP_TRUNC; break; }
                // chain: one bitmap byte per lane, popcounts summed by REDUX (the next
                // sparse row's offset needs only the total)
                const uint32_t pa = __popc(lds_u8_if(lane < BM, ps + rp + lane));
                const uint32_t pb = __popc(lds_u8_if(lane + 32 < BM, ps + rp + lane + 32));
                const uint32_t tot = __reduce_add_sync(0xffffffffu, pa + pb);
                // off the chain: consumer warp q's payload prefix = popcounts of bitmap
                // bytes [0, 4q) (exclusive scan of 4-byte group sums over lanes q < NW)
                {
                    uint32_t gs = pa;   // group q = lanes 4q..4q+3 of the byte counts
                    gs += __shfl_down_sync(0xffffffffu, gs, 1);
                    gs += __shfl_down_sync(0xffffffffu, gs, 2);
                    if (NW > 8) {       // groups 8..15 live in the second half (bytes 32..63)
                        uint32_t gh = pb;
                        gh += __shfl_down_sync(0xffffffffu, gh, 1);
                        gh += __shfl_down_sync(0xffffffffu, gh, 2);
                        const uint32_t hsrc = __shfl_sync(0xffffffffu, gh, (4 * lane - 32) & 31);
                        gs = __shfl_sync(0xffffffffu, gs, (4 * lane) & 31);
                        gs = lane >= 8 ? hsrc : gs;
                    } else {
                        gs = __shfl_sync(0xffffffffu, gs, (4 * lane) & 31);
                    }
                    uint32_t incl = gs;
#pragma unroll
                    for (int d = 1; d < NW; d <<= 1) {
                        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, d);
                        if (lane >= d) incl += t;
                    }
                    if (lane < NW) si.wpre[lane * 64 + (w - 1 - r)] = (uint16_t)(incl - gs);
                }
                if (size - rp - (uint32_t)BM < tot) { bad = r; bad_code = DEV_E_PAYLOAD_TRUNC; break; }
                if (r0 > r) acc0 += (uint32_t)BM + tot;
                if (r1 > r) acc1 += (uint32_t)BM + tot;
                acc += (uint32_t)BM + tot;
            }
            const uint32_t pr0 = pos0 + nd0 * (uint32_t)NC + acc0;
            const uint32_t pr1 = pos0 + nd1 * (uint32_t)NC + acc1;
            // dense rows truncated before the first sparse failure (reference order)
            const uint32_t t0 = __ballot_sync(0xffffffffu, d0 && r0 < bad && size - pr0 < (uint32_t)NC);
            const uint32_t t1 = __ballot_sync(0xffffffffu, d1 && r1 < bad && size - pr1 < (uint32_t)NC);
            if (t0 | t1) code = DEV_E_ROW_TRUNC;
            else if (bad_code) code = bad_code;
            else if (pos0 + (uint32_t)(__popc(dm0) + __popc(dm1)) * (uint32_t)NC + acc != size) code = DEV_E_SIZE;
            if (v0r) si.rowoff[w - 1 - r0] = pr0;
            if (v1r) si.rowoff[w - 1 - r1] = pr1;
            dmask = flags;  // flag bit (w-1-r) marks row r = plane w-1-r: bit p <-> plane p
        } else if (!code && pos != size) {
            code = DEV_E_SIZE;
        }
    }
    if (lane == 0) {
        si.code = code;
        si.w = w;
        si.hA = hA;
        si.z1 = z1;
        si.dmask = dmask;
    }
}

// The frame walker as its own one-block kernel, launched just before the decoder with
// programmatic dependent launch: it lets the decoder start at once
// (griddepcontrol.launch_dependents), and the decoder's producers wait on the per-batch
// ready flags it publishes.  Its own register and smem budget keep the next batch's table
// in flight without costing the decoder occupancy.
constexpr int kWalkThreads = 512;
__global__ void __launch_bounds__(kWalkThreads) walker_kernel(const uint8_t* __restrict__ arc, uint64_t len_arg,
                                                              const uint64_t* __restrict__ d_len, geometry g,
                                                              decode_ws ws, uint32_t cap, uint32_t emax, bool split) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uint64_t len = d_len ? *d_len : len_arg;
    extern __shared__ __align__(16) uint8_t wsmem[];
    uint4* raw = reinterpret_cast<uint4*>(wsmem);                 // 4 cap + 32 bytes
    uint32_t* pref = reinterpret_cast<uint32_t*>(wsmem + 4 * (size_t)cap + 32);  // cap entries
    uint64_t cursor;
    uint64_t b0;
    if (split) b0 = walk_frames_split(arc, len, g, ws, wsmem, emax, &cursor);
    else b0 = walk_frames_fast<4>(arc, len, g, ws, raw, pref, cap, emax, &cursor);
    walk_frames(arc, len, g, ws, raw, pref, cap, b0, cursor);
}

// Persistent, warp-specialized decode (the frame walker runs beside it, walker_kernel).
// In every block the last kProducers warps are producers: each takes chunk tickets, waits for
// the walker to publish its chunk's batch, streams the chunk bytes (16-B
// cp.async at the source's 16-B phase) into a ring of kDecodeSlots smem slots, parses
// and validates the staged chunk, and hands the slot to the NT consumer threads, which
// only gather, scan and store.  Staging and parsing of later chunks overlap the decode
// of the current one; the next chunk's offsets are fetched while a copy is in flight.
template <typename T, int NT>
__global__ void __launch_bounds__(NT + 32 * decode_cfg<T>::producers, decode_min_blocks<T, NT>()) decode_chunks_kernel(const uint8_t* __restrict__ arc, uint64_t len_arg,
                                                                const uint64_t* __restrict__ d_len,
                                                                geometry g, T* __restrict__ out,
                                                                decode_ws ws) {
    const uint64_t len = d_len ? *d_len : len_arg;
    constexpr int kProducers = decode_cfg<T>::producers;
    constexpr int kDecodeSlots = decode_cfg<T>::slots;
    using tr = lane_traits<T>;
    using B = typename tr::B;
    using S = typename tr::S;
    constexpr int W = tr::width;
    constexpr int nwarps = NT / 32;
    using SI = slot_info<T, B, nwarps>;

    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t n = g.chunk_n;
    const int NC = (int)((n - 1) / 8);
    const int BM = NC / 8;  // sparse bitmap bytes (bitplane.hpp:113-122)
    const uint32_t region = decode_region_bytes<T>(n);

    __shared__ __align__(8) uint64_t s_full[kDecodeSlots], s_empty[kDecodeSlots];
    __shared__ SI s_info[kDecodeSlots];

    if (threadIdx.x == 0) {
        for (int i = 0; i < kDecodeSlots; ++i) {
            mbar_init(&s_full[i], 32);       // every lane of the slot's producer warp
            mbar_init(&s_empty[i], nwarps);  // one per consumer warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if ((int)threadIdx.x >= NT) {
        // ===================== producer warps =====================
        const int lane = threadIdx.x & 31;
        const uint32_t pw = (threadIdx.x - NT) >> 5;  // producer pw fills iterations pw, pw + kProducers, ...
        const bool aligned = ((uintptr_t)arc & 15) == 0;
        // dynamic chunk tickets (measured better balanced than static striding); lane 0
        // waits for the chunk's batch frame and loads its offset and size
        uint32_t known_ready = 0;   // lane 0: batches [0, known_ready) seen published
        auto fetch = [&](uint32_t it, uint32_t& t, uint32_t& kind, uint64_t& off, uint32_t& size) {
            uint32_t tk = 0;
            if (lane == 0) tk = atomicAdd(ws.ticket, 1u);
            const uint64_t c = __shfl_sync(0xffffffffu, tk, 0);
            (void)it;
            t = (uint32_t)c;
            kind = c < g.n_chunks ? SLOT_CHUNK : SLOT_EXIT;
            off = 0;
            size = 0;
            if (kind == SLOT_CHUNK && lane == 0) {
                const uint32_t b = (uint32_t)g.batch_of(t);
                // the walker publishes batches in order with release stores, so one acquire
                // that saw batch b' published covers every batch <= b': no flag round trip
                // on the ticket -> offsets chain for those
                if (b + 1 > known_ready) {
                    while (ld_acquire32(&ws.ready[b]) == 0) {
                        if (*(volatile unsigned long long*)ws.abort_at <= b) {
                            kind = SLOT_SKIP;
                            break;
                        }
                        __nanosleep(64);
                    }
                    if (kind == SLOT_CHUNK) known_ready = b + 1;
                }
                if (kind == SLOT_CHUNK) {
                    off = ws.chunk_off[t];
                    size = ws.chunk_size[t];
                }
            }
            kind = __shfl_sync(0xffffffffu, kind, 0);
            off = __shfl_sync(0xffffffffu, off, 0);
            size = __shfl_sync(0xffffffffu, size, 0);
        };
        uint32_t t, kind, size;
        uint64_t off;
        fetch(pw, t, kind, off, size);
        for (uint32_t it = pw;; it += kProducers) {
            const int sl = (int)(it % kDecodeSlots);
            // the producer runs ahead: it parks on the slot's mbarrier (suspend hint) instead
            // of polling, leaving the issue slots to the consumers it waits for (A/B: polling
            // -0.2 %, 100-1000 ns sleeps -0.1 %)
            if (it >= (uint32_t)kDecodeSlots) mbar_wait(&s_empty[sl], ((it / kDecodeSlots) & 1) ^ 1);
            SI& si = s_info[sl];
            uint8_t* buf = smem + (size_t)sl * region;
            const uint32_t a = (uint32_t)(off & 15);
            const uint64_t end = (uint64_t)a + size;
            // a published chunk lies inside the archive unless an earlier entry of its table
            // was oversize (see walk_frames); that chunk's own error has the lower index
            if (kind == SLOT_CHUNK && (off > len || len - off < size)) kind = SLOT_BOUNDS;
            const bool staged = kind == SLOT_CHUNK && end <= region;
            if (staged) {
                const uint64_t base = off - a;
                const uint32_t nvec = (uint32_t)((end + 15) >> 4);
                for (uint32_t vv = lane; vv < nvec; vv += 32) {
                    const uint64_t gaddr = base + 16ull * vv;
                    if (aligned && gaddr + 16 <= len) {
                        cp_async16(buf + 16 * vv, arc + gaddr);
                    } else {  // ragged archive end: plain byte copies
                        for (uint32_t k = 0; k < 16; ++k)
                            if (gaddr + k < len) buf[16 * vv + k] = arc[gaddr + k];
                    }
                }
            }
            // the next chunk's offsets load while the copy is in flight
            uint32_t t2 = 0, kind2 = SLOT_EXIT, size2 = 0;
            uint64_t off2 = 0;
            if (kind != SLOT_EXIT) fetch(it + kProducers, t2, kind2, off2, size2);
            asm volatile("cp.async.wait_all;" ::: "memory");
            __syncwarp();
            if (kind == SLOT_CHUNK) parse_chunk<T, nwarps>(opaque_u32(smem_u32(buf + a)), staged ? buf + a : arc + off, size, !staged, NC, BM, si, lane);
            if (lane == 0) {
                si.kind = kind;
                si.chunk = t;
                si.off = off;
                si.size = size;
                if (kind == SLOT_CHUNK) {
                    // chunk-uniform values the consumers would otherwise each recompute
                    const uint32_t b = (uint32_t)g.batch_of(t);
                    const uint32_t ci = t - b * g.cpb;
                    const uint64_t left = g.values_in(b) - (uint64_t)ci * n;
                    si.v0 = (uint64_t)b * g.batch_values + (uint64_t)ci * n;
                    si.count = left < n ? (uint32_t)left : n;
                    const int al = si.hA > (uint32_t)tr::max_alpha ? 0 : (int)si.hA;
                    si.scale = pow10_of(T{}, al);
                    si.rscale = rpow10_of(T{}, al);   // RN(1 / 10^alpha), host-computed table
                }
            }
            __syncwarp();
            mbar_arrive(&s_full[sl]);
            if (kind == SLOT_EXIT) break;
            t = t2;
            kind = kind2;
            off = off2;
            size = size2;
        }
        return;
    }

    // ===================== consumer warps =====================
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool active = tid < NC;
    const uint32_t lt_mask = (1u << lane) - 1u;
    // a producer that ran out of chunks publishes one EXIT slot and stops; the other may
    // still hold a chunk for a later iteration, so consumers skip only the exited
    // producer's iterations and leave once every producer has exited
    uint32_t exited = 0;
    for (uint32_t it = 0;; ++it) {
        const uint32_t pw = it % kProducers;
        if ((exited >> pw) & 1u) continue;
        const int sl = (int)(it % kDecodeSlots);
        mbar_wait_cons(&s_full[sl], (it / kDecodeSlots) & 1);
        SI& si = s_info[sl];
        const uint32_t kind = si.kind;
        if (kind == SLOT_EXIT) {
            exited |= 1u << pw;
            if (exited == (1u << kProducers) - 1u) break;
            continue;
        }
        if (kind == SLOT_BOUNDS) {
            if (tid == 0) record_error(ws.error, si.chunk, DEV_E_SIZE);
        }
        const uint32_t code = kind == SLOT_CHUNK ? si.code : 0u;
        if (kind == SLOT_CHUNK && code != 0u) {
            if (tid == 0) record_error(ws.error, si.chunk, code);
        } else if (kind == SLOT_CHUNK) {
            const uint64_t v0 = si.v0;
            const uint32_t count = si.count;
            // the chunk's bytes as 32-bit offsets into smem[] (a generic img pointer made the
            // compiler rebuild each load address from the shared window, 3 extra ops per load)
            const uint32_t ib = opaque_u32(smem_u32(smem)) + (uint32_t)sl * region + (uint32_t)(si.off & 15);
            const uint32_t icol = ib + (uint32_t)tid, ibm = ib + ((uint32_t)tid >> 3);
            const uint32_t icol_s = active ? icol : ib;   // dense loads: an in-slot address for all
            const int w = (int)si.w;
            const uint32_t hA = si.hA;
            const bool case2 = hA > (uint32_t)tr::max_alpha;
            const uint64_t dmask = si.dmask;
            const B z1 = si.z1;

    // ---- planes -> lanes: thread t gathers byte t of every row (dense: verbatim;
    //      sparse: bitmap bit t, payload byte at warp prefix + ballot rank), one 8x8
    //      transpose per 8 planes, then a byte transpose assembles the lanes ----
    uint64_t yb[W / 8];
#pragma unroll
    for (int sb = 0; sb < W / 8; ++sb) yb[sb] = 0;
    const int nblk = (w + 7) >> 3;
#pragma unroll
    for (int sb = 0; sb < W / 8; ++sb) {
        if (sb >= nblk) break;
        const uint4 o03 = *reinterpret_cast<const uint4*>(&si.rowoff[8 * sb]);
        const uint4 o47 = *reinterpret_cast<const uint4*>(&si.rowoff[8 * sb + 4]);
        const uint32_t ro[8] = {o03.x, o03.y, o03.z, o03.w, o47.x, o47.y, o47.z, o47.w};
        const int kmax = w - 8 * sb;
        const uint32_t valid = kmax >= 8 ? 0xffu : ((1u << kmax) - 1u);
        const uint32_t dblk = (uint32_t)(dmask >> (8 * sb)) & valid;
        uint32_t xb[8];
        if (dblk == 0xffu) {
#pragma unroll
            for (int k = 0; k < 8; ++k) xb[k] = lds_u8(icol_s + ro[k]);   // inactive columns zeroed below
        } else {
            const uint4 wp = *reinterpret_cast<const uint4*>(&si.wpre[warp * 64 + 8 * sb]);
            const uint32_t wpre[8] = {wp.x & 0xffffu, wp.x >> 16, wp.y & 0xffffu, wp.y >> 16,
                                      wp.z & 0xffffu, wp.z >> 16, wp.w & 0xffffu, wp.w >> 16};
            const uint32_t bsh = 7u - ((uint32_t)tid & 7u);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                xb[k] = 0u;
                if (k >= kmax) continue;  // uniform: rows above w
                const bool dk = (dblk >> k) & 1u;
                const uint32_t bmb = lds_u8_if(!dk && active, ibm + ro[k]);
                const uint32_t bit = (bmb >> bsh) & 1u;
                const uint32_t m = __ballot_sync(0xffffffffu, bit);
                const uint32_t idx = dk ? icol + ro[k] : ib + ro[k] + BM + wpre[k] + __popc(m & lt_mask);
                xb[k] = lds_u8_if((dk && active) || bit, idx);
            }
        }
        // byte k of x = row byte of plane 8sb+k (xb[k] <= 0xff: selector 7 reads a zero byte)
        const uint32_t xl = __byte_perm(xb[0], xb[1], 0x7740) | __byte_perm(xb[2], xb[3], 0x4077);
        const uint32_t xh = __byte_perm(xb[4], xb[5], 0x7740) | __byte_perm(xb[6], xb[7], 0x4077);
        yb[sb] = active ? transpose8x8(((uint64_t)xh << 32) | xl) : 0ull;  // byte 7-j = byte sb of lane j
    }
    // byte transpose: lane j's byte sb = byte 7-j of yb[sb]
    B z[8];
    {
        auto tr4 = [](uint32_t h0, uint32_t h1, uint32_t h2, uint32_t h3, uint32_t o[4]) {
            // o[q] = [h0.b(q), h1.b(q), h2.b(q), h3.b(q)]
            const uint32_t p01l = __byte_perm(h0, h1, 0x5140), p01h = __byte_perm(h0, h1, 0x7362);
            const uint32_t p23l = __byte_perm(h2, h3, 0x5140), p23h = __byte_perm(h2, h3, 0x7362);
            o[0] = __byte_perm(p01l, p23l, 0x5410);
            o[1] = __byte_perm(p01l, p23l, 0x7632);
            o[2] = __byte_perm(p01h, p23h, 0x5410);
            o[3] = __byte_perm(p01h, p23h, 0x7632);
        };
        uint32_t lo[8], hi[8];
        uint32_t q[4];
        // low lane words: blocks 0..3; lane j = 7 - byte index
        tr4((uint32_t)(yb[0] >> 32), (uint32_t)(yb[1] >> 32), (uint32_t)(yb[2] >> 32), (uint32_t)(yb[3] >> 32), q);
        lo[3] = q[0]; lo[2] = q[1]; lo[1] = q[2]; lo[0] = q[3];
        tr4((uint32_t)yb[0], (uint32_t)yb[1], (uint32_t)yb[2], (uint32_t)yb[3], q);
        lo[7] = q[0]; lo[6] = q[1]; lo[5] = q[2]; lo[4] = q[3];
        if constexpr (W == 64) {
#pragma unroll
            for (int j = 0; j < 8; ++j) hi[j] = 0;
            if (nblk > 4) {
                tr4((uint32_t)(yb[4] >> 32), (uint32_t)(yb[5] >> 32), (uint32_t)(yb[6] >> 32), (uint32_t)(yb[7] >> 32), q);
                hi[3] = q[0]; hi[2] = q[1]; hi[1] = q[2]; hi[0] = q[3];
                tr4((uint32_t)yb[4], (uint32_t)yb[5], (uint32_t)yb[6], (uint32_t)yb[7], q);
                hi[7] = q[0]; hi[6] = q[1]; hi[5] = q[2]; hi[4] = q[3];
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) z[j] = (B)(((uint64_t)hi[j] << 32) | lo[j]);
        } else {
            (void)hi;
#pragma unroll
            for (int j = 0; j < 8; ++j) z[j] = (B)lo[j];
        }
    }

    // ---- inverse transform: wrapping inclusive scan (transform.hpp:97-100) ----
    // With w <= 28 every delta is below 2^27 in magnitude, so the thread-local prefix of
    // eight deltas fits 32 bits: unzigzag and accumulate in 32-bit, widen once.
    B d[8];
    B tsum = 0;
    if (sizeof(B) == 8 && w <= 28) {
        int32_t t32 = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t zz = (uint32_t)z[j];
            t32 += (int32_t)((zz >> 1) ^ (0u - (zz & 1u)));
            d[j] = (B)(int64_t)t32;
        }
        tsum = d[7];
    } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            tsum += unzigzag<B>(z[j]);
            d[j] = tsum;  // thread-local inclusive prefix
        }
    }
    B incl = tsum;
    if (sizeof(B) == 8 && w <= 23) {
        // |delta| <= 2^22, so a warp's 256 deltas sum below 2^30: scan in 32-bit
        int32_t i32 = (int32_t)tsum;
#pragma unroll
        for (int k = 1; k < 32; k <<= 1) {
            const int32_t t = __shfl_up_sync(0xffffffffu, i32, k);
            if (lane >= k) i32 += t;
        }
        incl = (B)(int64_t)i32;
    } else {
#pragma unroll
        for (int k = 1; k < 32; k <<= 1) {
            const B t = __shfl_up_sync(0xffffffffu, incl, k);
            if (lane >= k) incl += t;
        }
    }
    if (lane == 31) si.wtot[warp] = incl;
    consumer_sync<NT>();
    B before = z1;
#pragma unroll
    for (int q = 0; q < nwarps; ++q) before += q < warp ? si.wtot[q] : (B)0;
    before += incl - tsum;  // exclusive prefix of this thread
    const T scale = si.scale, rscale = si.rscale;
    // Case 1 divides by 10^alpha (numeric.hpp:159-162) without a division (dpds.cuh);
    // padded lanes are dropped (transform.hpp:96).  Values go through the slot (free once
    // every consumer passed the scan barrier) as [j][t] (conflict-free), then out with
    // lane-contiguous stores: a warp writes 256 consecutive bytes per instruction instead
    // of 32 scattered 8-B pieces.
    T* dst = out + v0;
    T* vstage = reinterpret_cast<T*>(smem + (size_t)sl * region);
    constexpr uint32_t SP = NT + 2;  // decode_stage_stride(NT)
    auto store = [&](auto to_value) {
#pragma unroll
        for (int j = 0; j < 8; ++j) vstage[j * SP + tid] = to_value((B)(before + d[j]));
        if (tid == 0) vstage[8 * SP] = to_value(z1);
    };
    constexpr int kMark = sizeof(T) == 8 ? kMarksteinMaxAlpha64 : kMarksteinMaxAlpha32;
    if (case2) {
        store([&](B gv) -> T { return value_of(unzigzag<B>(gv)); });
    } else if ((int)hA <= kMark) {
        store([&](B gv) -> T { return div_pow10_markstein(from_i64(T{}, (long long)(S)gv), scale, rscale); });
    } else {
        store([&](B gv) -> T { return inverse_scale_rn(from_i64(T{}, (long long)(S)gv), scale, rscale); });
    }
    consumer_sync<NT>();
    {
        // value i = tid + NT m (m = 0..8) is lane k = i - 1: thread k / 8, register k % 8;
        // NT is a multiple of 8, so k % 8 is fixed per thread and k / 8 steps by NT / 8
        const int kb = tid - 1;
        const T* vsrc = vstage + (kb & 7) * (int)SP + (kb >> 3);
        if (sizeof(T) == 8 && count == 8u * NT + 1u) {  // full f64 chunk (uniform): no bounds checks
#pragma unroll
            for (uint32_t m = 0; m < 8; ++m)
                dst[tid + NT * m] = (m == 0 && tid == 0) ? vstage[8 * SP] : vsrc[(NT / 8) * m];
            if (tid == 0) dst[8 * NT] = vsrc[NT];
        } else {
#pragma unroll
            for (uint32_t m = 0; m < 9; ++m) {
                const uint32_t i = (uint32_t)tid + NT * m;
                if (m * NT < 8u * NT + 1u && i < count) dst[i] = i == 0 ? vstage[8 * SP] : vsrc[(NT / 8) * m];
            }
        }
    }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[sl]);
    }
}

// Batch-offset index: one block walks the frames (read_batch,
// container.cpp:113-132) and writes index[b] = archive offset of batch b's frame,
// index[B] = end of the last frame.  Each size table is summed with independent
// lane-contiguous loads, so a batch costs about one DRAM round trip.  A frame that does not fit the archive records
// the same error codes as the decoder's walker.
__global__ void __launch_bounds__(256) index_frames_kernel(const uint8_t* __restrict__ arc, uint64_t len,
                                                           uint64_t header_bytes, uint64_t n_batches,
                                                           uint64_t* __restrict__ index,
                                                           unsigned long long* error) {
    __shared__ uint32_t s_cnt, s_code;
    __shared__ unsigned long long s_part[8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint64_t cursor = header_bytes;
    for (uint64_t b = 0; b < n_batches; ++b) {
        if (tid == 0) {
            index[b] = cursor;
            s_code = 0;
            if (len - cursor < 4) {
                s_code = DEV_E_BATCH_HDR_TRUNC;
            } else {
                s_cnt = ld_u32_le(arc + cursor);
                if (len - cursor < 4 + 4 * (uint64_t)s_cnt) s_code = DEV_E_TABLE_TRUNC;
            }
        }
        __syncthreads();
        if (s_code) {
            if (tid == 0) record_error(error, b, s_code);
            return;
        }
        const uint32_t cnt = s_cnt;
        const uint64_t table = cursor + 4;
        // sum of the u32 entries: lane-contiguous, independent loads (unrolled)
        unsigned long long sum = 0;
#pragma unroll 4
        for (uint32_t i = tid; i < cnt; i += blockDim.x) sum += ld_u32_le(arc + table + 4 * (uint64_t)i);
        for (int d = 16; d > 0; d >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, d);
        if (lane == 0) s_part[warp] = sum;
        __syncthreads();
        unsigned long long payload = 0;
        for (int q = 0; q < (int)(blockDim.x >> 5); ++q) payload += s_part[q];
        const uint64_t next = table + 4 * (uint64_t)cnt;
        if (len - next < payload) {
            if (tid == 0) record_error(error, b, DEV_E_PAYLOAD_BATCH_TRUNC);
            return;
        }
        cursor = next + payload;
        __syncthreads();
    }
    if (tid == 0) index[n_batches] = cursor;
}

cudaError_t launch_index(const uint8_t* d_archive, uint64_t len, uint64_t header_bytes, uint64_t n_batches,
                         uint64_t* d_index, unsigned long long* d_error, cudaStream_t st) {
    index_frames_kernel<<<1, 256, 0, st>>>(d_archive, len, header_bytes, n_batches, d_index, d_error);
    return cudaGetLastError();
}

template <typename T>
uint32_t decode_smem_bytes(uint32_t chunk_n) {
    return decode_cfg<T>::slots * decode_region_bytes<T>(chunk_n);
}

template <typename T>
cudaError_t launch_decode(const uint8_t* d_archive, uint64_t len, const geometry& g, T* d_out,
                          const decode_ws& ws, cudaStream_t st, cudaEvent_t ev0, cudaEvent_t ev1,
                          const uint64_t* d_len) {
    cudaError_t e;
    if (g.n_chunks == 0) return cudaSuccess;
    if ((e = cudaMemsetAsync(ws.ticket, 0, sizeof(uint32_t), st))) return e;
    if ((e = cudaMemsetAsync(ws.ready, 0, g.n_batches * sizeof(uint32_t), st))) return e;
    if ((e = cudaMemsetAsync(ws.abort_at, 0xff, sizeof(unsigned long long), st))) return e;
    const uint32_t threads = encode_block_threads(g.chunk_n);
    const uint32_t smem = decode_smem_bytes<T>(g.chunk_n);
    void (*kern)(const uint8_t*, uint64_t, const uint64_t*, geometry, T*, decode_ws);
    switch (threads) {
    case 32: kern = decode_chunks_kernel<T, 32>; break;
    case 64: kern = decode_chunks_kernel<T, 64>; break;
    case 96: kern = decode_chunks_kernel<T, 96>; break;
    case 128: kern = decode_chunks_kernel<T, 128>; break;
    case 160: kern = decode_chunks_kernel<T, 160>; break;
    case 192: kern = decode_chunks_kernel<T, 192>; break;
    case 224: kern = decode_chunks_kernel<T, 224>; break;
    case 256: kern = decode_chunks_kernel<T, 256>; break;
    case 512: kern = decode_chunks_kernel<T, 512>; break;
    case 1024: kern = decode_chunks_kernel<T, 1024>; break;
    default: kern = nullptr;
    }
    if (!kern) return cudaErrorInvalidConfiguration;
    if ((e = ensure_dynamic_smem((const void*)kern, smem))) return e;
    // persistent grid, every block co-resident; the walker kernel goes first and lets the
    // decoder launch immediately (programmatic dependent launch).  Occupancy and SM count
    // are cached per (device, kernel, smem): no queries per call.
    int per_sm = 0, sms = 0;
    if ((e = resident_blocks((const void*)kern, (int)threads + 32 * decode_cfg<T>::producers, smem, &per_sm, &sms)))
        return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    uint64_t grid = (uint64_t)per_sm * sms;
    if (grid > g.n_chunks) grid = g.n_chunks;
    if (grid < 1) grid = 1;
    // walker smem: the whole size table of a batch when it fits (fast path), else segments
    uint32_t cap = g.cpb + 64 < (24u << 10) ? g.cpb + 64 : (24u << 10);
    cap = (cap + 3) & ~3u;
    static const bool split_ok = std::getenv("FALCON_WALK_SERIAL") == nullptr;  // A/B knob
    // the two-role walk when every table fits the chain's registers and the u32 prefixes
    // of valid entries cannot wrap
    const uint32_t emax0 = (uint32_t)(lane_traits<T>::header + (lane_traits<T>::width + 7) / 8 +
                                      lane_traits<T>::width * ((g.chunk_n - 1) / 8));
    const bool split = ((uintptr_t)d_archive & 15) == 0 && (uint64_t)g.cpb + 8 <= 4ull * kWalkPF * kChainThreads &&
                       (uint64_t)g.cpb * emax0 < (1ull << 32) && split_ok;
    size_t wsm = 8 * (size_t)cap + 48;
    if (split && walk_split_smem(g.cpb) > wsm) wsm = walk_split_smem(g.cpb);
    if ((e = ensure_dynamic_smem((const void*)walker_kernel, (uint32_t)wsm))) return e;
    if (ev0 && (e = cudaEventRecord(ev0, st))) return e;
    const uint32_t emax = (uint32_t)(lane_traits<T>::header + (lane_traits<T>::width + 7) / 8 +
                                      lane_traits<T>::width * ((g.chunk_n - 1) / 8));  // max_encoded_chunk_size
    walker_kernel<<<1, kWalkThreads, wsm, st>>>(d_archive, len, d_len, g, ws, cap, emax, split);
    if ((e = cudaGetLastError())) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(threads + 32 * decode_cfg<T>::producers);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if ((e = cudaLaunchKernelEx(&cfg, kern, d_archive, len, d_len, g, d_out, ws))) return e;
    return ev1 ? cudaEventRecord(ev1, st) : cudaSuccess;
}

template cudaError_t launch_decode<double>(const uint8_t*, uint64_t, const geometry&, double*,
                                           const decode_ws&, cudaStream_t, cudaEvent_t, cudaEvent_t,
                                           const uint64_t*);
template cudaError_t launch_decode<float>(const uint8_t*, uint64_t, const geometry&, float*,
                                          const decode_ws&, cudaStream_t, cudaEvent_t, cudaEvent_t,
                                          const uint64_t*);
template uint32_t decode_smem_bytes<double>(uint32_t);
template uint32_t decode_smem_bytes<float>(uint32_t);

}  // namespace fb200
