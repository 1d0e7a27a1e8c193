// pipeline.cu -- host-resident Falcon: multi-stream pinned H2D / kernels / D2H.
//
// Compress keeps the reference's event-driven scheduler (pipeline.hpp:149-365):
// n_streams slots rotate in launch order; each slot copies a batch host->device,
// runs the encode kernels for that batch as a frames-only archive, and reads back
// the frame size (the paper's M-D2H).  A cycling `current` pointer accepts sizes
// strictly in launch order, assigns the archive offset and starts the payload D2H
// (P-D2H) plus the store stage, so bytes never depend on completion timing.  When a
// full scan makes no progress the coordinator blocks on the oldest in-flight slot
// (livelock safeguard, counted in blocking_waits).  CUDA streams + events replace the
// reference's worker-pool "streams" and one_shot_events.
//
// Decompress walks batch frames on the calling thread (read_batch, pipeline.hpp:395-417),
// then per batch: H2D of the frame, one decode launch, D2H of the values and the sink
// put on a host worker; at most n_streams batches in flight (pipeline.hpp:381-452).
//
// Host buffers that are already pinned are copied directly (no staging memcpy).
#include <algorithm>
#include <functional>
#include <thread>

#include "runtime.h"

using namespace fb200;

namespace {

struct error_box {
    std::mutex m;
    falcon_status status = FALCON_OK;
    std::string msg;
    std::atomic<bool> failed{false};
    void record(falcon_status s, const std::string& text) {
        std::lock_guard<std::mutex> l(m);
        if (status == FALCON_OK) {
            status = s;
            msg = text;
        }
        failed.store(true, std::memory_order_release);
    }
    falcon_status raise() { return set_error(status, msg); }
};

struct hook_call {
    const falcon_pipeline_options* opt;
    int stage;
    unsigned slot;
    uint64_t seq;
};

void CUDART_CB run_hook(void* p) {
    auto* h = static_cast<hook_call*>(p);
    h->opt->stage_delay(h->opt->stage_delay_user, h->stage, h->slot, h->seq);
}

falcon_status get_slots(falcon_ctx* ctx, unsigned n, std::vector<pipeline_slot*>& out) {
    while (ctx->slots.size() < n) ctx->slots.push_back(std::make_unique<pipeline_slot>());
    out.clear();
    for (unsigned i = 0; i < n; ++i) {
        FB_TRY(ctx->slots[i]->init());
        ctx->slots[i]->state = 0;
        ctx->slots[i]->done.fire();
        out.push_back(ctx->slots[i].get());
    }
    return FALCON_OK;
}

// Pageable <-> pinned staging copy split over the pool (a single memcpy thread moves
// ~10 GB/s, well below the ~55 GB/s host link): pieces of >= 4 MiB.
void parallel_copy(worker_pool& pool, void* dst, const void* src, uint64_t bytes) {
    const uint64_t piece = 4ull << 20;
    const unsigned parts = (unsigned)std::min<uint64_t>((bytes + piece - 1) / piece, pool.size() + 1ull);
    if (parts <= 1) {
        std::memcpy(dst, src, bytes);
        return;
    }
    const uint64_t step = ((bytes + parts - 1) / parts + 63) & ~63ull;
    pool.fork_join(parts, [&](unsigned i) {
        const uint64_t a = std::min<uint64_t>(bytes, i * step), b = std::min<uint64_t>(bytes, a + step);
        if (b > a) std::memcpy(static_cast<uint8_t*>(dst) + a, static_cast<const uint8_t*>(src) + a, b - a);
    });
}

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

// ---------------------------------------------------------------------------------
struct compress_io {
    falcon_read_fn read = nullptr;
    void* ruser = nullptr;
    const uint8_t* src = nullptr;  // buffer mode
    uint64_t src_count = 0;
    bool src_pinned = false;
    falcon_store_fn store = nullptr;
    void* suser = nullptr;
    uint8_t* dst = nullptr;        // buffer mode
    uint64_t dst_cap = 0;
    bool dst_pinned = false;
    bool frames_only = false;      // one shard of a multi-GPU call: frames at 0, no header
};

falcon_status run_compress(falcon_ctx* ctx, int prec, compress_io& io,
                           const falcon_pipeline_options& opt, falcon_pipeline_stats* stats_out) {
    FB_TRY(validate_options(opt.chunk_n, opt.batch_values));
    if (opt.n_streams == 0) return set_error(FALCON_ERR_INVALID, "stream count must be positive");
    const size_t esz = lane_bytes(prec);
    const uint32_t chunk_n = opt.chunk_n;
    const uint64_t bv = opt.batch_values;
    const unsigned N = opt.n_streams;
    worker_pool& pool = ctx->get_pool(opt.workers);
    std::vector<pipeline_slot*> slots;
    FB_TRY(get_slots(ctx, N, slots));
    std::vector<hook_call> hooks(N);
    error_box err;
    falcon_pipeline_stats stats{};

    // ---- source staging (pipeline.hpp:254-263) ----
    uint64_t src_pos = 0, stage_count = 0;
    const uint8_t* stage_ptr = nullptr;  // where the staged batch lives
    bool have_batch = false;
    const bool direct_in = io.src && io.src_pinned;
    auto refill = [&]() -> falcon_status {
        FB_NVTX("compress: source read / staging");
        if (io.src) {
            stage_count = std::min<uint64_t>(bv, io.src_count - src_pos);
            if (direct_in) {
                stage_ptr = io.src + src_pos * esz;
            } else if (stage_count) {
                // pageable caller buffer: staged into pinned memory by the pool's threads
                FB_TRY(ctx->stage.ensure(stage_count * esz));
                parallel_copy(pool, ctx->stage.p, io.src + src_pos * esz, stage_count * esz);
                stage_ptr = ctx->stage.as<uint8_t>();
            }
            src_pos += stage_count;
        } else {
            FB_TRY(ctx->stage.ensure(std::max<uint64_t>(bv, 1) * esz));
            uint64_t total = 0;
            while (total < bv) {  // read_full (pipeline.hpp:124-134)
                const int64_t k = io.read(io.ruser, ctx->stage.as<uint8_t>() + total * esz, bv - total);
                if (k < 0) return set_error(FALCON_ERR_CALLBACK, "value_source::read failed");
                if (k == 0) break;
                total += (uint64_t)k;
            }
            stage_count = total;
            stage_ptr = ctx->stage.as<uint8_t>();
        }
        have_batch = stage_count > 0;
        return FALCON_OK;
    };
    FB_TRY(refill());  // nothing in flight yet: a read error propagates directly

    unsigned active = 0, current = 0, next_slot = 0;
    uint64_t launch_counter = 0, write_cursor = io.frames_only ? 0 : 47, total_values = 0, batch_count = 0;

    auto launch = [&](pipeline_slot& s, unsigned i) -> falcon_status {
        FB_NVTX("compress: H2D + encode + size read-back (enqueue)");
        s.count = stage_count;
        s.seq = launch_counter++;
        geometry g;
        FB_TRY(make_geometry(s.count, chunk_n, bv, 0, g));
        const uint64_t fbound = frame_bound(prec, s.count, chunk_n);
        FB_TRY(s.d_in.ensure(s.count * esz));
        FB_TRY(s.d_out.ensure(fbound));
        FB_TRY(s.d_status.ensure(prec == FALCON_F64 ? encode_scratch_bytes<double>(g) : encode_scratch_bytes<float>(g)));
        const uint8_t* h_src = stage_ptr;
        if (!direct_in) {
            // swap the staged buffer into the slot (pipeline.hpp:281 s.input.swap(stage))
            std::swap(s.h_in.p, ctx->stage.p);
            std::swap(s.h_in.cap, ctx->stage.cap);
            h_src = s.h_in.as<uint8_t>();
        }
        cudaStream_t st = s.stream;
        FB_CUDA(cudaMemcpyAsync(s.d_in.p, h_src, s.count * esz, cudaMemcpyHostToDevice, st));
        uint8_t* misc = s.d_misc.as<uint8_t>();
        FB_CUDA(cudaMemsetAsync(misc + 8, 0xff, 8, st));
        auto* err = reinterpret_cast<unsigned long long*>(misc + 8);
        auto* tot = reinterpret_cast<uint64_t*>(misc + 16);
        const encode_ws ws = prec == FALCON_F64
                                 ? carve_encode_ws<double>(s.d_status.p, g, reinterpret_cast<uint32_t*>(misc), err, tot)
                                 : carve_encode_ws<float>(s.d_status.p, g, reinterpret_cast<uint32_t*>(misc), err, tot);
        const archive_header_bytes none{};
        cudaError_t e = prec == FALCON_F64
                            ? launch_encode<double>(s.d_in.as<double>(), g, s.d_out.as<uint8_t>(), fbound, ws, none, st)
                            : launch_encode<float>(s.d_in.as<float>(), g, s.d_out.as<uint8_t>(), fbound, ws, none, st);
        if (e) return set_error(FALCON_ERR_CUDA, std::string("encode launch: ") + cudaGetErrorString(e));
        FB_CUDA(cudaMemcpyAsync(&s.box->total, misc + 16, 8, cudaMemcpyDeviceToHost, st));
        FB_CUDA(cudaMemcpyAsync(&s.box->error, misc + 8, 8, cudaMemcpyDeviceToHost, st));
        if (opt.stage_delay) {
            hooks[i] = hook_call{&opt, FALCON_STAGE_COMPRESS, i, s.seq};
            FB_CUDA(cudaLaunchHostFunc(st, run_hook, &hooks[i]));
        }
        FB_CUDA(cudaEventRecord(s.ev_size, st));
        return FALCON_OK;
    };

    auto accept_size = [&](pipeline_slot& s) -> falcon_status {
        if (s.box->error != ~0ull) {
            const uint32_t code = (uint32_t)(s.box->error & 0xff);
            err.record(device_error_status(code), device_error_text(code));
        }
        s.frame = s.box->total;
        if (io.dst && write_cursor + s.frame > io.dst_cap)
            err.record(FALCON_ERR_CAPACITY, "output capacity too small for the compressed archive");
        s.offset = write_cursor;
        write_cursor += s.frame;
        total_values += s.count;
        ++batch_count;
        if (!err.failed.load()) {
            void* to = (io.dst && io.dst_pinned) ? io.dst + s.offset : s.h_out.p;
            if (!(io.dst && io.dst_pinned)) FB_TRY(s.h_out.ensure(s.frame));
            if (!(io.dst && io.dst_pinned)) to = s.h_out.p;
            FB_CUDA(cudaMemcpyAsync(to, s.d_out.p, s.frame, cudaMemcpyDeviceToHost, s.stream));
        }
        FB_CUDA(cudaEventRecord(s.ev_data, s.stream));
        return FALCON_OK;
    };

    auto start_store = [&](pipeline_slot& s, unsigned i) {
        s.done.reset();
        s.store_started = true;
        pool.submit([&, i] {
            FB_NVTX("compress: store batch");
            pipeline_slot& sl = *slots[i];
            if (!err.failed.load(std::memory_order_relaxed)) {
                if (io.store) {  // run_store (pipeline.hpp:237-252)
                    if (io.store(io.suser, sl.offset, sl.h_out.p, sl.frame) != 0)
                        err.record(FALCON_ERR_CALLBACK, "archive store callback failed");
                } else if (io.dst && !io.dst_pinned) {
                    std::memcpy(io.dst + sl.offset, sl.h_out.p, sl.frame);
                }
            }
            if (opt.stage_delay) opt.stage_delay(opt.stage_delay_user, FALCON_STAGE_STORE, i, sl.seq);
            sl.done.fire();
        });
    };

    falcon_status fatal = FALCON_OK;
    while (have_batch || active > 0) {
        if (err.failed.load(std::memory_order_acquire)) have_batch = false;
        bool progress = false;
        for (unsigned i = 0; i < N; ++i) {
            pipeline_slot& s = *slots[i];
            if (s.state == 0) {
                if (have_batch && i == next_slot) {
                    falcon_status ls = launch(s, i);
                    if (ls != FALCON_OK) {
                        err.record(ls, falcon_last_error());
                        have_batch = false;
                        // nothing was enqueued that needs draining beyond the stream itself
                        cudaStreamSynchronize(s.stream);
                        continue;
                    }
                    s.state = 1;
                    ++active;
                    next_slot = (next_slot + 1) % N;
                    progress = true;
                    falcon_status rs = refill();
                    if (rs != FALCON_OK) {
                        err.record(rs, falcon_last_error());
                        have_batch = false;
                    }
                }
            } else if (s.state == 1) {
                if (i == current) {
                    const cudaError_t q = cudaEventQuery(s.ev_size);
                    if (q == cudaSuccess) {
                        falcon_status as = accept_size(s);
                        if (as != FALCON_OK) {
                            err.record(as, falcon_last_error());
                            cudaStreamSynchronize(s.stream);
                        }
                        s.state = 2;
                        s.store_started = false;
                        current = (current + 1) % N;
                        progress = true;
                    } else if (q != cudaErrorNotReady) {
                        fatal = set_error(FALCON_ERR_CUDA, std::string("compress stream: ") + cudaGetErrorString(q));
                        err.record(fatal, falcon_last_error());
                        s.state = 2;
                        s.store_started = false;
                        current = (current + 1) % N;
                        progress = true;
                    }
                }
            } else {
                if (!s.store_started) {
                    const cudaError_t q = cudaEventQuery(s.ev_data);
                    if (q != cudaErrorNotReady) {
                        if (q != cudaSuccess)
                            err.record(FALCON_ERR_CUDA, std::string("compress stream: ") + cudaGetErrorString(q));
                        start_store(s, i);
                        progress = true;
                    }
                } else if (s.done.test()) {
                    --active;
                    s.state = 0;
                    progress = true;
                }
            }
        }
        if (!progress && active > 0) {
            // livelock safeguard (pipeline.hpp:329-342): block on the oldest slot
            pipeline_slot* oldest = nullptr;
            for (auto* s : slots)
                if (s->state != 0 && (!oldest || s->seq < oldest->seq)) oldest = s;
            ++stats.blocking_waits;
            if (oldest->state == 1) cudaEventSynchronize(oldest->ev_size);
            else if (!oldest->store_started) cudaEventSynchronize(oldest->ev_data);
            else oldest->done.wait();
        }
    }
    if (err.failed.load()) return err.raise();

    // header last (pipeline.hpp:351-358)
    const archive_header_bytes hdr = header_bytes_of(prec, chunk_n, bv, total_values, batch_count);
    if (io.frames_only) {
        // a shard: the multi-GPU caller writes the one header
    } else if (io.store) {
        if (io.store(io.suser, 0, hdr.b, 47) != 0)
            return set_error(FALCON_ERR_CALLBACK, "archive store callback failed");
    } else {
        if (io.dst_cap < 47) return set_error(FALCON_ERR_CAPACITY, "output capacity too small for the header");
        std::memcpy(io.dst, hdr.b, 47);
    }
    stats.batches = batch_count;
    stats.values = total_values;
    if (stats_out) *stats_out = stats;
    ctx->last_archive_bytes = write_cursor;
    return FALCON_OK;
}

// ---------------------------------------------------------------------------------
struct decompress_io {
    falcon_put_fn put = nullptr;
    void* puser = nullptr;
    uint8_t* dst = nullptr;  // buffer mode
    uint64_t dst_cap = 0;
    bool dst_pinned = false;
};

uint32_t rd32(const uint8_t* p) {
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

// Batches [b_begin, b_end) whose frames start at `cursor0`; values land at their absolute
// index (the whole archive: 0, batch_count, 47).  The trailing-bytes check belongs to the
// range that ends the archive.
falcon_status run_decompress_range(falcon_ctx* ctx, int prec, const uint8_t* arc, uint64_t len,
                                   const falcon_archive_info& h, uint64_t b_begin, uint64_t b_end,
                                   uint64_t cursor0, decompress_io& io, const falcon_pipeline_options& opt,
                                   falcon_pipeline_stats* stats_out);

falcon_status run_decompress(falcon_ctx* ctx, int prec, const uint8_t* arc, uint64_t len,
                             decompress_io& io, const falcon_pipeline_options& opt,
                             falcon_pipeline_stats* stats_out) {
    falcon_archive_info h;
    FB_TRY(falcon_read_header(arc, len, &h));
    return run_decompress_range(ctx, prec, arc, len, h, 0, h.batch_count, 47, io, opt, stats_out);
}

falcon_status run_decompress_range(falcon_ctx* ctx, int prec, const uint8_t* arc, uint64_t len,
                                   const falcon_archive_info& h, uint64_t b_begin, uint64_t b_end,
                                   uint64_t cursor0, decompress_io& io, const falcon_pipeline_options& opt,
                                   falcon_pipeline_stats* stats_out) {
    if (h.precision != prec)
        return set_error(FALCON_ERR_INVALID, "archive precision does not match the requested value type");
    if (opt.n_streams == 0) return set_error(FALCON_ERR_INVALID, "stream count must be positive");
    if (h.chunk_n > 4097)
        return set_error(FALCON_ERR_UNSUPPORTED, "chunk_n > 4097 is not supported by the sm_100a kernels of this build");
    if (io.dst && h.total_values > io.dst_cap)
        return set_error(FALCON_ERR_CAPACITY, "value capacity too small for the archive");
    const size_t esz = lane_bytes(prec);
    const uint64_t n = h.chunk_n;
    const unsigned N = opt.n_streams;
    worker_pool& pool = ctx->get_pool(opt.workers);
    std::vector<pipeline_slot*> slots;
    FB_TRY(get_slots(ctx, N, slots));
    error_box err;
    const bool direct_in = is_pinned(arc);
    const bool direct_out = io.dst && io.dst_pinned;

    auto drain = [&] {
        for (auto* s : slots) s->done.wait();
    };

    uint64_t cursor = cursor0;
    for (uint64_t b = b_begin; b < b_end; ++b) {
        if (err.failed.load(std::memory_order_acquire)) break;
        // read_batch (container.cpp:113-132)
        const char* werr = nullptr;
        uint64_t rem = len - cursor, cnt = 0, table_end = 0, payload = 0;
        if (rem < 4) {
            werr = "batch header truncated";
        } else {
            cnt = rd32(arc + cursor);
            table_end = 4 + 4 * cnt;
            if (rem < table_end) {
                werr = "batch size table truncated";
            } else {
                for (uint64_t i = 0; i < cnt; ++i) payload += rd32(arc + cursor + 4 + 4 * i);
                if (rem - table_end < payload) werr = "batch payload truncated";
            }
        }
        const uint64_t first = b * h.batch_values;
        const uint64_t count = std::min<uint64_t>(h.batch_values, h.total_values - first);
        const uint64_t chunks = (count + n - 1) / n;
        if (!werr && cnt != chunks) werr = "chunk count mismatch";
        if (werr) {
            drain();
            return set_error(FALCON_ERR_CORRUPT, std::string(werr) + " (batch " + std::to_string(b) + ")");
        }
        const uint64_t wire = table_end + payload;
        const unsigned i = (unsigned)(b % N);
        pipeline_slot& s = *slots[i];
        s.done.wait();  // counting_semaphore(n_streams) (pipeline.hpp:382, 418)
        s.done.reset();
        s.batch = b;
        s.first = first;
        s.count = count;
        geometry g;
        falcon_status gs = make_geometry(count, (uint32_t)n, h.batch_values, 0, g);
        auto fail_slot = [&](falcon_status st) {
            err.record(st, falcon_last_error());
            s.done.fire();
        };
        if (gs != FALCON_OK) { fail_slot(gs); break; }
        if (s.d_in.ensure(wire + 16) || s.d_out.ensure(count * esz) || s.d_off.ensure(chunks * 8) ||
            s.d_size.ensure(chunks * 4) || s.d_ready.ensure(8)) {
            fail_slot(FALCON_ERR_CUDA);
            break;
        }
        cudaStream_t st = s.stream;
        const uint8_t* h_src = arc + cursor;
        if (!direct_in) {
            if (s.h_in.ensure(wire)) { fail_slot(FALCON_ERR_CUDA); break; }
            parallel_copy(pool, s.h_in.p, arc + cursor, wire);
            h_src = s.h_in.as<uint8_t>();
        }
        uint8_t* misc = s.d_misc.as<uint8_t>();
        decode_ws ws{reinterpret_cast<uint32_t*>(misc), s.d_ready.as<uint32_t>(),
                     reinterpret_cast<unsigned long long*>(misc + 8), s.d_off.as<uint64_t>(),
                     s.d_size.as<uint32_t>(), reinterpret_cast<unsigned long long*>(misc + 16)};
        cudaError_t e = cudaMemcpyAsync(s.d_in.p, h_src, wire, cudaMemcpyHostToDevice, st);
        if (!e) e = cudaMemsetAsync(misc + 16, 0xff, 8, st);
        if (!e)
            e = prec == FALCON_F64
                    ? launch_decode<double>(s.d_in.as<uint8_t>(), wire, g, s.d_out.as<double>(), ws, st)
                    : launch_decode<float>(s.d_in.as<uint8_t>(), wire, g, s.d_out.as<float>(), ws, st);
        if (!e) e = cudaMemcpyAsync(&s.box->error, misc + 16, 8, cudaMemcpyDeviceToHost, st);
        void* vals_host = nullptr;
        if (!e) {
            if (direct_out) {
                vals_host = io.dst + first * esz;
            } else {
                if (s.h_out.ensure(count * esz)) { fail_slot(FALCON_ERR_CUDA); break; }
                vals_host = s.h_out.p;
            }
            e = cudaMemcpyAsync(vals_host, s.d_out.p, count * esz, cudaMemcpyDeviceToHost, st);
        }
        if (!e) e = cudaEventRecord(s.ev_data, st);
        if (e) {
            set_error(FALCON_ERR_CUDA, std::string("decompress enqueue: ") + cudaGetErrorString(e));
            cudaStreamSynchronize(st);
            fail_slot(FALCON_ERR_CUDA);
            break;
        }
        const uint64_t cpb = g.cpb;
        pool.submit([&, i, b, first, count, vals_host, cpb] {
            FB_NVTX("decompress: wait + put batch");
            pipeline_slot& sl = *slots[i];
            const cudaError_t q = cudaEventSynchronize(sl.ev_data);
            if (q != cudaSuccess) {
                err.record(FALCON_ERR_CUDA, std::string("decompress stream: ") + cudaGetErrorString(q));
            } else if (sl.box->error != ~0ull) {
                const uint32_t code = (uint32_t)(sl.box->error & 0xff);
                std::string m = device_error_text(code);
                if (code != DEV_E_TRAILING) m += " (batch " + std::to_string(b) + ")";
                (void)cpb;
                err.record(device_error_status(code), m);
            } else if (!err.failed.load(std::memory_order_relaxed)) {
                if (opt.stage_delay)
                    opt.stage_delay(opt.stage_delay_user, FALCON_STAGE_DECODE, (unsigned)(b % N), b);
                if (io.put) {
                    if (io.put(io.puser, first, vals_host, count) != 0)
                        err.record(FALCON_ERR_CALLBACK, "value_sink::put failed");
                } else if (io.dst && !direct_out) {
                    std::memcpy(io.dst + first * esz, vals_host, count * esz);
                }
            }
            sl.done.fire();
        });
        cursor += wire;
    }
    drain();
    if (err.failed.load()) return err.raise();
    if (b_end == h.batch_count && cursor != len)
        return set_error(FALCON_ERR_CORRUPT, "trailing bytes after final batch");
    if (stats_out) {
        stats_out->batches = b_end - b_begin;
        stats_out->values = std::min<uint64_t>(h.total_values, b_end * h.batch_values) -
                            std::min<uint64_t>(h.total_values, b_begin * h.batch_values);
        stats_out->blocking_waits = 0;
    }
    return FALCON_OK;
}

// read_batch over the whole archive on the host (container.cpp:113-132): frame offsets
// off[0..B], off[B] = end of the last frame; the reference's messages and batch suffix.
falcon_status walk_frames_host(const uint8_t* arc, uint64_t len, const falcon_archive_info& h,
                               std::vector<uint64_t>& off) {
    off.assign(h.batch_count + 1, 0);
    uint64_t cursor = 47;
    const uint64_t n = h.chunk_n;
    for (uint64_t b = 0; b < h.batch_count; ++b) {
        off[b] = cursor;
        const char* werr = nullptr;
        const uint64_t rem = len - cursor;
        uint64_t cnt = 0, table = 0, payload = 0;
        if (rem < 4) {
            werr = "batch header truncated";
        } else {
            cnt = rd32(arc + cursor);
            table = 4 + 4 * cnt;
            if (rem < table) {
                werr = "batch size table truncated";
            } else {
                for (uint64_t i = 0; i < cnt; ++i) payload += rd32(arc + cursor + 4 + 4 * i);
                if (rem - table < payload) werr = "batch payload truncated";
            }
        }
        const uint64_t count = std::min<uint64_t>(h.batch_values, h.total_values - b * h.batch_values);
        if (!werr && cnt != (count + n - 1) / n) werr = "chunk count mismatch";
        if (werr) return set_error(FALCON_ERR_CORRUPT, std::string(werr) + " (batch " + std::to_string(b) + ")");
        cursor += table + payload;
    }
    off[h.batch_count] = cursor;
    if (cursor != len) return set_error(FALCON_ERR_CORRUPT, "trailing bytes after final batch");
    return FALCON_OK;
}

// Runs fn(g) for every context on its own host thread; the error of the lowest-numbered
// failing context is returned (its message re-raised on the calling thread).
falcon_status run_on_contexts(unsigned n, const std::function<falcon_status(unsigned)>& fn) {
    std::vector<falcon_status> st(n, FALCON_OK);
    std::vector<std::string> msg(n);
    std::vector<std::thread> th;
    th.reserve(n);
    for (unsigned g = 0; g < n; ++g)
        th.emplace_back([&, g] {
            st[g] = fn(g);
            if (st[g] != FALCON_OK) msg[g] = falcon_last_error();
        });
    for (auto& t : th) t.join();
    for (unsigned g = 0; g < n; ++g)
        if (st[g] != FALCON_OK) return set_error(st[g], msg[g]);
    return FALCON_OK;
}

falcon_pipeline_options resolve(const falcon_pipeline_options* opt) {
    falcon_pipeline_options o;
    falcon_default_options(&o);
    return opt ? *opt : o;
}

}  // namespace

extern "C" {

falcon_status falcon_compress_stream(falcon_ctx* ctx, int precision, falcon_read_fn read,
                                     void* read_user, falcon_store_fn store, void* store_user,
                                     const falcon_pipeline_options* opt,
                                     falcon_pipeline_stats* stats) {
    FB_NVTX("falcon_compress_stream");
    if (!ctx || !read || !store) return set_error(FALCON_ERR_INVALID, "null argument");
    std::lock_guard<std::mutex> lock(ctx->api_mutex);
    device_guard dg(ctx->device);
    compress_io io;
    io.read = read;
    io.ruser = read_user;
    io.store = store;
    io.suser = store_user;
    const falcon_pipeline_options o = resolve(opt);
    return run_compress(ctx, precision, io, o, stats);
}

falcon_status falcon_compress_host(falcon_ctx* ctx, int precision, const void* values,
                                   uint64_t n_values, const falcon_pipeline_options* opt,
                                   uint8_t* out, uint64_t out_cap, uint64_t* out_bytes,
                                   falcon_pipeline_stats* stats) {
    FB_NVTX("falcon_compress_host");
    if (!ctx || (!values && n_values) || !out) return set_error(FALCON_ERR_INVALID, "null argument");
    std::lock_guard<std::mutex> lock(ctx->api_mutex);
    device_guard dg(ctx->device);
    compress_io io;
    io.src = static_cast<const uint8_t*>(values);
    io.src_count = n_values;
    io.src_pinned = is_pinned(values);
    io.dst = out;
    io.dst_cap = out_cap;
    io.dst_pinned = is_pinned(out);
    const falcon_pipeline_options o = resolve(opt);
    FB_TRY(run_compress(ctx, precision, io, o, stats));
    if (out_bytes) *out_bytes = ctx->last_archive_bytes;
    return FALCON_OK;
}

falcon_status falcon_compress_host_multi(falcon_ctx* const* ctxs, unsigned n_ctx, int precision,
                                         const void* values, uint64_t n_values,
                                         const falcon_pipeline_options* opt, uint8_t* out, uint64_t out_cap,
                                         uint64_t* out_bytes, falcon_pipeline_stats* stats) {
    FB_NVTX("falcon_compress_host_multi");
    if (!ctxs || n_ctx == 0 || (!values && n_values) || !out) return set_error(FALCON_ERR_INVALID, "null argument");
    for (unsigned g = 0; g < n_ctx; ++g)
        if (!ctxs[g]) return set_error(FALCON_ERR_INVALID, "null context");
    const falcon_pipeline_options o = resolve(opt);
    FB_TRY(validate_options(o.chunk_n, o.batch_values));
    const size_t esz = lane_bytes(precision);
    const uint64_t bv = o.batch_values;
    const uint64_t B = (n_values + bv - 1) / bv;
    // batch-range shards: context g owns batches [gB/G, (g+1)B/G)
    std::vector<uint64_t> b0(n_ctx + 1);
    for (unsigned g = 0; g <= n_ctx; ++g) b0[g] = B * g / n_ctx;
    std::vector<std::vector<uint8_t>> frames(n_ctx);
    std::vector<falcon_pipeline_stats> st(n_ctx);
    std::vector<uint64_t> bytes(n_ctx, 0);
    FB_TRY(run_on_contexts(n_ctx, [&](unsigned g) -> falcon_status {
        const uint64_t v0 = std::min(n_values, b0[g] * bv), v1 = std::min(n_values, b0[g + 1] * bv);
        if (v1 == v0) return FALCON_OK;
        falcon_ctx* ctx = ctxs[g];
        std::lock_guard<std::mutex> lock(ctx->api_mutex);
        device_guard dg(ctx->device);
        frames[g].resize(falcon_compress_bound(precision, v1 - v0, o.chunk_n, bv));
        compress_io io;
        io.src = static_cast<const uint8_t*>(values) + v0 * esz;
        io.src_count = v1 - v0;
        io.src_pinned = is_pinned(values);
        io.dst = frames[g].data();
        io.dst_cap = frames[g].size();
        io.frames_only = true;
        FB_TRY(run_compress(ctx, precision, io, o, &st[g]));
        bytes[g] = ctx->last_archive_bytes;
        return FALCON_OK;
    }));
    uint64_t total = 47;
    for (unsigned g = 0; g < n_ctx; ++g) total += bytes[g];
    if (total > out_cap) return set_error(FALCON_ERR_CAPACITY, "output capacity too small for the compressed archive");
    const archive_header_bytes hdr = header_bytes_of(precision, o.chunk_n, bv, n_values, B);
    std::memcpy(out, hdr.b, 47);
    uint64_t at = 47;
    for (unsigned g = 0; g < n_ctx; ++g) {
        if (bytes[g]) std::memcpy(out + at, frames[g].data(), bytes[g]);
        at += bytes[g];
    }
    if (out_bytes) *out_bytes = total;
    if (stats) {
        *stats = falcon_pipeline_stats{};
        for (auto& x : st) {
            stats->batches += x.batches;
            stats->values += x.values;
            stats->blocking_waits += x.blocking_waits;
        }
    }
    return FALCON_OK;
}

falcon_status falcon_decompress_host_multi(falcon_ctx* const* ctxs, unsigned n_ctx, int precision,
                                           const uint8_t* archive, uint64_t archive_bytes, void* values,
                                           uint64_t cap_values, uint64_t* n_values,
                                           const falcon_pipeline_options* opt, falcon_pipeline_stats* stats) {
    FB_NVTX("falcon_decompress_host_multi");
    if (!ctxs || n_ctx == 0 || (!archive && archive_bytes)) return set_error(FALCON_ERR_INVALID, "null argument");
    for (unsigned g = 0; g < n_ctx; ++g)
        if (!ctxs[g]) return set_error(FALCON_ERR_INVALID, "null context");
    falcon_archive_info h;
    FB_TRY(falcon_read_header(archive, archive_bytes, &h));
    if (h.precision != precision)
        return set_error(FALCON_ERR_INVALID, "archive precision does not match the requested value type");
    if (h.total_values > cap_values) return set_error(FALCON_ERR_CAPACITY, "value capacity too small for the archive");
    const falcon_pipeline_options o = resolve(opt);
    // the one sequential step: locate every frame (size tables only), then shard by batch
    std::vector<uint64_t> off;
    FB_TRY(walk_frames_host(archive, archive_bytes, h, off));
    const uint64_t B = h.batch_count;
    std::vector<falcon_pipeline_stats> st(n_ctx);
    FB_TRY(run_on_contexts(n_ctx, [&](unsigned g) -> falcon_status {
        const uint64_t lo = B * g / n_ctx, hi = B * (g + 1) / n_ctx;
        if (lo == hi) return FALCON_OK;
        falcon_ctx* ctx = ctxs[g];
        std::lock_guard<std::mutex> lock(ctx->api_mutex);
        device_guard dg(ctx->device);
        decompress_io io;
        io.dst = static_cast<uint8_t*>(values);
        io.dst_cap = cap_values;
        io.dst_pinned = is_pinned(values);
        return run_decompress_range(ctx, precision, archive, archive_bytes, h, lo, hi, off[lo], io, o, &st[g]);
    }));
    if (n_values) *n_values = h.total_values;
    if (stats) {
        *stats = falcon_pipeline_stats{};
        stats->batches = h.batch_count;
        stats->values = h.total_values;
    }
    return FALCON_OK;
}

falcon_status falcon_decompress_stream(falcon_ctx* ctx, int precision, const uint8_t* archive,
                                       uint64_t archive_bytes, falcon_put_fn put, void* put_user,
                                       const falcon_pipeline_options* opt,
                                       falcon_pipeline_stats* stats) {
    FB_NVTX("falcon_decompress_stream");
    if (!ctx || !put || (!archive && archive_bytes)) return set_error(FALCON_ERR_INVALID, "null argument");
    std::lock_guard<std::mutex> lock(ctx->api_mutex);
    device_guard dg(ctx->device);
    decompress_io io;
    io.put = put;
    io.puser = put_user;
    const falcon_pipeline_options o = resolve(opt);
    return run_decompress(ctx, precision, archive, archive_bytes, io, o, stats);
}

falcon_status falcon_decompress_host(falcon_ctx* ctx, int precision, const uint8_t* archive,
                                     uint64_t archive_bytes, void* values, uint64_t cap_values,
                                     uint64_t* n_values, const falcon_pipeline_options* opt,
                                     falcon_pipeline_stats* stats) {
    FB_NVTX("falcon_decompress_host");
    if (!ctx || (!archive && archive_bytes)) return set_error(FALCON_ERR_INVALID, "null argument");
    std::lock_guard<std::mutex> lock(ctx->api_mutex);
    device_guard dg(ctx->device);
    decompress_io io;
    io.dst = static_cast<uint8_t*>(values);
    io.dst_cap = cap_values;
    io.dst_pinned = is_pinned(values);
    const falcon_pipeline_options o = resolve(opt);
    falcon_pipeline_stats st{};
    FB_TRY(run_decompress(ctx, precision, archive, archive_bytes, io, o, &st));
    if (n_values) *n_values = st.values;
    if (stats) *stats = st;
    return FALCON_OK;
}

}  // extern "C"
