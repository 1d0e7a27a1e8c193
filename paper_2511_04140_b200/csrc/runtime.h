// runtime.h -- host runtime internals shared by the C-ABI translation units:
// status/message plumbing, device/pinned buffers, the host worker pool, the
// per-context scratch and pipeline slots.
#pragma once

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <deque>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include "../../include/falcon_b200.h"
#include "kernels.h"

namespace fb200 {

// ---- status plumbing -------------------------------------------------------
falcon_status set_error(falcon_status s, const std::string& msg);
const char* device_error_text(uint32_t code);
falcon_status device_error_status(uint32_t code);

#define FB_CUDA(x)                                                                          \
    do {                                                                                    \
        cudaError_t fb_e_ = (x);                                                            \
        if (fb_e_ != cudaSuccess)                                                           \
            return ::fb200::set_error(FALCON_ERR_CUDA, std::string(#x) + ": " +             \
                                                           cudaGetErrorString(fb_e_));      \
    } while (0)

#define FB_TRY(x)                                                                           \
    do {                                                                                    \
        falcon_status fb_s_ = (x);                                                          \
        if (fb_s_ != FALCON_OK) return fb_s_;                                               \
    } while (0)

// ---- NVTX: every C-ABI entry point and every host pipeline stage is a named range, so
//      an nsys / ncu timeline shows API calls, per-batch H2D / encode / D2H / store ----
struct nvtx_scope {
    explicit nvtx_scope(const char* name) { nvtxRangePushA(name); }
    ~nvtx_scope() { nvtxRangePop(); }
    nvtx_scope(const nvtx_scope&) = delete;
    nvtx_scope& operator=(const nvtx_scope&) = delete;
};
#define FB_NVTX(name) ::fb200::nvtx_scope fb_nvtx_scope_(name)

// ---- format helpers (host) ----------------------------------------------------
inline size_t lane_bytes(int prec) { return prec == FALCON_F64 ? 8 : 4; }
uint64_t max_chunk_bytes(int prec, uint32_t chunk_n);
uint64_t frame_bound(int prec, uint64_t count, uint32_t chunk_n);
falcon_status validate_options(uint32_t chunk_n, uint64_t batch_values);
falcon_status make_geometry(uint64_t n, uint32_t chunk_n, uint64_t bv, uint64_t header_bytes,
                            geometry& g);
archive_header_bytes header_bytes_of(int prec, uint32_t chunk_n, uint64_t bv, uint64_t total,
                                     uint64_t batches);

// ---- buffers ------------------------------------------------------------------
struct device_buffer {
    void* p = nullptr;
    size_t cap = 0;
    falcon_status ensure(size_t bytes);
    void release();
    ~device_buffer() { release(); }
    template <typename U> U* as() const { return static_cast<U*>(p); }
};

struct pinned_buffer {
    void* p = nullptr;
    size_t cap = 0;
    falcon_status ensure(size_t bytes);
    void release();
    ~pinned_buffer() { release(); }
    template <typename U> U* as() const { return static_cast<U*>(p); }
};

bool is_pinned(const void* p);

// ---- host task pool ------------------------------------------------------------
// Contract of the reference's worker_pool (include/falcon/worker_pool.hpp:14-38): N
// threads (0 = FALCON_WORKERS or the hardware thread count), FIFO jobs, joined on
// destruction.  Built here as a fixed-capacity ring of jobs plus a fork-join helper the
// pipeline uses to split pageable staging copies across threads.
class worker_pool {
public:
    explicit worker_pool(unsigned workers);
    ~worker_pool();
    worker_pool(const worker_pool&) = delete;
    worker_pool& operator=(const worker_pool&) = delete;
    void submit(std::function<void()> job);
    // run fn(0..parts-1) on the pool and the calling thread; returns when all are done
    void fork_join(unsigned parts, const std::function<void(unsigned)>& fn);
    unsigned size() const { return (unsigned)threads_.size(); }
    static unsigned default_workers();

private:
    void worker_main();
    std::mutex lock_;
    std::condition_variable has_job_, has_room_;
    std::vector<std::function<void()>> ring_;
    size_t head_ = 0, tail_ = 0;   // jobs [head_, tail_) modulo ring_.size()
    bool closing_ = false;
    std::vector<std::thread> threads_;
};

// Latched completion flag (pipeline.hpp:95-122 one_shot_event, host side).
class latch_flag {
public:
    void reset() {
        std::lock_guard<std::mutex> l(m_);
        set_ = false;
    }
    void fire() {
        {
            std::lock_guard<std::mutex> l(m_);
            set_ = true;
        }
        cv_.notify_all();
    }
    bool test() {
        std::lock_guard<std::mutex> l(m_);
        return set_;
    }
    void wait() {
        std::unique_lock<std::mutex> l(m_);
        cv_.wait(l, [&] { return set_; });
    }

private:
    std::mutex m_;
    std::condition_variable cv_;
    bool set_ = false;
};

// Small pinned mailbox a slot reads back after its kernels.
struct slot_mailbox {
    uint64_t total;
    unsigned long long error;
};

// One in-flight batch: a CUDA stream, its device buffers, pinned staging and events.
struct pipeline_slot {
    cudaStream_t stream = nullptr;
    cudaEvent_t ev_size = nullptr, ev_data = nullptr;
    device_buffer d_in, d_out, d_status, d_off, d_size, d_ready, d_misc;
    pinned_buffer h_in, h_out;
    slot_mailbox* box = nullptr;  // pinned
    // scheduling state (compress: pipeline.hpp:145 idle / m_pend / p_pend)
    int state = 0;
    uint64_t count = 0, seq = 0, offset = 0, frame = 0, first = 0, batch = 0;
    bool store_started = false;
    latch_flag done;
    falcon_status init();
    ~pipeline_slot();
};

}  // namespace fb200

struct falcon_ctx {
    int device = 0;
    // device-resident API scratch
    fb200::device_buffer enc_status, dec_off, dec_size, dec_ready, misc;
    fb200::pinned_buffer host_box;  // pinned mailbox for the sync device APIs
    fb200::device_buffer chunk_a, chunk_b;   // per-chunk operator scratch (chunk_workspace)
    std::mutex chunk_mutex;
    // host pipeline
    std::vector<std::unique_ptr<fb200::pipeline_slot>> slots;
    fb200::pinned_buffer stage;     // extra input staging buffer swapped into slots
    std::unique_ptr<fb200::worker_pool> pool;
    unsigned pool_workers = 0;
    std::mutex api_mutex;           // one API call at a time per context
    uint64_t last_archive_bytes = 0;
    uint64_t dec_err_cpb = 1, dec_err_first = 0;  // geometry of the last async decode's errors
    cudaEvent_t prof_ev[4] = {nullptr, nullptr, nullptr, nullptr};  // encode / decode kernel brackets
    fb200::worker_pool& get_pool(unsigned workers);
};
