// kernels.h -- host-side launch interface of the sm_100a codec kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "falcon_common.cuh"

namespace fb200 {

struct archive_header_bytes {
    uint8_t b[48];
};

// Scratch for one compress launch (device memory, owned by the caller/context).
// Carved out of one buffer by carve_encode_ws(); encode_scratch_bytes() sizes it.
struct encode_ws {
    uint8_t* images;              // [ring][slot] chunk images (16-B aligned slots), chunk c at c % ring
    uint64_t ring;                // image slots (O(wave), launch_encode)
    uint32_t slot;                // bytes per image slot
    uint32_t* sizes;              // [n_chunks] encoded chunk sizes
    uint64_t* tile_status;        // [n_tiles] placement look-back words
    uint64_t* batch_prefix;       // [n_batches] payload prefix of each batch | ready bit
    uint32_t* look;               // [n_chunks] sample verdicts (sample_chunks_kernel)
    uint32_t* ticket;             // placement tile ticket counter
    unsigned long long* error;    // (chunk << 8 | code), ~0 = none
    uint64_t* total;              // archive bytes, written by the placement kernel
};

// One encode launch: batches [b0, b0 + gridDim.y - 1) are encoded, and grid row 0 places
// `place_tiles` tiles (of blockDim.x chunks) that earlier launches finished.
struct encode_launch {
    uint32_t b0;
    uint32_t place_tiles;
    uint32_t enc_c0, enc_slot0;       // first chunk encoded here and its ring slot
    uint32_t place_c0, place_slot0;   // first chunk placed here and its ring slot
    uint32_t b_end;                   // first batch after this launch's wave
    uint32_t full_b;                  // batches [0, full_b) hold cpb full chunks each
    uint32_t pf_ahead;                // L2 prefetch distance in chunks (0: off)
};
template <typename T> uint32_t encode_slot_bytes(uint32_t chunk_n);
template <typename T> size_t encode_scratch_bytes(const geometry& g);
template <typename T>
encode_ws carve_encode_ws(void* scratch, const geometry& g, uint32_t* ticket,
                          unsigned long long* error, uint64_t* total);

// Scratch for one decompress launch.
struct decode_ws {
    uint32_t* ticket;             // chunk ticket counter
    uint32_t* ready;              // [n_batches] batch frame located (1) or not (0)
    unsigned long long* abort_at; // first batch the walker could not locate (~0 = none)
    uint64_t* chunk_off;          // [n_chunks] archive offset of each chunk
    uint32_t* chunk_size;         // [n_chunks]
    unsigned long long* error;
};

uint32_t encode_block_threads(uint32_t chunk_n);
template <typename T> uint32_t encode_smem_bytes(uint32_t chunk_n);
template <typename T> uint32_t decode_smem_bytes(uint32_t chunk_n);

// ev0/ev1 (optional) are recorded right before / after the main kernel (profiling hook).
template <typename T>
cudaError_t launch_encode(const T* d_in, const geometry& g, uint8_t* d_out, uint64_t out_cap,
                          const encode_ws& ws, const archive_header_bytes& hdr, cudaStream_t st,
                          cudaEvent_t ev0 = nullptr, cudaEvent_t ev1 = nullptr);

// d_archive points at the archive's first byte (the 47-byte header), `len` bytes long.
// d_len (optional): the archive length in device memory, read by the kernel instead of len.
template <typename T>
cudaError_t launch_decode(const uint8_t* d_archive, uint64_t len, const geometry& g, T* d_out,
                          const decode_ws& ws, cudaStream_t st, cudaEvent_t ev0 = nullptr,
                          cudaEvent_t ev1 = nullptr, const uint64_t* d_len = nullptr);

// index[b] = archive offset of batch b's frame (b < n_batches), index[n_batches] = end
cudaError_t launch_index(const uint8_t* d_archive, uint64_t len, uint64_t header_bytes, uint64_t n_batches,
                         uint64_t* d_index, unsigned long long* d_error, cudaStream_t st);

cudaError_t launch_selftest_dp(int prec, const void* v, uint64_t n, int A, int8_t* full,
                               int8_t* lit, int8_t* cert, int64_t* g, cudaStream_t st);

cudaError_t launch_selftest_div(int prec, const int64_t* g, uint64_t n, int alpha, void* out, cudaStream_t st);

// Counter-based field generator (field.cuh): values [first, first + count) into out.
cudaError_t launch_field(int prec, void* out, uint64_t first, uint64_t count, uint64_t seed, int dp,
                         cudaStream_t st);

// One-time upload of the pow10 / decade tables (numeric.hpp:17-41, numeric.cpp:10-39).
cudaError_t upload_tables();

}  // namespace fb200
