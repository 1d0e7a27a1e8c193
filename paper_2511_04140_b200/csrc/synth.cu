// synth.cu -- device generator for the counter-based field (field.cuh): the sharded
// configs produce their inputs in HBM, each rank only its own batch range.  Grid-stride,
// two values per thread per iteration with 16-B (f64) / 8-B (f32) stores.
#include "field.cuh"
#include "kernels.h"

namespace fb200 {

template <typename T>
__global__ void __launch_bounds__(256) field_kernel(T* __restrict__ out, uint64_t first, uint64_t count,
                                                    uint64_t seed, T scale) {
    const uint64_t stride = 2ull * gridDim.x * blockDim.x;
    for (uint64_t i = 2ull * (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x); i < count; i += stride) {
        // (T)units / 10^dp: one correctly rounded division, as inverse_scale does
        const T a = div_rn((T)field_units(seed, first + i), scale);
        if (i + 1 < count) {
            const T b = div_rn((T)field_units(seed, first + i + 1), scale);
            if ((reinterpret_cast<uintptr_t>(out + i) & (2 * sizeof(T) - 1)) == 0) {
                if constexpr (sizeof(T) == 8) *reinterpret_cast<double2*>(out + i) = make_double2(a, b);
                else *reinterpret_cast<float2*>(out + i) = make_float2(a, b);
            } else {
                out[i] = a;
                out[i + 1] = b;
            }
        } else {
            out[i] = a;
        }
    }
}

cudaError_t launch_field(int prec, void* out, uint64_t first, uint64_t count, uint64_t seed, int dp,
                         cudaStream_t st) {
    if (count == 0) return cudaSuccess;
    const uint64_t want = (count + 511) / 512;
    const unsigned grid = (unsigned)(want < 148ull * 16 ? want : 148ull * 16);
    if (prec == 0) {
        double p = 1;
        for (int i = 0; i < dp; ++i) p *= 10;
        field_kernel<double><<<grid, 256, 0, st>>>(static_cast<double*>(out), first, count, seed, p);
    } else {
        float p = 1;
        for (int i = 0; i < dp; ++i) p *= 10;
        field_kernel<float><<<grid, 256, 0, st>>>(static_cast<float*>(out), first, count, seed, p);
    }
    return cudaGetLastError();
}

}  // namespace fb200
