// selftest.cu -- device-side checks of the per-value analysis used by encode.cu,
// exposed through falcon_selftest_dp() so tests can compare it with the CPU oracle.
//   out_full[i] = dp_alpha_full(v[i])           (alpha or -1)
//   out_lit[i]  = literal reference loop         (dp_alpha: round(), IEEE division)
//   out_cert[i] = dp_certify(v[i], A) code      (0 undecided, 1 ok, 2 exception)
//   out_g[i]    = lane integer from certification (valid when code == 1)
// with bit 2 set when the encoder's one-sided certify_lean() accepts the value.  The
// branch-free certify_fast() must agree with dp_certify and certify_lean may only
// accept what dp_certify certifies, with the same integer (-1 is written otherwise,
// which the test treats as a failure).
#include "dpds.cuh"
#include "kernels.h"

namespace fb200 {

template <typename T>
__global__ void selftest_dp_kernel(const T* __restrict__ v, uint64_t n, int A, int8_t* out_full,
                                   int8_t* out_lit, int8_t* out_cert, int64_t* out_g) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const T x = v[i];
        const int af = dp_alpha_full<T>(x);
        out_full[i] = (int8_t)(dp_alpha_k<T, 4>(x) == af ? af : -2);  // -2: the 4-wide form disagrees
        out_lit[i] = (int8_t)dp_alpha<T>(x);
        typename fpx<T>::S gv = 0;
        const T p = fpx<T>::pow10(A);
        const int c1 = dp_certify<T>(x, A, p, &gv);
        typename fpx<T>::S gf = 0;
        int mg = 0;
        const int c2 = certify_fast(x, A, p, &gf, &mg);
        // certify_lean is one-sided: true only where dp_certify says CERT_OK, same integer
        typename fpx<T>::S gl = 0;
        uint32_t ah = 0;
        const bool lean = certify_lean(x, cert_params_for(T{}, A), &gl, &ah);
        const bool agree = c1 == c2 && (c1 != CERT_OK || gf == gv) && (!lean || (c1 == CERT_OK && gl == gv));
        out_cert[i] = (int8_t)(agree ? (c1 | (lean ? 4 : 0)) : -1);
        out_g[i] = (int64_t)gv;
    }
}

// out[i] = the decoder's division-free inverse scale of g[i] at scale alpha
template <typename T>
__global__ void selftest_div_kernel(const int64_t* __restrict__ g, uint64_t n, int alpha, T* __restrict__ out) {
    const T p = fpx<T>::pow10(alpha);
    const T rp = div_rn(T(1), p);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const T gd = sizeof(T) == 8 ? (T)__ll2double_rn(g[i]) : (T)__ll2float_rn(g[i]);
        out[i] = div_pow10_markstein(gd, p, rp);
    }
}

cudaError_t launch_selftest_div(int prec, const int64_t* g, uint64_t n, int alpha, void* out, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const unsigned blocks = (unsigned)((n + 255) / 256 < 148 * 32 ? (n + 255) / 256 : 148 * 32);
    if (prec == 0) selftest_div_kernel<double><<<blocks, 256, 0, st>>>(g, n, alpha, static_cast<double*>(out));
    else selftest_div_kernel<float><<<blocks, 256, 0, st>>>(g, n, alpha, static_cast<float*>(out));
    return cudaGetLastError();
}

cudaError_t launch_selftest_dp(int prec, const void* v, uint64_t n, int A, int8_t* f, int8_t* l,
                               int8_t* c, int64_t* g, cudaStream_t st) {
    const unsigned blocks = (unsigned)((n + 255) / 256 < 148 * 32 ? (n + 255) / 256 : 148 * 32);
    if (n == 0) return cudaSuccess;
    if (prec == 0)
        selftest_dp_kernel<double><<<blocks, 256, 0, st>>>(static_cast<const double*>(v), n, A, f, l, c, g);
    else
        selftest_dp_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float*>(v), n, A, f, l, c, g);
    return cudaGetLastError();
}

}  // namespace fb200
