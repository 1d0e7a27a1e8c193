// selftest.cu -- device-side checks of the per-value analysis used by encode.cu,
// exposed through falcon_selftest_dp() so tests can compare it with the CPU oracle.
//   out_full[i] = dp_alpha_full(v[i])           (alpha or -1)
//   out_lit[i]  = literal reference loop         (dp_alpha: round(), IEEE division)
//   out_cert[i] = dp_certify(v[i], A) code      (0 undecided, 1 ok, 2 exception)
//   out_g[i]    = lane integer from certification (valid when code == 1)
// and the branch-free encoder form certify_fast() must agree with dp_certify (code
// 3 is written when they disagree, which the test treats as a failure).
#include "dpds.cuh"
#include "kernels.h"

namespace fb200 {

template <typename T>
__global__ void selftest_dp_kernel(const T* __restrict__ v, uint64_t n, int A, int8_t* out_full,
                                   int8_t* out_lit, int8_t* out_cert, int64_t* out_g) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const T x = v[i];
        out_full[i] = (int8_t)dp_alpha_full<T>(x);
        out_lit[i] = (int8_t)dp_alpha<T>(x);
        typename fpx<T>::S gv = 0;
        const T p = fpx<T>::pow10(A);
        const int c1 = dp_certify<T>(x, A, p, &gv);
        typename fpx<T>::S gf = 0;
        int mg = 0;
        const int c2 = certify_fast(x, A, p, &gf, &mg);
        out_cert[i] = (int8_t)((c1 == c2 && (c1 != CERT_OK || gf == gv)) ? c1 : 3);
        out_g[i] = (int64_t)gv;
    }
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
