// tables.cu -- device copies of the numeric tables.
//   pow10:  exact 10^0..10^max_alpha built by repeated *10 (numeric.hpp:17-41)
//   decade: correctly rounded 10^k for k in [min_decade, max_decade], stored as IEEE
//           bit patterns (numeric.cpp:10-39 builds them with snprintf("1e%d") +
//           std::from_chars; glibc strtod/strtof are also correctly rounded, so the
//           tables are bit-identical).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "kernels.h"

namespace fb200 {

cudaError_t upload_tables() {
    double p64[23];
    float p32[11];
    double d = 1.0;
    for (int i = 0; i < 23; ++i, d *= 10.0) p64[i] = d;
    float f = 1.0f;
    for (int i = 0; i < 11; ++i, f *= 10.0f) p32[i] = f;
    // RN(1 / 10^a), the decoder's division-free inverse scale (dpds.cuh): IEEE division on
    // the host, correctly rounded like the device's div_rn
    double r64[23];
    float r32[11];
    for (int i = 0; i < 23; ++i) r64[i] = 1.0 / p64[i];
    for (int i = 0; i < 11; ++i) r32[i] = 1.0f / p32[i];
    uint64_t dec64[618];
    uint32_t dec32[78];
    dec64[617] = 0x7ff0000000000000ull;  // guard: only read for inf/nan lanes
    dec32[77] = 0x7f800000u;
    char buf[16];
    for (int k = -308; k <= 308; ++k) {
        std::snprintf(buf, sizeof buf, "1e%d", k);
        const double v = std::strtod(buf, nullptr);
        std::memcpy(&dec64[k + 308], &v, 8);
    }
    for (int k = -38; k <= 38; ++k) {
        std::snprintf(buf, sizeof buf, "1e%d", k);
        const float v = std::strtof(buf, nullptr);
        std::memcpy(&dec32[k + 38], &v, 4);
    }
    // certification parameters per candidate scale (dpds.cuh cert_params_for)
    cert_row64 c64[23];
    cert_row32 c32[11];
    for (int a = 0; a < 23; ++a) {
        uint64_t pb;
        std::memcpy(&pb, &p64[a], 8);
        const uint32_t L = (uint32_t)(dec64[308 - a] >> 32), U = (uint32_t)(dec64[308 + 15 - a] >> 32);
        c64[a].p = p64[a];
        c64[a].lo1 = L + 1u;
        c64[a].span = U > L + 1u ? U - L - 1u : 0u;
        c64[a].hk = (uint32_t)(pb >> 32) - (1076u << 20);
        c64[a].plo = (uint32_t)pb;
        c64[a].lim = (2074u - ((uint32_t)(pb >> 32) >> 20)) << 20;
        c64[a].pad = 0;
    }
    for (int a = 0; a < 11; ++a) {
        uint32_t pb;
        std::memcpy(&pb, &p32[a], 4);
        c32[a].p = p32[a];
        c32[a].lo = dec32[38 - a];
        c32[a].span = dec32[38 + 6 - a] - dec32[38 - a];
        c32[a].hk = pb - (151u << 23);
    }
    cudaError_t e;
    if ((e = cudaMemcpyToSymbol(g_cert_f64, c64, sizeof c64))) return e;
    if ((e = cudaMemcpyToSymbol(g_cert_f32, c32, sizeof c32))) return e;
    if ((e = cudaMemcpyToSymbol(g_pow10_f64, p64, sizeof p64))) return e;
    if ((e = cudaMemcpyToSymbol(g_pow10_f32, p32, sizeof p32))) return e;
    if ((e = cudaMemcpyToSymbol(g_rpow10_f64, r64, sizeof r64))) return e;
    if ((e = cudaMemcpyToSymbol(g_rpow10_f32, r32, sizeof r32))) return e;
    if ((e = cudaMemcpyToSymbol(g_decade_f64, dec64, sizeof dec64))) return e;
    return cudaMemcpyToSymbol(g_decade_f32, dec32, sizeof dec32);
}

}  // namespace fb200
