// kernels_all.cu -- single device translation unit (the tables in tables.cu are
// referenced by the encode/decode kernels without relocatable device code).
#define FB200_KERNEL_TU 1
#include "launch_cache.cuh"
#include "tables.cu"
#include "encode.cu"
#include "decode.cu"
#include "selftest.cu"
#include "synth.cu"
