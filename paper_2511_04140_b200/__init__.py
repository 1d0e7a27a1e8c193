"""B200-native Falcon (arXiv 2511.04140): lossless floating-point time-series codec.

The product is libfalcon_b200.so (sm_100a CUDA kernels + C ABI, include/falcon_b200.h)
and the C++ drop-in header include/falcon_b200/falcon.hpp.  This Python package is a
ctypes binding used by the tests and bench.
"""
from .falcon import (F32, F64, Codec, CorruptError, CudaError, FalconError, PipelineOptions,  # noqa: F401
                     PipelineStats, compress_bound, load, max_encoded_chunk_size, options,
                     read_header, synth)
from .falcon import compress_host_multi, decompress_host_multi  # noqa: F401
