"""B200-native sharded-parameter hot path of DeepCompile (arxiv 2504.09983).

    dc       — ctypes binding of include/dc.h (libdc_b200.so; no CPU fallback)
    runtime  — torch-side plumbing: allocates the shard store, symmetric
               buffers, streams; drives profile -> plan -> step through the C ABI
    build    — nvcc build of libdc_b200.so for sm_100a
"""
__all__ = ["dc", "runtime", "build"]
