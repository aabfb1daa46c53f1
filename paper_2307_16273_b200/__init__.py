"""zkdl-b200: B200-native (sm_100a) prover hot path of zkDL (arXiv 2307.16273).

The proving path is libzkdl.so (C ABI in include/zkdl.h, CUDA sources in csrc/);
`api` is its ctypes binding and `fcn` the FAC4DNN family driver.  There is no
CPU fallback: importing `api` without a built library raises.
"""
__all__ = ["api", "fcn", "build"]
