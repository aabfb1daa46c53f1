"""ctypes declarations of libzkdl.so (include/zkdl.h).  Argument marshalling only.

The library is loaded from this package directory (built in-tree by
`python -m paper_2307_16273_b200.build`).  There is no fallback: a missing
library raises ImportError, a missing device makes every call fail with
ZK_ERR_CUDA.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(HERE, "libzkdl.so")

STATUS = {0: "ZK_OK", -1: "ZK_ERR_ARG", -2: "ZK_ERR_RANGE", -3: "ZK_ERR_NONCANONICAL", -4: "ZK_ERR_OOM",
          -5: "ZK_ERR_CUDA", -6: "ZK_ERR_NCCL", -7: "ZK_ERR_UNIMPLEMENTED", -8: "ZK_ERR_INTERNAL",
          1: "ZK_REJECT"}


class ZkError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class MmShape(ctypes.Structure):
    _fields_ = [("logN", ctypes.c_uint32), ("logD1", ctypes.c_uint32), ("logD2", ctypes.c_uint32),
                ("logD3", ctypes.c_uint32), ("trans_a", ctypes.c_uint32), ("trans_b", ctypes.c_uint32)]


class View(ctypes.Structure):
    _fields_ = [("logN", ctypes.c_uint32), ("map", ctypes.c_void_p), ("u", ctypes.c_void_p)]


class CmView(ctypes.Structure):
    _fields_ = [("logN", ctypes.c_uint32), ("map", ctypes.c_void_p)]


class ProdStmt(ctypes.Structure):
    _fields_ = [("m", ctypes.c_uint32), ("n_eq", ctypes.c_uint32), ("n_tables", ctypes.c_uint32),
                ("i32_mask", ctypes.c_uint32), ("w", ctypes.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(SO_PATH):
        raise ImportError(f"libzkdl.so not built: run `python -m paper_2307_16273_b200.build` ({SO_PATH})")
    L = ctypes.CDLL(SO_PATH)
    c = ctypes
    vp, u64, u32, i32 = c.c_void_p, c.c_uint64, c.c_uint32, c.c_int
    sig = {
        "zk_ctx_create": ([i32, vp, c.POINTER(vp)], i32),
        "zk_ctx_destroy": ([vp], None),
        "zk_last_error": ([vp], c.c_char_p),
        "zk_version": ([], c.c_char_p),
        "zk_ctx_launch_count": ([vp], u64),
        "zk_ctx_synchronize": ([vp], i32),
        "zk_ctx_profile": ([vp, i32], i32),
        "zk_ctx_profile_read": ([vp, c.c_char_p, u64], i32),
        "zk_ctx_profile_filter": ([vp, c.c_char_p], i32),
        "zk_ctx_set_sm_budget": ([vp, u32], i32),
        "zk_ctx_set_persistent": ([vp, i32], i32),
        "zk_reindex_prove": ([vp, vp, vp, u32, u32, u32, vp, vp, vp, vp, c.POINTER(u64), vp, vp], i32),
        "zk_relu_merge": ([vp, vp, vp, vp, u32, u32, u32, vp, vp, vp, c.POINTER(u64), vp, vp], i32),
        "zk_relu_merge_dev": ([vp, vp, vp, vp, u32, u32, u32, vp, vp, c.POINTER(u64)], i32),
        "zk_hadamard_zero_prove": ([vp, vp, vp, vp, vp, u32, vp, c.POINTER(u64), vp, vp, vp], i32),
        "zk_transcript_new": ([vp, vp, c.POINTER(vp)], i32),
        "zk_transcript_absorb": ([vp, c.c_char_p, vp, u64], i32),
        "zk_transcript_challenges": ([vp, c.c_char_p, u32, vp], i32),
        "zk_transcript_state": ([vp, vp], i32),
        "zk_transcript_fork": ([vp, c.c_char_p, vp, c.POINTER(vp)], i32),
        "zk_transcript_absorb_state": ([vp, c.c_char_p, vp], i32),
        "zk_transcript_free": ([vp], None),
        "zk_embed_i32": ([vp, vp, u64, vp], i32),
        "zk_widen_i16": ([vp, vp, u64, vp], i32),
        "zk_undelta_i8": ([vp, vp, vp, u64, u32, u32, vp], i32),
        "zk_eq_table": ([vp, vp, u32, vp, vp], i32),
        "zk_mle_eval_i32": ([vp, vp, u32, vp, vp], i32),
        "zk_mle_eval_fr": ([vp, vp, u32, vp, vp], i32),
        "zk_fr_table_to_canonical": ([vp, vp, u64, vp], i32),
        "zk_fr_table_from_canonical": ([vp, vp, u64, vp], i32),
        "zk_matmul_reduce": ([vp, vp, vp, vp, MmShape, vp, vp, vp, vp], i32),
        "zk_sumcheck_prove": ([vp, vp, c.POINTER(ProdStmt), vp, vp, vp, vp, c.POINTER(u64), vp, vp], i32),
        "zk_relu_tables": ([vp, vp, vp, u64, u32, u32, vp, vp, vp, vp, vp, vp, vp], i32),
        "zk_relu_prove": ([vp, vp, vp, vp, u32, u32, u32, vp, c.POINTER(u64), vp, vp, vp], i32),
        "zk_matmul_prove": ([vp, vp, vp, vp, MmShape, vp, vp, vp, c.POINTER(u64)], i32),
        "zk_relu_prove_dev": ([vp, vp, vp, vp, u32, u32, u32, vp, c.POINTER(u64), vp], i32),
        "zk_transcript_state_dev": ([vp, vp], i32),
        "zk_sc_shard_create": ([vp, vp, c.POINTER(ProdStmt), vp, vp, u32, u32, c.POINTER(vp)], i32),
        "zk_sc_shard_partial": ([vp, vp], i32),
        "zk_sc_shard_finish": ([vp, vp], i32),
        "zk_sc_shard_rounds_done": ([vp], u32),
        "zk_sc_shard_local_log": ([vp], u32),
        "zk_sc_shard_export": ([vp, vp], i32),
        "zk_sc_shard_adopt": ([vp, vp], i32),
        "zk_sc_shard_result": ([vp, vp, c.POINTER(u64), vp, vp, vp], i32),
        "zk_sc_shard_free": ([vp], None),
        "zk_nccl_unique_id": ([vp], i32),
        "zk_ctx_attach_nccl": ([vp, vp, i32, i32], i32),
        "zk_ctx_detach_nccl": ([vp], i32),
        "zk_sc_shard_prove_nccl": ([vp, u32], i32),
        "zk_diag_fr_op": ([vp, i32, vp, vp, u64, vp], i32),
        "zk_diag_mul_bench": ([vp, vp, u32, u32, vp], i32),
        "zk_diag_rowdot": ([vp, vp, u64, u32, vp, vp, i32], i32),
        "zk_diag_fs_bench": ([vp, u32, i32, vp], i32),
        "zk_htr_init": ([vp, vp], i32),
        "zk_htr_absorb": ([vp, c.c_char_p, vp, u64], i32),
        "zk_htr_challenges": ([vp, c.c_char_p, u32, vp], i32),
        "zk_verify_sumcheck": ([vp, vp, u64, vp, vp, vp, vp, vp], i32),
        "zk_verify_hadamard_zero": ([vp, vp, u64, u32, vp, vp, vp], i32),
        "zk_verify_relu": ([vp, vp, u64, vp, vp, vp, vp], i32),
        "zk_verify_claim_merge": ([vp, u32, u32, u32, vp, vp, vp, vp, u64, vp, vp, vp], i32),
        "zk_claim_merge_dev": ([vp, vp, vp, vp, u32, u32, u32, u32, u32, u32, vp, vp, vp, vp, c.POINTER(u64)], i32),
        "zk_loss_grad_prove_dev": ([vp, vp, vp, vp, vp, u32, vp, c.POINTER(u64)], i32),
        "zk_rescale_prove_dev": ([vp, vp, vp, u32, u32, u32, vp, vp, c.POINTER(u64), vp], i32),
        "zk_verify_rescale": ([vp, vp, u64, vp, vp, vp, vp, vp, vp], i32),
        "zk_relu_prove_chained_dev": ([vp, vp, vp, vp, u32, u32, u32, vp, vp, c.POINTER(u64), vp], i32),
        "zk_loss_grad_prove": ([vp, vp, vp, vp, vp, u32, vp, vp], i32),
        "zk_verify_loss_grad": ([vp, u32, vp, vp, vp], i32),
        "zk_verify_relu_merge": ([vp, u32, u32, u32, vp, vp, vp, u64, vp, vp], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def declared_symbols(header: str | None = None) -> list:
    """Function names declared in include/zkdl.h (for the export test)."""
    import re
    header = header or os.path.join(os.path.dirname(HERE), "include", "zkdl.h")
    txt = open(header).read()
    return sorted(set(re.findall(r"^\s*(?:zk_status|void|const char\*|uint64_t|uint32_t)\s+(zk_\w+)\s*\(", txt, re.M)))
