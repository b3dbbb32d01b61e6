"""ctypes binding of libtmb200.so (include/tsetlin_b200.h).

The library is built in-tree (``make -C paper_2405_04212_b200/csrc``, or
``__graft_entry__.build()``).  There is deliberately no fallback: if the
shared object is missing or no sm_100 device is present, every compute call
raises ``TmbError``.
"""

from __future__ import annotations

import ctypes as ct
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# TMB_LIB: an alternative build of the same library (A/B timing experiments)
LIB_PATH = os.environ.get("TMB_LIB") or os.path.join(_HERE, "libtmb200.so")

u64, i64, i32, f64, vp = ct.c_uint64, ct.c_int64, ct.c_int, ct.c_double, ct.c_void_p

TMB_OK = 0
TMB_E_INVALID = -1
TMB_E_CUDA = -2
TMB_E_NO_DEVICE = -3
TMB_E_NOMEM = -4
TMB_E_UNSUPPORTED = -5


class TmbError(RuntimeError):
    """A libtmb200 call failed (message from tmb_last_error)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"libtmb200 error {code}: {msg}")
        self.code = code


class TrainCfg(ct.Structure):
    _fields_ = [("n_literals", i64), ("n_positions", i64), ("n_clauses", i64),
                ("n_classes", i64), ("n_blocks", i64), ("threshold", i64), ("budget", i64),
                ("s", f64), ("boost", ct.c_int32), ("state_min", ct.c_int32),
                ("state_max", ct.c_int32), ("flags", ct.c_int32), ("seed", u64)]


class TrainStats(ct.Structure):
    _fields_ = [("examples", u64), ("events", u64), ("type_i", u64), ("type_ii", u64),
                ("draws", u64), ("state_updates", u64)]


class SparseCfg(ct.Structure):
    _fields_ = [("n_literals", i64), ("n_clauses", i64), ("n_classes", i64),
                ("n_blocks", i64), ("threshold", i64), ("budget", i64), ("s", f64),
                ("boost", ct.c_int32), ("floor_", ct.c_int32), ("state_max", ct.c_int32),
                ("capacity", ct.c_int32), ("seed", u64), ("slab", i64)]


# name -> (restype, argtypes)
SIGNATURES = {
    "tmb_abi_version": (i32, []),
    "tmb_last_error": (ct.c_char_p, []),
    "tmb_device_info": (i32, [i32, vp, vp, vp, vp, vp]),
    "tmb_launch_count": (u64, []),
    "tmb_microbench_allreduce": (i32, [i32, i32, i32, i32, vp]),
    "tmb_microbench_sparse_event": (i32, [i32, i32, i32, i32, i32, i32, vp]),
    "tmb_microbench_feedback": (i32, [i32, i32, i32, i32, i32, vp]),
    "tmb_microbench_icache": (i32, [i32, i32, i32, vp]),
    "tmb_microbench_pipe": (i32, [i32, i32, i32, i32, vp, vp]),
    "tmb_microbench_pingpong": (i32, [i32, i32, vp, vp]),
    "tmb_derive_stream": (u64, [u64, u64]),
    "tmb_stream_u64_block": (i32, [u64, u64, i64, vp, vp]),
    "tmb_shuffle_permutation": (i32, [i64, u64, u64, vp, vp]),
    "tmb_clause_outputs": (i32, [vp, i64, i64, vp, i32, i64, vp, vp]),
    "tmb_clause_outputs_batch": (i32, [vp, i64, i64, vp, i64, i32, i64, vp, vp]),
    "tmb_bank_feedback": (i32, [vp, vp, i64, i64, i64, vp, vp, i64, i64, vp, vp, f64, i32,
                                i32, i32, u64, u64, vp, vp]),
    "tmb_bank_feedback_draws": (i32, [vp, vp, i64, i64, i64, vp, vp, i64, i64, vp, vp, f64,
                                      i32, i32, i32, u64, vp, i64, vp, vp]),
    "tmbh_clause_outputs": (i32, [vp, i64, i64, vp, i32, i64, vp]),
    "tmbh_clause_outputs_batch": (i32, [vp, i64, i64, vp, i64, i32, i64, vp]),
    "tmbh_bank_feedback": (i32, [vp, vp, i64, i64, i64, vp, vp, i64, i64, vp, vp, f64, i32,
                                 i32, i32, u64, u64, vp]),
    "tmb_pack_literals": (i32, [vp, i64, i64, i32, vp, vp]),
    "tmb_trainer_create": (i32, [vp, vp, vp, vp, i32, i32, vp]),
    "tmb_trainer_destroy": (i32, [vp]),
    "tmb_trainer_set_trace": (i32, [vp, vp]),
    "tmb_trainer_set_profile": (i32, [vp, vp]),
    "tmb_trainer_info": (i32, [vp, vp, vp, vp, vp]),
    "tmb_trainer_kernel": (i32, [vp, vp, vp]),
    "tmb_trainer_run": (i32, [vp, vp, vp, vp, i64, u64, vp, vp]),
    "tmb_rules_from_bank": (i32, [vp, vp, i64, i64, i64, i64, i32, vp, vp]),
    "tmb_rules_from_csr": (i32, [vp, vp, i64, vp, i64, i64, i32, vp]),
    "tmb_rules_destroy": (i32, [vp]),
    "tmb_rules_info": (i32, [vp, vp, vp]),
    "tmb_infer": (i32, [vp, vp, i64, vp, vp, vp, vp, vp]),
    "tmbh_infer": (i32, [vp, vp, i64, vp, vp, i64]),
    "tmb_infer_status": (i32, [vp]),
    "tmb_set_option": (i32, [ct.c_char_p, i64]),
    "tmb_explain": (i32, [vp, vp, i64, i32, vp, vp, vp, vp]),
    "tmb_infer_packed": (i32, [vp, vp, i64, i64, vp, vp, vp, vp, vp]),
    "tmb_sparse_create": (i32, [vp, vp, i64, vp]),
    "tmb_sparse_destroy": (i32, [vp]),
    "tmb_sparse_layout": (i32, [vp, vp]),
    "tmb_sparse_train": (i32, [vp, vp, vp, vp, vp, i64, u64, vp, vp]),
    "tmb_sparse_feedback": (i32, [vp, vp, i64, vp, i64, i64, vp, vp, u64, u64, vp, vp]),
    "tmb_sparse_get": (i32, [vp, vp, vp, vp, vp, vp, vp]),
    "tmb_sparse_set": (i32, [vp, vp, vp, vp, vp, vp, vp]),
    "tmb_sparse_infer": (i32, [vp, vp, vp, i64, vp, vp, vp]),
    "tmb_sparse_outputs": (i32, [vp, vp, vp, i64, vp, vp]),
}

_lib = None


def load():
    """Load libtmb200.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise TmbError(TMB_E_NO_DEVICE,
                           f"{LIB_PATH} is missing; build it with __graft_entry__.build() "
                           "(there is no CPU fallback)")
        lib = ct.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def call(name: str, *args) -> int:
    """Call an int-returning entry point and raise TmbError on failure."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != TMB_OK:
        msg = lib.tmb_last_error().decode(errors="replace")
        raise TmbError(rc, f"{name}: {msg}")
    return rc


def launch_count() -> int:
    return int(load().tmb_launch_count())
