"""ctypes binding of the in-tree C-ABI library `libsgns_b200.so` (include/sgns_b200.h).

There is no CPU fallback: importing a device entry point without the built
library, or calling one without a CUDA device, raises.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_NAME = "libsgns_b200.so"
LIB_PATH = os.environ.get("SGNS_LIB_OVERRIDE") or os.path.join(HERE, LIB_NAME)  # override: experiments

SGNS_F32, SGNS_F64 = 0, 1
SIGMOID_TABLE, SIGMOID_EXACT = 0, 1
RNG_SPLITMIX, RNG_PHILOX = 0, 1
SCHEDULE_STATIC, SCHEDULE_DYNAMIC = 0, 1

P = C.c_void_p
I32, I64, U64, F64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double


class SgnsWorker(C.Structure):
    _fields_ = [("next_sent", I64), ("lo", I64), ("hi", I64), ("epoch", I32), ("done", I32),
                ("rng", U64), ("alpha", F64), ("read_local", F64), ("trained_local", F64),
                ("kernel_counter", I64), ("words_read", I64), ("words_trained", I64),
                ("inputs", I64)]


class DriveParams(C.Structure):
    _fields_ = [
        ("dtype", I32), ("d_m_in", P), ("d_m_out", P), ("vocab", I64), ("ld", I64), ("dim", I32),
        ("d_ids", P), ("d_offsets", P), ("d_keep_probs", P), ("rng_mode", I32),
        ("d_slots", P), ("n_slots", I64), ("d_alias_thr", P), ("d_alias_idx", P), ("seed", U64),
        ("window", I32), ("dynamic", I32), ("k_neg", I32), ("batch_cap", I32),
        ("sigmoid_mode", I32), ("d_sig_table", P),
        ("alpha0", F64), ("floor_frac", F64), ("total_x_epochs", F64), ("refresh_words", I64),
        ("d_shared", P), ("epochs", I32), ("loss_every", I32), ("d_workers", P),
        ("n_workers", I32), ("word_budget", I64), ("d_loss_by_epoch", P),
        ("d_cells_by_epoch", P), ("update", I32), ("max_sentence", I32), ("trace_cap", I64),
        ("d_trace", P), ("d_trace_alpha", P), ("d_trace_count", P), ("d_error", P),
        ("warps_per_block", I32), ("token_base", I64), ("epoch_base", I32),
        ("schedule", I32), ("d_claim", P), ("claim_end", I64), ("shard_lo", I64),
        ("shard_hi", I64), ("words_base", I64), ("d_totals", P), ("d_loss_total", P),
        ("d_dirty", P),
    ]


class LibraryMissing(ImportError):
    pass


_lib: C.CDLL | None = None


def lib() -> C.CDLL:
    """Load (once) and return the C-ABI library; raise if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise LibraryMissing(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(nvcc -gencode arch=compute_100a,code=sm_100a); this package has no CPU fallback")
    L = C.CDLL(LIB_PATH)
    L.sgns_abi_version.restype = C.c_int
    L.sgns_error_string.restype = C.c_char_p
    L.sgns_error_string.argtypes = [I32]
    L.sgns_update_windows.restype = C.c_int
    L.sgns_update_windows.argtypes = [I32, P, P, P, P, I64, I32, I64, P, P, P, I32, I32, I32, P, P,
                                      I32, I32, P, P, P, P]
    L.sgns_drive.restype = C.c_int
    L.sgns_drive.argtypes = [C.POINTER(DriveParams), P]
    L.sgns_init_model.restype = C.c_int
    L.sgns_init_model.argtypes = [I32, P, P, I64, I32, I64, U64, P]
    L.sgns_expand_slots.restype = C.c_int
    L.sgns_expand_slots.argtypes = [P, I64, P, I64, P]
    L.sgns_build_alias.restype = C.c_int
    L.sgns_build_alias.argtypes = [P, I64, F64, P, P]
    L.sgns_resident_workers.restype = C.c_int
    L.sgns_resident_workers.argtypes = [I32, I32, I32, I32, I32, I32, C.POINTER(I32)]
    L.sgns_vocab_build.restype = C.c_int
    L.sgns_vocab_build.argtypes = [C.c_char_p, I32, I32, C.POINTER(P), C.POINTER(I64), C.POINTER(I64)]
    L.sgns_vocab_from_tokens.restype = C.c_int
    L.sgns_vocab_from_tokens.argtypes = [P, P, P, I64, C.POINTER(P)]
    L.sgns_vocab_export.restype = C.c_int
    L.sgns_vocab_export.argtypes = [P, P, P, P]
    L.sgns_vocab_free.restype = None
    L.sgns_vocab_free.argtypes = [P]
    L.sgns_encode.restype = C.c_int
    L.sgns_encode.argtypes = [P, C.c_char_p, I32, I32, C.POINTER(P), C.POINTER(I64), C.POINTER(I64)]
    L.sgns_encoded_export.restype = C.c_int
    L.sgns_encoded_export.argtypes = [P, P, P, P]
    L.sgns_encoded_free.restype = None
    L.sgns_encoded_free.argtypes = [P]
    L.sgns_write_vectors.restype = C.c_int
    L.sgns_write_vectors.argtypes = [C.c_char_p, P, P, I64, I32, P, I64, I32, I32, I32]
    L.sgns_vectors_header.restype = C.c_int
    L.sgns_vectors_header.argtypes = [C.c_char_p, C.POINTER(I64), C.POINTER(I32), C.POINTER(I64)]
    L.sgns_vectors_sniff.restype = C.c_int
    L.sgns_vectors_sniff.argtypes = [C.c_char_p, I64, I32, C.POINTER(I32)]
    L.sgns_parse_vectors.restype = C.c_int
    L.sgns_parse_vectors.argtypes = [C.c_char_p, I32, I64, I32, P, P, P, C.POINTER(I64), C.POINTER(I64)]
    L.sgns_unit_rows.restype = C.c_int
    L.sgns_unit_rows.argtypes = [P, I64, I64, I32, P, I64, P]
    L.sgns_analogy_top1.restype = C.c_int
    L.sgns_analogy_top1.argtypes = [P, I64, I64, I32, P, I64, P, P, P]
    L.sgns_struct_sizes.restype = C.c_int
    L.sgns_struct_sizes.argtypes = [C.POINTER(I32), C.POINTER(I32)]
    if L.sgns_abi_version() != 2:
        raise LibraryMissing("libsgns_b200.so ABI version mismatch; rebuild")
    wb, pb = I32(0), I32(0)
    L.sgns_struct_sizes(C.byref(wb), C.byref(pb))
    if (wb.value, pb.value) != (C.sizeof(SgnsWorker), C.sizeof(DriveParams)):
        raise LibraryMissing(f"struct layout mismatch: C ({wb.value}, {pb.value}) vs ctypes "
                             f"({C.sizeof(SgnsWorker)}, {C.sizeof(DriveParams)}); rebuild")
    _lib = L
    return L


EXPORTED = ("sgns_update_windows", "sgns_drive", "sgns_init_model", "sgns_expand_slots",
            "sgns_build_alias", "sgns_resident_workers", "sgns_error_string", "sgns_abi_version",
            "sgns_struct_sizes", "sgns_vocab_build", "sgns_vocab_from_tokens", "sgns_vocab_export",
            "sgns_vocab_free", "sgns_encode", "sgns_encoded_export", "sgns_encoded_free",
            "sgns_write_vectors", "sgns_vectors_header", "sgns_vectors_sniff", "sgns_parse_vectors",
            "sgns_unit_rows", "sgns_analogy_top1")


class SgnsError(RuntimeError):
    pass


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().sgns_error_string(rc).decode()
        if rc < 0:
            raise ValueError(f"{what}: {msg} (code {rc})")
        raise SgnsError(f"{what}: CUDA error {rc}: {msg}")
