"""ctypes binding of the C ABI in `include/lightbeam_b200.h` (the in-tree `_lightbeam_b200.so`).

There is deliberately no fallback: if the shared object is missing or no CUDA device is
visible, every entry point raises `DeviceError` -- the decode path never silently runs on
the CPU.  `build()` compiles the library in-tree with nvcc for sm_100a.
"""

from __future__ import annotations

import ctypes as C
import os
import sysconfig
import subprocess
from pathlib import Path

import numpy as np

from .errors import DeviceError

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB_PATH = PKG / "_lightbeam_b200.so"
# development A/B runs only (tools/ab_variants.py): load a variant build instead
if os.environ.get("LB_LIB_VARIANT"):
    LIB_PATH = PKG / f"_lightbeam_b200_{os.environ['LB_LIB_VARIANT']}.so"
INCLUDE = PKG.parent / "include"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-fmad=false",  # bit-exact fp64 score arithmetic: no contraction into FMA
    "-Xcompiler", "-fPIC,-ffp-contract=off",
    "-shared",
]
SOURCES = ["lb_kernels.cu", "lb_capi.cu", "lb_llm.cu"]


PYRES_PATH = PKG / f"_lb_results{sysconfig.get_config_var('EXT_SUFFIX')}"


def build_pyresults(force: bool = False) -> Path:
    """gcc -> the CPython result binding (csrc/lb_pyresults.c), skipped when up to date."""
    src = CSRC / "lb_pyresults.c"
    deps = [src, INCLUDE / "lightbeam_b200.h"]
    if not force and PYRES_PATH.exists() and PYRES_PATH.stat().st_mtime >= max(
            p.stat().st_mtime for p in deps):
        return PYRES_PATH
    cmd = [os.environ.get("CC", "gcc"), "-O2", "-shared", "-fPIC", "-std=c11",
           f"-I{sysconfig.get_paths()['include']}", f"-I{INCLUDE}", "-o", str(PYRES_PATH), str(src)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise DeviceError(f"result binding build failed ({' '.join(cmd)}):\n{res.stderr}")
    return PYRES_PATH


_PYRES = None


def pyresults():
    """The CPython result binding (built by build(); no pure-Python stand-in)."""
    global _PYRES
    if _PYRES is None:
        if not PYRES_PATH.exists():
            raise DeviceError(f"{PYRES_PATH.name} is missing: run __graft_entry__.build()")
        import importlib.util

        spec = importlib.util.spec_from_file_location("_lb_results", PYRES_PATH)
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _PYRES = mod
    return _PYRES


def build(verbose: bool = False, force: bool = False) -> Path:
    """nvcc -> paper_2603_14002_b200/_lightbeam_b200.so (skipped when up to date), plus the
    CPython result binding."""
    build_pyresults(force)
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h"))
    deps.append(INCLUDE / "lightbeam_b200.h")
    if not force and LIB_PATH.exists():
        newest = max(p.stat().st_mtime for p in deps)
        if LIB_PATH.stat().st_mtime >= newest:
            return LIB_PATH
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, *NVCC_FLAGS, "-o", str(LIB_PATH), *[str(CSRC / s) for s in SOURCES]]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    res = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    if res.returncode != 0:
        raise DeviceError(f"nvcc failed ({' '.join(cmd)}):\n{res.stderr}")
    if verbose:
        print(res.stderr)
    return LIB_PATH


class LbResultsView(C.Structure):
    """lb_results_view (include/lightbeam_b200.h)."""
    _fields_ = [
        ("n_trials", C.c_int32),
        ("total_nbest", C.c_int64),
        ("blob_bytes", C.c_int64),
        ("blob", C.c_void_p),
        ("status", C.c_void_p),
        ("best_text_off", C.c_void_p),
        ("best_text_len", C.c_void_p),
        ("best_score", C.c_void_p),
        ("nbest_count", C.c_void_p),
        ("nbest_text_off", C.c_void_p),
        ("nbest_text_len", C.c_void_p),
        ("nbest_score", C.c_void_p),
    ]


class LbConfig(C.Structure):
    _fields_ = [
        ("acoustic_scale", C.c_double),
        ("beam_prune_threshold", C.c_double),
        ("homophone_prune_threshold", C.c_double),
        ("token_insertion_bonus", C.c_double),
        ("word_boundary_bonus", C.c_double),
        ("ngram_weight", C.c_double),
        ("llm_weight", C.c_double),
        ("beam_size", C.c_int32),
        ("ortho_beams", C.c_int32),
        ("llm_rescore_interval", C.c_int32),
        ("llm_chunk_size", C.c_int32),
    ]


class LbTableDesc(C.Structure):
    _fields_ = [
        ("table", C.c_void_p),
        ("num_states", C.c_int32),
        ("vocab_size", C.c_int32),
        ("sink", C.c_int32),
        ("blank_id", C.c_int32),
        ("space_id", C.c_int32),
        ("comp_offsets", C.c_void_p),
        ("comp_surface", C.c_void_p),
        ("comp_lmword", C.c_void_p),
        ("n_comp", C.c_int32),
        ("surface_blob", C.c_char_p),
        ("surface_offsets", C.c_void_p),
        ("n_surfaces", C.c_int32),
    ]


class LbNgramDesc(C.Structure):
    _fields_ = [
        ("order", C.c_int32),
        ("n_grams", C.c_int64),
        ("words", C.c_void_p),
        ("probs", C.c_void_p),
        ("backoffs", C.c_void_p),
        ("bos_id", C.c_uint32),
        ("eos_word", C.c_int32),
        ("bos_backoff", C.c_double),
    ]


class LbStats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "frames", "beams_in", "beams_out", "ngram_calls", "ngram_probes", "boundary_beams",
        "history_nodes", "fallback_selects", "ngram_pairs_used")]


class LbLlmDesc(C.Structure):
    _fields_ = [
        ("n_layers", C.c_int32),
        ("n_heads", C.c_int32),
        ("n_kv_heads", C.c_int32),
        ("head_dim", C.c_int32),
        ("hidden", C.c_int32),
        ("vocab", C.c_int32),
        ("max_slots", C.c_int64),
        ("max_depth", C.c_int32),
        ("bos_token", C.c_int32),
        ("punct_tokens", C.c_int32 * 3),
        ("surface_tokens", C.c_void_p),
        ("surface_tokens_first", C.c_void_p),
        ("n_surfaces", C.c_int32),
        ("surface_token_off", C.c_void_p),
        ("surface_token_off_first", C.c_void_p),
        ("embedding", C.c_void_p),
        ("head_f32", C.c_void_p),
        ("precision", C.c_int32),
    ]


_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64
_D = C.c_double
_SIGS = {
    "lb_last_error": (C.c_char_p, []),
    "lb_device_count": (C.c_int, [_P]),
    "lb_model_create": (C.c_int, [C.POINTER(LbTableDesc), C.POINTER(LbNgramDesc), _I32, _P]),
    "lb_model_destroy": (C.c_int, [_P]),
    "lb_model_footprint": (C.c_int, [_P, _P]),
    "lb_model_lex_contiguous": (C.c_int, [_P, _P]),
    "lb_batch_create": (C.c_int, [_P, C.POINTER(LbConfig), _I32, _I32, _P, _P]),
    "lb_batch_destroy": (C.c_int, [_P]),
    "lb_batch_layout": (C.c_int, [_P, _P, _P, _P]),
    "lb_batch_set_logits": (C.c_int, [_P, _I32, _P, _P, _I32]),
    "lb_batch_set_logprobs": (C.c_int, [_P, _I32, _P, _P, _I32]),
    "lb_batch_get_logprobs": (C.c_int, [_P, _P]),
    "lb_batch_reset": (C.c_int, [_P]),
    "lb_batch_run": (C.c_int, [_P, _I32, _I32, _I32, _D]),
    "lb_batch_close": (C.c_int, [_P]),
    "lb_batch_device_ngram_fusion": (C.c_int, [_P, _I32, _D, _I32]),
    "lb_batch_gather_entries": (C.c_int, [_P, _P, _P]),
    "lb_batch_copy_entries": (C.c_int, [_P, _P, _P, _P, _P, _P, _P]),
    "lb_batch_apply_scores": (C.c_int, [_P, _P, _P, _P, _I32, _I32]),
    "lb_batch_status": (C.c_int, [_P, _P, _P]),
    "lb_batch_stats": (C.c_int, [_P, C.POINTER(LbStats)]),
    "lb_batch_clear_stats": (C.c_int, [_P]),
    "lb_batch_dump_beams": (C.c_int, [_P, _I32, _P, _P, _P, _P, _P, _P]),
    "lb_batch_enable_dump": (C.c_int, [_P, _I32]),
    "lb_batch_enable_phase_timing": (C.c_int, [_P, _I32]),
    "lb_batch_phase_cycles": (C.c_int, [_P, _P]),
    "lb_batch_dump_frame": (C.c_int, [_P, _I32, _I32, _P, _P, _P, _P, _P, _P]),
    "lb_batch_results_size": (C.c_int, [_P, _P, _P]),
    "lb_batch_results": (C.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "lb_batch_results_view": (C.c_int, [_P, _P]),
    "lb_batch_mark_begin": (C.c_int, [_P]),
    "lb_batch_mark_end": (C.c_int, [_P, _P, _P]),
    "lb_batch_sync": (C.c_int, [_P]),
    "lb_batch_after": (C.c_int, [_P, _P]),
    "lb_stream_create": (C.c_int, [_I32, _P]),
    "lb_stream_destroy": (C.c_int, [_P]),
    "lb_host_alloc": (C.c_int, [_I64, _P]),
    "lb_host_free": (C.c_int, [_P]),
    "lb_log_softmax_host": (C.c_int, [_P, _I64, _I32, _D, _P, _I32]),
    "lb_model_score_words": (C.c_int, [_P, _I32, _P, _P, _P, _P, _P, _P]),
    "lb_llm_create": (C.c_int, [_P, C.POINTER(LbLlmDesc), _P]),
    "lb_llm_destroy": (C.c_int, [_P]),
    "lb_llm_footprint": (C.c_int, [_P, _P]),
    "lb_llm_reset": (C.c_int, [_P]),
    "lb_llm_plan": (C.c_int, [_P, _I32, _I32, _P, _P]),
    "lb_llm_wave_rows": (C.c_int, [_P, _I32, _I64, _I32, _P, _P, _P, _P]),
    "lb_llm_finish": (C.c_int, [_P, _I32, _I32]),
    "lb_llm_plan_async": (C.c_int, [_P, _I32, _I32, _I32]),
    "lb_llm_wave_rows_async": (C.c_int, [_P, _I32, _P, _P, _P, _P]),
    "lb_llm_check": (C.c_int, [_P]),
    "lb_llm_reset_stats": (C.c_int, [_P]),
    "lb_llm_reset_device": (C.c_int, [_P]),
    "lb_launch_count": (C.c_int, [_P]),
    "lb_llm_rmsnorm": (C.c_int, [_P, _P, _P, _P, C.c_float, _I32, _P, _P]),
    "lb_llm_rope_kv": (C.c_int, [_P, _I32, _P, _I32, _P, _P, _P, _P, _P]),
    "lb_llm_layernorm": (C.c_int, [_P, _P, _P, _P, _P, C.c_float, _I32, _P, _P]),
    "lb_llm_gelu": (C.c_int, [_P, _P, _P, _I32, _I32, _P]),
    "lb_llm_attention": (C.c_int, [_P, _I32, _P, _I32, _P, _P, _P]),
    "lb_llm_swiglu": (C.c_int, [_P, _P, _I32, _I32, _P]),
    "lb_llm_lse": (C.c_int, [_P, _P, _I32, _I64, _P]),
    "lb_llm_lmhead_lse": (C.c_int, [_P, _P, _I32, _I64, _I32, _P, _I64, _I32, _P, _P]),
    "lb_llm_gateup_swiglu": (C.c_int, [_P, _P, _I32, _I64, _I32, _P, _I64, _I32, _P]),
    "lb_llm_stats": (C.c_int, [_P, _P]),
    "lb_llm_export": (C.c_int, [_P, _I64, _P, _P, _P, _P, _P, _P, _P]),
}

LLM_MAX_WAVES = 512

_lib = None


def exported_symbols() -> list[str]:
    return list(_SIGS)


def lib(require_device: bool = True):
    """The loaded library (raises DeviceError when it or a CUDA device is unavailable)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise DeviceError(
                f"{LIB_PATH.name} is not built; run __graft_entry__.build() (nvcc, sm_100a)")
        handle = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    if require_device:
        n = C.c_int32(0)
        if _lib.lb_device_count(C.byref(n)) != 0 or n.value < 1:
            raise DeviceError("no CUDA device visible: the LightBeam B200 decoder has no CPU path")
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        raise DeviceError(f"lightbeam_b200: {lib(False).lb_last_error().decode()} (rc={rc})")


def ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class PinnedArray(np.ndarray):
    """numpy view of page-locked host memory; freed when the last view goes away."""

    def __array_finalize__(self, obj):
        self._owner = getattr(obj, "_owner", None)


class _Pinned:
    def __init__(self, nbytes: int):
        p = C.c_void_p()
        check(lib().lb_host_alloc(nbytes, C.byref(p)))
        self.ptr = p

    def __del__(self):
        try:
            if self.ptr:
                lib(False).lb_host_free(self.ptr)
        except Exception:
            pass


def pinned_empty(shape, dtype=np.float32) -> np.ndarray:
    """Page-locked host array (fast, asynchronous H2D input staging for decode_batch_raw)."""
    dt = np.dtype(dtype)
    n = int(np.prod(shape)) * dt.itemsize
    owner = _Pinned(n)
    buf = (C.c_char * max(n, 1)).from_address(owner.ptr.value)
    arr = np.frombuffer(buf, dtype=dt, count=int(np.prod(shape))).reshape(shape).view(PinnedArray)
    arr._owner = owner
    return arr


def log_softmax_host(frames: np.ndarray, alpha: float, device: int = 0) -> np.ndarray:
    x = np.ascontiguousarray(frames, dtype=np.float32)
    out = np.empty(x.shape, dtype=np.float64)
    if x.size:
        check(lib().lb_log_softmax_host(ptr(x), x.shape[0], x.shape[1], alpha, ptr(out), device))
    return out
