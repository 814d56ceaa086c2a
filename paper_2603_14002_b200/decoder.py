"""Drop-in decode API over the CUDA beam-search kernels.

`decode(d, config, tt, lm, scorer, final_llm_only=False)` has the signature, arguments,
return type and error behaviour of the reference `lightbeam.decoder.decode`
(`pkg/src/lightbeam/decoder.py:408-460`): a `LogProbMatrix` (or fp64 `(T, V)` array) in, a
`DecodeResult` out, `DataValueError` on an empty matrix, `EmptyBeamError` when the beam dies,
`ScorerError` propagated from the scorer.  It accepts the reference's own `TransitionTable`,
`LmSession`/`NGramModel`, `DecodeConfig` and scorer objects as well as ours.

`decode_batch` / `decode_batch_raw` run many utterances at once -- one CTA per utterance --
which is how the GPU is meant to be fed.  Flow per batch:

    frames kernel over [0, e1]  -> fusion event e1 -> frames (e1, e2] -> ... -> closure
    -> final fusion -> ranking / n-best (host assembly in the C library)

Fusion events (`t > 0 and t % r == 0`, `decoder.py:428`) with a host scorer gather the word
histories on the device, send the unique texts through the scorer protocol, and apply the
scores with a device kernel.  With a `DeviceNgramScorer` the events happen inside the frames
kernel and the whole utterance is one launch plus closure and final fusion.  With a
`LlamaScorer` (llm.py) the events stay on the device: the word histories are mapped into the
LLM's prefix-trie KV cache, only new trie nodes run through the transformer, and the fusion
kernel reads the scores from the cache.
"""

from __future__ import annotations

import ctypes as C
import gc
import os
import threading
import time
import weakref
from dataclasses import dataclass

import numpy as np

from . import _native as N
from . import images
from .config import coerce_config
from .errors import DataValueError, DeviceError, EmptyBeamError, ShapeError
from .scorer import score_eos, score_texts

PUNCT_CODE = {".": 1, "?": 2, "!": 3}
PUNCT_CHAR = {0: "", 1: ".", 2: "?", 3: "!"}
_STATUS_MSG = {
    1: "all candidates pruned at frame {t}",
    2: "all hypotheses pruned at frame {t}",
    3: "no hypothesis survived end-of-utterance closure",
}


def _reference_result_type():
    """The reference's own `DecodeResult` (decoder.py:86-93) when `lightbeam` is loaded next to
    this package (errors.REFERENCE_ERRORS), so results are instances of the caller's type."""
    from .errors import REFERENCE_ERRORS

    if REFERENCE_ERRORS is None:
        return None
    try:
        from lightbeam.decoder import DecodeResult as ref
    except Exception:
        return None
    return ref


@dataclass
class DecodeResult:
    text: str
    score: float
    nbest: list
    frame_count: int
    wall_time_s: float
    llm_events: int


DecodeResult = _reference_result_type() or DecodeResult


class DeviceModel:
    """Device images of one (TransitionTable, NGramModel) pair, resident on one GPU."""

    MAX_CACHED_BATCHES = 2

    def __init__(self, tt, model, device: int = 0, image_path=None):
        """Compile the images from (tt, model), or -- with `image_path` -- load them from that
        file when it exists (skipping the compile) and write them there when it does not."""
        import os

        lib = N.lib()
        t0 = time.perf_counter()
        if image_path is not None and os.path.exists(image_path):
            tab, ng, bos_bo = images.load_images(image_path)
            self.image_source = "loaded"
        else:
            ng = images.compile_ngram(model)
            tab = images.compile_table(tt, model, ng)
            bos_bo = float(model.backoffs.get(("<s>",), 0.0))
            self.image_source = "compiled"
            if image_path is not None:
                tmp = f"{image_path}.{os.getpid()}.tmp"
                images.save_images(tmp, tab, ng, bos_bo)
                os.replace(tmp, image_path)  # atomic: concurrent ranks never read a partial file
        self.image_s = time.perf_counter() - t0
        self.ngram_image, self.table_image = ng, tab
        self.surfaces = tab.surfaces
        self.whitespace_free = tab.whitespace_free
        self.vocab_size = tab.table.shape[1]
        self.blank_id, self.space_id = tab.blank_id, tab.space_id
        self.device = device
        soff = tab.surface_off.astype(np.int64)
        td = N.LbTableDesc(
            N.ptr(tab.table), tab.table.shape[0], tab.table.shape[1], tab.sink, tab.blank_id,
            tab.space_id, N.ptr(tab.comp_off), N.ptr(tab.comp_surface), N.ptr(tab.comp_lmword),
            len(tab.comp_surface), tab.surface_blob, N.ptr(soff), len(tab.surfaces))
        nd = N.LbNgramDesc(ng.order, len(ng.probs), N.ptr(ng.words), N.ptr(ng.probs),
                           N.ptr(ng.backoffs), ng.bos_id, ng.eos_eff, bos_bo)
        handle = C.c_void_p()
        N.check(lib.lb_model_create(C.byref(td), C.byref(nd), device, C.byref(handle)))
        self.handle = handle
        # per host thread: batch handles are not thread-safe (SURVEY §8b threading row), so each
        # thread gets its own LRU of batches and its own pipeline pair
        self._per_thread: dict = {}
        self._lock = threading.Lock()

    def _mine(self) -> dict:
        tid = threading.get_ident()
        with self._lock:
            mine = self._per_thread.get(tid)
            if mine is None:
                # a new thread: first release the batches of threads that have exited
                alive = {t.ident for t in threading.enumerate()}
                for dead in [k for k in self._per_thread if k not in alive]:
                    self._destroy_batches(self._per_thread.pop(dead))
                mine = self._per_thread[tid] = {"lru": {}, "pipe": {}}
            return mine

    @staticmethod
    def _destroy_batches(per: dict):
        for b in list(per["lru"].values()) + [x[1] for x in per["pipe"].values()]:
            b.destroy()
        per["lru"].clear()
        per["pipe"].clear()

    def release(self):
        """Free every device batch (all threads) and the device images; idempotent."""
        with self._lock:
            per_all, self._per_thread = list(self._per_thread.values()), {}
        for per in per_all:
            self._destroy_batches(per)
        if getattr(self, "handle", None):
            N.lib(False).lb_model_destroy(self.handle)
            self.handle = None

    @property
    def lex_contiguous(self) -> bool:
        """Whether the frame kernel derives lexicon successors arithmetically (breadth-first
        trie) or looks them up in the compact image's successor list."""
        out = C.c_int32()
        N.check(N.lib().lb_model_lex_contiguous(self.handle, C.byref(out)))
        return bool(out.value)

    def footprint(self) -> int:
        out = C.c_int64()
        N.check(N.lib().lb_model_footprint(self.handle, C.byref(out)))
        return out.value

    def batch(self, cfg, n_trials: int, n_frames: int, own_stream: bool | None = None) -> "DeviceBatch":
        """A cached DeviceBatch for this config.  `own_stream`: the batch runs on its own CUDA
        stream (needed to capture whole decodes as CUDA graphs, LLM graph mode) instead of the
        legacy default stream; None = whichever batch the last decode of this config used."""
        base = tuple(getattr(cfg, f) for f in (
            "acoustic_scale", "beam_prune_threshold", "homophone_prune_threshold",
            "token_insertion_bonus", "word_boundary_bonus", "ngram_weight", "llm_weight",
            "beam_size", "ortho_beams", "llm_rescore_interval", "llm_chunk_size"))
        lru = self._mine()["lru"]
        if own_stream is None:
            own_stream = next((k[-1] for k in reversed(list(lru)) if k[:-1] == base), False)
        key = base + (own_stream,)
        got = lru.pop(key, None)
        if got is None or got.max_trials < n_trials or got.max_frames < n_frames:
            if got is not None:
                got.destroy()
            while len(lru) >= self.MAX_CACHED_BATCHES:  # evict the least recently used
                old = lru.pop(next(iter(lru)))
                old.destroy()
            stream = None
            if own_stream:
                import torch

                stream = torch.cuda.Stream(device=self.device)
            got = DeviceBatch(self, cfg, max(n_trials, 1), max(n_frames, 1),
                              stream=stream.cuda_stream if stream is not None else None)
            got._torch_stream = stream  # keep the stream alive with the batch
        lru[key] = got  # most recently used last
        return got

    def pipeline_batch(self, cfg, slot: int, n_trials: int, n_frames: int) -> "DeviceBatch":
        """One of the two DeviceBatch objects `decode_stream_raw` alternates between, each on its
        own CUDA stream."""
        key = (slot, cfg)
        pipe = self._mine()["pipe"]
        got = pipe.get(slot)
        if got is not None and (got[0] != key or got[1].max_trials < n_trials
                                or got[1].max_frames < n_frames):
            got[1].destroy()
            got = None
        if got is None:
            st = C.c_void_p()
            N.check(N.lib().lb_stream_create(self.device, C.byref(st)))
            b = DeviceBatch(self, cfg, max(n_trials, 1), max(n_frames, 1), stream=st.value)
            b._own_stream = st
            got = (key, b)
            pipe[slot] = got
        return got[1]

    def score_words(self, hist: list, words: list):
        """Device score_word for (history word ids, LM word id) pairs -- parity helper."""
        n = len(words)
        h = np.zeros((n, 3), dtype=np.uint32)
        hl = np.zeros(n, dtype=np.int32)
        for i, hh in enumerate(hist):
            h[i, : len(hh)] = hh
            hl[i] = len(hh)
        w = np.asarray(words, dtype=np.int32)
        inc = np.empty(n, dtype=np.float64)
        succ = np.empty((n, 3), dtype=np.uint32)
        sl = np.empty(n, dtype=np.int32)
        N.check(N.lib().lb_model_score_words(self.handle, n, N.ptr(h), N.ptr(hl), N.ptr(w),
                                             N.ptr(inc), N.ptr(succ), N.ptr(sl)))
        return inc, [tuple(int(x) for x in succ[i, : sl[i]]) for i in range(n)]

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


_MODELS: dict = {}
_MODELS_LOCK = threading.Lock()


def _drop_model(key):
    with _MODELS_LOCK:
        hit = _MODELS.pop(key, None)
    if hit is not None:
        hit[2].release()


_IMAGE_PATHS: dict = {}


def register_image_path(tt, lm, path) -> None:
    """Persist / reuse the device images of (tt, lm-model) at `path` (an .npz written by
    images.save_images): the next DeviceModel built for these components loads the file when
    it exists instead of compiling, and writes it when it does not.  `build_engine(...,
    image_cache=dir)` registers a path keyed by the component files' sha256."""
    model = getattr(lm, "model", lm)
    key = (id(tt), id(model))
    if path is None:  # unregister
        _IMAGE_PATHS.pop(key, None)
        return
    _IMAGE_PATHS[key] = str(path)
    weakref.finalize(tt, _IMAGE_PATHS.pop, key, None)


def device_model(tt, lm, device: int = 0) -> DeviceModel:
    """Cached DeviceModel for (tt, lm-model, device).  The cache holds its components only
    weakly: when the table or the n-gram model is collected, the entry is dropped and its
    device memory freed (`weakref.finalize`); `release_device_model` frees it explicitly."""
    model = getattr(lm, "model", lm)
    key = (id(tt), id(model), device)
    with _MODELS_LOCK:
        hit = _MODELS.get(key)
    if hit is not None:
        wt, wm, dm = hit
        if wt() is tt and wm() is model and dm.handle:
            return dm
        _drop_model(key)  # an id() reused by a new object, or a released entry
    dm = DeviceModel(tt, model, device, _IMAGE_PATHS.get((id(tt), id(model))))
    with _MODELS_LOCK:
        _MODELS[key] = (weakref.ref(tt), weakref.ref(model), dm)
    weakref.finalize(tt, _drop_model, key)
    weakref.finalize(model, _drop_model, key)
    return dm


def release_device_model(tt, lm, device: int = 0) -> None:
    """Free the cached device images and batches of (tt, lm-model, device), if any."""
    model = getattr(lm, "model", lm)
    _drop_model((id(tt), id(model), device))


class DeviceBatch:
    """One lb_batch: device beam state for up to `max_trials` utterances of `max_frames`."""

    def __init__(self, dm: DeviceModel, cfg, max_trials: int, max_frames: int, stream=None):
        self.dm = dm
        self.cfg = cfg
        self.max_trials, self.max_frames = max_trials, max_frames
        c = N.LbConfig(cfg.acoustic_scale, cfg.beam_prune_threshold, cfg.homophone_prune_threshold,
                       cfg.token_insertion_bonus, cfg.word_boundary_bonus, cfg.ngram_weight,
                       cfg.llm_weight, cfg.beam_size, cfg.ortho_beams, cfg.llm_rescore_interval,
                       cfg.llm_chunk_size)
        h = C.c_void_p()
        N.check(N.lib().lb_batch_create(dm.handle, C.byref(c), max_trials, max_frames,
                                        C.c_void_p(stream or 0), C.byref(h)))
        self.h = h
        self.stream_ptr = int(stream or 0)  # the CUDA stream every kernel of this batch runs on
        self.graph_launches = 0  # library kernels run inside CUDA-graph replays (LLM graph mode)
        self.n = 0
        self.frames = np.zeros(0, dtype=np.int32)

    def layout(self) -> dict:
        sm, gs, nt = C.c_int64(), C.c_int64(), C.c_int32()
        N.check(N.lib().lb_batch_layout(self.h, C.byref(sm), C.byref(gs), C.byref(nt)))
        return {"smem_bytes": sm.value, "gscratch_bytes": gs.value, "threads": nt.value}

    def destroy(self):
        sess = getattr(self, "_llm_session", None)
        if sess is not None:
            sess.destroy()
            self._llm_session = None
        if getattr(self, "h", None):
            N.lib(False).lb_batch_destroy(self.h)
            self.h = None
        st = getattr(self, "_own_stream", None)
        if st is not None and st.value:
            N.lib(False).lb_stream_destroy(st)
            self._own_stream = None

    # ---- inputs
    def _frames(self, frames) -> np.ndarray:
        fr = np.ascontiguousarray(frames, dtype=np.int32)
        if fr.size and (fr.min() < 0 or fr.max() > self.max_frames):
            raise ShapeError("frame counts exceed the batch capacity")
        self.n = len(fr)
        self.frames = fr
        return fr

    def _after_torch(self):
        """Inputs produced by torch on its current stream: order this batch's stream after it."""
        if self.stream_ptr and getattr(self, "_torch_stream", None) is not None:
            import torch

            self._torch_stream.wait_stream(torch.cuda.current_stream(self.dm.device))

    def load_logprobs(self, d: np.ndarray, frames, on_device_ptr: int | None = None):
        fr = self._frames(frames)
        if on_device_ptr is not None:
            self._after_torch()
            N.check(N.lib().lb_batch_set_logprobs(self.h, len(fr), C.c_void_p(on_device_ptr),
                                                  N.ptr(fr), 1))
            return
        x = np.ascontiguousarray(d, dtype=np.float64)
        if x.shape[1] != self.max_frames:
            pad = np.zeros((x.shape[0], self.max_frames, x.shape[2]), dtype=np.float64)
            pad[:, : x.shape[1]] = x
            x = pad
        N.check(N.lib().lb_batch_set_logprobs(self.h, len(fr), N.ptr(x), N.ptr(fr), 0))

    def load_logits(self, x: np.ndarray | None, frames, on_device_ptr: int | None = None):
        fr = self._frames(frames)
        if on_device_ptr is not None:
            self._after_torch()
            N.check(N.lib().lb_batch_set_logits(self.h, len(fr), C.c_void_p(on_device_ptr),
                                                N.ptr(fr), 1))
            return
        a = np.ascontiguousarray(x, dtype=np.float32)
        if a.shape[1] != self.max_frames:
            pad = np.zeros((a.shape[0], self.max_frames, a.shape[2]), dtype=np.float32)
            pad[:, : a.shape[1]] = a
            a = pad
        self._hold = a  # the copy is stream-ordered; keep the host buffer alive
        N.check(N.lib().lb_batch_set_logits(self.h, len(fr), N.ptr(a), N.ptr(fr), 0))

    def get_logprobs(self) -> np.ndarray:
        out = np.empty((self.n, self.max_frames, self.dm.vocab_size), dtype=np.float64)
        N.check(N.lib().lb_batch_get_logprobs(self.h, N.ptr(out)))
        return out

    # ---- search steps
    def reset(self):
        N.check(N.lib().lb_batch_reset(self.h))

    def run(self, t0: int, t1: int, fusion_mode: int = 0, scale: float = 0.0):
        N.check(N.lib().lb_batch_run(self.h, t0, t1, fusion_mode, scale))

    def close(self):
        N.check(N.lib().lb_batch_close(self.h))

    def device_fusion(self, final: bool, scale: float, min_frames: int = 0):
        N.check(N.lib().lb_batch_device_ngram_fusion(self.h, int(final), scale, min_frames))

    def gather(self):
        ne, nw = C.c_int64(), C.c_int64()
        lib = N.lib()
        N.check(lib.lb_batch_gather_entries(self.h, C.byref(ne), C.byref(nw)))
        n_e, n_w = ne.value, nw.value
        et = np.empty(n_e, dtype=np.int32)
        eb = np.empty(n_e, dtype=np.int32)
        wo = np.empty(n_e + 1, dtype=np.int64)
        words = np.empty(max(n_w, 1), dtype=np.int32)
        tot = np.empty(n_e, dtype=np.float64)
        pun = np.empty(n_e, dtype=np.int32)
        N.check(lib.lb_batch_copy_entries(self.h, N.ptr(et), N.ptr(eb), N.ptr(wo), N.ptr(words),
                                          N.ptr(tot), N.ptr(pun)))
        return et, eb, wo, words, tot, pun

    def apply_scores(self, scores, puncts, has_text, final: bool, min_frames: int):
        s = np.ascontiguousarray(scores, dtype=np.float64)
        p = np.ascontiguousarray(puncts, dtype=np.int32)
        h = np.ascontiguousarray(has_text, dtype=np.uint8)
        N.check(N.lib().lb_batch_apply_scores(self.h, N.ptr(s), N.ptr(p), N.ptr(h), int(final),
                                              min_frames))

    def status(self):
        st = np.empty(self.n, dtype=np.int32)
        ff = np.empty(self.n, dtype=np.int32)
        N.check(N.lib().lb_batch_status(self.h, N.ptr(st), N.ptr(ff)))
        return st, ff

    def stats(self) -> dict:
        s = N.LbStats()
        N.check(N.lib().lb_batch_stats(self.h, C.byref(s)))
        return {name: int(getattr(s, name)) for name, _ in N.LbStats._fields_}

    def clear_stats(self):
        N.check(N.lib().lb_batch_clear_stats(self.h))

    # frames_small_kernel (k <= 64) TIMING build: per barrier event, the critical (last-arriving)
    # warp's work since the previous release and the barrier's own release latency
    PHASES = ("A_work", "S1_sync", "scan_work", "hcum_sync", "collect_work", "S2_sync",
              "rank_work", "S3_sync", "F_work", "S4_sync", "recomb_work", "S5_sync",
              "keep_work", "S6_sync", "scatter_work", "frame_sync", "spec_overflow_permille",
              "ngram_warps_to_S3", "compute_to_S3", "ngover_work", "ng_scan", "ng_table",
              "ng_score", "ng_rounds_permille", "F1_work", "S3b_wait")

    def enable_phase_timing(self, on: bool = True):
        N.check(N.lib().lb_batch_enable_phase_timing(self.h, int(on)))

    def phase_cycles(self) -> dict:
        out = np.zeros(len(self.PHASES), dtype=np.uint64)
        N.check(N.lib().lb_batch_phase_cycles(self.h, N.ptr(out)))
        return {name: int(v) for name, v in zip(self.PHASES, out)}

    def enable_dump(self, on: bool = True):
        N.check(N.lib().lb_batch_enable_dump(self.h, int(on)))

    def dump_frame(self, trial: int, t: int):
        k = C.c_int32()
        K = self.cfg.beam_size
        sc = np.empty(K, dtype=np.float64)
        a = np.empty(K, dtype=np.uint64)
        b = np.empty(K, dtype=np.uint64)
        p = np.empty(K, dtype=np.int32)
        la = np.empty(K, dtype=np.int32)
        N.check(N.lib().lb_batch_dump_frame(self.h, trial, t, C.byref(k), N.ptr(sc), N.ptr(a),
                                            N.ptr(b), N.ptr(p), N.ptr(la)))
        n = k.value
        return [(int(a[i]), int(b[i]), int(p[i]), int(la[i]), float(sc[i])) for i in range(max(n, 0))]

    def beams(self, trial: int):
        k = C.c_int32()
        K = self.cfg.beam_size
        sc = np.empty(K, dtype=np.float64)
        a = np.empty(K, dtype=np.uint64)
        b = np.empty(K, dtype=np.uint64)
        p = np.empty(K, dtype=np.int32)
        la = np.empty(K, dtype=np.int32)
        N.check(N.lib().lb_batch_dump_beams(self.h, trial, C.byref(k), N.ptr(sc), N.ptr(a),
                                            N.ptr(b), N.ptr(p), N.ptr(la)))
        return [(int(a[i]), int(b[i]), int(p[i]), int(la[i]), float(sc[i])) for i in range(k.value)]

    def mark_begin(self):
        N.check(N.lib().lb_batch_mark_begin(self.h))
        self._graph_mark = self.graph_launches

    def mark_end(self):
        """(device ms since mark_begin, kernels launched since: by the library directly plus
        the library kernels inside CUDA-graph replays of whole decodes)."""
        ms, launches = C.c_float(), C.c_int64()
        N.check(N.lib().lb_batch_mark_end(self.h, C.byref(ms), C.byref(launches)))
        return ms.value, launches.value + self.graph_launches - getattr(self, "_graph_mark", 0)

    def sync(self):
        N.check(N.lib().lb_batch_sync(self.h))

    def after(self, prev: "DeviceBatch"):
        """Order this batch's later launches after everything already enqueued on `prev`."""
        N.check(N.lib().lb_batch_after(self.h, prev.h))

    def results(self):
        """[(text, score, nbest)] per trial (None for failed trials).  The library ranks and
        dedupes on the host (lb_batch_results_size); the CPython binding `_lb_results` builds the
        Python objects straight from the library's buffers (lb_batch_results_view)."""
        lib = N.lib()
        nbytes, ntot = C.c_int64(), C.c_int64()
        N.check(lib.lb_batch_results_size(self.h, C.byref(nbytes), C.byref(ntot)))
        view = N.LbResultsView()
        N.check(lib.lb_batch_results_view(self.h, C.byref(view)))
        return N.pyresults().assemble(C.addressof(view))


def _host_fusion(batch: DeviceBatch, scorer, cfg, final: bool, min_frames: int):
    """apply_llm (decoder.py:329-372) with a host scorer: device gather -> protocol -> device."""
    et, eb, wo, words, _tot, _pun = batch.gather()
    surf = batch.dm.surfaces
    n_e = len(et)
    texts = [" ".join([surf[w] for w in words[wo[i]: wo[i + 1]]]) for i in range(n_e)]
    live = batch.frames[et] > min_frames if n_e else np.zeros(0, dtype=bool)
    uniq: list = []
    seen: set = set()
    for i in range(n_e):
        tx = texts[i]
        if live[i] and tx and tx not in seen:
            seen.add(tx)
            uniq.append(tx)
    scores = np.zeros(n_e, dtype=np.float64)
    puncts = np.zeros(n_e, dtype=np.int32)
    has = np.zeros(n_e, dtype=np.uint8)
    if final:
        lut = dict(zip(uniq, score_eos(scorer, uniq, cfg.llm_chunk_size)))
    else:
        lut = {t: ("", s) for t, s in zip(uniq, score_texts(scorer, uniq, cfg.llm_chunk_size))}
    for i in range(n_e):
        tx = texts[i]
        if live[i] and tx:
            p, s = lut[tx]
            scores[i] = s
            puncts[i] = PUNCT_CODE.get(p, 0)
            has[i] = 1
    batch.apply_scores(scores, puncts, has, final, min_frames)


def _graph_mode(scorer) -> bool:
    """The scorer's decodes run as CUDA-graph replays (device LLM in graph mode)."""
    return bool(getattr(getattr(scorer, "device_llm_scorer", None), "graphs", False))


def _uses_device_scorer(scorer, model, dm: DeviceModel) -> bool:
    return getattr(scorer, "device_ngram_model", None) is model and dm.whitespace_free


def run_search(batch: DeviceBatch, cfg, scorer, model, final_llm_only: bool):
    """Everything after the inputs are on the device: frames, events, closure, final fusion."""
    for _ in _search_steps(batch, cfg, scorer, model, final_llm_only):
        pass


def run_search_many(batches, cfg, scorer, model, final_llm_only: bool):
    """run_search over several device batches (each on its own CUDA stream, e.g. the
    `pipeline_batch` pair) interleaved event by event: while the host waits for one batch's
    fusion plan, the other batch's frames and LLM forward keep the GPU busy."""
    gens = [_search_steps(b, cfg, scorer, model, final_llm_only) for b in batches]
    while gens:
        for g in list(gens):
            try:
                next(g)
            except StopIteration:
                gens.remove(g)


def _search_steps(batch: DeviceBatch, cfg, scorer, model, final_llm_only: bool):
    """run_search as a generator: yields after the launches of each fusion event (the host
    synchronises only inside an event's planning step)."""
    frames = batch.frames
    t_max = int(frames.max()) if len(frames) else 0
    r = cfg.llm_rescore_interval
    batch.reset()
    if _uses_device_scorer(scorer, model, batch.dm):
        scale = scorer.scale
        batch.run(0, t_max, 0 if final_llm_only else 1, scale)
        batch.close()
        batch.device_fusion(True, scale, 0)
        return
    llm = getattr(scorer, "device_llm_scorer", None)
    if llm is not None and batch.dm.whitespace_free:
        sess = llm.session(batch)
        if getattr(llm, "graphs", False) and batch.stream_ptr:
            _graph_search(batch, cfg, sess, final_llm_only, t_max)
            yield
            return
        sess.reset()
        fuse = sess.event
    else:
        def fuse(final, min_frames):
            _host_fusion(batch, scorer, cfg, final=final, min_frames=min_frames)
    t = 0
    if not final_llm_only:
        for e in range(r, t_max, r):  # events after frames e = r, 2r, ... (< the longest T)
            batch.run(t, e + 1)
            fuse(False, e)
            t = e + 1
            yield
    batch.run(t, t_max)
    batch.close()
    fuse(True, 0)
    yield


def _event_frames(t_max: int, r: int, final_llm_only: bool) -> list:
    """Interval fusion events after frames e = r, 2r, ... < the longest T (decoder.py:428)."""
    return [] if final_llm_only else list(range(r, t_max, r))


def _graph_search(batch: DeviceBatch, cfg, sess, final_llm_only: bool, t_max: int):
    """The whole decode of a batch with a device LLM scorer as ONE CUDA-graph replay: frames
    intervals, every fusion event (planning, a forward over a fixed row capacity, fusion),
    closure and the final pass, with no host synchronisation between events.  The first decode
    of a shape runs eagerly (it also measures the largest event) and captures the graph for the
    next ones; a replay whose event outgrows the captured rows is detected on the device
    (lb_llm_check) and the batch is decoded again eagerly, then re-captured with more rows."""
    import torch

    from .errors import DeviceError

    events = _event_frames(t_max, cfg.llm_rescore_interval, final_llm_only)
    key = (batch.n, tuple(int(x) for x in batch.frames), cfg.llm_rescore_interval,
           bool(final_llm_only))
    ent = sess.graphs.get(key)
    stream = torch.cuda.ExternalStream(batch.stream_ptr, device=sess.scorer.weights.device)
    if ent is not None:
        N.check(N.lib().lb_llm_reset_stats(sess.h))  # host half of the captured reset
        sess.waves_log = []
        with torch.cuda.stream(stream):  # replay on the batch's stream (ordered, timed there)
            ent["graph"].replay()
        batch.graph_launches += ent["kernels"]
        try:
            sess.check()
            return
        except DeviceError:  # an event had more rows than captured: redo eagerly, re-capture
            sess.graphs.pop(key, None)
    # eager decode (the result of this call) -- also sizes the graph's row capacity
    batch.reset()
    sess.reset()
    t = 0
    for e in events:
        batch.run(t, e + 1)
        sess.event(False, e)
        t = e + 1
    batch.run(t, t_max)
    batch.close()
    sess.event(True, 0)
    rows = max([max(w) if w else 0 for w in sess.waves_log] + [1])
    R = 64
    while R < 2 * rows:
        R *= 2
    if R > sess.scorer.row_chunk:
        return  # too large to pad every event: stay eager
    ws = sess.graph_workspace(R)
    c0, c1 = C.c_uint64(), C.c_uint64()
    N.check(N.lib().lb_launch_count(C.byref(c0)))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        batch.reset()
        N.check(N.lib().lb_llm_reset_device(sess.h))  # the host statistics stay this decode's
        t = 0
        for e in events:
            batch.run(t, e + 1)
            sess.event_async(False, e, R, ws)
            t = e + 1
        batch.run(t, t_max)
        batch.close()
        sess.event_async(True, 0, R, ws)
    N.check(N.lib().lb_launch_count(C.byref(c1)))
    sess.graphs[key] = {"graph": g, "rows": R, "ws": ws, "kernels": int(c1.value - c0.value)}


def _collect(batch: DeviceBatch, cfg, final_llm_only: bool, wall: float):
    st, ff = batch.status()
    res = batch.results()
    gc_on = gc.isenabled()
    if gc_on:  # ~256 result objects over ~15k fresh n-best objects: no collection in between
        gc.disable()
    try:
        return _collect_items(batch, cfg, final_llm_only, wall, st, ff, res)
    finally:
        if gc_on:
            gc.enable()


def _collect_items(batch, cfg, final_llm_only, wall, st, ff, res):
    out = []
    for i in range(batch.n):
        if batch.frames[i] == 0:  # decoder.py:421-422 (per item, so one bad item keeps the batch)
            out.append(DataValueError("cannot decode an empty log-probability matrix"))
            continue
        if st[i] != 0:
            if st[i] == 4:
                out.append(DeviceError("device word-history arena exhausted"))
            else:
                out.append(EmptyBeamError(_STATUS_MSG[int(st[i])].format(t=int(ff[i]))))
            continue
        text, score, nbest = res[i]
        t_i = int(batch.frames[i])
        events = 0 if final_llm_only else (t_i - 1) // cfg.llm_rescore_interval
        out.append(DecodeResult(text, score, nbest, t_i, wall, events))
    return out


def _stack(mats, dtype):
    frames = np.array([m.shape[0] for m in mats], dtype=np.int32)
    v = mats[0].shape[1]
    out = np.zeros((len(mats), int(frames.max()) if len(mats) else 0, v), dtype=dtype)
    for i, m in enumerate(mats):
        out[i, : m.shape[0]] = m
    return out, frames


def _prepare(cfg, tt, lm, device):
    cfg = coerce_config(cfg)
    model = getattr(lm, "model", lm)
    return cfg, model, device_model(tt, model, device)


def decode_batch(ds, config, tt, lm, scorer, final_llm_only: bool = False, device: int = 0):
    """Decode many fp64 log-prob matrices (LogProbMatrix / (T, V) arrays, or (B, T, V) + lengths
    via `ds=(array, frames)`).  Returns a list with a DecodeResult or the exception per item."""
    cfg, model, dm = _prepare(config, tt, lm, device)
    if isinstance(ds, tuple):
        arr, frames = np.asarray(ds[0], dtype=np.float64), np.asarray(ds[1], dtype=np.int32)
    else:
        mats = [np.asarray(getattr(d, "frames", d), dtype=np.float64) for d in ds]
        arr, frames = _stack(mats, np.float64)
    if arr.ndim != 3 or arr.shape[2] != dm.vocab_size:
        raise ShapeError(f"log-prob width must equal the table vocabulary ({dm.vocab_size})")
    t0 = time.perf_counter()
    batch = dm.batch(cfg, arr.shape[0], max(arr.shape[1], 1), own_stream=_graph_mode(scorer))
    batch.load_logprobs(arr, frames)
    run_search(batch, cfg, scorer, model, final_llm_only)
    return _collect(batch, cfg, final_llm_only, time.perf_counter() - t0)


def decode_batch_raw(raws, config, tt, lm, scorer, final_llm_only: bool = False, device: int = 0):
    """Raw fp32 logits in (RawLogits list or `(array, frames)`): the log-softmax prologue runs
    on the device (kernel K1) and feeds the search directly."""
    cfg, model, dm = _prepare(config, tt, lm, device)
    if isinstance(raws, tuple):
        arr, frames = np.asarray(raws[0], dtype=np.float32), np.asarray(raws[1], dtype=np.int32)
    else:
        mats = [np.asarray(getattr(r, "frames", r), dtype=np.float32) for r in raws]
        arr, frames = _stack(mats, np.float32)
    if arr.ndim != 3 or arr.shape[2] != dm.vocab_size:
        raise ShapeError(f"logit width must equal the table vocabulary ({dm.vocab_size})")
    t0 = time.perf_counter()
    batch = dm.batch(cfg, arr.shape[0], max(arr.shape[1], 1), own_stream=_graph_mode(scorer))
    batch.load_logits(arr, frames)
    run_search(batch, cfg, scorer, model, final_llm_only)
    return _collect(batch, cfg, final_llm_only, time.perf_counter() - t0)


def _raw_array(raws):
    if isinstance(raws, tuple):
        return np.asarray(raws[0], dtype=np.float32), np.asarray(raws[1], dtype=np.int32)
    return _stack([np.asarray(getattr(r, "frames", r), dtype=np.float32) for r in raws], np.float32)


_SERIAL_SEARCH = os.environ.get("LB_STREAM_OVERLAP", "0") != "1"


def decode_stream_raw(batches, config, tt, lm, scorer, final_llm_only: bool = False,
                      device: int = 0):
    """Generator over many batches of raw logits (each a RawLogits list or `(array, frames)`):
    yields each batch's list of DecodeResult / exception, in order.  Two device batches on two
    CUDA streams alternate, so batch i+1's H2D copy and search run on the GPU while the host
    assembles batch i's transcripts and n-best lists (with pinned host inputs the launches are
    asynchronous; a batch's host array must stay unmodified until its results are yielded).
    Results are identical to `decode_batch_raw` per batch."""
    cfg, model, dm = _prepare(config, tt, lm, device)
    pending: list = []  # [batch, t0, search generator or None when its launches are all issued]
    slot = 0

    def advance(until):  # step every in-flight search (event by event) until `until` is issued
        while until[2] is not None:
            for item in pending:
                if item[2] is not None:
                    try:
                        next(item[2])
                    except StopIteration:
                        item[2] = None

    for raws in batches:
        arr, frames = _raw_array(raws)
        if arr.ndim != 3 or arr.shape[2] != dm.vocab_size:
            raise ShapeError(f"logit width must equal the table vocabulary ({dm.vocab_size})")
        batch = dm.pipeline_batch(cfg, slot, arr.shape[0], max(arr.shape[1], 1))
        t0 = time.perf_counter()
        batch.load_logits(arr, frames)
        if _SERIAL_SEARCH and pending and pending[-1][2] is None:
            # the previous batch's launches are all issued: this batch's H2D copy and prologue
            # overlap its search, the search kernels themselves run back to back (two
            # persistent searches sharing the SMs and the L2 took ~20% longer per batch)
            batch.after(pending[-1][0])
        item = [batch, t0, _search_steps(batch, cfg, scorer, model, final_llm_only)]
        pending.append(item)
        try:  # launch right away (up to its first fusion event): the GPU never waits on the host
            next(item[2])
        except StopIteration:
            item[2] = None
        slot ^= 1
        if len(pending) == 2:
            advance(pending[0])
            b, t, _ = pending.pop(0)
            yield _collect(b, cfg, final_llm_only, time.perf_counter() - t)
    while pending:
        advance(pending[0])
        b, t, _ = pending.pop(0)
        yield _collect(b, cfg, final_llm_only, time.perf_counter() - t)


def decode(d, config, tt, lm, scorer, final_llm_only: bool = False) -> DecodeResult:
    """Drop-in for `lightbeam.decoder.decode` (decoder.py:408-460)."""
    frames = np.asarray(getattr(d, "frames", d), dtype=np.float64)
    if frames.ndim != 2 or frames.shape[0] == 0:
        raise DataValueError("cannot decode an empty log-probability matrix")
    res = decode_batch([frames], config, tt, lm, scorer, final_llm_only)[0]
    if isinstance(res, Exception):
        raise res
    return res
