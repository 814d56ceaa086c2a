"""Host "compilers": reference components -> flat arrays for the device images.

Lexicon (`TransitionTable`, reference `lexicon.py:84-209`):
- `table` int32 [S, V] as is (prefix ids are part of the contract; row padding to a 16-byte
  pitch happens on upload inside `lb_model_create`);
- completion CSR over states: for each state, the *distinct surfaces* of the words ending
  there, in completion order (the dedupe `decoder.py:197-206` does per call), each with its
  surface id and the LM word the n-gram model will score it as (`ngram.py:225-230`: the
  surface itself if it is a listed unigram, else `<unk>` if present, else -1 = kill).

N-gram model (`NGramModel`, reference `ngram.py:33-46`): every listed gram (probs or
backoffs) becomes one 32-byte record `{u32 words[4], f64 prob, f64 backoff}`; words are
dense LM ids (0xFFFFFFFF pads short grams), `prob` is `PROB_ABSENT` for a gram that only
carries a back-off, `backoff` is 0.0 when absent (the `.get(h, 0.0)` of `ngram.py:195`).
`lb_model_create` inserts them into an open-addressing table on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import FormatError, ShapeError

MAX_ORDER = 4
WORD_PAD = 0xFFFFFFFF
PROB_ABSENT_BITS = 0x7FF8DEAD00000000  # a quiet NaN no parser produces
MAX_VOCAB = 64  # candidate masks are one u64 per parent


@dataclass
class TableImage:
    table: np.ndarray  # int32 [S, V]
    sink: int
    blank_id: int
    space_id: int
    comp_off: np.ndarray  # int32 [S+1]
    comp_surface: np.ndarray  # int32 [n]
    comp_lmword: np.ndarray  # int32 [n]
    surfaces: list  # surface id -> str
    surface_blob: bytes  # utf-8 concatenation
    surface_off: np.ndarray  # int64 [n_surfaces+1]
    whitespace_free: bool  # all surfaces are split()-stable single tokens


@dataclass
class NgramImage:
    order: int
    words: np.ndarray  # uint32 [N, 4]
    probs: np.ndarray  # float64 [N]
    backoffs: np.ndarray  # float64 [N]
    word_id: dict  # str -> int
    bos_id: int
    eos_eff: int  # LM id `</s>` is scored as (or -1)
    unk_id: int  # -1 if absent


def compile_ngram(model) -> NgramImage:
    order = int(model.order)
    keys = set(model.probs)
    keys.update(model.backoffs)
    vocab = set()
    for g in keys:
        if len(g) > MAX_ORDER:
            raise FormatError(f"n-gram order {len(g)} > supported maximum {MAX_ORDER}")
        vocab.update(g)
    vocab.update(("<s>", "</s>", "<unk>"))
    names = sorted(vocab)
    wid = {w: i for i, w in enumerate(names)}
    n = len(keys)
    words = np.full((n, MAX_ORDER), WORD_PAD, dtype=np.uint32)
    probs = np.empty(n, dtype=np.float64)
    bos = np.zeros(n, dtype=np.float64)
    absent = np.array([PROB_ABSENT_BITS], dtype=np.uint64).view(np.float64)[0]
    get_p, get_b = model.probs.get, model.backoffs.get
    for row, g in enumerate(keys):
        words[row, : len(g)] = [wid[w] for w in g]
        p = get_p(g)
        probs[row] = absent if p is None else p
        bos[row] = get_b(g, 0.0)
    unk = wid["<unk>"] if model.unk_present else -1
    eos_eff = wid["</s>"] if ("</s>",) in model.probs else unk
    return NgramImage(order, words, probs, bos, wid, wid["<s>"], eos_eff, unk)


def lm_word_for(surface: str, model, img: NgramImage) -> int:
    if (surface,) in model.probs:
        return img.word_id[surface]
    return img.unk_id


def compile_table(tt, model, img: NgramImage) -> TableImage:
    table = np.ascontiguousarray(tt.table, dtype=np.int32)
    n_states, v = table.shape
    if v > MAX_VOCAB:
        raise ShapeError(f"vocabulary of {v} tokens exceeds the device limit of {MAX_VOCAB}")
    surf_id: dict = {}
    surfaces: list = []
    for e in tt.entries:
        if e.surface not in surf_id:
            surf_id[e.surface] = len(surfaces)
            surfaces.append(e.surface)
    counts = np.zeros(n_states + 1, dtype=np.int64)
    items_s: list = []
    items_w: list = []
    for state in tt.completion_states():
        seen: list = []
        for eid in tt.completions_at(state):
            s = tt.entries[eid].surface
            if s not in seen:
                seen.append(s)
        counts[state + 1] = len(seen)
        items_s.extend(surf_id[s] for s in seen)
        items_w.extend(lm_word_for(s, model, img) for s in seen)
    off = np.cumsum(counts).astype(np.int32)
    # the CSR must be filled in state order: completion_states() is sorted
    blobs = [s.encode("utf-8") for s in surfaces]
    soff = np.zeros(len(blobs) + 1, dtype=np.int64)
    soff[1:] = np.cumsum([len(b) for b in blobs])
    ws_free = all(s and s.split() == [s] for s in surfaces)
    return TableImage(
        table=table,
        sink=int(tt.sink),
        blank_id=int(tt.blank_id),
        space_id=int(tt.space_id),
        comp_off=off,
        comp_surface=np.asarray(items_s, dtype=np.int32),
        comp_lmword=np.asarray(items_w, dtype=np.int32),
        surfaces=surfaces,
        surface_blob=b"".join(blobs),
        surface_off=soff,
        whitespace_free=ws_free,
    )


# ------------------------------------------------------------------ persisted images
IMAGE_FORMAT = 1


def save_images(path, tab: TableImage, ng: NgramImage, bos_backoff: float) -> None:
    """Write both compiled images to one uncompressed .npz (plain arrays + a small header), so
    a later process uploads them without re-parsing or re-compiling the components.  The
    reference builders this replaces run per process: `load_arpa` (ngram.py:90-174, 2.4 s for
    1M n-grams) and `build_transition_table` (lexicon.py:149-209), plus compile_ngram /
    compile_table here."""
    import json

    names = [None] * len(ng.word_id)
    for w, i in ng.word_id.items():
        names[i] = w
    header = {"format": IMAGE_FORMAT, "sink": tab.sink, "blank_id": tab.blank_id,
              "space_id": tab.space_id, "whitespace_free": tab.whitespace_free,
              "order": ng.order, "bos_id": ng.bos_id, "eos_eff": ng.eos_eff, "unk_id": ng.unk_id,
              "bos_backoff": bos_backoff}
    lm_blob = "\n".join(names).encode("utf-8")
    with open(path, "wb") as fh:
        np.savez(fh, header=np.frombuffer(json.dumps(header).encode(), dtype=np.uint8),
                 table=tab.table, comp_off=tab.comp_off, comp_surface=tab.comp_surface,
                 comp_lmword=tab.comp_lmword,
                 surface_blob=np.frombuffer(tab.surface_blob, dtype=np.uint8),
                 surface_off=tab.surface_off, words=ng.words, probs=ng.probs,
                 backoffs=ng.backoffs, lm_names=np.frombuffer(lm_blob, dtype=np.uint8))


def load_images(path) -> tuple[TableImage, NgramImage, float]:
    """Inverse of save_images: (TableImage, NgramImage, back-off of `<s>`)."""
    import json

    with np.load(path, allow_pickle=False) as z:
        header = json.loads(bytes(z["header"]).decode())
        if header.get("format") != IMAGE_FORMAT:
            raise FormatError(f"{path}: image format {header.get('format')} != {IMAGE_FORMAT}")
        blob = bytes(z["surface_blob"])
        soff = z["surface_off"].astype(np.int64)
        surfaces = [blob[soff[i]:soff[i + 1]].decode("utf-8") for i in range(len(soff) - 1)]
        tab = TableImage(table=np.ascontiguousarray(z["table"], dtype=np.int32),
                         sink=header["sink"], blank_id=header["blank_id"],
                         space_id=header["space_id"], comp_off=z["comp_off"],
                         comp_surface=z["comp_surface"], comp_lmword=z["comp_lmword"],
                         surfaces=surfaces, surface_blob=blob, surface_off=soff,
                         whitespace_free=bool(header["whitespace_free"]))
        names = bytes(z["lm_names"]).decode("utf-8").split("\n")
        ng = NgramImage(order=header["order"], words=z["words"], probs=z["probs"],
                        backoffs=z["backoffs"], word_id={w: i for i, w in enumerate(names)},
                        bos_id=header["bos_id"], eos_eff=header["eos_eff"], unk_id=header["unk_id"])
    return tab, ng, float(header["bos_backoff"])
