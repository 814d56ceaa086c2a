"""CPU ORACLE for the LightBeam first-pass decoder -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline / `--impl reference`
legs may import this module, and only as the checker / the timed CPU port.  The product
(`paper_2603_14002_b200`) never imports it and has no CPU fallback.

What it is: a from-scratch numpy/Python restatement of the reference decode path
(`/root/reference/pkg/src/lightbeam/decoder.py:177-460`, `ngram.py:187-236`,
`scorer.py:269-325`, `logits.py:119-130`).  Every score is fp64 and every operation is done
in the reference's order, so results are bit-identical to the reference on the same inputs.
Each function cites the reference lines it restates.

Parity pinning: `tests/test_oracle_golden.py` replays the fixtures in `tests/golden/`, which
`tests/golden/make_golden.py` produced by running the *unmodified reference* in the build
container (the reference tree is not present on the GPU box).  The oracle must reproduce
every golden text, score, n-best list, event count and per-frame beam trace exactly.

Inputs are duck-typed: a transition table with `.table/.sink/.root/.blank_id/.space_id/
.entries/.completions_at()`, an n-gram model with `.order/.probs/.backoffs/.unk_present`,
any object with the `DecodeConfig` fields, and any scorer implementing `submit()` /
`next_request_id()`.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import NamedTuple

import numpy as np

NEG_INF = -1.0e30
GUARD = -1.0e29
H_INIT = (np.uint64(0xCBF29CE484222325), np.uint64(0x9AE16A3B2F90404F))  # decoder.py:38-39
H_MULT = (np.uint64(0x9E3779B97F4A7C15), np.uint64(0xC2B2AE3D27D4EB4F))  # decoder.py:40-41
PUNCT_ORDER = (".", "?", "!")


class OracleEmptyBeam(Exception):
    """Raised where the reference raises EmptyBeamError (decoder.py:267,314,394)."""


class OracleEmptyInput(Exception):
    """Raised where the reference raises DataValueError (decoder.py:421)."""


class OracleScorerError(Exception):
    """Raised where the reference raises ScorerError (scorer.py:297,318-323)."""


def log_softmax_scaled(frames, alpha: float) -> np.ndarray:
    """logits.py:119-130: alpha * (x - (m + log(sum(exp(x - m))))) in fp64, numpy row sums."""
    x = np.asarray(frames, dtype=np.float32).astype(np.float64)
    m = x.max(axis=1, keepdims=True)
    lse = m + np.log(np.exp(x - m).sum(axis=1, keepdims=True))
    return alpha * (x - lse)


class NgramOracle:
    """ngram.py:187-236. LM states are the history word tuples themselves (the reference's
    registry ids are session-local names for the same tuples)."""

    def __init__(self, model):
        self.order = model.order
        self.probs = model.probs
        self.backoffs = model.backoffs
        self.has_unk = model.unk_present
        self.memo: dict = {}

    def increment(self, hist: tuple, word: str):
        key = (hist, word)
        got = self.memo.get(key)
        if got is None:
            got = self._evaluate(hist, word)
            self.memo[key] = got
        return got

    def _evaluate(self, hist: tuple, word: str):
        if (word,) not in self.probs:  # ngram.py:225-230
            if not self.has_unk:
                return NEG_INF, ()
            word = "<unk>"
        n = len(hist)
        value, hit = NEG_INF, n + 1
        for i in range(n + 1):  # ngram.py:189-194: longest listed (h[i:], w)
            p = self.probs.get(hist[i:] + (word,))
            if p is not None:
                value, hit = p, i
                break
        for i in range(min(hit, n) - 1, -1, -1):  # right-nested bo(h0) + (bo(h1) + (... + p))
            value = self.backoffs.get(hist[i:], 0.0) + value
        if self.order <= 1:  # ngram.py:198-205
            succ = ()
        else:
            succ = (hist + (word,))[-(self.order - 1):]
            while succ and succ not in self.probs:
                succ = succ[1:]
        return value, succ

    def sequence(self, words, with_eos=False) -> float:
        """ngram.py:239-250 (score_sequence): left-to-right sum from ('<s>',)."""
        state, total = ("<s>",), 0.0
        for w in list(words) + (["</s>"] if with_eos else []):
            inc, state = self.increment(state, w)
            total += inc
        return total


def _roundtrip(scorer, texts, kind, chunk):
    """scorer.py:269-325: order-preserving dedupe, chunked submit, fan results back out."""
    if not texts:
        return []
    if chunk < 1:
        raise ValueError("chunk_size must be >= 1")
    pos: dict = {}
    uniq: list = []
    for t in texts:
        if t not in pos:
            pos[t] = len(uniq)
            uniq.append(t)
    # the request dataclass is whatever the scorer's module defines; build it duck-typed
    req_cls = _request_class(scorer)
    out: list = []
    for lo in range(0, len(uniq), chunk):
        part = tuple(uniq[lo:lo + chunk])
        resp = scorer.submit(req_cls(id=scorer.next_request_id(), kind=kind, texts=part))
        if kind == "score":
            if len(resp.scores) != len(part):
                raise OracleScorerError("scorer returned wrong number of scores")
            out.extend(resp.scores)
        else:
            if resp.puncts is None or len(resp.scores) != len(part) or len(resp.puncts) != len(part):
                raise OracleScorerError("score_eos reply missing puncts or wrong length")
            for p, s in zip(resp.puncts, resp.scores):
                if p not in PUNCT_ORDER:
                    raise OracleScorerError(f"invalid punctuation {p!r}")
                out.append((p, s))
    return [out[pos[t]] for t in texts]


def _request_class(scorer):
    import sys

    mod = sys.modules.get(type(scorer).__module__)
    cls = getattr(mod, "ScoreRequest", None)
    if cls is None:
        from paper_2603_14002_b200.scorer import ScoreRequest as cls  # plain dataclass
    return cls


class Entry(NamedTuple):
    """decoder.py:44-51 (OrthoEntry): weighted LM total, LM history, word node, creation seq."""

    total: float
    hist: tuple
    node: int
    seq: int
    punct: str = ""


@dataclass
class OracleResult:
    text: str
    score: float
    nbest: list
    frame_count: int
    wall_time_s: float
    llm_events: int
    trace: list = field(default_factory=list)


class OracleSearch:
    """One utterance's search state (decoder.py:96-147 BeamSet + WordHistory)."""

    def __init__(self, cfg, tt, model, scorer, trace: bool = False):
        self.cfg, self.tt, self.scorer = cfg, tt, scorer
        self.ng = NgramOracle(model)
        v = tt.table.shape[1]
        self.tokens = np.arange(v)
        self.phoneme = np.ones(v, dtype=bool)
        self.phoneme[[tt.blank_id, tt.space_id]] = False
        # decoder.py:112-125: one root hypothesis
        self.score = np.zeros(1, dtype=np.float64)
        self.last = np.array([tt.blank_id], dtype=np.int64)
        self.h1 = np.array([H_INIT[0]], dtype=np.uint64)
        self.h2 = np.array([H_INIT[1]], dtype=np.uint64)
        self.prefix = np.array([tt.root], dtype=np.int64)
        self.sets: list = [(Entry(0.0, ("<s>",), 0, 0),)]
        self.node_parent = [-1]
        self.node_word = [""]
        self._text_memo = {0: ""}
        self.seq = 1
        self.trace_on = trace
        self.trace: list = []

    # --- word history (decoder.py:54-83) ---
    def add_node(self, parent: int, word: str) -> int:
        self.node_parent.append(parent)
        self.node_word.append(word)
        return len(self.node_parent) - 1

    def text(self, node: int) -> str:
        got = self._text_memo.get(node)
        if got is None:
            words = []
            n = node
            while n > 0:
                words.append(self.node_word[n])
                n = self.node_parent[n]
            got = " ".join(reversed(words))
            self._text_memo[node] = got
        return got

    # --- n-gram shallow fusion at a word boundary (decoder.py:182-235) ---
    def word_boundary(self, j: int, completion_ids) -> None:
        cfg = self.cfg
        old = self.sets[j]
        surfaces: list = []
        for eid in completion_ids:
            s = self.tt.entries[eid].surface
            if s not in surfaces:
                surfaces.append(s)
        pool = []
        for e in old:
            for w in surfaces:
                inc, succ = self.ng.increment(e.hist, w)
                if inc <= GUARD:
                    continue
                pool.append((e.total + cfg.ngram_weight * inc, self.seq, succ, e.node, w))
                self.seq += 1
        if not pool:
            self.score[j] = NEG_INF
            return
        pool.sort(key=lambda c: (-c[0], c[1]))
        pool = pool[: cfg.ortho_beams]
        best = pool[0][0]
        floor = best - cfg.homophone_prune_threshold
        self.sets[j] = tuple(
            Entry(tot, succ, self.add_node(node, w), seq)
            for tot, seq, succ, node, w in pool
            if tot >= floor
        )
        self.score[j] += best - old[0].total

    # --- one frame (decoder.py:238-326) ---
    def frame(self, row: np.ndarray, t: int) -> None:
        cfg, tt = self.cfg, self.tt
        v = row.shape[0]
        blank, space = tt.blank_id, tt.space_id
        cand = self.score[:, None] + row[None, :]
        cand += cfg.token_insertion_bonus * (self.phoneme[None, :] & (self.tokens[None, :] != self.last[:, None]))
        cand[:, space] += cfg.word_boundary_bonus * (self.last != space)
        ok = tt.table[self.prefix] != tt.sink
        ok[:, blank] = True
        ok[np.arange(len(self.last)), self.last] = True
        cand[~ok] = NEG_INF

        flat = cand.ravel()
        top = np.argsort(-flat, kind="stable")[: min(cfg.beam_size, flat.size)]
        vals = flat[top]
        if vals[0] <= GUARD:
            raise OracleEmptyBeam(f"all candidates pruned at frame {t}")
        live = (vals >= vals[0] - cfg.beam_prune_threshold) & (vals > GUARD)
        top, vals = top[live], vals[live]

        par = top // v
        tok = top % v
        plast = self.last[par]
        ppre = self.prefix[par]
        emit = (tok != blank) & (tok != plast)
        step = tok.astype(np.uint64) + np.uint64(1)
        h1 = np.where(emit, self.h1[par] * H_MULT[0] + step, self.h1[par])
        h2 = np.where(emit, self.h2[par] * H_MULT[1] + step, self.h2[par])
        new_last = np.where(tok == blank, plast, tok)
        new_pre = np.where(emit, tt.table[ppre, tok], ppre)
        self.score = vals.astype(np.float64)
        self.sets = [self.sets[p] for p in par]

        for j in np.flatnonzero(emit & (tok == space)):
            self.word_boundary(int(j), tt.completions_at(int(ppre[j])))

        n = len(top)
        order = np.lexsort((np.arange(n), -self.score))
        premerge = None
        if self.trace_on:
            premerge = [(int(h1[j]), int(h2[j]), float(self.score[j])) for j in range(n)]
        seen = set()
        keep = []
        for j in order:
            if self.score[j] <= GUARD:
                continue
            key = (int(h1[j]), int(h2[j]))
            if key not in seen:
                seen.add(key)
                keep.append(int(j))
        if not keep:
            raise OracleEmptyBeam(f"all hypotheses pruned at frame {t}")
        idx = np.asarray(keep, dtype=np.int64)
        self.score = self.score[idx]
        self.last = new_last[idx]
        self.h1, self.h2 = h1[idx], h2[idx]
        self.prefix = new_pre[idx]
        self.sets = [self.sets[j] for j in keep]
        if self.trace_on:
            self.trace.append({"t": t, "kind": "step", "beams": self.snapshot(), "premerge": premerge,
                               "labels": tok[idx].tolist(), "parents": par[idx].tolist()})

    def snapshot(self):
        return [
            (int(self.h1[i]), int(self.h2[i]), int(self.prefix[i]), int(self.last[i]), float(self.score[i]))
            for i in range(len(self.score))
        ]

    # --- delayed fusion (decoder.py:329-372) ---
    def rescore(self, final: bool) -> None:
        cfg = self.cfg
        texts: list = []
        seen = set()
        for entries in self.sets:
            for e in entries:
                tx = self.text(e.node)
                if tx and tx not in seen:
                    seen.add(tx)
                    texts.append(tx)
        if final:
            lut = dict(zip(texts, _roundtrip(self.scorer, texts, "score_eos", cfg.llm_chunk_size)))
        else:
            lut = {tx: ("", s) for tx, s in
                   zip(texts, _roundtrip(self.scorer, texts, "score", cfg.llm_chunk_size))}
        for i, entries in enumerate(self.sets):
            prev = entries[0].total
            fresh = []
            for e in entries:
                tx = self.text(e.node)
                if not tx:
                    fresh.append(e._replace(total=0.0, punct=""))
                else:
                    p, s = lut[tx]
                    fresh.append(e._replace(total=cfg.llm_weight * s, punct=p if final else e.punct))
            fresh.sort(key=lambda e: (-e.total, e.seq))
            self.sets[i] = tuple(fresh)
            self.score[i] += fresh[0].total - prev
        if self.trace_on:
            self.trace.append({"kind": "final" if final else "llm", "beams": self.snapshot()})

    # --- end-of-utterance closure (decoder.py:375-405) ---
    def close(self) -> None:
        tt = self.tt
        for i in range(len(self.score)):
            st = int(self.prefix[i])
            if st == tt.root:
                continue
            ids = tt.completions_at(st)
            if ids:
                self.word_boundary(i, ids)
                self.prefix[i] = tt.root
            else:
                self.score[i] = NEG_INF
        alive = np.flatnonzero(self.score > GUARD)
        if len(alive) == 0:
            raise OracleEmptyBeam("no hypothesis survived end-of-utterance closure")
        if len(alive) < len(self.score):
            self.score = self.score[alive]
            self.last = self.last[alive]
            self.h1, self.h2 = self.h1[alive], self.h2[alive]
            self.prefix = self.prefix[alive]
            self.sets = [self.sets[j] for j in alive]
        if self.trace_on:
            self.trace.append({"kind": "close", "beams": self.snapshot()})

    # --- ranking and n-best (decoder.py:433-460) ---
    def results(self):
        ranked = np.lexsort((np.arange(len(self.score)), -self.score))
        pairs = []
        for i in ranked:
            entries = self.sets[i]
            best_lm = entries[0].total
            for e in entries:
                pairs.append((self.text(e.node) + e.punct, float(self.score[i] - best_lm + e.total)))
        pairs.sort(key=lambda p: -p[1])
        nbest, seen = [], set()
        for tx, s in pairs:
            if tx not in seen:
                seen.add(tx)
                nbest.append((tx, s))
        top = int(ranked[0])
        head = self.sets[top][0]
        return self.text(head.node) + head.punct, float(self.score[top]), nbest

    def entries_dump(self):
        """Per beam: [(text, total, punct, seq)] -- for GPU parity checks of ortho sets."""
        return [[(self.text(e.node), e.total, e.punct, e.seq) for e in ents] for ents in self.sets]


def decode(d, cfg, tt, model, scorer, final_llm_only: bool = False, trace: bool = False):
    """decoder.py:408-460. `d` is a LogProbMatrix-like object or an fp64 (T, V) array."""
    frames = getattr(d, "frames", d)
    frames = np.asarray(frames, dtype=np.float64)
    if frames.shape[0] == 0:
        raise OracleEmptyInput("cannot decode an empty log-probability matrix")
    t0 = time.perf_counter()
    search = OracleSearch(cfg, tt, model, scorer, trace=trace)
    events = 0
    r = cfg.llm_rescore_interval
    for t in range(frames.shape[0]):
        search.frame(frames[t], t)
        if t > 0 and t % r == 0 and not final_llm_only:
            search.rescore(final=False)
            events += 1
    search.close()
    search.rescore(final=True)
    text, score, nbest = search.results()
    return OracleResult(text, score, nbest, frames.shape[0], time.perf_counter() - t0, events,
                        search.trace)


def decode_with_state(d, cfg, tt, model, scorer, final_llm_only: bool = False):
    """Like `decode` but also returns the final OracleSearch (ortho sets for parity tests)."""
    frames = np.asarray(getattr(d, "frames", d), dtype=np.float64)
    if frames.shape[0] == 0:
        raise OracleEmptyInput("cannot decode an empty log-probability matrix")
    search = OracleSearch(cfg, tt, model, scorer)
    events = 0
    for t in range(frames.shape[0]):
        search.frame(frames[t], t)
        if t > 0 and t % cfg.llm_rescore_interval == 0 and not final_llm_only:
            search.rescore(final=False)
            events += 1
    search.close()
    search.rescore(final=True)
    text, score, nbest = search.results()
    return OracleResult(text, score, nbest, frames.shape[0], 0.0, events), search
