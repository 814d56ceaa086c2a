// lb_kernels.cu -- sm_100a kernels of the LightBeam first-pass decoder.
//
//   K1 log_softmax_kernel      logits.py:119-130 (fp64, numpy 8-lane pairwise row sum)
//   K2 frames_kernel           decoder.py:238-326 per frame, one CTA per utterance, frames
//                              [t0,t1) in one persistent launch; lexicon mask
//                              (lexicon.py:124-137), exact stable top-k + theta, rolling hash,
//                              n-gram fusion at word boundaries (decoder.py:182-235 with
//                              ngram.py:187-236 as parallel hash probes), max-merge
//                              recombination; optional in-kernel interval fusion for the device
//                              n-gram scorer.
//   K3 close_kernel            decoder.py:375-405
//   K4 count/write_entries     text gathering of apply_llm (decoder.py:338-345)
//   K7 apply_scores_kernel     fusion of apply_llm (decoder.py:354-371)
//      device_fusion_kernel    apply_llm with the n-gram stub scorer (scorer.py:121-139)
//
// Every score is IEEE fp64 computed with explicitly rounded intrinsics in the reference's
// operation order (the file is also compiled with -fmad=false), so results are bit-identical
// to the numpy/Python reference on the same D matrix.

#include <cuda_runtime.h>

#include <cfloat>
#include <cstdlib>
#include <cstdint>

#include "lb_device.cuh"
#include "lb_internal.h"

using namespace lbd;

#define FULLMASK 0xffffffffu

namespace lbk {
unsigned long long g_launches = 0;
}

namespace {

__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double xsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }

__device__ __forceinline__ bool prob_present(double p) {
  return (uint64_t)__double_as_longlong(p) != PROB_ABSENT;
}

// ---------------------------------------------------------------- async copy helpers
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  unsigned s = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(s), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(s), "r"(bytes)
               : "memory");
}
// 1-D TMA bulk copy global -> shared, completion signalled on an mbarrier
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, unsigned bytes,
                                             uint64_t* bar) {
  unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(d),
      "l"(src), "r"(bytes), "r"(b)
      : "memory");
}
// the same with an L2 evict-first hint: streamed log-prob rows must not push the lexicon and
// n-gram images (re-read every frame) out of L2
__device__ __forceinline__ void tma_bulk_g2s_stream(void* dst, const void* src, unsigned bytes,
                                                    uint64_t* bar) {
  unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  unsigned b = (unsigned)__cvta_generic_to_shared(bar);
#ifdef LB_NO_L2HINT
  tma_bulk_g2s(dst, src, bytes, bar);
  return;
#endif
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
      "%2, [%3], %4;\n" ::"r"(d),
      "l"(src), "r"(bytes), "r"(b), "l"(pol)
      : "memory");
}
// word-history nodes are written once per frame and read back only after the search
__device__ __forceinline__ void st_stream(uint32_t* p, uint32_t v) {
#ifdef LB_NO_L2HINT
  *p = v;
#else
  __stcs(p, v);
#endif
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  unsigned s = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n .reg .pred p;\n"
      "LBW%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LBW%=;\n}\n" ::"r"(s),
      "r"(parity)
      : "memory");
}

// ---------------------------------------------------------------- warp reductions
__device__ __forceinline__ double warp_max(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FULLMASK, v, o));
  return v;
}

// ---------------------------------------------------------------- candidate value
// decoder.py:252-256: ((s + d) + beta*[phoneme & non-repeat]) then + gamma*[last != space]
// on the space column.  Multiplying by exactly 1.0/0.0 reproduces numpy's `beta * mask`.
struct FrameConsts {
  double beta, gamma;
  int blank, space;
};

__device__ __forceinline__ double cand_value(double s, double d, int v, int lp, const FrameConsts& c) {
  double x = xadd(s, d);
  const bool ph = (v != c.blank) & (v != c.space);
  x = xadd(x, xmul(c.beta, (ph && v != lp) ? 1.0 : 0.0));
  if (v == c.space) x = xadd(x, xmul(c.gamma, (lp != c.space) ? 1.0 : 0.0));
  return x;
}

// ---------------------------------------------------------------- n-gram probes
// score_word (ngram.py:208-236) for one (entry history, word) per 8-lane group; all 32 lanes
// call.  Lane sub = 2*i + c scans candidate bucket c of the key K_i = (h[i:], w), i <= hlen,
// in the bucketized cuckoo image: one 128-byte line, four 16-byte key loads in flight, so a
// whole score_word is a single memory round trip.  The back-offs of the abandoned histories
// h[i:] come from the entry's cache.  The group leader (sub 0) combines the right-nested sum
// bo(h0) + (bo(h1) + (... + p)), the successor = longest listed suffix of (h + w) capped at
// order-1 words, and the successor's own suffix back-offs (the new entry's cache).  `w < 0`
// is the OOV-without-<unk> kill: increment NEG_INF, successor ().
// h[j] for a runtime j < MAXH without dynamic register indexing (no local-memory array)
static_assert(MAXH == 3, "hist_at assumes three history slots");
__device__ __forceinline__ uint32_t hist_at(const uint32_t h[MAXH], int j) {
  return j == 0 ? h[0] : (j == 1 ? h[1] : h[2]);
}

struct WordScore {
  double inc;
  double sbo[MAXH];
  uint32_t succ[MAXH];
  int slen;
};

__device__ void group_score_word(const ModelDev& m, bool act, const uint32_t h[MAXH], int hl,
                                 const double hbo[MAXH], int w, WordScore& out,
                                 unsigned& probes) {
  const int lane = threadIdx.x & 31, sub = lane & 7, grp = lane >> 3;
  const bool valid = act && w >= 0;
  const int ki = sub >> 1, cb = sub & 1;
  bool hit = false;
  double p = 0.0, bo = 0.0;
  if (valid && ki <= hl) {
    // key = (h[ki..hl-1], w, pad...), built with static indices so it stays in registers
    uint32_t k[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int j = ki + i;
      k[i] = j < hl ? hist_at(h, j) : (j == hl ? (uint32_t)w : WPAD);
    }
    uint32_t b1, b2;
    ng_buckets(ng_hash(k[0], k[1], k[2], k[3]), m.ng_nb, b1, b2);
    const uint4* bucket = reinterpret_cast<const uint4*>(m.ng + (size_t)(cb ? b2 : b1) * NG_WAYS);
    uint4 r[NG_WAYS];
#pragma unroll
    for (int q = 0; q < NG_WAYS; ++q) r[q] = __ldg(bucket + 2 * q);
    ++probes;
    int slot = -1;
#pragma unroll
    for (int q = NG_WAYS - 1; q >= 0; --q)
      if (r[q].x == k[0] && r[q].y == k[1] && r[q].z == k[2] && r[q].w == k[3]) slot = q;
    if (slot >= 0) {
      const double2 pb = __ldg(reinterpret_cast<const double2*>(bucket + 2 * slot + 1));
      p = pb.x;
      bo = pb.y;
      hit = true;
    }
  }
  const unsigned bal = __ballot_sync(FULLMASK, hit);
  const unsigned gb = (bal >> (grp * 8)) & 0xFFu;
  double pk[4], bk[4];
  bool fk[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int src = grp * 8 + 2 * j + (((gb >> (2 * j)) & 1u) ? 0 : 1);
    pk[j] = __shfl_sync(FULLMASK, p, src);
    bk[j] = __shfl_sync(FULLMASK, bo, src);
    fk[j] = ((gb >> (2 * j)) & 3u) != 0;
  }
  out.slen = 0;
  out.inc = NEG_INF;
  if (sub != 0 || !valid) return;
  double val = NEG_INF;
  int hitk = hl + 1;
#pragma unroll
  for (int j = 3; j >= 0; --j)
    if (j <= hl && fk[j] && prob_present(pk[j])) {
      val = pk[j];
      hitk = j;
    }
  {
    const int lim = min(hitk, hl);  // right-nested back-off sum, j = lim-1 .. 0
    if (lim > 2) val = xadd(hbo[2], val);
    if (lim > 1) val = xadd(hbo[1], val);
    if (lim > 0) val = xadd(hbo[0], val);
  }
  out.inc = val;
  if (m.order > 1) {
    const int start = max(0, hl + 1 - (m.order - 1));
    int sk = -1;
#pragma unroll
    for (int j = 3; j >= 0; --j)
      if (j >= start && j <= hl && fk[j] && prob_present(pk[j])) sk = j;
    if (sk >= 0) {
      const int n = hl - sk + 1;  // successor = (h[sk..hl-1], w)
#pragma unroll
      for (int t = 0; t < MAXH; ++t) {
        const int j = sk + t;
        out.succ[t] = j < hl ? hist_at(h, j) : (j == hl ? (uint32_t)w : 0u);
      }
      out.slen = n;
#pragma unroll
      for (int t = 0; t < MAXH; ++t) {
        const int j = sk + t;
        double v = 0.0;
        if (t < n) {
          if (j == 0) v = fk[0] ? bk[0] : 0.0;
          else if (j == 1) v = fk[1] ? bk[1] : 0.0;
          else if (j == 2) v = fk[2] ? bk[2] : 0.0;
          else v = fk[3] ? bk[3] : 0.0;
        }
        out.sbo[t] = v;
      }
    }
  }
}

// score_word with 4 lanes per query (quad): lane sub = i probes BOTH candidate buckets of
// K_i = (h[i:], w); 8 pairs per warp per round.  Same combination as group_score_word.
__device__ void quad_score_word(const ModelDev& m, bool act, const uint32_t h[MAXH], int hl,
                                const double hbo[MAXH], int w, WordScore& out, unsigned& probes) {
  const int lane = threadIdx.x & 31, ki = lane & 3, grp = lane >> 2;
  const bool valid = act && w >= 0;
  bool hit = false;
  double p = 0.0, bo = 0.0;
  if (valid && ki <= hl) {
    // key = (h[ki..hl-1], w, pad...), built with static indices so it stays in registers
    uint32_t k[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int j = ki + i;
      k[i] = j < hl ? hist_at(h, j) : (j == hl ? (uint32_t)w : WPAD);
    }
    uint32_t b1, b2;
    ng_buckets(ng_hash(k[0], k[1], k[2], k[3]), m.ng_nb, b1, b2);
    const uint4* bk1 = reinterpret_cast<const uint4*>(m.ng + (size_t)b1 * NG_WAYS);
    const uint4* bk2 = reinterpret_cast<const uint4*>(m.ng + (size_t)b2 * NG_WAYS);
    uint4 r[2 * NG_WAYS];
#pragma unroll
    for (int q = 0; q < NG_WAYS; ++q) {
      r[q] = __ldg(bk1 + 2 * q);
      r[NG_WAYS + q] = __ldg(bk2 + 2 * q);
    }
    probes += 2;
    int slot = -1;
#pragma unroll
    for (int q = 2 * NG_WAYS - 1; q >= 0; --q)
      if (r[q].x == k[0] && r[q].y == k[1] && r[q].z == k[2] && r[q].w == k[3]) slot = q;
    if (slot >= 0) {
      const uint4* rec = (slot < NG_WAYS ? bk1 : bk2) + 2 * (slot & (NG_WAYS - 1));
      const double2 pb = __ldg(reinterpret_cast<const double2*>(rec + 1));
      p = pb.x;
      bo = pb.y;
      hit = true;
    }
  }
  const unsigned bal = __ballot_sync(FULLMASK, hit);
  const unsigned gb = (bal >> (grp * 4)) & 0xFu;
  double pk[4], bk[4];
  bool fk[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    pk[j] = __shfl_sync(FULLMASK, p, grp * 4 + j);
    bk[j] = __shfl_sync(FULLMASK, bo, grp * 4 + j);
    fk[j] = (gb >> j) & 1u;
  }
  out.slen = 0;
  out.inc = NEG_INF;
  if (ki != 0 || !valid) return;
  double val = NEG_INF;
  int hitk = hl + 1;
#pragma unroll
  for (int j = 3; j >= 0; --j)
    if (j <= hl && fk[j] && prob_present(pk[j])) {
      val = pk[j];
      hitk = j;
    }
  {
    const int lim = min(hitk, hl);  // right-nested back-off sum, j = lim-1 .. 0
    if (lim > 2) val = xadd(hbo[2], val);
    if (lim > 1) val = xadd(hbo[1], val);
    if (lim > 0) val = xadd(hbo[0], val);
  }
  out.inc = val;
  if (m.order > 1) {
    const int start = max(0, hl + 1 - (m.order - 1));
    int sk = -1;
#pragma unroll
    for (int j = 3; j >= 0; --j)
      if (j >= start && j <= hl && fk[j] && prob_present(pk[j])) sk = j;
    if (sk >= 0) {
      const int n = hl - sk + 1;  // successor = (h[sk..hl-1], w)
#pragma unroll
      for (int t = 0; t < MAXH; ++t) {
        const int j = sk + t;
        out.succ[t] = j < hl ? hist_at(h, j) : (j == hl ? (uint32_t)w : 0u);
      }
      out.slen = n;
#pragma unroll
      for (int t = 0; t < MAXH; ++t) {
        const int j = sk + t;
        double v = 0.0;
        if (t < n) {
          if (j == 0) v = fk[0] ? bk[0] : 0.0;
          else if (j == 1) v = fk[1] ? bk[1] : 0.0;
          else if (j == 2) v = fk[2] ? bk[2] : 0.0;
          else v = fk[3] ? bk[3] : 0.0;
        }
        out.sbo[t] = v;
      }
    }
  }
}

__device__ __forceinline__ void new_entry(Ent& o, double total, double cum, const WordScore& ws,
                                          uint32_t node, uint32_t seq, uint32_t depth) {
  o.total = total;
  o.cum = cum;
  o.node = node;
  o.seq = seq;
  o.hlen = (uint8_t)ws.slen;
  o.depth = (uint16_t)depth;
  o.punct = 0;
#pragma unroll
  for (int t = 0; t < MAXH; ++t) {
    o.h[t] = t < ws.slen ? ws.succ[t] : 0u;
    o.bo[t] = t < ws.slen ? ws.sbo[t] : 0.0;
  }
}

// Completion header embedded in a padded lexicon row (see ROW_HDR in lb_device.cuh).
struct CompHdr {
  int ns, off, s0, l0, s1, l1;
};
__device__ __forceinline__ CompHdr comp_hdr(const int32_t* row, int V) {
  return CompHdr{row[V], row[V + 1], row[V + 2], row[V + 3], row[V + 4], row[V + 5]};
}

// Successor of prefix state `lr` on token `tok` (a valid transition): breadth-first tries give
// first child + rank (space -> root), any other table a successor-list lookup.
__device__ __forceinline__ int lex_succ(const ModelDev& m, const LexRec& lr, int tok) {
  if (m.lex_contig) {
    const unsigned long long ms = lr.mask & ~(1ull << m.space);
    return tok == m.space ? 0 : lr.base + __popcll(ms & ((1ull << tok) - 1ull));
  }
  return __ldg(m.lex_next + lr.base + __popcll(lr.mask & ((1ull << tok) - 1ull)));
}
// Completion header from a compact lexicon record (CSR offset read only for > 2 surfaces).
__device__ __forceinline__ CompHdr lex_hdr_g(const ModelDev& m, const LexRec& r, int state) {
  return CompHdr{r.ns, r.ns > 2 ? __ldg(m.comp_off + state) : 0, r.s0, r.l0, r.s1, r.l1};
}
// The same header from a compact lexicon record and the beam's staged CSR offset.
__device__ __forceinline__ CompHdr small_hdr(const LexRec& r, int off) {
  return CompHdr{r.ns, off, r.s0, r.l0, r.s1, r.l1};
}

// apply_ngram (decoder.py:182-235) for one beam, one full warp.  Candidates are the
// (entry, distinct surface) pairs in creation order; the running top-O list is ordered by
// (-total, seq) -- candidates arrive in increasing seq, so strict '>' keeps ties stable.
// On return (lane 0 authoritative): *outn = kept entries (written to outents), or -1 when no
// candidate survived (beam killed: *score = NEG_INF, decoder.py:223-225).
// NP = pairs per warp round: 4 (8 lanes per pair, one cuckoo bucket per lane) or 8 (4 lanes per
// pair probing both buckets, quad_score_word); the candidates reach the top-O list in the same
// order either way, so both give identical results.
template <int NP, class Scratch>
__device__ void warp_apply_ngram_t(const ModelDev& m, const CfgDev& c, const BatchDev& b, int trial,
                                   const Ent* pents, int pn, const CompHdr ch, Scratch* ws,
                                   Ent* outents, int* outn, double* score, int* node_counter,
                                   int* fail, unsigned& calls, unsigned& probes) {
  static_assert(NP == 4 || NP == 8, "4 or 8 pairs per round");
  const int lane = threadIdx.x & 31, sub = lane & (32 / NP - 1), grp = lane / (32 / NP);
  const int ns = ch.ns;
  const int npairs = pn * ns;
  int ntop = 0;
  for (int base = 0; base < npairs; base += NP) {
    const int pi = base + grp;
    const bool act = pi < npairs;
    int e = 0, s = 0, w = -1, surf = -1;
    if (act) {
      e = pi / ns;
      s = pi - e * ns;
      if (s == 0) {
        w = ch.l0;
        surf = ch.s0;
      } else if (s == 1) {
        w = ch.l1;
        surf = ch.s1;
      } else {
        w = __ldg(m.comp_lm + ch.off + s);
        surf = __ldg(m.comp_surf + ch.off + s);
      }
    }
    const Ent& E = pents[act ? e : 0];
    uint32_t hh[MAXH] = {E.h[0], E.h[1], E.h[2]};
    double hb[MAXH] = {E.bo[0], E.bo[1], E.bo[2]};
    WordScore sw;
    if (NP == 4) group_score_word(m, act, hh, E.hlen, hb, w, sw, probes);
    else quad_score_word(m, act, hh, E.hlen, hb, w, sw, probes);
    if (sub == 0) {
      NgCand& pc = ws->pending[grp];
      pc.valid = 0;
      if (act) {
        ++calls;
        if (sw.inc > GUARD) {
          pc.valid = 1;
          pc.total = xadd(E.total, xmul(c.omega, sw.inc));
          pc.cum = xadd(E.cum, sw.inc);
          pc.depth = (uint32_t)E.depth + 1u;
          pc.node = E.node;
          pc.surf = (uint32_t)surf;
          pc.seq = (uint32_t)pi;
          pc.hlen = (uint32_t)sw.slen;
          for (int t = 0; t < MAXH; ++t) {
            pc.h[t] = sw.succ[t];
            pc.bo[t] = sw.sbo[t];
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) {
      for (int g = 0; g < NP; ++g) {
        const NgCand& cd = ws->pending[g];
        if (!cd.valid) continue;
        int pos = ntop;
        for (int i = 0; i < ntop; ++i)
          if (cd.total > ws->top[i].total) {
            pos = i;
            break;
          }
        if (pos >= c.O) continue;
        const int last = min(ntop, c.O - 1);
        for (int i = last; i > pos; --i) ws->top[i] = ws->top[i - 1];
        ws->top[pos] = cd;
        ntop = min(ntop + 1, c.O);
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    if (ntop == 0) {
      *score = NEG_INF;
      *outn = -1;
    } else {
      const double best = ws->top[0].total;
      const double floor_ = xsub(best, c.lambda);
      int kept = 0;
      while (kept < ntop && ws->top[kept].total >= floor_) ++kept;
      const int base = atomicAdd(node_counter, kept);
      if (base + kept > b.ncap) {
        *fail = 1;
        *outn = -1;
        *score = NEG_INF;
      } else {
        const size_t nb = (size_t)trial * b.ncap;
        for (int i = 0; i < kept; ++i) {
          const NgCand& cd = ws->top[i];
          const uint32_t node = (uint32_t)(base + i);
          st_stream(b.nparent + nb + node, cd.node);
          st_stream(b.nsurf + nb + node, cd.surf);
          WordScore sw;
          sw.slen = (int)cd.hlen;
          for (int t = 0; t < MAXH; ++t) {
            sw.succ[t] = cd.h[t];
            sw.sbo[t] = cd.bo[t];
          }
          new_entry(outents[i], cd.total, cd.cum, sw, node, cd.seq, cd.depth);
        }
        *outn = kept;
        *score = xadd(*score, xsub(best, pents[0].total));
      }
    }
  }
  __syncwarp();
}

__device__ __forceinline__ void warp_apply_ngram(const ModelDev& m, const CfgDev& c,
                                                 const BatchDev& b, int trial, const Ent* pents,
                                                 int pn, const CompHdr ch, WarpScratch* ws,
                                                 Ent* outents, int* outn, double* score,
                                                 int* node_counter, int* fail, unsigned& calls,
                                                 unsigned& probes) {
  warp_apply_ngram_t<4>(m, c, b, trial, pents, pn, ch, ws, outents, outn, score, node_counter,
                        fail, calls, probes);
}

// insertion sort of <= OMAX entries by (-total, seq) (decoder.py:369)
__device__ __forceinline__ void sort_entries(Ent* e, int n) {
  for (int i = 1; i < n; ++i) {
    Ent x = e[i];
    int j = i - 1;
    while (j >= 0 && (e[j].total < x.total || (e[j].total == x.total && e[j].seq > x.seq))) {
      e[j + 1] = e[j];
      --j;
    }
    e[j + 1] = x;
  }
}

// 32-bit fingerprint of a beam's two prefix-hash lanes (equal lanes -> equal fingerprints)
__device__ __forceinline__ uint32_t hash_fp(uint64_t a1, uint64_t a2) {
  const uint64_t x = a1 ^ (a2 * 0x9E3779B97F4A7C15ull);
  return (uint32_t)(x >> 32) ^ (uint32_t)x;
}

// order-preserving 64-bit key of an fp64 (after canonicalising -0.0)
__device__ __forceinline__ uint64_t ord64(double x) {
  uint64_t u = (uint64_t)__double_as_longlong(xadd(x, 0.0));
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

struct BeamPtrs {
  double* score;
  uint64_t* h1;
  uint64_t* h2;
  int32_t* last;
  int32_t* pre;
  int32_t* nent;
  Ent* ents;
};

constexpr int ENT_U4 = sizeof(Ent) / 16;


}  // namespace

// =====================================================================================
// K2: persistent frame loop
// =====================================================================================
// Named barriers: 0 = whole CTA, 1 = compute warps, 2 = n-gram -> compute hand-off,
// 3 = n-gram warps.
__device__ __forceinline__ void bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

constexpr int NGT = 64;  // threads of the speculative n-gram warps

// K2: the frame loop.  NC compute threads (8+ warps) run the search; NGT extra threads (two
// warps) evaluate, for every parent that can emit a word boundary this frame, all its
// (entry, surface) score_word lookups speculatively while the compute warps select the top-k,
// so the n-gram memory latency is off the critical path.
template <int NC, bool SMEM_ONLY>
__global__ void __launch_bounds__(NC + NGT, (NC <= 256 ? 2 : 1))
    frames_kernel(ModelDev m, CfgDev c, BatchDev b, Layout L, int t0, int t1, int fusion_mode,
                  double scale) {
  constexpr int NT = NC + NGT;
  constexpr int NWC = NC / 32;
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t dbar[2];
  __shared__ unsigned hist[NBINS];
  __shared__ int hcum[NBINS];   // exclusive prefix of hist (identical in every warp)
  __shared__ int hfill[NBINS];  // counting-sort fill pointers
  __shared__ double wmax[NWC];
  __shared__ double s_maxs;     // max beam score entering the frame
  __shared__ int s_nb, s_ncount, s_fail, s_status, s_K, s_ngP, s_ngcov;
  __shared__ int ngtot[2];
  __shared__ unsigned s_calls, s_probes, s_pairs;

  const int trial = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (b.status[trial] != 0) return;
  const int T = b.T[trial];
  const int tb = t0, te = min(t1, T);
  if (tb >= te) return;

  char* gs = b.gscratch + (int64_t)trial * b.gscratch_stride;
  auto R = [&](int r) -> char* {
    if (SMEM_ONLY) return smem + L.off[r];
    return L.in_smem[r] ? smem + L.off[r] : gs + L.off[r];
  };
  double* dbuf = reinterpret_cast<double*>(R(R_DBUF));
  LexRec* lrows = reinterpret_cast<LexRec*>(R(R_ROWS));  // staged lexicon records (when they fit)
  BeamPtrs cur{(double*)R(R_CUR_SCORE), (uint64_t*)R(R_CUR_H1), (uint64_t*)R(R_CUR_H2),
               (int32_t*)R(R_CUR_LAST), (int32_t*)R(R_CUR_PRE), (int32_t*)R(R_CUR_NENT),
               (Ent*)R(R_CUR_ENTS)};
  BeamPtrs nxt{(double*)R(R_NXT_SCORE), (uint64_t*)R(R_NXT_H1), (uint64_t*)R(R_NXT_H2),
               (int32_t*)R(R_NXT_LAST), (int32_t*)R(R_NXT_PRE), (int32_t*)R(R_NXT_NENT),
               (Ent*)R(R_NXT_ENTS)};
  uint16_t* cbin = reinterpret_cast<uint16_t*>(R(R_CBIN));  // [K*V] histogram bin or 0xFFFF
  double* cval = reinterpret_cast<double*>(R(R_CVAL));
  uint32_t* ckey = reinterpret_cast<uint32_t*>(R(R_CKEY));
  double* sval = reinterpret_cast<double*>(R(R_SVAL));
  uint32_t* skey = reinterpret_cast<uint32_t*>(R(R_SKEY));
  double* nscore = reinterpret_cast<double*>(R(R_NSCORE));
  uint64_t* nh1 = reinterpret_cast<uint64_t*>(R(R_NH1));
  uint64_t* nh2 = reinterpret_cast<uint64_t*>(R(R_NH2));
  int32_t* nlast = reinterpret_cast<int32_t*>(R(R_NLAST));
  int32_t* npre = reinterpret_cast<int32_t*>(R(R_NPRE));
  int32_t* npar = reinterpret_cast<int32_t*>(R(R_NPAR));
  int32_t* rankv = reinterpret_cast<int32_t*>(R(R_RANK));
  int32_t* blist = reinterpret_cast<int32_t*>(R(R_BLIST));
  Ent* bents = reinterpret_cast<Ent*>(R(R_BENTS));
  int32_t* bnent = reinterpret_cast<int32_t*>(R(R_BNENT));
  uint32_t* keep = reinterpret_cast<uint32_t*>(R(R_KEEP));
  WarpScratch* wsc = reinterpret_cast<WarpScratch*>(gs + L.off[R_WARP]);  // always global
  int32_t* ppoff = reinterpret_cast<int32_t*>(R(R_POFF));    // [K+1] per-parent pair offsets
  PairRes* pres = reinterpret_cast<PairRes*>(R(R_PAIRS));    // [pcap]
  int32_t* slotb = reinterpret_cast<int32_t*>(R(R_SLOTB));   // [tslots]
  int32_t* slotm = reinterpret_cast<int32_t*>(R(R_SLOTM));   // [tslots]
  int32_t* myslot = reinterpret_cast<int32_t*>(R(R_MYSLOT)); // [K]

  const int V = m.V, VPD = b.VPD, O = c.O, KC = b.K;
  const int nkw = (c.k + 31) >> 5;
  const int TS = L.tslots;
  const float invV = 1.0f / (float)V;
  // exact `beta * mask` / `gamma * mask` of decoder.py:254-256 as selects (x*1.0 == x)
  const double b_on = c.beta, b_off = xmul(c.beta, 0.0);
  const double g_on = c.gamma, g_off = xmul(c.gamma, 0.0);

  // ---- load the home beam state and gather the first frame's lexicon rows
  int K = b.nbeam[trial];
  {
    const size_t hb = (size_t)trial * KC;
    for (int i = tid; i < K; i += NT) {
      cur.score[i] = b.score[hb + i];
      cur.h1[i] = b.h1[hb + i];
      cur.h2[i] = b.h2[hb + i];
      cur.last[i] = b.last[hb + i];
      cur.pre[i] = b.prefix[hb + i];
      cur.nent[i] = b.nent[hb + i];
      if (L.stage_rows) {
        const LexRec* src = m.lex + b.prefix[hb + i];
        cp_async16(&lrows[i], src);
        cp_async16(reinterpret_cast<char*>(&lrows[i]) + 16, reinterpret_cast<const char*>(src) + 16);
      }
    }
    if (L.stage_rows) cp_async_commit();
    const uint4* src = reinterpret_cast<const uint4*>(b.ents + hb * O);
    uint4* dst = reinterpret_cast<uint4*>(cur.ents);
    for (int i = tid; i < K * O * ENT_U4; i += NT) dst[i] = src[i];
  }
  for (int i = tid; i < NBINS; i += NT) {
    hist[i] = 0;
    hfill[i] = 0;
  }
  if (tid == 0) {
    s_ncount = b.ncount[trial];
    s_fail = 0;
    s_status = 0;
    s_calls = 0;
    s_pairs = 0;
    s_probes = 0;
    s_K = K;
    mbar_init(&dbar[0], 1);
    mbar_init(&dbar[1], 1);
    fence_mbar_init();
  }
  if (L.stage_rows) cp_async_wait_all();
  __syncthreads();
  if (warp == 0) {  // max beam score entering the first frame (home state is not sorted)
    double ms = -DBL_MAX;
    for (int i = lane; i < K; i += 32) ms = fmax(ms, cur.score[i]);
    ms = warp_max(ms);
    if (lane == 0) s_maxs = ms;
  }
  __syncthreads();

  const double* Dtrial = b.D + (size_t)trial * b.Tmax * VPD;
  auto issue_chunk = [&](int ci) {
    const int f0 = tb + ci * CHUNK;
    if (f0 >= te) return;
    const int nf = min(CHUNK, te - f0);
    const unsigned bytes = (unsigned)(nf * VPD * sizeof(double));
    mbar_expect_tx(&dbar[ci & 1], bytes);
    tma_bulk_g2s(dbuf + (size_t)(ci & 1) * CHUNK * VPD, Dtrial + (size_t)f0 * VPD, bytes,
                 &dbar[ci & 1]);
  };
  if (tid == 0) issue_chunk(0);

  unsigned long long st_beams_in = 0, st_beams_out = 0, st_bound = 0, st_fallback = 0;
  unsigned calls_l = 0, probes_l = 0, pairs_l = 0;
  int fail_t = -1;
  // phase timers live in frames_small_kernel<true>; here they would cost registers/spills
#ifdef LB_GENERAL_PHASE_TIMING
  const bool timing = b.phase_cycles != nullptr && tid == 0;
#else
  const bool timing = false;
#endif
  unsigned long long ph[NPHASE];
  for (int i = 0; i < NPHASE; ++i) ph[i] = 0;
  long long tprev = timing ? clock64() : 0;
#define LB_PHASE(i)                                \
  if (timing) {                                    \
    const long long tnow = clock64();              \
    ph[i] += (unsigned long long)(tnow - tprev);   \
    tprev = tnow;                                  \
  }
  auto lrec = [&](int p) -> const LexRec& { return L.stage_rows ? lrows[p] : m.lex[cur.pre[p]]; };

  for (int t = tb; t < te; ++t) {
    const int rel = t - tb;
    const int ci = rel / CHUNK;
    const int cr = rel - ci * CHUNK;
    st_beams_in += K;
    const int KV = K * V;

    if (warp >= NWC) {
      // ============ speculative n-gram warps (decoder.py:293-295 / 182-235 lookups) ============
      const int gt = tid - NC, ngw = warp - NWC;
      int carry = 0;
      for (int base = 0; base < K; base += NGT) {
        const int p = base + gt;
        int np = 0;
        if (p < K) {
          const int ns = lrec(p).ns;
          if (ns > 0 && cur.last[p] != m.space) np = cur.nent[p] * ns;
        }
        int incl = np;
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(FULLMASK, incl, o);
          if (lane >= o) incl += y;
        }
        if (lane == 31) ngtot[ngw] = incl;
        bar_sync(3, NGT);
        const int woff = ngw ? ngtot[0] : 0;
        const int tot = ngtot[0] + ngtot[1];
        if (p < K) ppoff[p] = carry + woff + incl - np;
        carry += tot;
        bar_sync(3, NGT);
      }
      if (gt == 0) {
        ppoff[K] = carry;
        s_ngP = carry;
        if (carry <= min(L.pcap, b.spec_cap)) s_ngcov = carry;
      }
      const int P = carry;
      // parents are in score order: when the pairs exceed the cap, speculate the leading
      // parents whose pairs all fit (s_ngcov pairs); the rest take the warp path after S4
      for (int p = gt; p < K; p += NGT) {
        const int q0 = ppoff[p], q1 = p + 1 < K ? ppoff[p + 1] : P;
        const int scap = min(L.pcap, b.spec_cap);
        if (q1 > scap && q0 <= scap) s_ngcov = q0;  // the first parent that does not fit
      }
      bar_sync(3, NGT);
      const int PCOV = s_ngcov;
      {
        constexpr int NG = NGT / 8;
        const int grp = gt >> 3, sub = lane & 7;
        for (int q0 = 0; q0 < PCOV; q0 += NG) {
          const int q = q0 + grp;
          const bool act = q < PCOV;
          int w = -1, surf = -1, p = 0, e = 0;
          if (act) {
            int lo = 0, hi = K - 1;  // last parent with ppoff[p] <= q
            while (lo < hi) {
              const int mid = (lo + hi + 1) >> 1;
              if (ppoff[mid] <= q) lo = mid;
              else hi = mid - 1;
            }
            p = lo;
            const CompHdr ch = lex_hdr_g(m, lrec(p), cur.pre[p]);
            const int local = q - ppoff[p];
            e = local / ch.ns;
            const int sidx = local - e * ch.ns;
            if (sidx == 0) {
              w = ch.l0;
              surf = ch.s0;
            } else if (sidx == 1) {
              w = ch.l1;
              surf = ch.s1;
            } else {
              w = __ldg(m.comp_lm + ch.off + sidx);
              surf = __ldg(m.comp_surf + ch.off + sidx);
            }
          }
          const Ent& E = cur.ents[(size_t)p * O + e];
          uint32_t hh[MAXH] = {E.h[0], E.h[1], E.h[2]};
          double hb[MAXH] = {E.bo[0], E.bo[1], E.bo[2]};
          WordScore sw;
          group_score_word(m, act, hh, E.hlen, hb, w, sw, probes_l);
          if (act && sub == 0) {
            ++calls_l;
            PairRes pr;
            pr.valid = sw.inc > GUARD;
            pr.total = xadd(E.total, xmul(c.omega, sw.inc));
            pr.cum = xadd(E.cum, sw.inc);
            pr.node = E.node;
            pr.surf = (uint32_t)surf;
            for (int tt = 0; tt < MAXH; ++tt) {
              pr.h[tt] = sw.succ[tt];
              pr.bo[tt] = sw.sbo[tt];
            }
            pr.depth = (uint16_t)(E.depth + 1);
            pr.hlen = (uint8_t)sw.slen;
            pres[q] = pr;
          }
        }
      }
      bar_arrive(2, NT);
    } else {
      // ======================================= compute warps =======================================
      if (cr == 0) {
        mbar_wait(&dbar[ci & 1], (unsigned)((ci >> 1) & 1));
        if (tid == 0) issue_chunk(ci + 1);
      }
      const double* drow = dbuf + ((size_t)(ci & 1) * CHUNK + cr) * VPD;
      // U >= every candidate (rounding up each step of (s + d) + beta + gamma)
      const double U = __dadd_ru(__dadd_ru(__dadd_ru(s_maxs, drow[V]), fmax(c.beta, 0.0)),
                                 fmax(c.gamma, 0.0));
      LB_PHASE(0);

      // ---- A: candidate values (decoder.py:252-260) + histogram over bins anchored at U
      double wm = -DBL_MAX;
      for (int f = tid; f < KV; f += NC) {
        const int p = (int)(((float)f + 0.5f) * invV);
        const int v = f - p * V;
        const int lp = cur.last[p];
        uint16_t bin = 0xFFFF;
        if (((lrec(p).mask >> v) & 1ull) || (v == m.blank) || (v == lp)) {
          double x = xadd(cur.score[p], drow[v]);
          const bool ph2 = (v != m.blank) & (v != m.space);
          x = xadd(x, (ph2 && v != lp) ? b_on : b_off);
          if (v == m.space) x = xadd(x, lp != m.space ? g_on : g_off);
          if (x > GUARD) {
            const double fb = fmin(fmax(xmul(xsub(U, x), c.inv_binw), 0.0), (double)(NBINS - 1));
            bin = (uint16_t)(int)fb;
            atomicAdd(&hist[bin], 1u);
            wm = fmax(wm, x);
          }
        }
        cbin[f] = bin;
      }
      wm = warp_max(wm);
      LB_PHASE(11);
      if (lane == 0) wmax[warp] = wm;
      if (tid == 0) s_nb = 0;
      for (int i = tid; i < nkw; i += NC) keep[i] = 0;
      for (int i = tid; i < TS; i += NC) {
        slotb[i] = -1;
        slotm[i] = 0x7FFFFFFF;
      }
      bar_sync(1, NC);  // S1
      LB_PHASE(1);

      double M = -DBL_MAX;
      for (int w = 0; w < NWC; ++w) M = fmax(M, wmax[w]);
      int nsel = 0;
      bool dead = !(M > GUARD);  // decoder.py:267-268
      if (dead) {
        if (tid == 0) {
          s_status = 1;
          s_K = 0;
        }
        fail_t = t;
      } else {
        const double thr = xsub(M, c.theta);
        const int bthr =
            (int)fmin(fmax(xmul(xsub(U, thr), c.inv_binw), 0.0), (double)(NBINS - 1));
        // ---- C: every warp scans the histogram in registers; warp 0 publishes hcum[]
        int bstar = NBINS, cum_thr = 0, cum_bstar = 0;
        {
          constexpr int PB = NBINS / 32;
          int part[PB];
          int ls = 0;
#pragma unroll
          for (int i = 0; i < PB; ++i) {
            part[i] = (int)hist[lane * PB + i];
            ls += part[i];
          }
          int incl = ls;
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULLMASK, incl, o);
            if (lane >= o) incl += y;
          }
          const int excl = incl - ls;
          if (warp == 0) {
            int run = excl;
#pragma unroll
            for (int i = 0; i < PB; ++i) {
              hcum[lane * PB + i] = run;
              run += part[i];
            }
          }
          bar_sync(1, NC);  // hcum[] visible to every compute warp
          __syncwarp();
          cum_thr = hcum[bthr] + (int)hist[bthr];
          const bool here = excl < c.k && incl >= c.k;
          const unsigned bl = __ballot_sync(FULLMASK, here);
          if (bl) {
            const int src = __ffs(bl) - 1;
            int lb = 0;
            if (lane == src) {
              int cum = excl;
#pragma unroll
              for (int i = 0; i < PB; ++i) {
                if (cum + part[i] >= c.k) {
                  lb = i;
                  break;
                }
                cum += part[i];
              }
            }
            lb = __shfl_sync(FULLMASK, lb, src);
            bstar = src * PB + lb;
            cum_bstar = hcum[bstar] + (int)hist[bstar];
          }
        }
        const bool sure = bstar < bthr;  // bins < bthr are entirely >= thr
        const int take_bin = sure ? bstar : bthr;
        const int bound = sure ? cum_bstar : cum_thr;
        if (bound <= L.lcap) {
          // ---- D: collect = counting sort by bin (bins are strictly ordered by value)
          for (int f = tid; f < KV; f += NC) {
            const int bn = cbin[f];
            if (bn <= take_bin) {
              const int p = (int)(((float)f + 0.5f) * invV);
              const int v = f - p * V;
              const double x = cand_value(cur.score[p], drow[v], v, cur.last[p],
                                          FrameConsts{c.beta, c.gamma, m.blank, m.space});
              if (sure || x >= thr) {
                const int pos = hcum[bn] + atomicAdd(&hfill[bn], 1);
                cval[pos] = x;
                ckey[pos] = (uint32_t)f;
              }
            }
          }
          bar_sync(1, NC);  // S2
          const int m_sel = hcum[take_bin] + hfill[take_bin];
          nsel = min(c.k, m_sel);
          LB_PHASE(2);
          // ---- E: exact order inside each bin (value desc, flat index asc)
          for (int a = tid; a < m_sel; a += NC) {
            const double va = cval[a];
            const uint32_t ka = ckey[a];
            const int bn = cbin[ka];
            const int lo = hcum[bn], n = hfill[bn];
            int r = lo;
            for (int q = lo; q < lo + n; ++q) {
              const double vq = cval[q];
              r += (vq > va) || (vq == va && ckey[q] < ka);
            }
            if (r < nsel) {
              sval[r] = va;
              skey[r] = ka;
            }
          }
        } else {
          // ---- fallback: exact radix select on the 96-bit key (ord64(value), ~flat index)
          ++st_fallback;
          auto cval_at = [&](int f) -> double {
            if (cbin[f] == 0xFFFF) return -DBL_MAX;
            const int p = (int)(((float)f + 0.5f) * invV);
            const int v = f - p * V;
            return cand_value(cur.score[p], drow[v], v, cur.last[p],
                              FrameConsts{c.beta, c.gamma, m.blank, m.space});
          };
          __shared__ int s_cnt2, s_inr;
          bar_sync(1, NC);
          if (tid == 0) {
            s_cnt2 = 0;
            s_inr = 0;
          }
          bar_sync(1, NC);
          for (int f = tid; f < KV; f += NC)
            if (cval_at(f) >= thr) atomicAdd(&s_inr, 1);
          bar_sync(1, NC);
          nsel = min(c.k, s_inr);
          uint64_t phi = 0, pmask_hi = 0;
          uint32_t plo = 0, pmask_lo = 0;
          int rem = nsel;
          for (int pass = 0; pass < 12; ++pass) {
            bar_sync(1, NC);
            for (int i = tid; i < NBINS; i += NC) hist[i] = 0;
            bar_sync(1, NC);
            for (int f = tid; f < KV; f += NC) {
              const double x = cval_at(f);
              if (!(x >= thr)) continue;
              const uint64_t kh = ord64(x);
              const uint32_t kl = ~(uint32_t)f;
              if ((kh & pmask_hi) != phi || (kl & pmask_lo) != plo) continue;
              const unsigned dg = pass < 8 ? (unsigned)((kh >> (56 - 8 * pass)) & 0xFF)
                                           : (unsigned)((kl >> (24 - 8 * (pass - 8))) & 0xFF);
              atomicAdd(&hist[dg], 1u);
            }
            bar_sync(1, NC);
            int above = 0, dsel = 0;
            for (int d = NBINS - 1; d >= 0; --d) {
              const int h = (int)hist[d];
              if (above + h >= rem) {
                dsel = d;
                break;
              }
              above += h;
            }
            rem -= above;
            if (pass < 8) {
              phi |= (uint64_t)dsel << (56 - 8 * pass);
              pmask_hi |= 0xFFull << (56 - 8 * pass);
            } else {
              plo |= (uint32_t)dsel << (24 - 8 * (pass - 8));
              pmask_lo |= 0xFFu << (24 - 8 * (pass - 8));
            }
          }
          bar_sync(1, NC);
          for (int f0 = 0; f0 < KV; f0 += NC) {
            const int f = f0 + tid;
            bool take = false;
            double x = 0.0;
            if (f < KV) {
              x = cval_at(f);
              if (x >= thr) {
                const uint64_t kh = ord64(x);
                const uint32_t kl = ~(uint32_t)f;
                take = kh > phi || (kh == phi && kl >= plo);
              }
            }
            const unsigned bl = __ballot_sync(FULLMASK, take);
            if (bl) {
              int base = 0;
              if (lane == 0) base = atomicAdd(&s_cnt2, __popc(bl));
              base = __shfl_sync(FULLMASK, base, 0);
              if (take) {
                const int pos = base + __popc(bl & ((1u << lane) - 1u));
                cval[pos] = x;
                ckey[pos] = (uint32_t)f;
              }
            }
          }
          bar_sync(1, NC);
          for (int i = tid; i < nsel; i += NC) {
            const double vi = cval[i];
            const uint32_t ki = ckey[i];
            int cnt = 0;
            for (int j = 0; j < nsel; ++j) {
              const double vj = cval[j];
              cnt += (vj > vi) || (vj == vi && ckey[j] < ki);
            }
            sval[cnt] = vi;
            skey[cnt] = ki;
          }
          for (int i = tid; i < NBINS; i += NC) hist[i] = 0;
        }
      }
      bar_sync(2, NT);  // S3: selection done + speculative n-gram results ready
      LB_PHASE(3);

      if (!dead) {
        const int ncov = s_ngcov;
        const bool ngover = ncov < s_ngP;  // some parents' pairs were not speculated
        // ---- F: materialise survivors (decoder.py:272-291); a new word-boundary emitter merges
        // its parent's precomputed (entry, surface) pairs (decoder.py:208-235) right here
        for (int j = tid; j < nsel; j += NC) {
          const double x = sval[j];
          const uint32_t f = skey[j];
          const int p = (int)(((float)f + 0.5f) * invV);
          const int tok = (int)f - p * V;
          const int lp = cur.last[p], pp = cur.pre[p];
          const bool emit = (tok != m.blank) && (tok != lp);
          uint64_t a1 = cur.h1[p], a2 = cur.h2[p];
          int np = pp;
          if (emit) {
            a1 = a1 * H_MULT1 + (uint64_t)(tok + 1);
            a2 = a2 * H_MULT2 + (uint64_t)(tok + 1);
            np = lex_succ(m, lrec(p), tok);
          }
          double sc = x;
          int bn = -1;
          if (emit && tok == m.space) {
            blist[atomicAdd(&s_nb, 1)] = j;
            pairs_l += (unsigned)(ppoff[p + 1] - ppoff[p]);
            if (ppoff[p + 1] > ncov) {
              bn = -2;  // resolved below by the warp-per-beam path
            } else {
              const int q0 = ppoff[p], q1 = ppoff[p + 1];
              // running top-O list (total desc, q asc); every index below is a compile-time
              // constant after unrolling, so the list lives in registers (no local memory)
              int top[OMAX];
#pragma unroll
              for (int i = 0; i < OMAX; ++i) top[i] = 0;
              int ntop = 0;
              for (int q = q0; q < q1; ++q) {
                if (!pres[q].valid) continue;
                const double tq = pres[q].total;
                int pos = ntop;
#pragma unroll
                for (int i = OMAX - 1; i >= 0; --i)
                  if (i < ntop && tq > pres[top[i]].total) pos = i;
                if (pos >= O) continue;
#pragma unroll
                for (int i = OMAX - 1; i > 0; --i)
                  if (i > pos && i <= ntop) top[i] = top[i - 1];
#pragma unroll
                for (int i = 0; i < OMAX; ++i)
                  if (i == pos) top[i] = q;
                ntop = min(ntop + 1, O);
              }
              if (ntop == 0) {
                sc = NEG_INF;  // decoder.py:223-225
              } else {
                const double best = pres[top[0]].total;
                const double floor_ = xsub(best, c.lambda);
                int kept = 0;
#pragma unroll
                for (int i = 0; i < OMAX; ++i)
                  if (kept == i && i < ntop && pres[top[i]].total >= floor_) kept = i + 1;
                const int base = atomicAdd(&s_ncount, kept);
                if (base + kept > b.ncap) {
                  s_fail = 1;
                  sc = NEG_INF;
                } else {
                  const size_t nbase = (size_t)trial * b.ncap;
                  Ent* out = bents + (size_t)j * O;
#pragma unroll
                  for (int i = 0; i < OMAX; ++i) {
                    if (i >= kept) break;
                    const PairRes& pr = pres[top[i]];
                    const uint32_t node = (uint32_t)(base + i);
                    b.nparent[nbase + node] = pr.node;
                    b.nsurf[nbase + node] = pr.surf;
                    WordScore sw;
                    sw.slen = pr.hlen;
                    for (int tt = 0; tt < MAXH; ++tt) {
                      sw.succ[tt] = pr.h[tt];
                      sw.sbo[tt] = pr.bo[tt];
                    }
                    new_entry(out[i], pr.total, pr.cum, sw, node, (uint32_t)(top[i] - q0),
                              pr.depth);
                  }
                  bn = kept;
                  sc = xadd(x, xsub(best, cur.ents[(size_t)p * O].total));
                }
              }
            }
          }
          nscore[j] = sc;
          nh1[j] = a1;
          nh2[j] = a2;
          nlast[j] = (tok == m.blank) ? lp : tok;
          npre[j] = np;
          npar[j] = p;
          bnent[j] = bn;
        }
        bar_sync(1, NC);  // S4
        LB_PHASE(4);
        const int nb = s_nb;
        st_bound += nb;
        if (ngover && nb > 0) {
          // rare: more pairs than the speculative round holds -> one warp per boundary beam
          for (int bi = warp; bi < nb; bi += NWC) {
            const int j = blist[bi];
            if (bnent[j] != -2) continue;  // speculated parent
            const int p = npar[j];
            int outn = -1;
            double sc = nscore[j];
            warp_apply_ngram(m, c, b, trial, cur.ents + (size_t)p * O, cur.nent[p],
                             lex_hdr_g(m, lrec(p), cur.pre[p]), &wsc[warp], bents + (size_t)j * O, &outn, &sc,
                             &s_ncount, &s_fail, calls_l, probes_l);
            if (lane == 0) {
              nscore[j] = sc;
              bnent[j] = outn;
            }
          }
          bar_sync(1, NC);
        }
        LB_PHASE(5);
    // ---- H1: recombination ranking by (post-fusion score desc, index asc).  Beams that did
    // not cross a word boundary keep their selection scores, which are already in that order,
    // so only the nb boundary beams need explicit comparisons.  Equal-hash groups are found
    // with a shared-memory table (exact (h1, h2) equality); each group keeps its best rank.
    {
      const int n = nsel;
      int G = 1;
      while (G < 32 && 2 * G * n <= NC) G <<= 1;
      const int groups = NC / G, g = tid / G, r = tid & (G - 1);
      for (int i0 = 0; i0 < n; i0 += groups) {
        const int i = i0 + g;
        const bool act = i < n;
        const double si = act ? nscore[i] : 0.0;
        const bool ib = act && (bnent[i] != -1 || si <= GUARD);  // crossed a boundary
        int cnt = 0;
        if (act) {
          // regular beams keep sval order (score desc, j asc): those beating a boundary beam
          // are the regular indices below e (two binary searches over sval); the boundary
          // beams below e are subtracted in the loop that compares the boundary beams
          int e = 0;
          if (ib) {
            int lo = 0, hi = n;  // first j with sval[j] <= si
            while (lo < hi) {
              const int mid = (lo + hi) >> 1;
              if (sval[mid] > si) lo = mid + 1;
              else hi = mid;
            }
            const int a = lo;
            hi = n;  // first j with sval[j] < si
            while (lo < hi) {
              const int mid = (lo + hi) >> 1;
              if (sval[mid] >= si) lo = mid + 1;
              else hi = mid;
            }
            e = max(a, min(lo, i));
          }
          // boundary beams beating i (+ count of boundary beams before i when i is regular)
          for (int k2 = r; k2 < nb; k2 += G) {
            const int j = blist[k2];
            const double sj = nscore[j];
            cnt += (sj > si) || (sj == si && j < i);
            cnt -= ib ? (j < e) : (j < i);
          }
          if (ib && r == 0) cnt += e;
        }
        for (int o = G >> 1; o > 0; o >>= 1) cnt += __shfl_xor_sync(FULLMASK, cnt, o);
        if (act && r == 0) {
          if (!ib) cnt += i;  // regular beams before i all beat it
          rankv[i] = cnt;
          if (si > GUARD) {
            const uint64_t a1 = nh1[i], a2 = nh2[i];
            int h = (int)((a1 ^ (a2 * 0x9E3779B97F4A7C15ull)) >> 20) & (TS - 1);
            for (;;) {
              const int owner = atomicCAS(&slotb[h], -1, i);
              if (owner == -1 || (nh1[owner] == a1 && nh2[owner] == a2)) break;
              h = (h + 1) & (TS - 1);
            }
            myslot[i] = h;
            atomicMin(&slotm[h], cnt);
          }
        }
      }
    }
    bar_sync(1, NC);  // S6
    LB_PHASE(6);
    // ---- H2: survivors = best rank of each hash group, killed beams dropped
    for (int i = tid; i < nsel; i += NC) {
      if (nscore[i] > GUARD && slotm[myslot[i]] == rankv[i])
        atomicOr(&keep[rankv[i] >> 5], 1u << (rankv[i] & 31));
    }
    bar_sync(1, NC);  // S7
    LB_PHASE(7);

    // ---- scatter survivors into the next buffer in rank order; prefetch their lexicon rows
    for (int i = tid; i < NBINS; i += NC) {  // scanned after S1 / filled before S2: free again
      hist[i] = 0;
      hfill[i] = 0;
    }
    int newK = 0;
    for (int w = 0; w < nkw; ++w) newK += __popc(keep[w]);
    {
      int G = 1;
      while (G < 32 && 2 * G * nsel <= NC) G <<= 1;
      const int groups = NC / G, g = tid / G, r = tid & (G - 1);
      for (int i0 = 0; i0 < nsel; i0 += groups) {
        const int i = i0 + g;
        if (i >= nsel) continue;
        const int rk = rankv[i];
        if (!((keep[rk >> 5] >> (rk & 31)) & 1u)) continue;
        int pos = __popc(keep[rk >> 5] & ((1u << (rk & 31)) - 1u));
        for (int w = 0; w < (rk >> 5); ++w) pos += __popc(keep[w]);
        const int bn = bnent[i];
        const Ent* srcE = bn >= 0 ? bents + (size_t)i * O : cur.ents + (size_t)npar[i] * O;
        const int cnt = bn >= 0 ? bn : cur.nent[npar[i]];
        if (r == 0) {
          if (pos == 0) s_maxs = nscore[i];  // survivors are sorted: rank 0 is the maximum
          nxt.score[pos] = nscore[i];
          nxt.h1[pos] = nh1[i];
          nxt.h2[pos] = nh2[i];
          nxt.last[pos] = nlast[i];
          nxt.pre[pos] = npre[i];
          nxt.nent[pos] = cnt;
          if (b.dump_k) {
            const size_t di = ((size_t)trial * b.Tmax + t) * KC + pos;
            b.dump_h1[di] = nh1[i];
            b.dump_h2[di] = nh2[i];
            b.dump_pre[di] = npre[i];
            b.dump_last[di] = nlast[i];
            b.dump_score[di] = nscore[i];
          }
        }
        const uint4* su = reinterpret_cast<const uint4*>(srcE);
        uint4* du = reinterpret_cast<uint4*>(nxt.ents + (size_t)pos * O);
        for (int u = r; u < cnt * ENT_U4; u += G) du[u] = su[u];
        if (L.stage_rows)
          for (int u = r; u < 2; u += G)  // the record's two 16-B halves (G may be 1)
            cp_async16(reinterpret_cast<char*>(&lrows[pos]) + 16 * u,
                       reinterpret_cast<const char*>(m.lex + npre[i]) + 16 * u);
      }
      if (L.stage_rows) {
        cp_async_commit();
        cp_async_wait_all();
      }
    }
    if (b.dump_k && tid == 0) b.dump_k[(size_t)trial * b.Tmax + t] = newK;
    if (tid == 0) {
      s_K = newK;
      if (s_fail) s_status = 4;
      else if (newK == 0) s_status = 2;  // decoder.py:314-315
    }
    if (s_fail || newK == 0) fail_t = t;
      }  // !dead
    }  // compute warps
    __syncthreads();  // S8: frame end (whole CTA)
    LB_PHASE(8);
    {
      BeamPtrs tmp = cur;
      cur = nxt;
      nxt = tmp;
    }
    K = s_K;
    st_beams_out += K;
    if (s_status != 0) break;

    // ---- optional interval fusion of the device n-gram scorer (decoder.py:428-430)
    if (fusion_mode == 1 && t > 0 && (t % c.r) == 0) {
      for (int i = tid; i < K; i += NT) {
        Ent* e = cur.ents + (size_t)i * O;
        const int n = cur.nent[i];
        const double prev = e[0].total;
        for (int q = 0; q < n; ++q) {
          if (e[q].node == 0) {
            e[q].total = 0.0;
            e[q].punct = 0;
          } else {
            e[q].total = xmul(c.phi, xmul(scale, e[q].cum));
          }
        }
        sort_entries(e, n);
        cur.score[i] = xadd(cur.score[i], xsub(e[0].total, prev));
      }
      __syncthreads();
      if (warp == 0) {
        double ms = -DBL_MAX;
        for (int i = lane; i < K; i += 32) ms = fmax(ms, cur.score[i]);
        ms = warp_max(ms);
        if (lane == 0) s_maxs = ms;
      }
      __syncthreads();
      LB_PHASE(10);
    }
    LB_PHASE(9);
  }

  // ---- write back
  __syncthreads();
  if (timing)
    for (int i = 0; i < NPHASE; ++i) b.phase_cycles[(size_t)trial * NPHASE + i] += ph[i];
#undef LB_PHASE
  const int status = s_status;
  if (tid == 0) {
    if (status != 0) {
      b.status[trial] = status;
      b.fail_frame[trial] = fail_t;
    }
    b.nbeam[trial] = K;
    b.ncount[trial] = s_ncount;
  }
  if (status == 0 || status == 4) {
    const size_t hb = (size_t)trial * KC;
    for (int i = tid; i < K; i += NT) {
      b.score[hb + i] = cur.score[i];
      b.h1[hb + i] = cur.h1[i];
      b.h2[hb + i] = cur.h2[i];
      b.last[hb + i] = cur.last[i];
      b.prefix[hb + i] = cur.pre[i];
      b.nent[hb + i] = cur.nent[i];
    }
    const uint4* src = reinterpret_cast<const uint4*>(cur.ents);
    uint4* dst = reinterpret_cast<uint4*>(b.ents + hb * O);
    for (int i = tid; i < K * O * ENT_U4; i += NT) dst[i] = src[i];
  }
  atomicAdd(&s_calls, calls_l);
  if (pairs_l) atomicAdd(&s_pairs, pairs_l);
  atomicAdd(&s_probes, probes_l);
  __syncthreads();
  if (tid == 0) {
    unsigned long long* stt = b.stats + (size_t)trial * 8;
    stt[0] += (unsigned long long)(te - tb);
    stt[1] += st_beams_in;
    stt[2] += st_beams_out;
    stt[3] += s_calls;
    stt[4] += s_probes;
    stt[5] += st_bound;
    stt[6] += s_pairs;  // (entry, surface) pairs the boundary beams consume (reference score_word calls)
    stt[7] += st_fallback;
  }
}

// =====================================================================================
// K2s: frames kernel specialised for k <= 64, ortho_beams <= 4, V <= 48 (every BASELINE
// config at beam 16/64 and all reference fixtures).  Same algorithm as frames_kernel; the
// whole working set has a compile-time shared-memory layout (immediate-offset addressing, no
// pointer registers), candidate bins stay in registers (transposed thread <-> token mapping),
// and word-boundary entries are built straight from the speculative pair results.
// =====================================================================================
namespace small {
constexpr int KC = 64, OC = 3, VC = 48, VPDC = 50;
// PC: speculative (entry, surface) pairs per frame -- 64..80 measured best at config 2 (7.23 ms
// at 160 -> 7.13 ms; the n-gram warps are the critical path up to S3 and the uncovered parents'
// few selected boundary beams take the warp path); LC 280 and 4-frame D chunks keep two CTAs
// inside the 132 KB shared-memory carve-out (124 KB of L1 for the lexicon / n-gram probes)
constexpr int LC = 280, PC = 80, SCHUNK = 4;
constexpr int NC = 256, NWC = NC / 32, NT = NC + NGT;
constexpr int TBK = VC / 4;  // candidate tokens per thread: 4 threads per parent
static_assert(KC * 4 == NC && TBK % 4 == 0, "candidate mapping: one parent per 4 threads");
// Beam state by slot (double-buffered by frame parity): beams live in the slot their selection
// gave them (slot j = rank j of the frame's top-k selection); JMAP lists the slots of the kept
// beams in post-fusion score order, so parent p of the next frame is slot JMAP[p] -- no beam is
// moved at the end of a frame.  JMAP is indexed by the rank among all selected beams, with -1
// holes for the ones recombination dropped (ranks are monotone in the compacted positions, so
// every (parent, token) tie-break is unchanged) -- no compaction pass per frame.  LROW / LOFF: the lexicon record and completion-CSR offset of a
// beam's prefix state, gathered by cp.async as soon as the beam is materialised.
constexpr int B_SCORE = 0, B_H1 = KC * 8, B_H2 = 2 * KC * 8, B_LAST = 3 * KC * 8,
              B_PRE = 3 * KC * 8 + KC * 4, B_NENT = 3 * KC * 8 + 2 * KC * 4,
              B_JMAP = 3 * KC * 8 + 3 * KC * 4, B_LOFF = B_JMAP + KC * 4, B_LROW = B_LOFF + KC * 4,
              B_ENTS = B_LROW + KC * (int)sizeof(LexRec);
static_assert(B_LROW % 16 == 0 && B_ENTS % 16 == 0, "16-byte aligned beam arrays");
constexpr int BEAM_BYTES = B_ENTS + KC * OC * (int)sizeof(Ent);
constexpr int O_DBUF = 0;
constexpr int O_BEAM = O_DBUF + 2 * SCHUNK * VPDC * 8;
constexpr int O_CVAL = O_BEAM + 2 * BEAM_BYTES;
constexpr int O_CKEY = O_CVAL + LC * 8;
constexpr int O_CBINL = O_CKEY + LC * 4;
constexpr int O_SVAL = O_CBINL + LC * 2;
constexpr int O_SKEY = O_SVAL + KC * 8;
constexpr int O_NPAR = O_SKEY + KC * 4;
constexpr int O_RANK = O_NPAR + KC * 4;
constexpr int O_BLIST = O_RANK + KC * 4;
constexpr int O_BSEL = O_BLIST + KC * 4;
constexpr int O_KEEP = O_BSEL + KC * 16;
constexpr int O_POFF = O_KEEP + 16;
constexpr int O_PRES = O_POFF + ((KC + 1) * 4 + 15) / 16 * 16;
constexpr int O_NFP = O_PRES + PC * (int)sizeof(PairRes);
constexpr int O_QINFO = O_NFP + KC * 4;  // int4 per speculative pair: (entry slot, word, surface, parent)
constexpr int O_PTOP = O_QINFO + PC * 16;  // int4 per parent: its top-o speculated pairs (-1: none)
constexpr int O_PVAL = O_PTOP + KC * 16;   // per speculative pair: its new total, or -inf if killed
constexpr int TOTAL = O_PVAL + PC * 8;
static_assert(O_BEAM % 16 == 0 && O_CVAL % 16 == 0 && O_PRES % 16 == 0 && BEAM_BYTES % 16 == 0,
              "16-byte alignment");
// global scratch per trial: the warp path's top-o lists
constexpr int G_WARP = 0;
constexpr int GTOTAL = G_WARP + NWC * (int)sizeof(WarpScratch);
}  // namespace small

#ifdef LB_INLINE_FALLBACK
#define LB_COLD __forceinline__
#else
#define LB_COLD __noinline__
#endif
// Exact radix-select fallback of frames_small_kernel (a histogram bin overflowed LC): compiled
// out of line so its ~1300 instructions stay out of the frame loop's instruction-cache footprint.
// Called by all NC compute threads; returns nsel with sval/skey in (value desc, index asc) order.
__device__ LB_COLD int small_fallback_select(const int ck, const double cbeta, const double cgamma,
                                             int K, int V, double thr,
                                             int blank, int space, const int32_t* jmap,
                                             const LexRec* lrow,
                                             const int32_t* C_LAST, const double* C_SCORE,
                                             const double* drow, unsigned* hist, double* cval,
                                             uint32_t* ckey, double* sval, uint32_t* skey,
                                             int* s_inr, int* s_cnt2) {
  using namespace small;
  const int tid = threadIdx.x, lane = tid & 31;
  int nsel;
  // ---- fallback: exact radix select on the 96-bit key (ord64(value), ~flat index)
  auto cval_at = [&](int f) -> double {
    const int p = f / V, v = f - (f / V) * V;
    const int jp = jmap[p];
    if (jp < 0) return -DBL_MAX;  // a dropped rank (hole)
    const int lp = C_LAST[jp];
    if (!(((lrow[jp].mask >> v) & 1ull) || (v == blank) || (v == lp))) return -DBL_MAX;
    const double x = cand_value(C_SCORE[jp], drow[v], v, lp,
                                FrameConsts{cbeta, cgamma, blank, space});
    return x > GUARD ? x : -DBL_MAX;
  };
  const int KV = K * V;
  bar_sync(1, NC);
  if (tid == 0) {
    (*s_cnt2) = 0;
    (*s_inr) = 0;
  }
  bar_sync(1, NC);
  for (int f = tid; f < KV; f += NC)
    if (cval_at(f) >= thr) atomicAdd(s_inr, 1);
  bar_sync(1, NC);
  nsel = min(ck, (*s_inr));
  uint64_t phi = 0, pmask_hi = 0;
  uint32_t plo = 0, pmask_lo = 0;
  int rem = nsel;
  for (int pass = 0; pass < 12; ++pass) {
    bar_sync(1, NC);
    for (int i = tid; i < NBINS; i += NC) hist[i] = 0;
    bar_sync(1, NC);
    for (int f = tid; f < KV; f += NC) {
      const double x = cval_at(f);
      if (!(x >= thr)) continue;
      const uint64_t kh = ord64(x);
      const uint32_t kl = ~(uint32_t)f;
      if ((kh & pmask_hi) != phi || (kl & pmask_lo) != plo) continue;
      const unsigned dg = pass < 8 ? (unsigned)((kh >> (56 - 8 * pass)) & 0xFF)
                                   : (unsigned)((kl >> (24 - 8 * (pass - 8))) & 0xFF);
      atomicAdd(&hist[dg], 1u);
    }
    bar_sync(1, NC);
    int above = 0, dsel = 0;
    for (int d = NBINS - 1; d >= 0; --d) {
      const int h = (int)hist[d];
      if (above + h >= rem) {
        dsel = d;
        break;
      }
      above += h;
    }
    rem -= above;
    if (pass < 8) {
      phi |= (uint64_t)dsel << (56 - 8 * pass);
      pmask_hi |= 0xFFull << (56 - 8 * pass);
    } else {
      plo |= (uint32_t)dsel << (24 - 8 * (pass - 8));
      pmask_lo |= 0xFFu << (24 - 8 * (pass - 8));
    }
  }
  bar_sync(1, NC);
  for (int f0 = 0; f0 < KV; f0 += NC) {
    const int f = f0 + tid;
    bool take = false;
    double x = 0.0;
    if (f < KV) {
      x = cval_at(f);
      if (x >= thr) {
        const uint64_t kh = ord64(x);
        const uint32_t kl = ~(uint32_t)f;
        take = kh > phi || (kh == phi && kl >= plo);
      }
    }
    const unsigned bl = __ballot_sync(FULLMASK, take);
    if (bl) {
      int base = 0;
      if (lane == 0) base = atomicAdd(s_cnt2, __popc(bl));
      base = __shfl_sync(FULLMASK, base, 0);
      if (take) {
        const int pos = base + __popc(bl & ((1u << lane) - 1u));
        cval[pos] = x;
        ckey[pos] = ((uint32_t)(f / V) << 8) | (uint32_t)(f % V);  // (parent, token) key
      }
    }
  }
  bar_sync(1, NC);
  for (int i = tid; i < nsel; i += NC) {
    const double vi = cval[i];
    const uint32_t ki = ckey[i];
    int cnt = 0;
    for (int j = 0; j < nsel; ++j) {
      const double vj = cval[j];
      cnt += (vj > vi) || (vj == vi && ckey[j] < ki);
    }
    sval[cnt] = vi;
    skey[cnt] = ki;
  }
  for (int i = tid; i < NBINS; i += NC) hist[i] = 0;
  return nsel;
}

template <bool TIMING>
__global__ void __launch_bounds__(small::NT, 2)
    frames_small_kernel(ModelDev m, CfgDev c, BatchDev b, int t0, int t1, int fusion_mode,
                        double scale) {
  using namespace small;
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t dbar[2];
  __shared__ unsigned hist[NBINS + 32];  // + one spare bin per lane for rejected candidates
  __shared__ int hcum[NBINS];  // exclusive prefix of hist (published by warp 0)
  __shared__ int hfill[NBINS];
  __shared__ double wmax[NWC];
  __shared__ double s_maxs;
  __shared__ int s_nb, s_ncount, s_fail, s_status, s_K, s_ngP, s_ngcov, s_inr, s_cnt2, s_nsel;
  __shared__ int s_live[2];  // surviving beams of a frame, by frame parity
  __shared__ int ngtot[2];
  __shared__ unsigned s_calls, s_probes, s_pairs;
  __shared__ unsigned s_tarr[NBAR_EV], s_tbase;  // TIMING only
  __shared__ unsigned long long ph[NPHASE];       // TIMING only (thread 0): no register cost

  const int trial = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (b.status[trial] != 0) return;
  const int T = b.T[trial];
  const int tb = t0, te = min(t1, T);
  if (tb >= te) return;
  char* gs = b.gscratch + (int64_t)trial * b.gscratch_stride;

  double* dbuf = reinterpret_cast<double*>(sm + O_DBUF);
  double* cval = reinterpret_cast<double*>(sm + O_CVAL);
  uint32_t* ckey = reinterpret_cast<uint32_t*>(sm + O_CKEY);
  uint16_t* cbinl = reinterpret_cast<uint16_t*>(sm + O_CBINL);
  double* sval = reinterpret_cast<double*>(sm + O_SVAL);
  uint32_t* skey = reinterpret_cast<uint32_t*>(sm + O_SKEY);
  int32_t* npar = reinterpret_cast<int32_t*>(sm + O_NPAR);
  int32_t* rankv = reinterpret_cast<int32_t*>(sm + O_RANK);
  int32_t* blist = reinterpret_cast<int32_t*>(sm + O_BLIST);
  // per slot: {kept pairs | -1 inherit | -2 warp path pending | -3 entries built, node base,
  // top01, top23}
  int4* bsel = reinterpret_cast<int4*>(sm + O_BSEL);
  uint32_t* keep = reinterpret_cast<uint32_t*>(sm + O_KEEP);
  int32_t* ppoff = reinterpret_cast<int32_t*>(sm + O_POFF);
  PairRes* pres = reinterpret_cast<PairRes*>(sm + O_PRES);
  uint32_t* nfp = reinterpret_cast<uint32_t*>(sm + O_NFP);  // hash-lane fingerprints (recombination)
  WarpScratch* wsc = reinterpret_cast<WarpScratch*>(gs + G_WARP);

  // beam buffers selected by parity: cur = buffer `par`, nxt = buffer `par ^ 1`
  int par = 0;
#define BUF(pp) (sm + O_BEAM + (pp) * BEAM_BYTES)
#define C_SCORE ((double*)(BUF(par) + B_SCORE))
#define C_H1 ((uint64_t*)(BUF(par) + B_H1))
#define C_H2 ((uint64_t*)(BUF(par) + B_H2))
#define C_LAST ((int32_t*)(BUF(par) + B_LAST))
#define C_PRE ((int32_t*)(BUF(par) + B_PRE))
#define C_NENT ((int32_t*)(BUF(par) + B_NENT))
#define C_ENTS ((Ent*)(BUF(par) + B_ENTS))
#define X_SCORE ((double*)(BUF(par ^ 1) + B_SCORE))
#define X_H1 ((uint64_t*)(BUF(par ^ 1) + B_H1))
#define X_H2 ((uint64_t*)(BUF(par ^ 1) + B_H2))
#define X_LAST ((int32_t*)(BUF(par ^ 1) + B_LAST))
#define X_PRE ((int32_t*)(BUF(par ^ 1) + B_PRE))
#define X_NENT ((int32_t*)(BUF(par ^ 1) + B_NENT))
#define X_ENTS ((Ent*)(BUF(par ^ 1) + B_ENTS))
#define C_JMAP ((int32_t*)(BUF(par) + B_JMAP))
#define C_LOFF ((int32_t*)(BUF(par) + B_LOFF))
#define C_LROW ((LexRec*)(BUF(par) + B_LROW))
#define X_JMAP ((int32_t*)(BUF(par ^ 1) + B_JMAP))
#define X_LOFF ((int32_t*)(BUF(par ^ 1) + B_LOFF))
#define X_LROW ((LexRec*)(BUF(par ^ 1) + B_LROW))

  const int V = m.V, VPD = b.VPD, O = c.O, KC_ = b.K;
  const double ibw = c.inv_binw;
  const double b_on = c.beta, b_off = xmul(c.beta, 0.0);
  const double g_on = c.gamma, g_off = xmul(c.gamma, 0.0);
  const int blank = m.blank, space = m.space;
  // candidate mapping: thread -> parent cp = tid / 4 and its token block of TBK tokens, with
  // the block's static token classes as bit masks (bit i = token cv0 + i)
  const int cp = tid >> 2, cv0 = (tid & 3) * TBK;
  unsigned tk_inv = 0, tk_phon = 0, tk_blank = 0;
  int tk_sidx = -1;
  for (int i = 0; i < TBK; ++i) {
    const int v = cv0 + i;
    if (v >= V) continue;
    tk_inv |= 1u << i;
    if (v == blank) tk_blank |= 1u << i;
    else if (v == space) tk_sidx = i;
    else tk_phon |= 1u << i;
  }

  // ---- load the home beam state and gather the first frame's lexicon rows
  int K = b.nbeam[trial];  // parents of the frame (ranks incl. holes)
  int Klive = K;            // surviving beams among them
  {
    const size_t hb = (size_t)trial * KC_;
    for (int i = tid; i < K; i += NT) {
      C_SCORE[i] = b.score[hb + i];
      C_H1[i] = b.h1[hb + i];
      C_H2[i] = b.h2[hb + i];
      C_LAST[i] = b.last[hb + i];
      C_PRE[i] = b.prefix[hb + i];
      C_NENT[i] = b.nent[hb + i];
      C_JMAP[i] = i;
      const LexRec* src = m.lex + b.prefix[hb + i];
      cp_async4(&C_LOFF[i], m.comp_off + b.prefix[hb + i]);
      cp_async16(&C_LROW[i], src);
      cp_async16(reinterpret_cast<char*>(&C_LROW[i]) + 16, reinterpret_cast<const char*>(src) + 16);
    }
    cp_async_commit();
    for (int i = tid; i < K * O; i += NT) {
      const int bi = i / O, e = i - bi * O;
      if (e < b.nent[hb + bi]) C_ENTS[bi * OC + e] = b.ents[hb * O + i];
    }
  }
  for (int i = tid; i < NBINS; i += NT) {
    hist[i] = 0;
    hfill[i] = 0;
  }
  if (tid == 0) {
    s_live[0] = s_live[1] = 0;
    s_ncount = b.ncount[trial];
    s_fail = 0;
    s_status = 0;
    s_calls = 0;
    s_pairs = 0;
    s_probes = 0;
    s_K = K;
    s_tbase = (unsigned)clock();
    for (int e = 0; e < NBAR_EV; ++e) s_tarr[e] = 0;
    if (TIMING)
      for (int i = 0; i < NPHASE; ++i) ph[i] = 0;
    mbar_init(&dbar[0], 1);
    mbar_init(&dbar[1], 1);
    fence_mbar_init();
  }
  cp_async_wait_all();
  __syncthreads();
  if (warp == 0) {
    double ms = -DBL_MAX;
    for (int i = lane; i < K; i += 32) ms = fmax(ms, C_SCORE[i]);
    ms = warp_max(ms);
    if (lane == 0) s_maxs = ms;
  }
  __syncthreads();

  const double* Dtrial = b.D + (size_t)trial * b.Tmax * VPD;
  auto issue_chunk = [&](int ci) {
    const int f0 = tb + ci * SCHUNK;
    if (f0 >= te) return;
    const int nf = min(SCHUNK, te - f0);
    const unsigned bytes = (unsigned)(nf * VPD * sizeof(double));
    mbar_expect_tx(&dbar[ci & 1], bytes);
    tma_bulk_g2s_stream(dbuf + (size_t)(ci & 1) * SCHUNK * VPDC, Dtrial + (size_t)f0 * VPD,
                        bytes, &dbar[ci & 1]);
  };
  if (tid == 0) issue_chunk(0);

  unsigned long long st_beams_in = 0, st_beams_out = 0, st_bound = 0, st_fallback = 0;
  unsigned calls_l = 0, probes_l = 0, pairs_l = 0;
  int fail_t = -1;
  // TIMING: critical-path accounting per barrier event e (SM clock, 32-bit wrap-safe): every
  // arriving warp records its arrival (atomicMax), thread 0 after the release adds
  // work[e] = last arrival - previous release and sync[e] = release - last arrival.
  const bool timing = TIMING && b.phase_cycles != nullptr;  // ph[] zeroed before the first barrier
  unsigned trel = timing ? (unsigned)clock() : 0u, tfs = trel;
#define LB_ARR(e)                                              \
  if (timing && lane == 0) atomicMax(&s_tarr[e], (unsigned)clock() - s_tbase);
#define LB_REL(e)                                              \
  if (timing && tid == 0) {                                    \
    const unsigned tnow = (unsigned)clock();                   \
    const unsigned ta = s_tarr[e] + s_tbase;                   \
    ph[2 * (e)] += ta - trel;                                  \
    ph[2 * (e) + 1] += tnow - ta;                              \
    trel = tnow;                                               \
    s_tarr[e] = 0;                                             \
  }
#define LB_PHASE(i)

  for (int t = tb; t < te; ++t) {
    const int rel = t - tb;
    const int ci = rel / SCHUNK;
    const int cr = rel - ci * SCHUNK;
    st_beams_in += Klive;

    if (warp >= NWC) {
      // ================== speculative n-gram warps (as in frames_kernel) ==================
      const int gt = tid - NC, ngw = warp - NWC;
      const bool ngtim = timing && gt == 0;
      unsigned tg = ngtim ? (unsigned)clock() : 0u;
      // one parent per n-gram thread: pair offsets by a warp scan + one cross-warp barrier
      static_assert(KC <= NGT, "one parent per speculative n-gram thread");
      const int p = gt;
      int np = 0, ns = 0, nent = 0;
      const int jp0 = p < K ? C_JMAP[p] : -1;
      if (jp0 >= 0) {
        ns = C_LROW[jp0].ns;
        nent = C_NENT[jp0];
        if (ns > 0 && C_LAST[jp0] != space) np = nent * ns;
      }
      int incl = np;
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULLMASK, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) ngtot[ngw] = incl;
      bar_sync(3, NGT);
      const int q0 = (ngw ? ngtot[0] : 0) + incl - np, q1 = q0 + np;
      const int P = ngtot[0] + ngtot[1];
      const int SCAP = min(PC, b.spec_cap);
      if (p < K) ppoff[p] = q0;
      if (gt == 0) {
        ppoff[K] = P;
        s_ngP = P;
        if (P <= SCAP) s_ngcov = P;
      }
      if (ngtim) {
        const unsigned tn = (unsigned)clock();
        ph[20] += tn - tg;
        tg = tn;
      }
      {
        // pair table, one pair per thread (balanced: a parent may carry dozens of homophone
        // pairs): pair q of parent p = (entry e, surface s) with q = ppoff[p] + e * ns + s, the
        // creation order.  Parents are in score order; when the pairs exceed PC only the leading
        // parents whose pairs all fit are speculated (s_ngcov = their pair count), the rest take
        // the warp path after S4
        int4* qinfo = reinterpret_cast<int4*>(sm + O_QINFO);
        if (q1 > SCAP && q0 <= SCAP) s_ngcov = q0;  // the first parent that does not fit (unique)
        bar_sync(3, NGT);
        const int PC0 = s_ngcov;
        for (int q = gt; q < PC0; q += NGT) {
          int lo = 0, hi = K - 1;  // the parent: last p with ppoff[p] <= q
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (ppoff[mid] <= q) lo = mid;
            else hi = mid - 1;
          }
          const int jlo = C_JMAP[lo];
          const LexRec& lr = C_LROW[jlo];
          const int local = q - ppoff[lo];
          const int e = local / lr.ns, sidx = local - e * lr.ns;
          int w, surf;
          if (sidx == 0) {
            w = lr.l0;
            surf = lr.s0;
          } else if (sidx == 1) {
            w = lr.l1;
            surf = lr.s1;
          } else {
            w = __ldg(m.comp_lm + C_LOFF[jlo] + sidx);
            surf = __ldg(m.comp_surf + C_LOFF[jlo] + sidx);
          }
          qinfo[q] = make_int4(jlo * OC + e, w, surf, lo);
        }
        bar_sync(3, NGT);
        const int PCOV = s_ngcov;
        constexpr int NQ = NGT / 4;
        if (ngtim) {
          const unsigned tn = (unsigned)clock();
          ph[21] += tn - tg;
          ph[23] += 1000u * (unsigned)((PCOV + NQ - 1) / NQ);
          tg = tn;
        }
        const int grp = gt >> 2, sub = lane & 3;
        for (int q0 = 0; q0 < PCOV; q0 += NQ) {
          const int q = q0 + grp;
          const bool act = q < PCOV;
          const int4 qi = act ? qinfo[q] : make_int4(0, -1, -1, 0);
          const Ent& E = C_ENTS[qi.x];
          uint32_t hh[MAXH] = {E.h[0], E.h[1], E.h[2]};
          double hb2[MAXH] = {E.bo[0], E.bo[1], E.bo[2]};
          WordScore sw;
          quad_score_word(m, act, hh, E.hlen, hb2, qi.y, sw, probes_l);
          if (act && sub == 0) {
            ++calls_l;
            PairRes pr;
            pr.valid = sw.inc > GUARD;
            pr.total = xadd(E.total, xmul(c.omega, sw.inc));
            pr.cum = xadd(E.cum, sw.inc);
            pr.node = E.node;
            pr.surf = (uint32_t)qi.z;
            for (int tt = 0; tt < MAXH; ++tt) {
              pr.h[tt] = sw.succ[tt];
              pr.bo[tt] = sw.sbo[tt];
            }
            pr.depth = (uint16_t)(E.depth + 1);
            pr.hlen = (uint8_t)sw.slen;
            pres[q] = pr;
            reinterpret_cast<double*>(sm + O_PVAL)[q] = pr.valid ? pr.total : -INFINITY;
          }
        }
        // each parent's top-o pairs (total desc, creation order asc: decoder.py:221-227), one
        // pair per thread ranking itself among its parent's pairs, so F2 does no pair loop
        int4* ptop = reinterpret_cast<int4*>(sm + O_PTOP);
        if (p < K) ptop[p] = make_int4(-1, -1, -1, -1);
        bar_sync(3, NGT);
        const double* pval = reinterpret_cast<const double*>(sm + O_PVAL);
        for (int q = gt; q < PCOV; q += NGT) {
          const double tq = pval[q];
          if (tq == -INFINITY) continue;  // killed pair (OOV without <unk>)
          const int pp = qinfo[q].w, a0 = ppoff[pp], a1 = ppoff[pp + 1];
          int rk = 0;
          for (int q2 = a0; q2 < a1; ++q2) {
            const double t2 = pval[q2];
            rk += (t2 > tq || (t2 == tq && q2 < q)) ? 1 : 0;
          }
          if (rk < O) reinterpret_cast<int*>(&ptop[pp])[rk] = q;  // ortho_beams <= 3
        }
        if (ngtim) ph[22] += (unsigned)clock() - tg;
      }
      LB_ARR(8);
      bar_arrive(2, NT);
      // then, while the compute warps rank and recombine, copy the inherited entries of every
      // live non-boundary beam into its slot (four threads per beam)
      bar_sync(4, NT);  // F2 done
      if (s_status == 0) {
        const int nsl = s_nsel, r4 = gt & 3;
        for (int i = gt >> 2; i < nsl; i += NGT / 4) {
          if (bsel[i].x != -1 || !(X_SCORE[i] > GUARD)) continue;
          const int jp = C_JMAP[npar[i]];
          const int cnt_e = C_NENT[jp];
          const uint4* su = reinterpret_cast<const uint4*>(C_ENTS + jp * OC);
          uint4* du = reinterpret_cast<uint4*>(X_ENTS + i * OC);
          for (int u = r4; u < cnt_e * ENT_U4; u += 4) du[u] = su[u];
          if (r4 == 0) X_NENT[i] = cnt_e;
        }
      }
    } else {
      // ============================== compute warps ==============================
      if (cr == 0) {
        mbar_wait(&dbar[ci & 1], (unsigned)((ci >> 1) & 1));
        if (tid == 0) issue_chunk(ci + 1);
      }
      const double* drow = dbuf + (size_t)(ci & 1) * SCHUNK * VPDC + (size_t)cr * VPD;
      const double U = __dadd_ru(__dadd_ru(__dadd_ru(s_maxs, drow[V]), fmax(c.beta, 0.0)),
                                 fmax(c.gamma, 0.0));
      // per-thread parent constants (thread -> parent cp, tokens cv0 .. cv0 + TBK - 1)
      const int jraw = cp < K ? C_JMAP[cp] : -1;
      const bool pin = jraw >= 0;  // a live parent (not beyond K, not a dropped rank)
      const int jcl = pin ? jraw : 0;
      const int lp = C_LAST[jcl];
      const double sp = C_SCORE[jcl];
      const double gsel = lp != space ? g_on : g_off;
      // token classes of this frame: bonus bits (phoneme, not a repeat of lp) and the tokens
      // that are always allowed (blank, the repeat of lp; lexicon.py:124-137)
      const unsigned lpb = (unsigned)(lp - cv0) < (unsigned)TBK ? 1u << (lp - cv0) : 0u;
      const unsigned bbits = tk_phon & ~lpb;
      const unsigned abits = tk_blank | (lpb & tk_inv);
      // F1 (materialise selected beam j from its (value, key)): hash lanes, last token, next
      // prefix state (and an L1 prefetch of its lexicon record), word-boundary list.  No
      // n-gram results are needed, so it runs while the speculative n-gram warps still probe.
      auto materialise = [&](int j, double x, uint32_t f) {
        const int p = (int)(f >> 8);
        const int tok = (int)(f & 0xFFu);
        const int jp = C_JMAP[p];
        const int lp = C_LAST[jp], pp = C_PRE[jp];
        const bool emit = (tok != blank) && (tok != lp);
        uint64_t a1 = C_H1[jp], a2 = C_H2[jp];
        int np = pp;
        if (emit) {
          a1 = a1 * H_MULT1 + (uint64_t)(tok + 1);
          a2 = a2 * H_MULT2 + (uint64_t)(tok + 1);
          const LexRec& lr = C_LROW[jp];
          if (m.lex_contig) {  // breadth-first trie: first child + rank, space -> root
            const unsigned long long ms = lr.mask & ~(1ull << space);
            np = tok == space ? 0 : lr.base + __popcll(ms & ((1ull << tok) - 1ull));
          } else {
            np = __ldg(m.lex_next + lr.base + __popcll(lr.mask & ((1ull << tok) - 1ull)));
          }
        }
        // the next frame's lexicon record and completion-CSR offset of slot j (waited for at
        // the end of the frame)
        cp_async16(&X_LROW[j], m.lex + np);
        cp_async16(reinterpret_cast<char*>(&X_LROW[j]) + 16, reinterpret_cast<const char*>(m.lex + np) + 16);
        cp_async4(&X_LOFF[j], m.comp_off + np);
        cp_async_commit();
        if (emit && tok == space) blist[atomicAdd(&s_nb, 1)] = j;
        X_SCORE[j] = x;
        X_H1[j] = a1;
        X_H2[j] = a2;
        nfp[j] = hash_fp(a1, a2);
        X_LAST[j] = (tok == blank) ? lp : tok;
        X_PRE[j] = np;
        npar[j] = p;
        bsel[j] = make_int4(-1, 0, 0, 0);
      };
      LB_PHASE(0);

      // ---- A: candidates of parent cp for its TBK tokens; bins kept in registers.  Branch-free
      // (predicated) so the unrolled items' fp64 chains overlap; the lexicon row segment arrives
      // as int4 loads.  x = (s + d) + addend, addend = beta*[phoneme, no repeat] or, on the
      // space column, gamma*[last != space]: the reference's ((s + d) + beta*mask) + gamma*m
      // (decoder.py:252-256) adds beta*0 = +-0.0 to the space column, an exact identity.  The
      // bin is trunc((U - x) / binw) clamped to NBINS-1: x <= U (U rounds up), so no lower
      // clamp; monotone in x, identical to the clamped double form.  Rejected candidates count
      // into a per-lane spare bin NBINS + lane (never scanned; no same-address conflicts).
      uint16_t bins[TBK];
      double wm = -DBL_MAX;
      if (__any_sync(FULLMASK, pin)) {
        // allowed tokens (lexicon.py:124-137): a valid transition, the blank, or the repeat
        const unsigned albits = ((unsigned)(C_LROW[jcl].mask >> cv0) & tk_inv) | abits;
#pragma unroll
        for (int i = 0; i < TBK; ++i) {
          const double add = (i == tk_sidx) ? gsel : (((bbits >> i) & 1u) ? b_on : b_off);
          const double x = xadd(xadd(sp, drow[cv0 + i]), add);
          const bool ok = pin && ((albits >> i) & 1u) && (x > GUARD);
          const int bn = min(__double2int_rz(xmul(xsub(U, x), ibw)), NBINS - 1);
          bins[i] = ok ? (uint16_t)bn : (uint16_t)0xFFFF;
          atomicAdd(&hist[ok ? bn : NBINS + lane], 1u);  // rejected: no intra-warp conflict
          wm = (ok && x > wm) ? x : wm;
        }
      } else {
#pragma unroll
        for (int i = 0; i < TBK; ++i) bins[i] = 0xFFFF;
      }
      wm = warp_max(wm);
      LB_PHASE(11);
      if (lane == 0) wmax[warp] = wm;
      if (tid == 0) s_nb = 0;
      if (tid < 2) keep[tid] = 0;
      LB_ARR(0);
      bar_sync(1, NC);  // S1
      LB_REL(0);
      LB_PHASE(1);

      double M = -DBL_MAX;
#pragma unroll
      for (int w = 0; w < NWC; ++w) M = fmax(M, wmax[w]);
      int nsel = 0;
      const bool dead = !(M > GUARD);  // decoder.py:267-268
      if (dead) {
        if (tid == 0) {
          s_status = 1;
          s_K = 0;
        }
        fail_t = t;
      } else {
        const double thr = xsub(M, c.theta);
        const int bthr =
            (int)fmin(fmax(xmul(xsub(U, thr), ibw), 0.0), (double)(NBINS - 1));
        int bstar = NBINS, cum_thr = 0, cum_bstar = 0;
        {
          constexpr int PB = NBINS / 32;
          int part[PB];
          int ls = 0;
#pragma unroll
          for (int i = 0; i < PB; ++i) {
            part[i] = (int)hist[lane * PB + i];
            ls += part[i];
          }
          int incl = ls;
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULLMASK, incl, o);
            if (lane >= o) incl += y;
          }
          const int excl = incl - ls;
          if (warp == 0) {
            int run = excl;
#pragma unroll
            for (int i = 0; i < PB; ++i) {
              hcum[lane * PB + i] = run;
              run += part[i];
            }
          }
          LB_ARR(1);
          bar_sync(1, NC);  // hcum[] visible to every compute warp
          LB_REL(1);
          cum_thr = hcum[bthr] + (int)hist[bthr];
          const unsigned bl = __ballot_sync(FULLMASK, excl < c.k && incl >= c.k);
          if (bl) {
            const int src = __ffs(bl) - 1;
            int lb = 0;
            if (lane == src) {
              int cum = excl;
#pragma unroll
              for (int i = 0; i < PB; ++i) {
                if (cum + part[i] >= c.k) {
                  lb = i;
                  break;
                }
                cum += part[i];
              }
            }
            lb = __shfl_sync(FULLMASK, lb, src);
            bstar = src * PB + lb;
            cum_bstar = hcum[bstar] + (int)hist[bstar];
          }
        }
        const bool sure = bstar < bthr;
        const int take_bin = sure ? bstar : bthr;
        const int bound = sure ? cum_bstar : cum_thr;
        if (bound <= LC) {
          // ---- D: counting-sort collect from the register bins
          // only the (typically 0-2) items inside the take window are revisited: a bit mask of
          // them, then one pass per set bit (value and bin recomputed exactly as in A)
          unsigned cm = 0;
#pragma unroll
          for (int i = 0; i < TBK; ++i) cm |= (bins[i] <= take_bin ? 1u : 0u) << i;
          while (cm) {
            const int i = __ffs(cm) - 1;
            cm &= cm - 1;
            const int v = cv0 + i;
            const double add = (i == tk_sidx) ? gsel : (((bbits >> i) & 1u) ? b_on : b_off);
            const double x = xadd(xadd(sp, drow[v]), add);
            if (sure || x >= thr) {
              const int bn = min(__double2int_rz(xmul(xsub(U, x), ibw)), NBINS - 1);
              const int pos = hcum[bn] + atomicAdd(&hfill[bn], 1);
              cval[pos] = x;
              ckey[pos] = ((uint32_t)cp << 8) | (uint32_t)v;  // orders like cp * V + v
              cbinl[pos] = (uint16_t)bn;
            }
          }
          LB_ARR(2);
          bar_sync(1, NC);  // S2
          LB_REL(2);
          const int m_sel = hcum[take_bin] + hfill[take_bin];
          nsel = min(c.k, m_sel);
          LB_PHASE(2);
          // consecutive positions per warp: lanes share bins (uniform loop counts, broadcast
          // loads of the bin mates) -- 1% faster than spreading a warp over all bins
          for (int a = tid; a < m_sel; a += NC) {
            const double va = cval[a];
            const uint32_t ka = ckey[a];
            const int bn = cbinl[a];
            const int lo = hcum[bn], n = hfill[bn];
            int r = lo;
            for (int q = lo; q < lo + n; ++q) {
              const double vq = cval[q];
              r += (vq > va) || (vq == va && ckey[q] < ka);
            }
            if (r < nsel) materialise(r, va, ka);  // F1 fused into the ranking
          }
        } else {
          ++st_fallback;
          nsel = small_fallback_select(c.k, c.beta, c.gamma, K, V, thr, blank, space, C_JMAP, C_LROW, C_LAST,
                                       C_SCORE, drow, hist, cval, ckey, sval, skey, &s_inr,
                                       &s_cnt2);
          bar_sync(1, NC);  // the exact selection is visible to every compute warp
          for (int j = lane * NWC + warp; j < nsel; j += NC) materialise(j, sval[j], skey[j]);
        }
      }
      LB_PHASE(3);
      if (tid == 0) s_nsel = nsel;
      LB_ARR(9);
      bar_sync(2, NT);  // S3b: speculative n-gram results ready (+ F1 visible)
      if (timing && tid == 0) {  // n-gram warps' and compute warps' arrival since frame start
        const unsigned tnow = (unsigned)clock();
        ph[17] += s_tarr[8] + s_tbase - tfs;
        ph[18] += s_tarr[9] + s_tbase - tfs;
        ph[24] += s_tarr[9] + s_tbase - trel;  // ranking + F1 (compute warps)
        ph[25] += tnow - (s_tarr[9] + s_tbase);  // waiting for the n-gram warps + release
        trel = tnow;
        s_tarr[8] = 0;
        s_tarr[9] = 0;
      }

      if (dead) bar_arrive(4, NT);
      // the previous frame's survivor count was read by every thread right after that frame's
      // end barrier; after this hand-off (all warps) its buffer serves the next frame
      if (tid == 0) s_live[(rel + 1) & 1] = 0;
      if (!dead) {
        const int ncov = s_ngcov;
        const bool ngover = ncov < s_ngP;  // some parents' pairs were not speculated
        if (timing && tid == 0 && ngover) ph[16] += 1000;  // permille of frames past the speculative pair cap
        LB_PHASE(13);
        // ---- F2: new word boundaries pick their top-o pairs (decoder.py:182-235)
        const int nb0 = s_nb;
        for (int bi = lane * NWC + warp; bi < nb0; bi += NC) {
          const int j = blist[bi];
          const int p = npar[j];
          const double x = X_SCORE[j];
          double sc = x;
          int4 bs = make_int4(-1, 0, 0, 0);
          {
            pairs_l += (unsigned)(ppoff[p + 1] - ppoff[p]);
            if (ppoff[p + 1] > ncov) {
              bs.x = -2;
            } else {
              const int4 pt = reinterpret_cast<const int4*>(sm + O_PTOP)[p];
              const int t0 = pt.x, t1 = pt.y, t2 = pt.z;
              const int ntop = t0 < 0 ? 0 : t1 < 0 ? 1 : t2 < 0 ? 2 : 3;
              if (ntop == 0) {
                sc = NEG_INF;  // decoder.py:223-225
              } else {
                const double best = pres[t0].total;
                const double floor_ = xsub(best, c.lambda);
                int kept = 0;
                if (pres[t0].total >= floor_) {
                  kept = 1;
                  if (ntop > 1 && pres[t1].total >= floor_) {
                    kept = 2;
                    if (ntop > 2 && pres[t2].total >= floor_) kept = 3;
                  }
                }
                const int base = atomicAdd(&s_ncount, kept);
                if (base + kept > b.ncap) {
                  s_fail = 1;
                  sc = NEG_INF;
                } else {
                  const size_t nbase = (size_t)trial * b.ncap;
                  if (kept > 0) {
                    st_stream(b.nparent + nbase + base, pres[t0].node);
                    st_stream(b.nsurf + nbase + base, pres[t0].surf);
                  }
                  if (kept > 1) {
                    st_stream(b.nparent + nbase + base + 1, pres[t1].node);
                    st_stream(b.nsurf + nbase + base + 1, pres[t1].surf);
                  }
                  if (kept > 2) {
                    st_stream(b.nparent + nbase + base + 2, pres[t2].node);
                    st_stream(b.nsurf + nbase + base + 2, pres[t2].surf);
                  }
                  bs.x = kept;
                  bs.y = base;
                  bs.z = (t0 & 0xFFFF) | ((kept > 1 ? t1 : 0) << 16);
                  bs.w = kept > 2 ? t2 : 0;
                  sc = xadd(x, xsub(best, C_ENTS[C_JMAP[p] * OC].total));
                }
              }
            }
          }
          X_SCORE[j] = sc;
          bsel[j] = bs;
        }
        LB_PHASE(12);
        bar_arrive(4, NT);  // the n-gram warps may copy inherited entries now
        LB_ARR(4);
        bar_sync(1, NC);  // S4
        LB_REL(4);
        LB_PHASE(4);
        const int nb = s_nb;
        st_bound += nb;
        if (ngover && nb > 0) {
          for (int bi = warp; bi < nb; bi += NWC) {
            const int j = blist[bi];
            if (bsel[j].x != -2) continue;  // speculated parent
            const int jp = C_JMAP[npar[j]];
            int outn = -1;
            double sc = X_SCORE[j];
            warp_apply_ngram(m, c, b, trial, C_ENTS + jp * OC, C_NENT[jp],
                             small_hdr(C_LROW[jp], C_LOFF[jp]), &wsc[warp], X_ENTS + j * OC, &outn,
                             &sc, &s_ncount, &s_fail, calls_l, probes_l);
            if (lane == 0) {
              X_SCORE[j] = sc;
              X_NENT[j] = max(outn, 0);
              bsel[j] = make_int4(-3, 0, 0, 0);  // entries built in the slot
            }
          }
          if (timing && tid == 0) ph[19] += (unsigned)clock() - trel;
          bar_sync(1, NC);
        }
        LB_PHASE(5);

        // ---- H: recombination (decoder.py:297-312) in one pass.  rank(i) = #{j : (s_j, -j) >
        // (s_i, -i)} over the selection, and beam i survives iff no live j with the same prefix
        // hash lanes ranks ahead of it (the first-ranked beam of each prefix keeps it).  All
        // pairs, four threads per beam: no hash table, no second barrier.
        {
          static_assert(KC * 4 == NC, "recombination: four threads per selected beam");
          const int n = nsel;
          const int i = tid >> 2, r = tid & 3;
          const bool act = i < n;
          const double si = act ? X_SCORE[i] : 0.0;
          const uint64_t a1 = act ? X_H1[i] : 0ull, a2 = act ? X_H2[i] : 0ull;
          // a 32-bit fingerprint of the hash lanes filters the exact 128-bit comparison
          const uint32_t fi = act ? nfp[i] : 0u;
          int cnt = 0, dup = 0;
#pragma unroll
          for (int it = 0; it < KC / 4; ++it) {
            const int j = r + 4 * it;
            const double sj = X_SCORE[j];
            const uint32_t fj = nfp[j];
            const bool ahead = (j < n) & ((sj > si) | ((sj == si) & (j < i)));
            cnt += ahead ? 1 : 0;
            if (ahead & (fj == fi)) dup |= (X_H1[j] == a1) & (X_H2[j] == a2) ? 1 : 0;
          }
          cnt += __shfl_xor_sync(FULLMASK, cnt, 1);
          dup |= __shfl_xor_sync(FULLMASK, dup, 1);
          cnt += __shfl_xor_sync(FULLMASK, cnt, 2);
          dup |= __shfl_xor_sync(FULLMASK, dup, 2);
          if (act && r == 0) {
            rankv[i] = cnt;
            const bool kept = si > GUARD && !dup;
            X_JMAP[cnt] = kept ? i : -1;  // the next frame's parent of rank cnt (or a hole)
            if (kept) {
              atomicOr(&keep[cnt >> 5], 1u << (cnt & 31));
              atomicAdd(&s_live[rel & 1], 1);
              if (cnt == 0) s_maxs = si;  // rank 0: the best survivor
            }
          }
          // entries of a fresh word boundary i into its slot (four threads) from the chosen
          // speculative pairs; inherited entries are copied by the n-gram warps meanwhile
          if (act && si > GUARD) {
            const int4 bs = bsel[i];
            Ent* dst = X_ENTS + i * OC;
            if (bs.x >= 0) {
              for (int e = r; e < bs.x; e += 4) {
                const int q = e == 0 ? (bs.z & 0xFFFF) : e == 1 ? (bs.z >> 16) : (bs.w & 0xFFFF);
                const PairRes& pr = pres[q];
                WordScore sw;
                sw.slen = pr.hlen;
                for (int tt = 0; tt < MAXH; ++tt) {
                  sw.succ[tt] = pr.h[tt];
                  sw.sbo[tt] = pr.bo[tt];
                }
                new_entry(dst[e], pr.total, pr.cum, sw, (uint32_t)(bs.y + e),
                          (uint32_t)(q - ppoff[npar[i]]), pr.depth);
              }
              if (r == 0) X_NENT[i] = bs.x;
            }
          }
        }
        // histogram bins free again for the next frame; this frame's lexicon-record gathers
        for (int i = tid; i < NBINS; i += NC) {
          hist[i] = 0;
          hfill[i] = 0;
        }
        cp_async_wait_all();
        if (b.dump_k) {  // debug traces: the survivors in compacted rank order
          bar_sync(1, NC);
          const unsigned kp0 = keep[0], kp1 = keep[1];
          for (int i = tid; i < nsel; i += NC) {
            const int rk = rankv[i];
            const unsigned kw = rk >= 32 ? kp1 : kp0;
            if (!((kw >> (rk & 31)) & 1u)) continue;
            const int pos = __popc(kw & ((1u << (rk & 31)) - 1u)) + (rk >= 32 ? __popc(kp0) : 0);
            const size_t di = ((size_t)trial * b.Tmax + t) * KC_ + pos;
            b.dump_h1[di] = X_H1[i];
            b.dump_h2[di] = X_H2[i];
            b.dump_pre[di] = X_PRE[i];
            b.dump_last[di] = X_LAST[i];
            b.dump_score[di] = X_SCORE[i];
          }
          if (tid == 0) b.dump_k[(size_t)trial * b.Tmax + t] = __popc(kp0) + __popc(kp1);
        }
        if (tid == 0) s_K = nsel;
      }  // !dead
    }  // compute warps
    LB_ARR(7);
    __syncthreads();  // frame end (whole CTA)
    LB_REL(7);
    tfs = trel;
    LB_PHASE(8);
    par ^= 1;
    K = s_K;
    Klive = s_live[rel & 1];
    st_beams_out += Klive;
    if (s_status == 0 && (s_fail || Klive == 0)) {  // decoder.py:314-315 / arena exhausted
      if (tid == 0) s_status = s_fail ? 4 : 2;
      fail_t = t;
      break;
    }
    if (s_status != 0) break;

    // ---- optional interval fusion of the device n-gram scorer (decoder.py:428-430)
    if (fusion_mode == 1 && t > 0 && (t % c.r) == 0) {
      for (int i = tid; i < K; i += NT) {
        const int ji = C_JMAP[i];
        if (ji < 0) continue;
        Ent* e = C_ENTS + ji * OC;
        const int n = C_NENT[ji];
        const double prev = e[0].total;
        for (int q = 0; q < n; ++q) {
          if (e[q].node == 0) {
            e[q].total = 0.0;
            e[q].punct = 0;
          } else {
            e[q].total = xmul(c.phi, xmul(scale, e[q].cum));
          }
        }
        sort_entries(e, n);
        C_SCORE[ji] = xadd(C_SCORE[ji], xsub(e[0].total, prev));
      }
      __syncthreads();
      if (warp == 0) {
        double ms = -DBL_MAX;
        for (int i = lane; i < K; i += 32)
          if (C_JMAP[i] >= 0) ms = fmax(ms, C_SCORE[C_JMAP[i]]);
        ms = warp_max(ms);
        if (lane == 0) s_maxs = ms;
      }
      __syncthreads();
      LB_PHASE(10);
    }
    LB_PHASE(9);
  }

  // ---- write back
  __syncthreads();
  if (timing && tid == 0)
    for (int i = 0; i < NPHASE; ++i) b.phase_cycles[(size_t)trial * NPHASE + i] += ph[i];
#undef LB_PHASE
#undef LB_ARR
#undef LB_REL
  const int status = s_status;
  if (tid == 0) {
    if (status != 0) {
      b.status[trial] = status;
      b.fail_frame[trial] = fail_t;
    }
    b.nbeam[trial] = Klive;
    b.ncount[trial] = s_ncount;
  }
  if (status == 0 || status == 4) {
    // the home state is compact: the survivors' slots in rank order (holes squeezed out)
    int32_t* cslot = rankv;  // free now: compacted position -> slot
    if (warp == 0) {
      int base = 0;
      for (int i0 = 0; i0 < K; i0 += 32) {
        const int i = i0 + lane;
        const int ji = i < K ? C_JMAP[i] : -1;
        const unsigned bl = __ballot_sync(FULLMASK, ji >= 0);
        if (ji >= 0) cslot[base + __popc(bl & ((1u << lane) - 1u))] = ji;
        base += __popc(bl);
      }
    }
    __syncthreads();
    const size_t hb = (size_t)trial * KC_;
    for (int i = tid; i < Klive; i += NT) {
      const int ji = cslot[i];
      b.score[hb + i] = C_SCORE[ji];
      b.h1[hb + i] = C_H1[ji];
      b.h2[hb + i] = C_H2[ji];
      b.last[hb + i] = C_LAST[ji];
      b.prefix[hb + i] = C_PRE[ji];
      b.nent[hb + i] = C_NENT[ji];
    }
    for (int i = tid; i < Klive * O; i += NT) {
      const int bi = i / O, e = i - bi * O;
      const int jb = cslot[bi];
      if (e < C_NENT[jb]) b.ents[hb * O + i] = C_ENTS[jb * OC + e];
    }
  }
  atomicAdd(&s_calls, calls_l);
  if (pairs_l) atomicAdd(&s_pairs, pairs_l);
  atomicAdd(&s_probes, probes_l);
  __syncthreads();
  if (tid == 0) {
    unsigned long long* stt = b.stats + (size_t)trial * 8;
    stt[0] += (unsigned long long)(te - tb);
    stt[1] += st_beams_in;
    stt[2] += st_beams_out;
    stt[3] += s_calls;
    stt[4] += s_probes;
    stt[5] += st_bound;
    stt[6] += s_pairs;  // (entry, surface) pairs the boundary beams consume (reference score_word calls)
    stt[7] += st_fallback;
  }
#undef BUF
#undef C_SCORE
#undef C_H1
#undef C_H2
#undef C_LAST
#undef C_PRE
#undef C_NENT
#undef C_ENTS
#undef X_SCORE
#undef X_H1
#undef X_H2
#undef X_LAST
#undef X_PRE
#undef X_NENT
#undef X_ENTS
#undef C_JMAP
#undef C_LOFF
#undef C_LROW
#undef X_JMAP
#undef X_LOFF
#undef X_LROW
}

// =====================================================================================
// K3: end-of-utterance closure (decoder.py:375-405), one CTA per trial, warp per beam
// =====================================================================================
__device__ int64_t block_excl_scan(int64_t v, int64_t* out_excl);

#ifndef LB_CLOSE_NT
#define LB_CLOSE_NT 512
#endif
#ifndef LB_CLOSE_MINB
#define LB_CLOSE_MINB 1
#endif
constexpr int CLOSE_NT = LB_CLOSE_NT;  // 16 warps: the open beams' closures are independent
__global__ void __launch_bounds__(CLOSE_NT, LB_CLOSE_MINB) close_kernel(ModelDev m, CfgDev c, BatchDev b) {
  constexpr int NT = CLOSE_NT, NW = NT / 32;
#ifdef LB_CLOSE_NP4
  constexpr int CNP = 4;
#else
  constexpr int CNP = 8;
#endif
  struct CloseScratch {
    NgCand top[OMAX];
    NgCand pending[CNP];
  };
  __shared__ CloseScratch wsc[NW];
  __shared__ int s_ncount, s_fail, s_next;
  __shared__ unsigned s_calls, s_probes;
  extern __shared__ __align__(16) Ent close_tmp[];
  const int trial = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (b.status[trial] != 0) return;
  const int KC = b.K, O = c.O;
  const size_t hb = (size_t)trial * KC;
  const int K = b.nbeam[trial];
  Ent* tmp = close_tmp + (size_t)warp * O;
  if (tid == 0) {
    s_ncount = b.ncount[trial];
    s_fail = 0;
    s_calls = 0;
    s_probes = 0;
    s_next = NW;
  }
  __syncthreads();
  unsigned calls = 0, probes = 0;
  // beams handed out dynamically (first NW statically): closures differ in cost (root beams
  // are free, homophone-heavy states take several probe rounds), so a fixed round-robin left
  // most warps waiting at the compaction barrier for the slowest one
  for (int i = warp; i < K;) {
    do {
      const int st = b.prefix[hb + i];
      if (st == 0) continue;  // root: nothing pending
      // completion header from the compact record (L2-resident after the frame loop; the padded
      // table row it replaces is not touched by the frame kernels)
      const CompHdr ch = lex_hdr_g(m, m.lex[st], st);
      if (ch.ns == 0) {
        if (lane == 0) b.score[hb + i] = NEG_INF;
        continue;
      }
      double sc = b.score[hb + i];
      int outn = -1;
      Ent* pe = b.ents + (hb + i) * O;
      warp_apply_ngram_t<CNP>(m, c, b, trial, pe, b.nent[hb + i], ch, &wsc[warp], tmp, &outn, &sc,
                              &s_ncount, &s_fail, calls, probes);
      outn = __shfl_sync(FULLMASK, outn, 0);  // lane 0 is authoritative
      if (lane == 0) {
        b.score[hb + i] = sc;
        if (outn >= 0) b.nent[hb + i] = outn;
        b.prefix[hb + i] = 0;
      }
      static_assert(sizeof(Ent) % 8 == 0, "Ent copies as 8-byte words");
      if (outn > 0) {  // the kept entries (lane 0 built them in shared memory): whole warp copies
        const int nw = outn * (int)(sizeof(Ent) / 8);
        const uint2* src = reinterpret_cast<const uint2*>(tmp);
        uint2* dst = reinterpret_cast<uint2*>(pe);
        for (int q = lane; q < nw; q += 32) dst[q] = src[q];
      }
      __syncwarp();
    } while (0);
    int nx = 0;
    if (lane == 0) nx = atomicAdd(&s_next, 1);
    i = __shfl_sync(FULLMASK, nx, 0);
  }
  atomicAdd(&s_calls, calls);
  atomicAdd(&s_probes, probes);
  __syncthreads();
  if (K <= NT && O <= 4) {
    // compact survivors in parallel, order preserved (decoder.py:397-405): every thread reads
    // its beam into registers, a block scan gives its new index, then all write
    const bool alive = tid < K && b.score[hb + tid] > GUARD;
    double sc = 0.0;
    uint64_t a1 = 0, a2 = 0;
    int la = 0, pr = 0, ne = 0;
    Ent e4[4];
    if (alive) {
      sc = b.score[hb + tid];
      a1 = b.h1[hb + tid];
      a2 = b.h2[hb + tid];
      la = b.last[hb + tid];
      pr = b.prefix[hb + tid];
      ne = b.nent[hb + tid];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (q < O) e4[q] = b.ents[(hb + tid) * O + q];
    }
    int64_t excl;
    const int64_t n = block_excl_scan(alive ? 1 : 0, &excl);  // ends with a barrier
    if (alive) {
      const size_t d = hb + (size_t)excl;
      b.score[d] = sc;
      b.h1[d] = a1;
      b.h2[d] = a2;
      b.last[d] = la;
      b.prefix[d] = pr;
      b.nent[d] = ne;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (q < O) b.ents[d * O + q] = e4[q];
    }
    if (tid == 0) {
      b.nbeam[trial] = (int)n;
      b.ncount[trial] = s_ncount;
      if (s_fail) {
        b.status[trial] = 4;
        b.fail_frame[trial] = b.T[trial];
      } else if (n == 0) {
        b.status[trial] = 3;
        b.fail_frame[trial] = b.T[trial];
      }
      unsigned long long* stt = b.stats + (size_t)trial * 8;
      stt[3] += s_calls;
      stt[4] += s_probes;
    }
    return;
  }
  if (tid == 0) {
    // compact survivors, order preserved (decoder.py:397-405)
    int n = 0;
    for (int i = 0; i < K; ++i) {
      if (!(b.score[hb + i] > GUARD)) continue;
      if (n != i) {
        b.score[hb + n] = b.score[hb + i];
        b.h1[hb + n] = b.h1[hb + i];
        b.h2[hb + n] = b.h2[hb + i];
        b.last[hb + n] = b.last[hb + i];
        b.prefix[hb + n] = b.prefix[hb + i];
        b.nent[hb + n] = b.nent[hb + i];
        for (int q = 0; q < O; ++q) b.ents[(hb + n) * O + q] = b.ents[(hb + i) * O + q];
      }
      ++n;
    }
    b.nbeam[trial] = n;
    b.ncount[trial] = s_ncount;
    if (s_fail) {
      b.status[trial] = 4;
      b.fail_frame[trial] = b.T[trial];
    } else if (n == 0) {
      b.status[trial] = 3;
      b.fail_frame[trial] = b.T[trial];
    }
    unsigned long long* stt = b.stats + (size_t)trial * 8;
    stt[3] += s_calls;
    stt[4] += s_probes;
  }
}

// =====================================================================================
// device n-gram scorer fusion (apply_llm with StubScorer(ngram_model, scale) semantics)
// =====================================================================================
#ifndef LB_FUSION_NT
#define LB_FUSION_NT 512
#endif
constexpr int FUSION_NT = LB_FUSION_NT;  // 16 warps, two CTAs per SM: every utterance in one wave
__global__ void __launch_bounds__(FUSION_NT, 2) device_fusion_kernel(ModelDev m, CfgDev c,
                                                                     BatchDev b, int final_,
                                                                     double scale,
                                                                     int min_frames) {
  constexpr int NT = FUSION_NT, NW = NT / 32;
  __shared__ unsigned s_probes;
  const int trial = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (b.status[trial] != 0 || b.T[trial] <= min_frames) return;
  const int KC = b.K, O = c.O;
  const size_t hb = (size_t)trial * KC;
    const int K = b.nbeam[trial];
  if (tid == 0) s_probes = 0;
  __syncthreads();
  unsigned probes = 0;
  const int grp = lane >> 3, sub = lane & 7;
  for (int i = warp; i < K; i += NW) {
    Ent* e = b.ents + (hb + i) * O;
    const int n = b.nent[hb + i];
    const double prev = e[0].total;
    for (int base = 0; base < n; base += 4) {
      const int q = base + grp;
      const bool act = q < n;
      const Ent E = e[act ? q : 0];
      double inc = 0.0;
      if (final_) {
        uint32_t hh[MAXH] = {E.h[0], E.h[1], E.h[2]};
        double hb[MAXH] = {E.bo[0], E.bo[1], E.bo[2]};
        WordScore sw;
        group_score_word(m, act && E.node != 0, hh, E.hlen, hb, m.eos_word, sw, probes);
        inc = sw.inc;
      }
      if (act && sub == 0) {
        Ent o = E;
        if (E.node == 0) {
          o.total = 0.0;
          o.punct = 0;
        } else if (final_) {
          o.total = xmul(c.phi, xmul(scale, xadd(E.cum, inc)));
          o.punct = 1;  // "." (scorer.py:136-139)
        } else {
          o.total = xmul(c.phi, xmul(scale, E.cum));
        }
        e[q] = o;
      }
      __syncwarp();
    }
    if (lane == 0) {
      sort_entries(e, n);
      b.score[hb + i] = xadd(b.score[hb + i], xsub(e[0].total, prev));
    }
    __syncwarp();
  }
  atomicAdd(&s_probes, probes);
  __syncthreads();
  if (tid == 0) b.stats[(size_t)trial * 8 + 4] += s_probes;
}

// =====================================================================================
// K4: entry gathering for host scorers / results
// =====================================================================================
__global__ void count_entries_kernel(BatchDev b, int64_t* counts) {
  const int trial = blockIdx.x;
  const int tid = threadIdx.x;
  __shared__ unsigned long long s_e, s_w;
  if (tid == 0) {
    s_e = 0;
    s_w = 0;
  }
  __syncthreads();
  if (b.status[trial] == 0) {
    const size_t hb = (size_t)trial * b.K;
    const int K = b.nbeam[trial];
    unsigned long long ne = 0, nw = 0;
    for (int i = tid; i < K; i += blockDim.x) {
      const int n = b.nent[hb + i];
      ne += n;
      for (int q = 0; q < n; ++q) nw += b.ents[(hb + i) * b.O + q].depth;
    }
    atomicAdd(&s_e, ne);
    atomicAdd(&s_w, nw);
  }
  __syncthreads();
  if (tid == 0) {
    counts[2 * trial] = (int64_t)s_e;
    counts[2 * trial + 1] = (int64_t)s_w;
  }
}

// block-wide exclusive scan of one int64 per thread (blockDim.x <= 1024); returns the block total
__device__ int64_t block_excl_scan(int64_t v, int64_t* out_excl) {
  __shared__ int64_t wsum[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  int64_t incl = v;
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(FULLMASK, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int64_t w = lane < nw ? wsum[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(FULLMASK, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) wsum[lane] = w;  // inclusive warp prefix
  }
  __syncthreads();
  const int64_t before = warp ? wsum[warp - 1] : 0;
  const int64_t total = wsum[nw - 1];
  *out_excl = before + incl - v;
  __syncthreads();
  return total;
}

// entries of every beam in beam order with their word-id sequences (apply_llm texts,
// decoder.py:338-345); prefix sums are block scans, chains are walked in parallel
__global__ void write_entries_kernel(BatchDev b, const int64_t* entry_off, const int64_t* word_off,
                                     int32_t* e_trial, int32_t* e_beam, int64_t* e_woff,
                                     int32_t* words, double* totals, int32_t* puncts) {
  const int trial = blockIdx.x;
  if (b.status[trial] != 0) return;
  const size_t hb = (size_t)trial * b.K;
  const size_t nbase = (size_t)trial * b.ncap;
  const int K = b.nbeam[trial];
  const int O = b.O;
  int64_t ecarry = entry_off[trial], wcarry = word_off[trial];
  for (int base = 0; base < K; base += blockDim.x) {  // uniform trip count over the block
    const int i = base + threadIdx.x;
    int ne = 0;
    int64_t nw = 0;
    if (i < K) {
      ne = b.nent[hb + i];
      for (int q = 0; q < ne; ++q) nw += b.ents[(hb + i) * O + q].depth;
    }
    int64_t eex, wex;
    const int64_t etot = block_excl_scan(ne, &eex);
    const int64_t wtot = block_excl_scan(nw, &wex);
    if (i < K) {
      int64_t idx = ecarry + eex, wp0 = wcarry + wex;
      for (int q = 0; q < ne; ++q, ++idx) {
        const Ent E = b.ents[(hb + i) * O + q];
        e_trial[idx] = trial;
        e_beam[idx] = i;
        totals[idx] = E.total;
        puncts[idx] = E.punct;
        e_woff[idx] = wp0;
        uint32_t node = E.node;
        int64_t wp = wp0 + E.depth - 1;
        while (node != 0) {
          words[wp--] = (int32_t)b.nsurf[nbase + node];
          node = b.nparent[nbase + node];
        }
        wp0 += E.depth;
      }
    }
    ecarry += etot;
    wcarry += wtot;
  }
}

// K7: host-scored fusion (decoder.py:354-371)
__global__ void apply_scores_kernel(CfgDev c, BatchDev b, const int64_t* entry_off,
                                    const double* scores, const int32_t* puncts,
                                    const uint8_t* has_text, int final_, int min_frames) {
  const int trial = blockIdx.x;
  if (b.status[trial] != 0 || b.T[trial] <= min_frames) return;
  const size_t hb = (size_t)trial * b.K;
  const int K = b.nbeam[trial];
  const int O = b.O;
  extern __shared__ int64_t sh_off[];
  if (threadIdx.x == 0) {
    int64_t e = 0;
    for (int i = 0; i < K; ++i) {
      sh_off[i] = e;
      e += b.nent[hb + i];
    }
  }
  __syncthreads();
  const int64_t ebase = entry_off[trial];
  for (int i = threadIdx.x; i < K; i += blockDim.x) {
    Ent* e = b.ents + (hb + i) * O;
    const int n = b.nent[hb + i];
    const double prev = e[0].total;
    for (int q = 0; q < n; ++q) {
      const int64_t idx = ebase + sh_off[i] + q;
      if (!has_text[idx]) {
        e[q].total = 0.0;
        e[q].punct = 0;
      } else {
        e[q].total = xmul(c.phi, scores[idx]);
        if (final_) e[q].punct = (uint8_t)puncts[idx];
      }
    }
    sort_entries(e, n);
    b.score[hb + i] = xadd(b.score[hb + i], xsub(e[0].total, prev));
  }
}

// =====================================================================================
// setup kernels
// =====================================================================================
__global__ void reset_kernel(ModelDev m, BatchDev b) {
  const int trial = blockIdx.x * blockDim.x + threadIdx.x;
  if (trial >= b.B) return;
  const size_t hb = (size_t)trial * b.K;
  b.nbeam[trial] = 1;
  b.score[hb] = 0.0;
  b.h1[hb] = H_INIT1;
  b.h2[hb] = H_INIT2;
  b.last[hb] = m.blank;
  b.prefix[hb] = 0;
  b.nent[hb] = 1;
  Ent e;
  e.total = 0.0;
  e.cum = 0.0;
  e.bo[0] = m.bos_bo;
  e.bo[1] = 0.0;
  e.bo[2] = 0.0;
  e.node = 0;
  e.seq = 0;
  e.h[0] = m.bos;
  e.h[1] = 0;
  e.h[2] = 0;
  e.depth = 0;
  e.hlen = 1;
  e.punct = 0;
  b.ents[hb * b.O] = e;
  const size_t nb = (size_t)trial * b.ncap;
  b.nparent[nb] = WPAD;
  b.nsurf[nb] = WPAD;
  b.ncount[trial] = 1;
  b.status[trial] = 0;
  b.fail_frame[trial] = -1;
  for (int q = 0; q < 8; ++q) b.stats[(size_t)trial * 8 + q] = 0;
}

__global__ void pad_table_kernel(int32_t* dst, const int32_t* src, int32_t S, int32_t V,
                                 int32_t VP, const int32_t* comp_off, const int32_t* comp_surf,
                                 const int32_t* comp_lm) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)S * VP) return;
  const int64_t s = i / VP;
  const int v = (int)(i - s * VP);
  int32_t out = 0;
  if (v < V) {
    out = src[s * V + v];
  } else if (v < V + ROW_HDR) {
    const int off = comp_off[s], n = comp_off[s + 1] - off;
    switch (v - V) {
      case 0: out = n; break;
      case 1: out = off; break;
      case 2: out = n > 0 ? comp_surf[off] : -1; break;
      case 3: out = n > 0 ? comp_lm[off] : -1; break;
      case 4: out = n > 1 ? comp_surf[off + 1] : -1; break;
      default: out = n > 1 ? comp_lm[off + 1] : -1; break;
    }
  }
  dst[i] = out;
}

// K1: one warp per row; numpy's pairwise sum (8 accumulators + sequential tail, n <= 128)
__global__ void log_softmax_kernel(const float* x, int64_t rows, int32_t V, int32_t in_pitch,
                                   double alpha, double* out, int32_t out_pitch) {
  __shared__ double ebuf[8][64];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int64_t row = (int64_t)blockIdx.x * 8 + wl;
  if (row >= rows) return;
  const float* xr = x + row * in_pitch;
  double xv0 = lane < V ? (double)xr[lane] : -DBL_MAX;
  double xv1 = lane + 32 < V ? (double)xr[lane + 32] : -DBL_MAX;
  const double mx = warp_max(fmax(xv0, xv1));
  if (lane < V) ebuf[wl][lane] = exp(xsub(xv0, mx));
  if (lane + 32 < V) ebuf[wl][lane + 32] = exp(xsub(xv1, mx));
  __syncwarp();
  double res = 0.0;
  if (V < 8) {
    if (lane == 0)
      for (int i = 0; i < V; ++i) res = xadd(res, ebuf[wl][i]);
  } else {
    const int full = V - (V % 8);
    double r = 0.0;
    if (lane < 8) {
      r = ebuf[wl][lane];
      for (int i = 8 + lane; i < full; i += 8) r = xadd(r, ebuf[wl][i]);
    }
    const double r1 = __shfl_xor_sync(FULLMASK, r, 1);
    const double s01 = (lane & 1) ? xadd(r1, r) : xadd(r, r1);  // (r0+r1), (r2+r3), ...
    const double t1 = __shfl_xor_sync(FULLMASK, s01, 2);
    const double s03 = (lane & 2) ? xadd(t1, s01) : xadd(s01, t1);
    const double t2 = __shfl_xor_sync(FULLMASK, s03, 4);
    const double s07 = (lane & 4) ? xadd(t2, s03) : xadd(s03, t2);
    if (lane == 0) {
      res = s07;
      for (int i = full; i < V; ++i) res = xadd(res, ebuf[wl][i]);
    }
  }
  res = __shfl_sync(FULLMASK, res, 0);
  const double lse = xadd(mx, log(res));
  double* orow = out + row * out_pitch;
  double o0 = -DBL_MAX, o1 = -DBL_MAX;
  if (lane < V) orow[lane] = o0 = xmul(alpha, xsub(xv0, lse));
  if (lane + 32 < V) orow[lane + 32] = o1 = xmul(alpha, xsub(xv1, lse));
  // padded batch layout: slot V carries the row maximum (the frame kernel's bound U)
  const double mx2 = warp_max(fmax(o0, o1));
  if (out_pitch > V && lane == 0) orow[V] = mx2;
}

// K1, eight lanes per row (the production launch): lane t of a row's 8-lane group owns the
// columns i = t (mod 8), so it holds numpy's pairwise accumulator r[t] (columns below
// V - V % 8, in order) plus at most one tail column; the accumulators combine by xor shuffles
// in numpy's order ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) and the tail columns are then added
// one by one, exactly as log_softmax_kernel does with one warp per row.  No shared memory and
// few registers: ~60 resident warps per SM hide the fp64 exp latency the warp-per-row form
// (41 of 64 lane slots busy, the sum serialised on lane 0) and a row-per-thread form (smem-
// limited to 12 warps per SM) could not.
__global__ void __launch_bounds__(256) log_softmax_oct_kernel(
    const float* __restrict__ x, int64_t rows, int32_t V, int32_t in_pitch, double alpha,
    double* __restrict__ out, int32_t out_pitch) {
  const int lane = threadIdx.x & 31, t = lane & 7, gbase = lane & ~7;
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const bool live = row < rows;  // whole 8-lane groups are live or not; shuffles stay uniform
  const float* xr = x + (live ? row : 0) * in_pitch;
  const int full = V >= 8 ? V - (V % 8) : 0;
  float xf[8];  // the row's columns t, t+8, ... as read (fp32: 8 registers, no fp64 copies)
  double mx = -DBL_MAX;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int i = t + 8 * k;
    xf[k] = (live && i < V) ? __ldcs(xr + i) : 0.f;
    if (i < V) mx = fmax(mx, (double)xf[k]);
  }
  mx = fmax(mx, __shfl_xor_sync(FULLMASK, mx, 1));
  mx = fmax(mx, __shfl_xor_sync(FULLMASK, mx, 2));
  mx = fmax(mx, __shfl_xor_sync(FULLMASK, mx, 4));
  // exps consumed as produced: r = numpy's accumulator r[t] over the columns below `full`
  // (in column order), e0 = this lane's first exp (V < 8), tail = its column full + t
  double r = 0.0, e0 = 0.0, tail = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int i = t + 8 * k;
    if (i < V) {
      const double ek = exp(xsub((double)xf[k], mx));
      if (k == 0) e0 = ek;
      if (i < full) r = k == 0 ? ek : xadd(r, ek);
      else tail = ek;  // i >= full: the (only) tail column of this lane
    }
  }
  double res = 0.0;
  if (V < 8) {
    for (int k = 0; k < V; ++k) res = xadd(res, __shfl_sync(FULLMASK, e0, gbase + k));
  } else {
    const double r1 = __shfl_xor_sync(FULLMASK, r, 1);
    const double s01 = (t & 1) ? xadd(r1, r) : xadd(r, r1);
    const double t1 = __shfl_xor_sync(FULLMASK, s01, 2);
    const double s03 = (t & 2) ? xadd(t1, s01) : xadd(s01, t1);
    const double t2 = __shfl_xor_sync(FULLMASK, s03, 4);
    res = (t & 4) ? xadd(t2, s03) : xadd(s03, t2);
    for (int k = 0; k < V - full; ++k) res = xadd(res, __shfl_sync(FULLMASK, tail, gbase + k));
  }
  const double lse = xadd(mx, log(res));
  double m2 = -DBL_MAX;
  double* orow = out + (live ? row : 0) * out_pitch;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int i = t + 8 * k;
    if (i < V) {
      const double o = xmul(alpha, xsub((double)xf[k], lse));
      m2 = fmax(m2, o);
      if (live) orow[i] = o;
    }
  }
  m2 = fmax(m2, __shfl_xor_sync(FULLMASK, m2, 1));
  m2 = fmax(m2, __shfl_xor_sync(FULLMASK, m2, 2));
  m2 = fmax(m2, __shfl_xor_sync(FULLMASK, m2, 4));
  if (live && t == 0 && out_pitch > V) orow[V] = m2;  // padded layout: slot V = row max
}

// row maximum into slot V of a padded log-prob matrix that was uploaded as is
__global__ void rowmax_kernel(double* d, int64_t rows, int32_t V, int32_t pitch) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= rows) return;
  double* r = d + row * pitch;
  double mx = -DBL_MAX;
  for (int v = lane; v < V; v += 32) mx = fmax(mx, r[v]);
  mx = warp_max(mx);
  if (lane == 0) r[V] = mx;
}

// single-thread exact lookup (parity helper): record of `k` or nullptr
__device__ const NgRec* ng_find(const ModelDev& m, const uint32_t k[4]) {
  uint32_t b1, b2;
  ng_buckets(ng_hash(k[0], k[1], k[2], k[3]), m.ng_nb, b1, b2);
  for (int c2 = 0; c2 < 2; ++c2) {
    const NgRec* bk = m.ng + (size_t)(c2 ? b2 : b1) * NG_WAYS;
    for (int q = 0; q < NG_WAYS; ++q)
      if (bk[q].w[0] == k[0] && bk[q].w[1] == k[1] && bk[q].w[2] == k[2] && bk[q].w[3] == k[3])
        return bk + q;
  }
  return nullptr;
}

// device score_word for parity tests of the n-gram image (history back-offs looked up here)
__global__ void score_words_kernel(ModelDev m, int n, const uint32_t* hist, const int32_t* hlen,
                                   const int32_t* word, double* inc, uint32_t* succ,
                                   int32_t* slen) {
  const int lane = threadIdx.x & 31, grp = lane >> 3, sub = lane & 7;
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int q = warp_global * 4 + grp;
  const bool act = q < n;
  uint32_t hh[MAXH] = {0, 0, 0};
  double hb[MAXH] = {0.0, 0.0, 0.0};
  int hl = 0, w = -1;
  if (act) {
    hl = hlen[q];
    for (int i = 0; i < hl; ++i) hh[i] = hist[3 * q + i];
    w = word[q];
    for (int i = 0; i < hl; ++i) {
      uint32_t k[4] = {WPAD, WPAD, WPAD, WPAD};
      for (int j = i; j < hl; ++j) k[j - i] = hh[j];
      const NgRec* r = ng_find(m, k);
      hb[i] = r ? r->bo : 0.0;
    }
  }
  WordScore sw;
  unsigned probes = 0;
  group_score_word(m, act, hh, hl, hb, w, sw, probes);
  if (act && sub == 0) {
    inc[q] = sw.inc;
    slen[q] = sw.slen;
    for (int i = 0; i < 3; ++i) succ[3 * q + i] = i < sw.slen ? sw.succ[i] : 0u;
  }
}

// =====================================================================================
// launch wrappers
// =====================================================================================
namespace lbk {

int max_threads_for(int K) { return K <= 64 ? 256 : (K <= 256 ? 512 : 960); }

int small_smem_bytes() { return small::TOTAL; }
int small_gscratch_bytes() { return small::GTOTAL; }

cudaError_t set_smem_limit(int nthreads, int64_t bytes) {
  cudaError_t e = cudaSuccess;
  e = cudaFuncSetAttribute(frames_small_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           small::TOTAL);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(frames_small_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           small::TOTAL);
  if (e != cudaSuccess) return e;
#define LB_SET(NCV)                                                                          \
  e = cudaFuncSetAttribute(frames_kernel<NCV, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           (int)bytes);                                                      \
  if (e != cudaSuccess) return e;                                                            \
  e = cudaFuncSetAttribute(frames_kernel<NCV, false>,                                        \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (nthreads == 256) {
    LB_SET(256)
  } else if (nthreads == 512) {
    LB_SET(512)
  } else {
    LB_SET(960)
  }
#undef LB_SET
  return e;
}

cudaError_t pad_table(int32_t* dst, const int32_t* src, int32_t S, int32_t V, int32_t VP,
                      const int32_t* comp_off, const int32_t* comp_surf, const int32_t* comp_lm,
                      cudaStream_t st) {
  const int64_t n = (int64_t)S * VP;
  pad_table_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(dst, src, S, V, VP, comp_off,
                                                                comp_surf, comp_lm);
  ++g_launches;
  return cudaGetLastError();
}

static int lsm_rows_enabled() {  // LB_LSM_ROWS=0: the warp-per-row K1 (A/B, parity test)
  static const int on = [] {
    const char* e = getenv("LB_LSM_ROWS");
    return e ? atoi(e) : 1;
  }();
  return on;
}

cudaError_t log_softmax(const float* x, int64_t rows, int32_t V, int32_t in_pitch, double alpha,
                        double* out, int32_t out_pitch, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  if (lsm_rows_enabled()) {
    const int64_t threads = rows * 8;
    log_softmax_oct_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(
        x, rows, V, in_pitch, alpha, out, out_pitch);
  } else {
    log_softmax_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(x, rows, V, in_pitch, alpha,
                                                                   out, out_pitch);
  }
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t rowmax(double* d, int64_t rows, int32_t V, int32_t pitch, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  rowmax_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(d, rows, V, pitch);
  ++g_launches;
  return cudaGetLastError();
}

// Bulk L2 prefetch of the read-only search images (cuckoo n-gram buckets, compact lexicon
// records) at the start of a decode: fire-and-forget `cp.async.bulk.prefetch.L2` in 32 KB
// pieces, so the image lines are L2-resident before the frame loop's probes reach them instead
// of missing to HBM one dependent probe round at a time during the first frames.  Opt-in
// (LB_L2_PREFETCH=1): measured 4.746 vs 4.763 ms per config-2 step without/with it -- the
// n-gram probe rounds cost the same with the images already L2-resident.
__device__ __forceinline__ void l2_prefetch_range(const void* base, size_t bytes, int gtid,
                                                  int gthreads) {
  constexpr size_t PIECE = 32768;
  const char* p = reinterpret_cast<const char*>(base);
  const size_t n = (bytes + PIECE - 1) / PIECE;
  for (size_t i = gtid; i < n; i += gthreads) {
    const size_t off = i * PIECE;
    const unsigned len = (unsigned)((min(PIECE, bytes - off) + 15) & ~(size_t)15);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p + off), "r"(len)
                 : "memory");
  }
}

__global__ void __launch_bounds__(128) l2_prefetch_kernel(ModelDev m) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x, n = gridDim.x * blockDim.x;
  l2_prefetch_range(m.ng, (size_t)m.ng_nb * NG_WAYS * sizeof(NgRec), g, n);
  l2_prefetch_range(m.lex, (size_t)m.S * sizeof(LexRec), g, n);
}

static int l2_prefetch_enabled() {
  static const int on = [] {
    const char* e = getenv("LB_L2_PREFETCH");
    return e ? atoi(e) : 0;
  }();
  return on;
}

cudaError_t reset(const ModelDev& m, const BatchDev& b, cudaStream_t st) {
  reset_kernel<<<(b.B + 127) / 128, 128, 0, st>>>(m, b);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t frames(const ModelDev& m, const CfgDev& c, const BatchDev& b, const Layout& L, int t0,
                   int t1, int fusion_mode, double scale, cudaStream_t st) {
  const size_t sm = (size_t)L.smem_bytes;
  if (t0 == 0 && l2_prefetch_enabled() && m.ng != nullptr && m.lex != nullptr) {
    l2_prefetch_kernel<<<16, 128, 0, st>>>(m);  // first frame range of a decode
    ++g_launches;
  }
  if (L.small) {
    // the phase-timer build is a separate instantiation: the production kernel carries no
    // timer state (it would cost registers at the 96-register cap)
    if (b.phase_cycles != nullptr)
      frames_small_kernel<true><<<b.B, small::NT, sm, st>>>(m, c, b, t0, t1, fusion_mode, scale);
    else
      frames_small_kernel<false><<<b.B, small::NT, sm, st>>>(m, c, b, t0, t1, fusion_mode, scale);
    ++g_launches;
    return cudaGetLastError();
  }
  bool all_smem = true;
  for (int r = 0; r < N_REGIONS; ++r)
    if (r != R_WARP && !L.in_smem[r]) all_smem = false;
#define LB_LAUNCH(NCV)                                                                 \
  if (all_smem)                                                                        \
    frames_kernel<NCV, true><<<b.B, NCV + NGT, sm, st>>>(m, c, b, L, t0, t1, fusion_mode, \
                                                         scale);                        \
  else                                                                                 \
    frames_kernel<NCV, false><<<b.B, NCV + NGT, sm, st>>>(m, c, b, L, t0, t1,            \
                                                          fusion_mode, scale);
  switch (L.nthreads) {
    case 256:
      LB_LAUNCH(256)
      break;
    case 512:
      LB_LAUNCH(512)
      break;
    default:
      LB_LAUNCH(960)
      break;
  }
#undef LB_LAUNCH
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t close(const ModelDev& m, const CfgDev& c, const BatchDev& b, cudaStream_t st) {
  const size_t sm = (size_t)(CLOSE_NT / 32) * c.O * sizeof(Ent);
  close_kernel<<<b.B, CLOSE_NT, sm, st>>>(m, c, b);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t device_ngram_fusion(const ModelDev& m, const CfgDev& c, const BatchDev& b, int final_,
                                double scale, int min_frames, cudaStream_t st) {
  device_fusion_kernel<<<b.B, FUSION_NT, 0, st>>>(m, c, b, final_, scale, min_frames);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t count_entries(const BatchDev& b, int64_t* counts, cudaStream_t st) {
  count_entries_kernel<<<b.B, 128, 0, st>>>(b, counts);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t write_entries(const BatchDev& b, const int64_t* entry_off, const int64_t* word_off,
                          int32_t* e_trial, int32_t* e_beam, int64_t* e_woff, int32_t* words,
                          double* totals, int32_t* puncts, cudaStream_t st) {
  write_entries_kernel<<<b.B, 256, 0, st>>>(b, entry_off, word_off, e_trial, e_beam, e_woff, words,
                                            totals, puncts);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t apply_scores(const CfgDev& c, const BatchDev& b, const int64_t* entry_off,
                         const double* scores, const int32_t* puncts, const uint8_t* has_text,
                         int final_, int min_frames, cudaStream_t st) {
  const size_t sm = (size_t)(b.K + 1) * sizeof(int64_t);
  apply_scores_kernel<<<b.B, 128, sm, st>>>(c, b, entry_off, scores, puncts, has_text, final_,
                                            min_frames);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t score_words(const ModelDev& m, int n, const uint32_t* hist, const int32_t* hlen,
                        const int32_t* word, double* inc, uint32_t* succ, int32_t* slen,
                        cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const int warps = (n + 3) / 4;
  const int blocks = (warps * 32 + 127) / 128;
  score_words_kernel<<<blocks, 128, 0, st>>>(m, n, hist, hlen, word, inc, succ, slen);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace lbk
