// lb_device.cuh -- device-side data layout shared by the kernels and the C ABI.
//
// Layout in HBM (per model, read-only, shared by every batch/stream):
//   table   int32 [S][VP]   lexicon automaton, rows padded to a 16-byte pitch (VP = ceil4(V))
//   comp_*  int32 CSR       per state: distinct completing surfaces + their LM word ids
//   ng      NgRec [2^b]     open-addressing hash of every listed n-gram (32 B = one sector)
// Per batch (B trials):
//   D       f64 [B][Tmax][VPD]  scaled log-probs (VPD = ceil2(V): 16-byte rows for TMA bulk)
//   beams   SoA [B][K]      score, hash lanes, last token, prefix state, entry count
//   ents    Ent [B][K][O]   ortho entries (word-level sub-hypotheses)
//   nodes   SoA [B][cap]    append-only word-history trie: parent, surface, depth, n-gram sum
#pragma once
#include <cstdint>

namespace lbd {

constexpr double NEG_INF = -1.0e30;   // ngram.py:26
constexpr double GUARD = -1.0e29;     // ngram.py:27
constexpr uint64_t H_INIT1 = 0xCBF29CE484222325ull;  // decoder.py:38-41
constexpr uint64_t H_INIT2 = 0x9AE16A3B2F90404Full;
constexpr uint64_t H_MULT1 = 0x9E3779B97F4A7C15ull;
constexpr uint64_t H_MULT2 = 0xC2B2AE3D27D4EB4Full;
constexpr uint32_t WPAD = 0xFFFFFFFFu;    // unused word slot / empty hash slot marker
constexpr uint64_t PROB_ABSENT = 0x7FF8DEAD00000000ull;
constexpr int NBINS = 256;   // selection histogram bins
constexpr int CHUNK = 8;     // frames per TMA-staged D chunk
constexpr int OMAX = 8;      // max ortho_beams supported
constexpr int MAXH = 3;      // max LM history words (order <= 4)

struct __align__(32) NgRec {
  uint32_t w[4];
  double prob;  // PROB_ABSENT bits: gram carries only a back-off
  double bo;    // 0.0 if absent
};

// One ortho entry (OrthoEntry, decoder.py:44-51) plus two running sums carried with it so
// no fusion step has to walk or load the word history: `cum` is the raw n-gram sum
// sum(inc) from <s> (= score_sequence of its words), `depth` the number of words.
// `bo[i]` caches backoffs.get(h[i:], 0.0) for the entry's own LM history (ngram.py:195): the
// lookups that created the entry already returned those records, so the next score_word
// only needs the (h[i:], w) probability lookups.
struct __align__(16) Ent {
  double total;     // weighted LM total (OrthoEntry.lm_total)
  double cum;       // raw n-gram log-prob of the word sequence (ngram.py:239-250 order)
  double bo[MAXH];  // back-off weights of h[0:], h[1:], h[2:]
  uint32_t node;    // word-history node
  uint32_t seq;     // creation rank inside the apply_ngram call that made it
  uint32_t h[MAXH]; // LM history word ids (OrthoEntry.lm_state)
  uint16_t depth;   // words in the history
  uint8_t hlen;
  uint8_t punct;    // LB_PUNCT_*
};
static_assert(sizeof(Ent) == 64, "Ent must be 64 bytes");

// Lexicon rows are padded to VP = ceil4(V + 6) int32 and carry a completion header after the
// V transitions, so the row gather of a frame also brings the word-boundary data:
//   row[V+0] = number of distinct completing surfaces, row[V+1] = CSR offset,
//   row[V+2], row[V+3] = (surface, LM word) of the first, row[V+4], row[V+5] of the second.
constexpr int ROW_HDR = 6;

// Compact lexicon record (the k <= 64 frames kernel): one 32-byte sector per state instead of a
// 192-byte padded row.  mask bit v <=> table[s][v] != sink; the successors of the set bits, in
// token order, are lex_next[base ...] (next state of token v = lex_next[base + popc(mask & ((1 <<
// v) - 1))]); then the completion header: count of distinct surfaces and the first two
// (surface, LM word) pairs (the rest through comp_off / comp_surf / comp_lm).
struct __align__(16) LexRec {
  unsigned long long mask;
  int32_t base, ns, s0, l0, s1, l1;
};
static_assert(sizeof(LexRec) == 32, "LexRec is one 32-byte sector");

struct ModelDev {
  const int32_t* table;
  const LexRec* lex;        // [S] compact records
  const int32_t* lex_next;  // successors of the valid transitions, per state in token order
  // 1 when every state's non-space successors are consecutive ids in token order and a valid
  // space transition leads to the root (breadth-first tries, lexicon.py:149-209): then
  // LexRec.base is the first child and next(s, v) = base + rank, with no successor load
  int32_t lex_contig;
  int32_t S, V, VP;  // VP: int32 row pitch (multiple of 4)
  int32_t sink, blank, space;
  const int32_t* comp_off;
  const int32_t* comp_surf;
  const int32_t* comp_lm;
  const NgRec* ng;     // bucketized cuckoo table: ng_nb buckets x 4 records (128 B each)
  uint32_t ng_nb;
  int32_t order;
  uint32_t bos;
  int32_t eos_word;
  double bos_bo;       // backoffs.get(("<s>",), 0.0): the initial entry's cached back-off
};
constexpr int NG_WAYS = 4;

struct CfgDev {
  double theta, lambda, beta, gamma, omega, phi;
  double inv_binw;  // NBINS / (min(theta, 24) + 12): histogram span below the upper bound U
  double bonus_up;  // max(beta, 0) + max(gamma, 0), for U = max s + max D + bonus_up
  int32_t k, O, r;
};

struct BatchDev {
  int32_t B, Tmax, K, O, VPD;
  const int32_t* T;  // frames per trial
  const double* D;   // [B][Tmax][VPD]
  // beam home state
  int32_t* nbeam;
  double* score;
  uint64_t* h1;
  uint64_t* h2;
  int32_t* last;
  int32_t* prefix;
  int32_t* nent;
  Ent* ents;
  // word history
  uint32_t* nparent;
  uint32_t* nsurf;
  int32_t* ncount;
  int32_t ncap;
  int32_t* status;
  int32_t* fail_frame;
  unsigned long long* stats;  // [B][8]
  // global spill scratch for large beams (per trial)
  char* gscratch;
  int64_t gscratch_stride;
  // optional per-frame beam dump for parity bisection: [B][Tmax][K] of (h1,h2,prefix,last,score)
  uint64_t* dump_h1;
  uint64_t* dump_h2;
  int32_t* dump_pre;
  int32_t* dump_last;
  double* dump_score;
  int32_t* dump_k;  // [B][Tmax]
  // optional per-phase cycle counters of the frames kernel: [B][NPHASE] (thread 0, clock64)
  unsigned long long* phase_cycles;
  // speculative n-gram pair budget of frames_small_kernel per frame (<= its shared-memory cap)
  int32_t spec_cap;
};
constexpr int NPHASE = 26;
constexpr int NBAR_EV = 10;  // frames_small_kernel TIMING: barrier events per frame

// Byte layout of the per-CTA working set; each region lives in shared memory or, when the
// beam is too wide for 227 KB, in the trial's global scratch (generic pointers either way).
enum Region {
  R_DBUF = 0,
  R_ROWS,
  R_CUR_SCORE, R_CUR_H1, R_CUR_H2, R_CUR_LAST, R_CUR_PRE, R_CUR_NENT, R_CUR_ENTS,
  R_NXT_SCORE, R_NXT_H1, R_NXT_H2, R_NXT_LAST, R_NXT_PRE, R_NXT_NENT, R_NXT_ENTS,
  R_CV, R_CBIN,
  R_CVAL, R_CKEY,
  R_SVAL, R_SKEY,
  R_NSCORE, R_NH1, R_NH2, R_NLAST, R_NPRE, R_NPAR, R_RANK, R_BLIST,
  R_BENTS, R_BNENT,
  R_KEEP,
  R_WARP,
  R_POFF, R_PAIRS, R_SLOTB, R_SLOTM, R_MYSLOT,
  N_REGIONS
};

struct Layout {
  int64_t off[N_REGIONS];
  int32_t in_smem[N_REGIONS];
  int64_t smem_bytes;
  int64_t gscratch_bytes;
  int32_t lcap;        // candidate list capacity
  int32_t stage_rows;  // rows staged through shared memory
  int32_t nthreads;    // compute threads (the kernel adds two speculative n-gram warps)
  int32_t pcap;        // n-gram (entry, surface) pair capacity of one flattened round
  int32_t tslots;      // recombination hash-table slots (power of two >= 2k)
  int32_t small;       // 1: the specialised kernel (k <= 64, o <= 4, V <= 48) with its own layout
};

// one evaluated (entry, surface) pair of the flattened n-gram phase
struct PairRes {
  double total;  // entry.total + omega * inc
  double cum;    // entry.cum + inc
  double bo[MAXH];
  uint32_t node, surf;
  uint32_t h[MAXH];
  uint16_t depth;
  uint8_t hlen, valid;
};

struct NgCand {
  double total;
  double cum;
  double bo[MAXH];
  uint32_t node, surf, seq, hlen;
  uint32_t h[MAXH];
  uint32_t valid;
  uint32_t depth, pad;
};

struct WarpScratch {
  NgCand top[OMAX];
  NgCand pending[4];
};

// splitmix64 finaliser
__host__ __device__ inline uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__host__ __device__ inline uint64_t ng_hash(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  uint64_t lo = (uint64_t)a | ((uint64_t)b << 32);
  uint64_t hi = (uint64_t)c | ((uint64_t)d << 32);
  return mix64(lo ^ mix64(hi ^ 0x5BD1E9955BD1E995ull));
}

// the two candidate buckets of a key (multiply-shift range reduction, distinct buckets)
__host__ __device__ inline void ng_buckets(uint64_t h, uint32_t nb, uint32_t& b1, uint32_t& b2) {
  b1 = (uint32_t)(((uint64_t)(uint32_t)h * nb) >> 32);
  b2 = (uint32_t)(((uint64_t)(uint32_t)(h >> 32) * nb) >> 32);
  if (b2 == b1) b2 = (b1 + 1 == nb) ? 0u : b1 + 1u;
}

}  // namespace lbd
