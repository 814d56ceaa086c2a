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
constexpr int CHUNK = 16;    // frames per TMA-staged D chunk
constexpr int OMAX = 8;      // max ortho_beams supported
constexpr int MAXH = 3;      // max LM history words (order <= 4)

struct __align__(32) NgRec {
  uint32_t w[4];
  double prob;  // PROB_ABSENT bits: gram carries only a back-off
  double bo;    // 0.0 if absent
};

struct __align__(16) Ent {
  double total;     // weighted LM total (OrthoEntry.lm_total)
  uint32_t node;    // word-history node
  uint32_t seq;     // creation rank inside the apply_ngram call that made it
  uint32_t h[MAXH]; // LM history word ids (OrthoEntry.lm_state)
  uint8_t hlen;
  uint8_t punct;    // LB_PUNCT_*
  uint16_t pad;
};
static_assert(sizeof(Ent) == 32, "Ent must be 32 bytes");

struct ModelDev {
  const int32_t* table;
  int32_t S, V, VP;  // VP: int32 row pitch (multiple of 4)
  int32_t sink, blank, space;
  const int32_t* comp_off;
  const int32_t* comp_surf;
  const int32_t* comp_lm;
  const NgRec* ng;
  uint64_t ng_mask;
  int32_t order;
  uint32_t bos;
  int32_t eos_word;
};

struct CfgDev {
  double theta, lambda, beta, gamma, omega, phi;
  double inv_binw;  // NBINS / theta
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
  uint32_t* ndepth;
  double* ncum;
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
};

// Byte layout of the per-CTA working set; each region lives in shared memory or, when the
// beam is too wide for 227 KB, in the trial's global scratch (generic pointers either way).
enum Region {
  R_DBUF = 0,
  R_ROWS,
  R_CUR_SCORE, R_CUR_H1, R_CUR_H2, R_CUR_LAST, R_CUR_PRE, R_CUR_NENT, R_CUR_ENTS,
  R_NXT_SCORE, R_NXT_H1, R_NXT_H2, R_NXT_LAST, R_NXT_PRE, R_NXT_NENT, R_NXT_ENTS,
  R_MASK,
  R_CVAL, R_CKEY,
  R_SVAL, R_SKEY,
  R_NSCORE, R_NH1, R_NH2, R_NLAST, R_NPRE, R_NPAR, R_RANK, R_BLIST,
  R_BENTS, R_BNENT,
  R_KEEP,
  R_WARP,
  N_REGIONS
};

struct Layout {
  int64_t off[N_REGIONS];
  int32_t in_smem[N_REGIONS];
  int64_t smem_bytes;
  int64_t gscratch_bytes;
  int32_t lcap;        // candidate list capacity
  int32_t stage_rows;  // rows staged through shared memory
  int32_t nthreads;
};

struct NgCand {
  double total;
  double inc;
  uint32_t node, surf, seq, hlen;
  uint32_t h[MAXH];
  uint32_t valid;
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

}  // namespace lbd
