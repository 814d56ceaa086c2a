// lb_capi.cu -- the extern "C" boundary (include/lightbeam_b200.h): model/batch lifetime,
// device memory, launch orchestration, and host-side result assembly (ranking + n-best,
// decoder.py:433-460).  No torch types cross this boundary.

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <string_view>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/lightbeam_b200.h"
#include "lb_device.cuh"
#include "lb_internal.h"
#include "lb_structs.h"

using namespace lbd;

namespace {
thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(expr)                                                                   \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess)                                                         \
      return fail(LB_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

template <typename T>
cudaError_t dalloc(T** p, size_t n) {
  if (n == 0) n = 1;
  return cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T));
}

int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// Cuckoo insertion with random-walk eviction; every key ends in one of its two buckets.
bool cuckoo_build(const lb_ngram_desc* nd, uint32_t nb, std::vector<NgRec>& tab, int* max_kicks) {
  NgRec empty;
  for (int q = 0; q < 4; ++q) empty.w[q] = WPAD;
  empty.prob = 0.0;
  empty.bo = 0.0;
  tab.assign((size_t)nb * NG_WAYS, empty);
  uint64_t rng = 0x2545F4914F6CDD1Dull;
  int worst = 0;
  for (int64_t i = 0; i < nd->n_grams; ++i) {
    NgRec cur;
    for (int q = 0; q < 4; ++q) cur.w[q] = nd->words[4 * i + q];
    cur.prob = nd->probs[i];
    cur.bo = nd->backoffs[i];
    bool placed = false;
    int kicks = 0;
    for (; kicks < 2000 && !placed; ++kicks) {
      uint32_t b[2];
      ng_buckets(ng_hash(cur.w[0], cur.w[1], cur.w[2], cur.w[3]), nb, b[0], b[1]);
      for (int c2 = 0; c2 < 2 && !placed; ++c2)
        for (int q = 0; q < NG_WAYS; ++q) {
          NgRec& slot = tab[(size_t)b[c2] * NG_WAYS + q];
          if (slot.w[0] == WPAD) {
            slot = cur;
            placed = true;
            break;
          }
        }
      if (placed) break;
      rng ^= rng << 13;
      rng ^= rng >> 7;
      rng ^= rng << 17;
      NgRec& victim = tab[(size_t)b[rng & 1] * NG_WAYS + ((rng >> 1) & (NG_WAYS - 1))];
      std::swap(cur, victim);
    }
    if (!placed) return false;
    worst = std::max(worst, kicks);
  }
  *max_kicks = worst;
  return true;
}
}  // namespace



namespace lbh {
int set_error(int code, const std::string& msg) { return fail(code, msg); }
}  // namespace lbh

extern "C" {

const char* lb_last_error(void) { return g_err.c_str(); }

int lb_device_count(int32_t* out) {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  *out = n;
  return LB_OK;
}

int lb_model_create(const lb_table_desc* td, const lb_ngram_desc* nd, int32_t device,
                    lb_model** out) {
  if (!td || !nd || !out) return fail(LB_ERR_ARG, "null argument");
  if (td->vocab_size < 3 || td->vocab_size > 64)
    return fail(LB_ERR_ARG, "vocab_size must be in [3, 64]");
  if (nd->order < 1 || nd->order > 4) return fail(LB_ERR_ARG, "n-gram order must be 1..4");
  CK(cudaSetDevice(device));
  lb_model* m = new lb_model();
  m->device = device;
  const int32_t S = td->num_states, V = td->vocab_size;
  const int32_t VP = (int32_t)round_up(V + ROW_HDR, 4);
  CK(dalloc(&m->d_comp_off, (size_t)S + 1));
  CK(cudaMemcpy(m->d_comp_off, td->comp_offsets, ((size_t)S + 1) * sizeof(int32_t),
                cudaMemcpyHostToDevice));
  CK(dalloc(&m->d_comp_surf, (size_t)td->n_comp));
  CK(dalloc(&m->d_comp_lm, (size_t)td->n_comp));
  if (td->n_comp > 0) {
    CK(cudaMemcpy(m->d_comp_surf, td->comp_surface, (size_t)td->n_comp * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(m->d_comp_lm, td->comp_lmword, (size_t)td->n_comp * 4, cudaMemcpyHostToDevice));
  }
  // lexicon table: rows padded to VP with the completion header after the V transitions
  int32_t* tmp = nullptr;
  CK(dalloc(&tmp, (size_t)S * V));
  CK(cudaMemcpy(tmp, td->table, (size_t)S * V * sizeof(int32_t), cudaMemcpyHostToDevice));
  CK(dalloc(&m->d_table, (size_t)S * VP));
  CK(lbk::pad_table(m->d_table, tmp, S, V, VP, m->d_comp_off, m->d_comp_surf, m->d_comp_lm, 0));
  CK(cudaDeviceSynchronize());
  CK(cudaFree(tmp));
  // compact lexicon image (LexRec per state + successor list), built on the host
  int64_t n_next = 0;
  int32_t contig = 1;
  {
    std::vector<lbd::LexRec> lex((size_t)S);
    std::vector<int32_t> nexts;
    nexts.reserve((size_t)S * 2);
    for (int32_t s = 0; s < S; ++s) {
      const int32_t* row = td->table + (size_t)s * V;
      lbd::LexRec& r = lex[(size_t)s];
      r.mask = 0ull;
      r.base = (int32_t)nexts.size();
      for (int32_t v = 0; v < V; ++v)
        if (row[v] != td->sink) {
          r.mask |= 1ull << v;
          nexts.push_back(row[v]);
        }
      const int32_t off = td->comp_offsets[s], n = td->comp_offsets[s + 1] - off;
      r.ns = n;
      r.s0 = n > 0 ? td->comp_surface[off] : -1;
      r.l0 = n > 0 ? td->comp_lmword[off] : -1;
      r.s1 = n > 1 ? td->comp_surface[off + 1] : -1;
      r.l1 = n > 1 ? td->comp_lmword[off + 1] : -1;
    }
    n_next = (int64_t)nexts.size();
    // breadth-first tries: successors of each state (space excluded) are consecutive ids
    for (int32_t s = 0; s < S && contig; ++s) {
      const int32_t* row = td->table + (size_t)s * V;
      int32_t expect = -1;
      for (int32_t v = 0; v < V && contig; ++v) {
        if (row[v] == td->sink) continue;
        if (v == td->space_id) {
          if (row[v] != 0) contig = 0;
        } else if (v == td->blank_id) {
          contig = 0;
        } else {
          if (expect >= 0 && row[v] != expect) contig = 0;
          expect = row[v] + 1;
        }
      }
    }
    if (contig)
      for (int32_t s = 0; s < S; ++s) {
        lbd::LexRec& r = lex[(size_t)s];
        const unsigned long long ms = r.mask & ~(1ull << td->space_id);
        r.base = ms ? td->table[(size_t)s * V + __builtin_ctzll(ms)] : 0;
      }
    CK(dalloc(&m->d_lex, (size_t)S));
    CK(cudaMemcpy(m->d_lex, lex.data(), (size_t)S * sizeof(lbd::LexRec), cudaMemcpyHostToDevice));
    CK(dalloc(&m->d_lex_next, (size_t)std::max<int64_t>(n_next, 1)));
    if (n_next > 0)
      CK(cudaMemcpy(m->d_lex_next, nexts.data(), (size_t)n_next * 4, cudaMemcpyHostToDevice));
  }
  // n-gram image: bucketized cuckoo table (4 records per 128-byte bucket, 2 candidate buckets)
  // built on the host -- deterministic and a few hundred ms for 1M grams
  std::vector<NgRec> tab;
  uint32_t nb = (uint32_t)std::max<int64_t>(8, (int64_t)(nd->n_grams / (NG_WAYS * 0.85)) + 1);
  for (int attempt = 0;; ++attempt) {
    if (cuckoo_build(nd, nb, tab, &m->max_probe)) break;
    if (attempt > 20) return fail(LB_ERR_CAPACITY, "cuckoo n-gram table build failed");
    nb = (uint32_t)(nb * 1.15) + 1;
  }
  m->ng_cap = (int64_t)nb * NG_WAYS;
  CK(dalloc(&m->d_ng, tab.size()));
  CK(cudaMemcpy(m->d_ng, tab.data(), tab.size() * sizeof(NgRec), cudaMemcpyHostToDevice));
  const int64_t cap = m->ng_cap;
  m->bytes = (int64_t)S * VP * 4 + ((int64_t)S + 1) * 4 + (int64_t)td->n_comp * 8 +
             cap * (int64_t)sizeof(NgRec) + (int64_t)S * (int64_t)sizeof(lbd::LexRec) + n_next * 4;
  ModelDev& d = m->dev;
  d.table = m->d_table;
  d.lex = m->d_lex;
  d.lex_next = m->d_lex_next;
  d.lex_contig = contig;
  d.S = S;
  d.V = V;
  d.VP = VP;
  d.sink = td->sink;
  d.blank = td->blank_id;
  d.space = td->space_id;
  d.comp_off = m->d_comp_off;
  d.comp_surf = m->d_comp_surf;
  d.comp_lm = m->d_comp_lm;
  d.ng = m->d_ng;
  d.ng_nb = nb;
  d.bos_bo = nd->bos_backoff;
  d.order = nd->order;
  d.bos = nd->bos_id;
  d.eos_word = nd->eos_word;
  m->surfaces.resize(td->n_surfaces);
  for (int32_t i = 0; i < td->n_surfaces; ++i)
    m->surfaces[i].assign(td->surface_blob + td->surface_offsets[i],
                          (size_t)(td->surface_offsets[i + 1] - td->surface_offsets[i]));
  *out = m;
  return LB_OK;
}

int lb_model_destroy(lb_model* m) {
  if (!m) return LB_OK;
  cudaSetDevice(m->device);
  cudaFree(m->d_table);
  cudaFree(m->d_comp_off);
  cudaFree(m->d_comp_surf);
  cudaFree(m->d_comp_lm);
  cudaFree(m->d_lex);
  cudaFree(m->d_lex_next);
  cudaFree(m->d_ng);
  delete m;
  return LB_OK;
}

int lb_model_lex_contiguous(const lb_model* m, int32_t* out) {
  if (!m || !out) return fail(LB_ERR_ARG, "null argument");
  *out = m->dev.lex_contig;
  return LB_OK;
}

int lb_model_footprint(const lb_model* m, int64_t* bytes) {
  if (!m || !bytes) return fail(LB_ERR_ARG, "null argument");
  *bytes = m->bytes;
  return LB_OK;
}

}  // extern "C"

namespace {

// Place the per-CTA working set: shared memory first, spilling the bulkiest regions to the
// trial's global scratch when a wide beam would not fit in 227 KB.
void plan_layout(lb_batch* b) {
  const int64_t K = b->K, O = b->O, VP = b->m->dev.VP, VPD = b->VPD;
  int nt = lbk::max_threads_for((int)K);
  if (const char* env = std::getenv("LB_THREADS")) {
    const int v = std::atoi(env);
    if (v == 256 || v == 512 || v == 960) nt = v;
  }
  const int64_t lcap = std::max<int64_t>(2 * K, K + 256);
  int64_t sz[N_REGIONS] = {};
  sz[R_DBUF] = 2 * CHUNK * VPD * 8;
  sz[R_ROWS] = K * (int64_t)sizeof(LexRec);  // compact lexicon record per beam
  const int64_t beam[7] = {K * 8, K * 8, K * 8, K * 4, K * 4, K * 4, K * O * (int64_t)sizeof(Ent)};
  for (int i = 0; i < 7; ++i) {
    sz[R_CUR_SCORE + i] = beam[i];
    sz[R_NXT_SCORE + i] = beam[i];
  }
  sz[R_CV] = 0;
  sz[R_CBIN] = round_up(K * b->m->dev.V * 2, 16);
  sz[R_CVAL] = lcap * 8;
  sz[R_CKEY] = lcap * 4;
  sz[R_SVAL] = K * 8;
  sz[R_SKEY] = K * 4;
  sz[R_NSCORE] = K * 8;
  sz[R_NH1] = K * 8;
  sz[R_NH2] = K * 8;
  for (int r : {R_NLAST, R_NPRE, R_NPAR, R_RANK, R_BLIST, R_BNENT}) sz[r] = K * 4;
  sz[R_BENTS] = K * O * (int64_t)sizeof(Ent);
  sz[R_KEEP] = ((K + 31) / 32) * 4;
  sz[R_WARP] = (nt / 32) * (int64_t)sizeof(WarpScratch);
  const int64_t pcap = std::max<int64_t>(128, K);
  int64_t ts = 64;
  while (ts < 2 * K) ts <<= 1;
  sz[R_POFF] = (K + 1) * 4;
  sz[R_PAIRS] = pcap * (int64_t)sizeof(PairRes);
  sz[R_SLOTB] = ts * 4;
  sz[R_SLOTM] = ts * 4;
  sz[R_MYSLOT] = K * 4;
  const int64_t budget = 200 * 1024;  // leave room for static shared memory
  int in_smem[N_REGIONS];
  for (int i = 0; i < N_REGIONS; ++i) in_smem[i] = 1;
  in_smem[R_WARP] = 0;  // scratch of the rare warp-per-beam n-gram path: global (L1-cached)
  // bulkiest / least latency-critical first; a beam of several hundred (the b2t25 profile's
  // 900) keeps the log-prob stage, the 32-B lexicon record per beam (read by every candidate)
  // and the small per-frame arrays in shared memory
  const int spill_order[] = {R_BENTS, R_NXT_ENTS, R_CUR_ENTS, R_CV, R_CVAL, R_CKEY,
                             R_NXT_H1, R_NXT_H2, R_CUR_H1, R_CUR_H2, R_NH1, R_NH2,
                             R_PAIRS, R_CBIN, R_SLOTB, R_SLOTM, R_NSCORE, R_SVAL, R_SKEY,
                             R_NLAST, R_NPRE, R_NPAR, R_BNENT, R_MYSLOT, R_BLIST, R_RANK, R_ROWS,
                             R_NXT_LAST, R_NXT_PRE, R_NXT_NENT, R_CUR_LAST, R_CUR_PRE,
                             R_CUR_NENT, R_NXT_SCORE, R_CUR_SCORE, R_POFF, R_KEEP};
  auto total = [&]() {
    int64_t t = 0;
    for (int i = 0; i < N_REGIONS; ++i)
      if (in_smem[i]) t += round_up(sz[i], 16);
    return t;
  };
  for (int r : spill_order) {
    if (total() <= budget) break;
    in_smem[r] = 0;
  }
  int64_t so = 0, go = 0;
  for (int i = 0; i < N_REGIONS; ++i) {
    if (in_smem[i]) {
      b->L.off[i] = so;
      so += round_up(sz[i], 16);
    } else {
      b->L.off[i] = go;
      go += round_up(sz[i], 16);
    }
    b->L.in_smem[i] = in_smem[i];
  }
  b->L.smem_bytes = so;
  b->L.gscratch_bytes = go;
  b->L.lcap = (int32_t)lcap;
  b->L.stage_rows = in_smem[R_ROWS];
  b->L.nthreads = nt;
  b->L.pcap = (int32_t)pcap;
  b->L.tslots = (int32_t)ts;
  b->L.small = 0;
  const char* env = std::getenv("LB_KERNEL");
  const bool want_small = !(env && std::strcmp(env, "general") == 0);
  if (want_small && K <= 64 && O <= 3 && b->m->dev.V <= 48 && b->m->dev.VP <= 56 && VPD <= 50) {
    b->L.small = 1;
    b->L.smem_bytes = lbk::small_smem_bytes();
    b->L.gscratch_bytes = lbk::small_gscratch_bytes();
  }
}

void fill_cfg(lb_batch* b) {
  const lb_config& c = b->cfg;
  CfgDev& d = b->cdev;
  d.theta = c.beam_prune_threshold;
  d.lambda = c.homophone_prune_threshold;
  d.beta = c.token_insertion_bonus;
  d.gamma = c.word_boundary_bonus;
  d.omega = c.ngram_weight;
  d.phi = c.llm_weight;
  const double span = std::min(c.beam_prune_threshold, 24.0) + 12.0;
  d.inv_binw = (double)NBINS / span;
  d.bonus_up = std::max(c.token_insertion_bonus, 0.0) + std::max(c.word_boundary_bonus, 0.0);
  d.k = c.beam_size;
  d.O = c.ortho_beams;
  d.r = c.llm_rescore_interval;
}

}  // namespace

extern "C" {

static int batch_alloc(lb_batch* b, int32_t max_trials, int32_t max_frames);

int lb_batch_create(lb_model* m, const lb_config* cfg, int32_t max_trials, int32_t max_frames,
                    void* stream, lb_batch** out) {
  if (!m || !cfg || !out) return fail(LB_ERR_ARG, "null argument");
  if (max_trials < 1 || max_frames < 1) return fail(LB_ERR_ARG, "empty batch");
  if (cfg->beam_size < 1 || cfg->beam_size > 4096) return fail(LB_ERR_ARG, "beam_size out of range");
  if (cfg->ortho_beams < 1 || cfg->ortho_beams > OMAX)
    return fail(LB_ERR_ARG, "ortho_beams must be in [1, 8]");
  CK(cudaSetDevice(m->device));
  lb_batch* b = new lb_batch();
  b->m = m;
  b->cfg = *cfg;
  b->st = reinterpret_cast<cudaStream_t>(stream);
  b->Bmax = max_trials;
  b->Tmax = max_frames;
  b->K = cfg->beam_size;
  b->O = cfg->ortho_beams;
  b->VPD = (int32_t)round_up(m->dev.V + 1, 2);  // slot V: row maximum
  fill_cfg(b);
  plan_layout(b);
  if (b->L.smem_bytes > 200 * 1024) {
    delete b;
    return fail(LB_ERR_ARG, "beam_size too wide for the per-CTA shared-memory layout");
  }
  // every failure after this point frees what was allocated so far (lb_batch_destroy skips
  // null pointers), so an OOM during creation does not leak device memory
  const int rc = batch_alloc(b, max_trials, max_frames);
  if (rc != LB_OK) {
    lb_batch_destroy(b);
    return rc;
  }
  *out = b;
  return LB_OK;
}

static int batch_alloc(lb_batch* b, int32_t max_trials, int32_t max_frames) {
  CK(lbk::set_smem_limit(b->L.nthreads, b->L.smem_bytes));
  const size_t B = (size_t)max_trials, K = (size_t)b->K, O = (size_t)b->O;
  int64_t ncap = (int64_t)max_frames * b->K * b->O + 1;
  const int64_t budget_nodes = (int64_t)16e9 / (8 * (int64_t)B);
  ncap = std::min<int64_t>(ncap, std::max<int64_t>(4096, budget_nodes));
  ncap = std::min<int64_t>(ncap, (int64_t)1 << 30);
  BatchDev& d = b->dev;
  // speculative n-gram pairs per frame (leading parents in score order; the rest of the
  // selected word-boundary beams take the warp path).  Measured: config 2 (k = 64) flat at
  // 64..80 (7.13 ms vs 7.23 at 160); k = 256: 42.7 ms at 64 vs 56.0 ms at 256 (full).
  d.spec_cap = 64;
  if (const char* e = std::getenv("LB_SPEC_CAP")) d.spec_cap = std::max(0, std::atoi(e));
  d.Tmax = max_frames;
  d.K = b->K;
  d.O = b->O;
  d.VPD = b->VPD;
  d.ncap = (int32_t)ncap;
  CK(dalloc(&b->d_T, B));
  CK(dalloc(&b->d_D, B * max_frames * b->VPD));
  CK(dalloc(&d.nbeam, B));
  CK(dalloc(&d.score, B * K));
  CK(dalloc(&d.h1, B * K));
  CK(dalloc(&d.h2, B * K));
  CK(dalloc(&d.last, B * K));
  CK(dalloc(&d.prefix, B * K));
  CK(dalloc(&d.nent, B * K));
  CK(dalloc(&d.ents, B * K * O));
  CK(dalloc(&d.nparent, B * ncap));
  CK(dalloc(&d.nsurf, B * ncap));
  CK(dalloc(&d.ncount, B));
  CK(dalloc(&d.status, B));
  CK(dalloc(&d.fail_frame, B));
  CK(dalloc(&d.stats, B * 8));
  CK(cudaMemset(d.stats, 0, B * 8 * sizeof(unsigned long long)));
  CK(dalloc(&d.gscratch, std::max<int64_t>(16, b->L.gscratch_bytes) * B));
  d.gscratch_stride = std::max<int64_t>(16, b->L.gscratch_bytes);
  CK(dalloc(&b->d_counts, 2 * B));
  CK(dalloc(&b->d_entry_off, B + 1));
  CK(dalloc(&b->d_word_off, B + 1));
  d.T = b->d_T;
  d.D = b->d_D;
  CK(cudaEventCreate(&b->ev0));
  CK(cudaEventCreate(&b->ev1));
  CK(cudaEventCreateWithFlags(&b->evd, cudaEventDisableTiming));
  b->T_host.assign(B, 0);
  return LB_OK;
}

int lb_batch_layout(lb_batch* b, int64_t* smem_bytes, int64_t* gscratch_bytes,
                    int32_t* nthreads) {
  if (!b) return fail(LB_ERR_ARG, "null argument");
  if (smem_bytes) *smem_bytes = b->L.smem_bytes;
  if (gscratch_bytes) *gscratch_bytes = b->L.gscratch_bytes;
  if (nthreads) *nthreads = b->L.nthreads;
  return LB_OK;
}

int lb_batch_destroy(lb_batch* b) {
  if (!b) return LB_OK;
  cudaSetDevice(b->m->device);
  cudaStreamSynchronize(b->st);
  BatchDev& d = b->dev;
  void* ptrs[] = {b->d_T, b->d_D, b->d_x, d.nbeam, d.score, d.h1, d.h2, d.last, d.prefix, d.nent,
                  d.ents, d.nparent, d.nsurf, d.ncount, d.status,
                  d.fail_frame, d.stats, d.gscratch, b->d_counts, b->d_entry_off,
                  b->d_word_off, b->d_e_trial, b->d_e_beam, b->d_e_woff, b->d_words,
                  b->d_totals, b->d_puncts, b->d_scores_in, b->d_puncts_in, b->d_has_text,
                  d.dump_h1, d.dump_h2, d.dump_pre, d.dump_last, d.dump_score, d.dump_k,
                  d.phase_cycles};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  void* hptrs[] = {b->h_beam, b->h_punct, b->h_woff, b->h_tot, b->h_words, b->h_misc, b->h_sc};
  for (void* p : hptrs)
    if (p) cudaFreeHost(p);
  if (b->ev0) cudaEventDestroy(b->ev0);
  if (b->ev1) cudaEventDestroy(b->ev1);
  if (b->evd) cudaEventDestroy(b->evd);
  delete b;
  return LB_OK;
}

static int set_trials(lb_batch* b, int32_t n, const int32_t* frames) {
  if (n < 1 || n > b->Bmax) return fail(LB_ERR_ARG, "n_trials out of range");
  for (int32_t i = 0; i < n; ++i)
    if (frames[i] < 0 || frames[i] > b->Tmax) return fail(LB_ERR_ARG, "frames out of range");
  b->n_trials = n;
  b->dev.B = n;
  b->T_host.assign(frames, frames + n);
  CK(cudaMemcpyAsync(b->d_T, frames, n * sizeof(int32_t), cudaMemcpyHostToDevice, b->st));
  return LB_OK;
}

int lb_batch_set_logprobs(lb_batch* b, int32_t n, const double* x, const int32_t* frames,
                          int32_t on_device) {
  if (!b || !x || !frames) return fail(LB_ERR_ARG, "null argument");
  int rc = set_trials(b, n, frames);
  if (rc) return rc;
  const int V = b->m->dev.V;
  CK(cudaMemcpy2DAsync(b->d_D, b->VPD * sizeof(double), x, V * sizeof(double), V * sizeof(double),
                       (size_t)n * b->Tmax,
                       on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, b->st));
  CK(lbk::rowmax(b->d_D, (int64_t)n * b->Tmax, V, b->VPD, b->st));
  return LB_OK;
}

int lb_batch_set_logits(lb_batch* b, int32_t n, const float* x, const int32_t* frames,
                        int32_t on_device) {
  if (!b || !x || !frames) return fail(LB_ERR_ARG, "null argument");
  int rc = set_trials(b, n, frames);
  if (rc) return rc;
  const int V = b->m->dev.V;
  const size_t rows = (size_t)n * b->Tmax;
  const float* src = x;
  if (!on_device) {
    if (!b->d_x) CK(dalloc(&b->d_x, (size_t)b->Bmax * b->Tmax * V));
    CK(cudaMemcpyAsync(b->d_x, x, rows * V * sizeof(float), cudaMemcpyHostToDevice, b->st));
    src = b->d_x;
  }
  CK(lbk::log_softmax(src, (int64_t)rows, V, V, b->cfg.acoustic_scale, b->d_D, b->VPD, b->st));
  return LB_OK;
}

int lb_batch_get_logprobs(lb_batch* b, double* out) {
  if (!b || !out) return fail(LB_ERR_ARG, "null argument");
  const int V = b->m->dev.V;
  CK(cudaMemcpy2DAsync(out, V * sizeof(double), b->d_D, b->VPD * sizeof(double), V * sizeof(double),
                       (size_t)b->n_trials * b->Tmax, cudaMemcpyDeviceToHost, b->st));
  CK(cudaStreamSynchronize(b->st));
  return LB_OK;
}

int lb_batch_reset(lb_batch* b) {
  if (!b || b->n_trials < 1) return fail(LB_ERR_STATE, "no trials loaded");
  CK(lbk::reset(b->m->dev, b->dev, b->st));
  return LB_OK;
}

int lb_batch_run(lb_batch* b, int32_t t_begin, int32_t t_end, int32_t fusion_mode,
                 double scorer_scale) {
  if (!b || b->n_trials < 1) return fail(LB_ERR_STATE, "no trials loaded");
  if (t_begin < 0 || t_end > b->Tmax || t_begin > t_end) return fail(LB_ERR_ARG, "bad frame range");
  if (t_begin == t_end) return LB_OK;
  CK(lbk::frames(b->m->dev, b->cdev, b->dev, b->L, t_begin, t_end, fusion_mode, scorer_scale,
                 b->st));
  return LB_OK;
}

int lb_batch_close(lb_batch* b) {
  if (!b || b->n_trials < 1) return fail(LB_ERR_STATE, "no trials loaded");
  CK(lbk::close(b->m->dev, b->cdev, b->dev, b->st));
  return LB_OK;
}

int lb_batch_device_ngram_fusion(lb_batch* b, int32_t final_, double scale, int32_t min_frames) {
  if (!b || b->n_trials < 1) return fail(LB_ERR_STATE, "no trials loaded");
  CK(lbk::device_ngram_fusion(b->m->dev, b->cdev, b->dev, final_, scale, min_frames, b->st));
  return LB_OK;
}

int lb_batch_gather_entries(lb_batch* b, int64_t* n_entries, int64_t* n_words) {
  if (!b || b->n_trials < 1) return fail(LB_ERR_STATE, "no trials loaded");
  const int B = b->n_trials;
  CK(lbk::count_entries(b->dev, b->d_counts, b->st));
  std::vector<int64_t> counts(2 * (size_t)B);
  CK(cudaMemcpyAsync(counts.data(), b->d_counts, counts.size() * 8, cudaMemcpyDeviceToHost, b->st));
  CK(cudaStreamSynchronize(b->st));
  b->h_entry_off.assign(B + 1, 0);
  b->h_word_off.assign(B + 1, 0);
  for (int i = 0; i < B; ++i) {
    b->h_entry_off[i + 1] = b->h_entry_off[i] + counts[2 * i];
    b->h_word_off[i + 1] = b->h_word_off[i] + counts[2 * i + 1];
  }
  const int64_t ne = b->h_entry_off[B], nw = b->h_word_off[B];
  if (ne > b->cap_entries) {
    const int64_t cap = std::max<int64_t>(ne, 2 * b->cap_entries);
    for (void* p : {(void*)b->d_e_trial, (void*)b->d_e_beam, (void*)b->d_e_woff,
                    (void*)b->d_totals, (void*)b->d_puncts, (void*)b->d_scores_in,
                    (void*)b->d_puncts_in, (void*)b->d_has_text})
      if (p) cudaFree(p);
    CK(dalloc(&b->d_e_trial, cap));
    CK(dalloc(&b->d_e_beam, cap));
    CK(dalloc(&b->d_e_woff, cap + 1));
    CK(dalloc(&b->d_totals, cap));
    CK(dalloc(&b->d_puncts, cap));
    CK(dalloc(&b->d_scores_in, cap));
    CK(dalloc(&b->d_puncts_in, cap));
    CK(dalloc(&b->d_has_text, cap));
    b->cap_entries = cap;
  }
  if (nw > b->cap_words) {
    const int64_t cap = std::max<int64_t>(nw, 2 * b->cap_words);
    if (b->d_words) cudaFree(b->d_words);
    CK(dalloc(&b->d_words, cap));
    b->cap_words = cap;
  }
  CK(cudaMemcpyAsync(b->d_entry_off, b->h_entry_off.data(), (B + 1) * 8, cudaMemcpyHostToDevice, b->st));
  CK(cudaMemcpyAsync(b->d_word_off, b->h_word_off.data(), (B + 1) * 8, cudaMemcpyHostToDevice, b->st));
  CK(lbk::write_entries(b->dev, b->d_entry_off, b->d_word_off, b->d_e_trial, b->d_e_beam,
                        b->d_e_woff, b->d_words, b->d_totals, b->d_puncts, b->st));
  b->n_entries = ne;
  b->n_words = nw;
  if (n_entries) *n_entries = ne;
  if (n_words) *n_words = nw;
  return LB_OK;
}

int lb_batch_copy_entries(lb_batch* b, int32_t* entry_trial, int32_t* entry_beam,
                          int64_t* word_offsets, int32_t* words, double* totals, int32_t* puncts) {
  if (!b) return fail(LB_ERR_ARG, "null argument");
  const int64_t ne = b->n_entries, nw = b->n_words;
  if (ne > 0) {
    if (entry_trial) CK(cudaMemcpyAsync(entry_trial, b->d_e_trial, ne * 4, cudaMemcpyDeviceToHost, b->st));
    if (entry_beam) CK(cudaMemcpyAsync(entry_beam, b->d_e_beam, ne * 4, cudaMemcpyDeviceToHost, b->st));
    if (word_offsets) CK(cudaMemcpyAsync(word_offsets, b->d_e_woff, ne * 8, cudaMemcpyDeviceToHost, b->st));
    if (totals) CK(cudaMemcpyAsync(totals, b->d_totals, ne * 8, cudaMemcpyDeviceToHost, b->st));
    if (puncts) CK(cudaMemcpyAsync(puncts, b->d_puncts, ne * 4, cudaMemcpyDeviceToHost, b->st));
  }
  if (nw > 0 && words) CK(cudaMemcpyAsync(words, b->d_words, nw * 4, cudaMemcpyDeviceToHost, b->st));
  CK(cudaStreamSynchronize(b->st));
  if (word_offsets) word_offsets[ne] = nw;
  return LB_OK;
}

int lb_batch_apply_scores(lb_batch* b, const double* scores, const int32_t* puncts,
                          const uint8_t* has_text, int32_t final_, int32_t min_frames) {
  if (!b || !scores || !has_text) return fail(LB_ERR_ARG, "null argument");
  const int64_t ne = b->n_entries;
  if (ne > 0) {
    CK(cudaMemcpyAsync(b->d_scores_in, scores, ne * 8, cudaMemcpyHostToDevice, b->st));
    CK(cudaMemcpyAsync(b->d_has_text, has_text, ne, cudaMemcpyHostToDevice, b->st));
    if (puncts) CK(cudaMemcpyAsync(b->d_puncts_in, puncts, ne * 4, cudaMemcpyHostToDevice, b->st));
    else CK(cudaMemsetAsync(b->d_puncts_in, 0, ne * 4, b->st));
  }
  CK(lbk::apply_scores(b->cdev, b->dev, b->d_entry_off, b->d_scores_in, b->d_puncts_in,
                       b->d_has_text, final_, min_frames, b->st));
  return LB_OK;
}

int lb_batch_status(lb_batch* b, int32_t* status, int32_t* fail_frame) {
  if (!b) return fail(LB_ERR_ARG, "null argument");
  const int B = b->n_trials;
  if (status) CK(cudaMemcpyAsync(status, b->dev.status, B * 4, cudaMemcpyDeviceToHost, b->st));
  if (fail_frame) CK(cudaMemcpyAsync(fail_frame, b->dev.fail_frame, B * 4, cudaMemcpyDeviceToHost, b->st));
  CK(cudaStreamSynchronize(b->st));
  return LB_OK;
}

int lb_batch_stats(lb_batch* b, lb_stats* out) {
  if (!b || !out) return fail(LB_ERR_ARG, "null argument");
  const int B = b->n_trials;
  std::vector<unsigned long long> s((size_t)B * 8);
  std::vector<int32_t> nc(B);
  CK(cudaMemcpyAsync(s.data(), b->dev.stats, s.size() * 8, cudaMemcpyDeviceToHost, b->st));
  CK(cudaMemcpyAsync(nc.data(), b->dev.ncount, B * 4, cudaMemcpyDeviceToHost, b->st));
  CK(cudaStreamSynchronize(b->st));
  std::memset(out, 0, sizeof(*out));
  for (int i = 0; i < B; ++i) {
    out->frames += s[8 * i + 0];
    out->beams_in += s[8 * i + 1];
    out->beams_out += s[8 * i + 2];
    out->ngram_calls += s[8 * i + 3];
    out->ngram_probes += s[8 * i + 4];
    out->boundary_beams += s[8 * i + 5];
    out->fallback_selects += s[8 * i + 7];
    out->ngram_pairs_used += s[8 * i + 6];
    out->history_nodes += (uint64_t)std::max(0, nc[i] - 1);
  }
  return LB_OK;
}

int lb_batch_clear_stats(lb_batch* b) {
  if (!b) return fail(LB_ERR_ARG, "null argument");
  CK(cudaMemsetAsync(b->dev.stats, 0, (size_t)b->Bmax * 8 * 8, b->st));
  return LB_OK;
}

int lb_batch_dump_beams(lb_batch* b, int32_t trial, int32_t* k, double* scores, uint64_t* h1,
                        uint64_t* h2, int32_t* prefix, int32_t* last) {
  if (!b || trial < 0 || trial >= b->n_trials) return fail(LB_ERR_ARG, "bad trial");
  int32_t kk = 0;
  CK(cudaMemcpyAsync(&kk, b->dev.nbeam + trial, 4, cudaMemcpyDeviceToHost, b->st));
  CK(cudaStreamSynchronize(b->st));
  const size_t hb = (size_t)trial * b->K;
  *k = kk;
  if (kk > 0) {
    CK(cudaMemcpyAsync(scores, b->dev.score + hb, kk * 8, cudaMemcpyDeviceToHost, b->st));
    CK(cudaMemcpyAsync(h1, b->dev.h1 + hb, kk * 8, cudaMemcpyDeviceToHost, b->st));
    CK(cudaMemcpyAsync(h2, b->dev.h2 + hb, kk * 8, cudaMemcpyDeviceToHost, b->st));
    CK(cudaMemcpyAsync(prefix, b->dev.prefix + hb, kk * 4, cudaMemcpyDeviceToHost, b->st));
    CK(cudaMemcpyAsync(last, b->dev.last + hb, kk * 4, cudaMemcpyDeviceToHost, b->st));
  }
  CK(cudaStreamSynchronize(b->st));
  return LB_OK;
}

int lb_batch_enable_phase_timing(lb_batch* b, int32_t on) {
  if (!b) return fail(LB_ERR_ARG, "null argument");
  BatchDev& d = b->dev;
  if (on && !d.phase_cycles) {
    CK(dalloc(&d.phase_cycles, (size_t)b->Bmax * NPHASE));
    CK(cudaMemset(d.phase_cycles, 0, (size_t)b->Bmax * NPHASE * 8));
  } else if (!on && d.phase_cycles) {
    cudaFree(d.phase_cycles);
    d.phase_cycles = nullptr;
  }
  return LB_OK;
}

int lb_batch_phase_cycles(lb_batch* b, uint64_t* out /* [NPHASE] summed over trials */) {
  if (!b || !b->dev.phase_cycles) return fail(LB_ERR_STATE, "phase timing not enabled");
  std::vector<unsigned long long> v((size_t)b->n_trials * NPHASE);
  CK(cudaMemcpy(v.data(), b->dev.phase_cycles, v.size() * 8, cudaMemcpyDeviceToHost));
  for (int i = 0; i < NPHASE; ++i) out[i] = 0;
  for (int t = 0; t < b->n_trials; ++t)
    for (int i = 0; i < NPHASE; ++i) out[i] += v[(size_t)t * NPHASE + i];
  return LB_OK;
}

int lb_batch_enable_dump(lb_batch* b, int32_t on) {
  if (!b) return fail(LB_ERR_ARG, "null argument");
  BatchDev& d = b->dev;
  if (on && !d.dump_k) {
    const size_t n = (size_t)b->Bmax * b->Tmax * b->K;
    CK(dalloc(&d.dump_h1, n));
    CK(dalloc(&d.dump_h2, n));
    CK(dalloc(&d.dump_pre, n));
    CK(dalloc(&d.dump_last, n));
    CK(dalloc(&d.dump_score, n));
    CK(dalloc(&d.dump_k, (size_t)b->Bmax * b->Tmax));
    CK(cudaMemset(d.dump_k, 0xFF, (size_t)b->Bmax * b->Tmax * 4));
  } else if (!on && d.dump_k) {
    for (void* p : {(void*)d.dump_h1, (void*)d.dump_h2, (void*)d.dump_pre, (void*)d.dump_last,
                    (void*)d.dump_score, (void*)d.dump_k})
      cudaFree(p);
    d.dump_h1 = d.dump_h2 = nullptr;
    d.dump_pre = d.dump_last = d.dump_k = nullptr;
    d.dump_score = nullptr;
  }
  return LB_OK;
}

int lb_batch_dump_frame(lb_batch* b, int32_t trial, int32_t t, int32_t* k, double* scores,
                        uint64_t* h1, uint64_t* h2, int32_t* prefix, int32_t* last) {
  if (!b || !b->dev.dump_k) return fail(LB_ERR_STATE, "dump not enabled");
  if (trial < 0 || trial >= b->n_trials || t < 0 || t >= b->Tmax) return fail(LB_ERR_ARG, "bad index");
  const BatchDev& d = b->dev;
  int32_t kk = 0;
  CK(cudaMemcpyAsync(&kk, d.dump_k + (size_t)trial * b->Tmax + t, 4, cudaMemcpyDeviceToHost, b->st));
  CK(cudaStreamSynchronize(b->st));
  *k = kk;
  if (kk > 0) {
    const size_t base = ((size_t)trial * b->Tmax + t) * b->K;
    CK(cudaMemcpyAsync(scores, d.dump_score + base, kk * 8, cudaMemcpyDeviceToHost, b->st));
    CK(cudaMemcpyAsync(h1, d.dump_h1 + base, kk * 8, cudaMemcpyDeviceToHost, b->st));
    CK(cudaMemcpyAsync(h2, d.dump_h2 + base, kk * 8, cudaMemcpyDeviceToHost, b->st));
    CK(cudaMemcpyAsync(prefix, d.dump_pre + base, kk * 4, cudaMemcpyDeviceToHost, b->st));
    CK(cudaMemcpyAsync(last, d.dump_last + base, kk * 4, cudaMemcpyDeviceToHost, b->st));
    CK(cudaStreamSynchronize(b->st));
  }
  return LB_OK;
}

// ------------------------------------------------------------------ results (host assembly)
extern "C++" {
// Pinned host staging for the result gather (D2H at full link speed, reused across calls).
template <typename T>
static int pinned_reserve(T*& p, int64_t& cap, int64_t n) {
  if (n <= cap) return LB_OK;
  if (p) cudaFreeHost(p);
  p = nullptr;
  const int64_t c = std::max<int64_t>(n, 2 * cap);
  if (cudaHostAlloc(reinterpret_cast<void**>(&p), (size_t)std::max<int64_t>(c, 1) * sizeof(T),
                    cudaHostAllocDefault) != cudaSuccess)
    return fail(LB_ERR_CUDA, "cudaHostAlloc failed for result staging");
  cap = c;
  return LB_OK;
}

// Persistent worker pool for the host-side result assembly (spawning threads per call cost
// ~1 ms per config-2 batch).  run(n, f) calls f(0..n-1) on the workers and the caller.
class HostPool {
 public:
  explicit HostPool(int nw) {
    for (int w = 0; w < nw; ++w) th_.emplace_back([this] { loop(); });
  }
  template <typename F>
  void run(int n, F&& f) {
    if (n <= 0) return;
    std::function<void(int)> fn(f);
    // one job at a time: batches driven from different host threads share the pool, and a
    // caller that finds it busy runs its job inline instead of waiting
    std::unique_lock<std::mutex> owner(run_mu_, std::try_to_lock);
    if (!owner.owns_lock() || th_.empty() || n == 1) {
      for (int i = 0; i < n; ++i) fn(i);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = &fn;
      n_ = n;
      next_.store(0);
      ++gen_;
    }
    cv_.notify_all();
    for (int i; (i = next_.fetch_add(1)) < n;) fn(i);
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [&] { return active_ == 0; });
    job_ = nullptr;
  }

 private:
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* f;
      int n;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        f = job_;
        n = n_;
        if (!f) continue;
        ++active_;
      }
      for (int i; (i = next_.fetch_add(1)) < n;) (*f)(i);
      std::lock_guard<std::mutex> lk(mu_);
      if (--active_ == 0) done_.notify_all();
    }
  }
  std::vector<std::thread> th_;
  std::mutex run_mu_, mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  int n_ = 0, active_ = 0;
  uint64_t gen_ = 0;
  std::atomic<int> next_{0};
};

static HostPool& host_pool() {
  // never destroyed: workers block on the condition variable until process exit
  static HostPool* pool = new HostPool(
      std::max(0, std::min(15, (int)std::thread::hardware_concurrency() - 1)));
  return *pool;
}

// Text of an entry = " ".join(surfaces) + punct.  When every surface is non-empty, unique, free
// of ' ' and does not end in ".?!", (word ids, punct) -> text is injective, so the n-best text
// dedupe (decoder.py:444-449) can compare word-id sequences and build strings only for the
// entries that survive.
static bool texts_injective(const lb_model* m) {
  for (const auto& x : m->surfaces) {
    if (x.empty() || x.find(' ') != std::string::npos) return false;
    const char last = x.back();
    if (last == '.' || last == '?' || last == '!') return false;
  }
  return true;
}

}  // extern "C++"

int lb_batch_results_size(lb_batch* b, int64_t* blob_bytes, int64_t* total_nbest) {
  if (!b || b->n_trials < 1) return fail(LB_ERR_STATE, "no trials loaded");
  int rc = lb_batch_gather_entries(b, nullptr, nullptr);
  if (rc) return rc;
  const int B = b->n_trials;
  const int64_t ne = b->n_entries, nw = b->n_words;
  rc = pinned_reserve(b->h_beam, b->hcap_e1, ne);
  if (!rc) rc = pinned_reserve(b->h_punct, b->hcap_e2, ne);
  if (!rc) rc = pinned_reserve(b->h_woff, b->hcap_e3, ne + 1);
  if (!rc) rc = pinned_reserve(b->h_tot, b->hcap_e4, ne);
  if (!rc) rc = pinned_reserve(b->h_words, b->hcap_w, nw);
  if (!rc) rc = pinned_reserve(b->h_misc, b->hcap_m, 2 * (int64_t)B);
  if (!rc) rc = pinned_reserve(b->h_sc, b->hcap_s, (int64_t)B * b->K);
  if (rc) return rc;
  int32_t* e_beam = b->h_beam;
  int32_t* puncts = b->h_punct;
  int64_t* woff = b->h_woff;
  double* totals = b->h_tot;
  int32_t* words = b->h_words;
  int32_t* nbeam = b->h_misc;
  int32_t* status = b->h_misc + B;
  double* scores = b->h_sc;
  CK(cudaMemcpyAsync(nbeam, b->dev.nbeam, B * 4, cudaMemcpyDeviceToHost, b->st));
  CK(cudaMemcpyAsync(status, b->dev.status, B * 4, cudaMemcpyDeviceToHost, b->st));
  CK(cudaMemcpyAsync(scores, b->dev.score, (size_t)B * b->K * 8, cudaMemcpyDeviceToHost, b->st));
  rc = lb_batch_copy_entries(b, nullptr, e_beam, woff, words, totals, puncts);  // synchronises
  if (rc) return rc;
  static const char* PUN[4] = {"", ".", "?", "!"};
  static const int PUNLEN[4] = {0, 1, 1, 1};
  const auto& surf = b->m->surfaces;
  if (b->injective < 0) b->injective = texts_injective(b->m) ? 1 : 0;
  const bool fast = b->injective == 1;
  // phase A (parallel over trials): ranking + n-best dedupe -> selected entries, scores and
  // text byte lengths; no strings are built on the injective path
  struct TrialOut {
    int64_t best_e = -1;
    double best_score = 0.0;
    std::vector<int64_t> ents;
    std::vector<double> scores;
    std::vector<int32_t> lens;
    int32_t best_len = 0;
    size_t bytes = 0;
  };
  std::vector<TrialOut> outs(B);
  auto text_len = [&](int64_t e) {
    int64_t len = PUNLEN[puncts[e] & 3];
    for (int64_t w = woff[e]; w < woff[e + 1]; ++w) len += (int64_t)surf[words[w]].size() + (w > woff[e]);
    return (int32_t)len;
  };
  auto write_text = [&](int64_t e, char* dst) {
    for (int64_t w = woff[e]; w < woff[e + 1]; ++w) {
      if (w > woff[e]) *dst++ = ' ';
      const std::string& x = surf[words[w]];
      std::memcpy(dst, x.data(), x.size());
      dst += x.size();
    }
    const int pl = PUNLEN[puncts[e] & 3];
    if (pl) *dst++ = PUN[puncts[e] & 3][0];
    *dst = '\0';
  };
  auto text_of = [&](int64_t e) {
    std::string s2((size_t)text_len(e) + 1, '\0');
    write_text(e, &s2[0]);
    s2.pop_back();
    return s2;
  };
  auto same_words = [&](int64_t x, int64_t y) {
    if ((puncts[x] & 3) != (puncts[y] & 3)) return false;
    const int64_t nx = woff[x + 1] - woff[x];
    if (nx != woff[y + 1] - woff[y]) return false;
    return std::memcmp(words + woff[x], words + woff[y], (size_t)nx * 4) == 0;
  };
  auto assemble = [&](int t) {
    if (status[t] != 0) return;
    TrialOut& to = outs[t];
    const int K = nbeam[t];
    const int64_t e0 = b->h_entry_off[t], e1 = b->h_entry_off[t + 1];
    std::vector<int64_t> first(K + 1, e1);
    for (int64_t e = e1 - 1; e >= e0; --e) first[e_beam[e]] = e;
    first[K] = e1;
    for (int i = K - 1; i >= 0; --i)
      if (first[i] > first[i + 1]) first[i] = first[i + 1];
    const double* sc = scores + (size_t)t * b->K;
    std::vector<int> order(K);
    for (int i = 0; i < K; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return sc[x] > sc[y]; });
    struct Pair {
      int64_t e;
      double score;
    };
    std::vector<Pair> pairs;
    pairs.reserve(e1 - e0);
    for (int i : order) {
      const double best_lm = totals[first[i]];
      for (int64_t e = first[i]; e < first[i + 1]; ++e) pairs.push_back({e, (sc[i] - best_lm) + totals[e]});
    }
    std::stable_sort(pairs.begin(), pairs.end(),
                     [](const Pair& x, const Pair& y) { return x.score > y.score; });
    to.best_score = sc[order[0]];
    to.best_e = first[order[0]];
    to.best_len = text_len(to.best_e);
    to.bytes = (size_t)to.best_len + 1;
    to.ents.reserve(pairs.size());
    auto keep = [&](const Pair& pr) {
      const int32_t len = text_len(pr.e);
      to.ents.push_back(pr.e);
      to.scores.push_back(pr.score);
      to.lens.push_back(len);
      to.bytes += (size_t)len + 1;
    };
    if (fast) {
      // dedupe on (word ids, punct): FNV hash buckets, exact comparison on hash match
      std::unordered_map<uint64_t, std::vector<int64_t>> seen;
      seen.reserve(pairs.size() * 2);
      for (const Pair& pr : pairs) {
        uint64_t h = 0xCBF29CE484222325ull ^ (uint64_t)(puncts[pr.e] & 3);
        for (int64_t w = woff[pr.e]; w < woff[pr.e + 1]; ++w) h = (h ^ (uint32_t)words[w]) * 0x100000001B3ull;
        auto& bucket = seen[h];
        bool dup = false;
        for (int64_t o : bucket)
          if (same_words(o, pr.e)) {
            dup = true;
            break;
          }
        if (dup) continue;
        bucket.push_back(pr.e);
        keep(pr);
      }
      return;
    }
    std::vector<std::string> texts(e1 - e0);
    for (int64_t e = e0; e < e1; ++e) texts[e - e0] = text_of(e);
    std::unordered_set<std::string_view> seen;
    seen.reserve(pairs.size() * 2);
    for (const Pair& pr : pairs)
      if (seen.insert(std::string_view(texts[pr.e - e0])).second) keep(pr);
  };
  host_pool().run(B, assemble);
  // phase B (serial): blob layout -- per successful trial its best text then its n-best texts,
  // each followed by a NUL (offsets/lengths exclude the separators)
  std::vector<size_t> tb(B + 1, 0);
  std::vector<int64_t> tn(B + 1, 0);
  for (int t = 0; t < B; ++t) {
    tb[t + 1] = tb[t] + outs[t].bytes;
    tn[t + 1] = tn[t] + (int64_t)outs[t].ents.size();
  }
  const size_t total = tb[B];
  const int64_t nn = tn[B];
  if (total > b->blob_cap) {
    b->blob_cap = std::max(total, 2 * b->blob_cap);
    b->blob.reset(new char[b->blob_cap]);
  }
  b->blob_len = total;
  b->best_off.assign(B, 0);
  b->best_len.assign(B, 0);
  b->best_score.assign(B, 0.0);
  b->nb_count.assign(B, 0);
  b->nb_off.resize(nn);
  b->nb_len.resize(nn);
  b->nb_score.resize(nn);
  // phase C (parallel over trials): texts written in place
  char* blob = b->blob.get();
  host_pool().run(B, [&](int t) {
    if (status[t] != 0) return;
    const TrialOut& to = outs[t];
    size_t at = tb[t];
    b->best_off[t] = (int64_t)at;
    b->best_len[t] = to.best_len;
    b->best_score[t] = to.best_score;
    write_text(to.best_e, blob + at);
    at += (size_t)to.best_len + 1;
    const int64_t q0 = tn[t];
    b->nb_count[t] = (int32_t)to.ents.size();
    for (size_t i = 0; i < to.ents.size(); ++i) {
      b->nb_off[q0 + i] = (int64_t)at;
      b->nb_len[q0 + i] = to.lens[i];
      b->nb_score[q0 + i] = to.scores[i];
      write_text(to.ents[i], blob + at);
      at += (size_t)to.lens[i] + 1;
    }
  });
  *blob_bytes = (int64_t)total;
  *total_nbest = nn;
  return LB_OK;
}

int lb_batch_results(lb_batch* b, char* blob, int64_t* best_text_off, int32_t* best_text_len,
                     double* best_score, int32_t* nbest_count, int64_t* nbest_text_off,
                     int32_t* nbest_text_len, double* nbest_score) {
  if (!b) return fail(LB_ERR_ARG, "null argument");
  const int B = b->n_trials;
  if (blob && b->blob_len) std::memcpy(blob, b->blob.get(), b->blob_len);
  for (int t = 0; t < B; ++t) {
    if (best_text_off) best_text_off[t] = b->best_off[t];
    if (best_text_len) best_text_len[t] = b->best_len[t];
    if (best_score) best_score[t] = b->best_score[t];
    if (nbest_count) nbest_count[t] = b->nb_count[t];
  }
  const size_t n = b->nb_score.size();
  for (size_t i = 0; i < n; ++i) {
    if (nbest_text_off) nbest_text_off[i] = b->nb_off[i];
    if (nbest_text_len) nbest_text_len[i] = b->nb_len[i];
    if (nbest_score) nbest_score[i] = b->nb_score[i];
  }
  return LB_OK;
}

int lb_batch_results_view(lb_batch* b, lb_results_view* out) {
  if (!b || !out) return fail(LB_ERR_ARG, "null argument");
  const int B = b->n_trials;
  if ((int)b->best_off.size() != B || !b->h_misc) return fail(LB_ERR_STATE, "call lb_batch_results_size first");
  out->n_trials = B;
  out->total_nbest = (int64_t)b->nb_score.size();
  out->blob_bytes = (int64_t)b->blob_len;
  out->blob = b->blob.get();
  out->status = b->h_misc + B;
  out->best_text_off = b->best_off.data();
  out->best_text_len = b->best_len.data();
  out->best_score = b->best_score.data();
  out->nbest_count = b->nb_count.data();
  out->nbest_text_off = b->nb_off.data();
  out->nbest_text_len = b->nb_len.data();
  out->nbest_score = b->nb_score.data();
  return LB_OK;
}

int lb_stream_create(int32_t device, void** out) {
  if (!out) return fail(LB_ERR_ARG, "null argument");
  CK(cudaSetDevice(device));
  cudaStream_t st = nullptr;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  *out = st;
  return LB_OK;
}

int lb_stream_destroy(void* stream) {
  if (stream) cudaStreamDestroy(reinterpret_cast<cudaStream_t>(stream));
  return LB_OK;
}

int lb_host_alloc(int64_t bytes, void** out) {
  if (!out || bytes < 0) return fail(LB_ERR_ARG, "bad arguments");
  CK(cudaHostAlloc(out, (size_t)std::max<int64_t>(bytes, 1), cudaHostAllocPortable));
  return LB_OK;
}

int lb_host_free(void* p) {
  if (p) CK(cudaFreeHost(p));
  return LB_OK;
}

int lb_launch_count(uint64_t* out) {
  if (!out) return fail(LB_ERR_ARG, "null argument");
  *out = lbk::g_launches;
  return LB_OK;
}

int lb_batch_mark_begin(lb_batch* b) {
  if (!b) return fail(LB_ERR_ARG, "null argument");
  b->launch_mark = lbk::g_launches;
  CK(cudaEventRecord(b->ev0, b->st));
  return LB_OK;
}

int lb_batch_mark_end(lb_batch* b, float* ms, int64_t* launches) {
  if (!b) return fail(LB_ERR_ARG, "null argument");
  CK(cudaEventRecord(b->ev1, b->st));
  CK(cudaEventSynchronize(b->ev1));
  float t = 0.f;
  CK(cudaEventElapsedTime(&t, b->ev0, b->ev1));
  if (ms) *ms = t;
  if (launches) *launches = (int64_t)(lbk::g_launches - b->launch_mark);
  return LB_OK;
}

int lb_batch_after(lb_batch* b, lb_batch* prev) {
  if (!b || !prev) return fail(LB_ERR_ARG, "null argument");
  if (b == prev || b->st == prev->st) return LB_OK;  // one stream is already ordered
  CK(cudaEventRecord(prev->evd, prev->st));
  CK(cudaStreamWaitEvent(b->st, prev->evd, 0));
  return LB_OK;
}

int lb_batch_sync(lb_batch* b) {
  if (!b) return fail(LB_ERR_ARG, "null argument");
  CK(cudaStreamSynchronize(b->st));
  return LB_OK;
}

int lb_log_softmax_host(const float* x, int64_t rows, int32_t cols, double alpha, double* out,
                        int32_t device) {
  if (!x || !out || cols < 1 || cols > 64) return fail(LB_ERR_ARG, "bad arguments");
  CK(cudaSetDevice(device));
  float* dx = nullptr;
  double* dy = nullptr;
  CK(dalloc(&dx, (size_t)rows * cols));
  CK(dalloc(&dy, (size_t)rows * cols));
  CK(cudaMemcpy(dx, x, (size_t)rows * cols * 4, cudaMemcpyHostToDevice));
  CK(lbk::log_softmax(dx, rows, cols, cols, alpha, dy, cols, 0));
  CK(cudaMemcpy(out, dy, (size_t)rows * cols * 8, cudaMemcpyDeviceToHost));
  cudaFree(dx);
  cudaFree(dy);
  return LB_OK;
}

int lb_model_score_words(lb_model* m, int32_t n, const uint32_t* hist, const int32_t* hist_len,
                         const int32_t* word, double* inc, uint32_t* succ, int32_t* succ_len) {
  if (!m || n < 0) return fail(LB_ERR_ARG, "bad arguments");
  if (n == 0) return LB_OK;
  CK(cudaSetDevice(m->device));
  uint32_t *dh = nullptr, *ds = nullptr;
  int32_t *dl = nullptr, *dw = nullptr, *dsl = nullptr;
  double* di = nullptr;
  CK(dalloc(&dh, (size_t)n * 3));
  CK(dalloc(&ds, (size_t)n * 3));
  CK(dalloc(&dl, (size_t)n));
  CK(dalloc(&dw, (size_t)n));
  CK(dalloc(&dsl, (size_t)n));
  CK(dalloc(&di, (size_t)n));
  CK(cudaMemcpy(dh, hist, (size_t)n * 12, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dl, hist_len, (size_t)n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dw, word, (size_t)n * 4, cudaMemcpyHostToDevice));
  CK(lbk::score_words(m->dev, n, dh, dl, dw, di, ds, dsl, 0));
  CK(cudaMemcpy(inc, di, (size_t)n * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(succ, ds, (size_t)n * 12, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(succ_len, dsl, (size_t)n * 4, cudaMemcpyDeviceToHost));
  for (void* p : {(void*)dh, (void*)ds, (void*)dl, (void*)dw, (void*)dsl, (void*)di}) cudaFree(p);
  return LB_OK;
}

}  // extern "C"
