// lb_llm.cu -- delayed LLM fusion on the device: the prefix-trie KV cache behind a
// Llama-architecture scorer and the kernels around its transformer body.
//
// Reference semantics (what is computed):
//   apply_llm            decoder.py:329-372  (texts of every ortho entry, replace lm_total by
//                        llm_weight * score, final pass picks punctuation, beam delta)
//   score_texts/score_eos  scorer.py:285-325 (dedupe, chunking: results are chunk-invariant)
//   sidecar convention   sidecar/src/model.ts:35-47,116-137 (BOS + tokens of the sentence-cased
//                        text, score = sum of natural-log next-token probabilities, empty text
//                        scores 0, eos = best of text+".", "?", "!" with strict > so ties -> ".")
//
// How (B200 design): every text at a fusion event is a path in the decoder's word-history
// trie, and one word is one token, so the token sequences of all texts of all utterances form
// one prefix trie.  Each trie node ("slot") is evaluated once per batch decode:
//   - slots are hash-consed on (parent slot, token) so equal texts share one slot;
//   - a slot's log-prob needs only its parent's final hidden state and log-sum-exp
//     (lp = h_parent . E[token] - lse_parent), so the transformer forward runs only for slots
//     that get children or need end-of-sentence punctuation ("forward set"), all of one event
//     in one pass in slot-id order, which is a dependency order (a row attends to K/V written in
//     the same layer by its new ancestors, or by earlier events: tree-causal prefill);
//   - attention reads K/V straight from the slot cache through per-row ancestor chains (page
//     size one token), so surviving beams never copy or reorder KV: the cache is indexed by
//     text, not by beam, and a beam reorder is free.
// Text score = cum[slot] = sum of lp along the path in root-to-leaf order (fp64), exactly the
// order of the sidecar's full-sequence sum.
//
// Kernels:
//   map_nodes_kernel      word-history nodes of live entries -> slots (per utterance CTA,
//                         unmapped ancestors resolved parent-first, global hash-consing)
//   schedule_kernel       cum-needed slots and the forward set of this event
//   flag_count/blk_scan/compact_kernel   forward set in slot-id (= dependency) order
//   wave_rows_kernel      tokens, positions, ancestor chains of a wave's rows
//   add_rmsnorm_kernel    residual add + RMSNorm (fp32 residual stream, bf16 GEMM operand)
//   rope_kv_kernel        rotary embedding of q/k, K/V written into the slot cache
//   chain_attn_kernel     causal GQA attention of one new token over its ancestor chain
//   swiglu_kernel         silu(gate) * up
//   lse_kernel            K6: row log-sum-exp of the LM-head logits (128k vocab)
//   lp_kernel / cum_kernel  K6 gather: next-token log-prob and running text score
//   punct_kernel          end-of-sentence punctuation log-probs of final texts
//   llm_apply_kernel      K7: fusion into the ortho entries and beam scores
#include <cuda.h>  // CUtensorMap (TMA descriptors; the encoder is fetched at run time)
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/lightbeam_b200.h"
#include "lb_device.cuh"
#include "lb_internal.h"
#include "lb_structs.h"

using namespace lbd;
typedef __nv_bfloat16 bf16;

#define FULLMASK 0xffffffffu

namespace {

constexpr int MAX_LEVELS = LB_LLM_MAX_WAVES;

struct LlmDev {
  int32_t L, NH, NKV, HD, H, vocab;
  int64_t cap;        // slot capacity
  int32_t max_depth;  // deepest slot (tokens after BOS); chain pitch = max_depth + 1
  int32_t* s_parent;
  int32_t* s_token;
  int32_t* s_depth;
  int32_t* s_fwd;  // 0 none, 1 scheduled, 2 forwarded (K/V, hidden, lse present)
  int32_t* s_cum;  // 0 none, 1 scheduled, 2 score ready
  int32_t* s_pun;  // 0 none, 1 punctuation log-probs present
  double* s_lp;
  double* s_cumv;
  double* s_plp;  // [cap][3]
  float* s_lse;
  float* s_h;  // [cap][H] final normed hidden state (fp32: the next-token dot products)
  void* kc;    // [L][cap][NKV*HD] bf16, or fp32 when split
  void* vc;
  int32_t split;  // 1: bf16x2 precision (activations as hi+lo bf16 pairs, fp32 q/K/V)
  int32_t* htab;
  uint32_t hmask;
  int32_t* ctr;  // see C_* below
  int32_t* node_slot;  // [B][ncap]
  int32_t* nlist;      // [B][nlist_cap] claimed nodes of this event
  int32_t* nlist_depth;
  int32_t nlist_cap;
  int32_t* fwd_list;
  int32_t* cum_list;
  int32_t* wave_slots;
  int32_t* blk;        // [ceil(cap / 1024)] compaction block offsets
  const int32_t* tok_low;  // surface tokens after an earlier word, CSR over tok_low_off
  const int32_t* tok_cap;  // surface tokens as the sentence-cased first word, CSR over tok_cap_off
  const int32_t* tok_low_off;
  const int32_t* tok_cap_off;
  int32_t n_surf;
  int32_t bos_tok;
  int32_t punct_tok[3];
  const bf16* emb;
  const float* head32;  // fp32 LM head for the lp / punct dot products (nullptr: emb)
};

enum {
  C_SLOTS = 0,   // slots allocated
  C_ERR = 1,     // bit 1: slot capacity, 2: node list, 4: depth
  C_NFWD = 2,    // forward-set size of this event
  C_NCUM = 3,    // cum-needed slots of this event
  C_BOS = 4,     // 1: BOS slot still to be forwarded
  C_EVENTS = 5,  // graph-mode (async) events, forward rows, largest event: device-side stats
  C_ROWS = 6,
  C_MAXROWS = 7,
  C_NCTR = 8
};

__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double xsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }

__device__ __forceinline__ int ld_vol(const int32_t* p) { return *(const volatile int32_t*)p; }

__device__ __forceinline__ float warp_sum(float v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULLMASK, v, o);
  return v;
}
__device__ __forceinline__ float warp_maxf(float v) {
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(FULLMASK, v, o));
  return v;
}

// insertion sort of <= OMAX entries by (-total, seq) (decoder.py:369)
__device__ __forceinline__ void sort_ents(Ent* e, int n) {
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

// ------------------------------------------------------------------ slot hash-consing
// Slot ids live in an open-addressing table; a key (parent slot, token) is compared through
// the slot's own fields, which the inserting thread publishes before its CAS.
__device__ int hashcons(const LlmDev& l, int ps, int tok, int depth) {
  const uint64_t key = ((uint64_t)(uint32_t)ps << 32) | (uint32_t)tok;
  uint32_t h = (uint32_t)mix64(key) & l.hmask;
  int mine = -1;
  for (uint32_t probe = 0; probe <= l.hmask; ++probe) {
    int v = ld_vol(l.htab + h);
    if (v < 0) {
      if (mine < 0) {
        mine = atomicAdd(l.ctr + C_SLOTS, 1);
        if (mine >= l.cap - 1) {  // slot cap-1: scratch row of padded graph-mode rows
          atomicOr(l.ctr + C_ERR, 1);
          return -1;
        }
        l.s_parent[mine] = ps;
        l.s_token[mine] = tok;
        l.s_depth[mine] = depth;
        l.s_fwd[mine] = 0;
        l.s_cum[mine] = 0;
        l.s_pun[mine] = 0;
        __threadfence();
      }
      v = atomicCAS(l.htab + h, -1, mine);
      if (v < 0) return mine;
    }
    __threadfence();
    if (ld_vol(l.s_parent + v) == ps && ld_vol(l.s_token + v) == tok) {
      if (mine >= 0) l.s_parent[mine] = -2;  // lost an insert race: tombstone the spare slot
      return v;
    }
    h = (h + 1) & l.hmask;
  }
  atomicOr(l.ctr + C_ERR, 1);
  return -1;
}

// ------------------------------------------------------------------ event planning
// Node -> slot for every node on the word-history path of a live entry.  Nodes without a slot
// are claimed (-1 -> -2) by exactly one walker, listed, then resolved level by level: a node
// is ready once its parent has a slot.
__global__ void __launch_bounds__(256) map_nodes_kernel(BatchDev b, LlmDev l, int min_frames) {
  const int trial = blockIdx.x;
  if (b.status[trial] != 0 || b.T[trial] <= min_frames) return;
  __shared__ int s_n, s_more;
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  const size_t hb = (size_t)trial * b.K;
  const size_t nb = (size_t)trial * b.ncap;
  const size_t lb = (size_t)trial * l.nlist_cap;
  int32_t* ns = l.node_slot + nb;
  const int K = b.nbeam[trial], O = b.O;
  for (int i = threadIdx.x; i < K * O; i += blockDim.x) {
    const int beam = i / O, q = i - beam * O;
    if (q >= b.nent[hb + beam]) continue;
    const Ent& E = b.ents[(hb + beam) * O + q];
    uint32_t n = E.node;
    int d = E.depth;
    while (true) {
      if (ld_vol(ns + n) != -1) break;
      if (atomicCAS(ns + n, -1, -2) != -1) break;
      const int idx = atomicAdd(&s_n, 1);
      if (idx < l.nlist_cap) {
        l.nlist[lb + idx] = (int)n;
        l.nlist_depth[lb + idx] = d;
      } else {
        atomicOr(l.ctr + C_ERR, 2);
      }
      n = b.nparent[nb + n];
      --d;
    }
  }
  __syncthreads();
  const int nn = min(s_n, l.nlist_cap);
  for (int iter = 0; iter < 4 * 1024; ++iter) {
    if (threadIdx.x == 0) s_more = 0;
    __syncthreads();
    for (int j = threadIdx.x; j < nn; j += blockDim.x) {
      const int n = l.nlist[lb + j];
      if (ld_vol(ns + n) >= 0) continue;
      const int p = (int)b.nparent[nb + n];
      const int ps = ld_vol(ns + p);
      if (ps < 0) {
        s_more = 1;
        continue;
      }
      const int d = l.nlist_depth[lb + j];
      // the word's tokens hang below its parent's slot one slot per token (word-level
      // tokenizers: one; char-level: " w o r d"); the node maps to the last one
      const int surf = (int)b.nsurf[nb + n];
      const int32_t* toff = d == 1 ? l.tok_cap_off : l.tok_low_off;
      const int32_t* toks = d == 1 ? l.tok_cap : l.tok_low;
      int s = ps;
      for (int k = toff[surf]; k < toff[surf + 1]; ++k) {
        const int dep = ld_vol(l.s_depth + s) + 1;
        if (dep > l.max_depth) {
          atomicOr(l.ctr + C_ERR, 4);
          s = -1;
          break;
        }
        s = hashcons(l, s, toks[k], dep);
        if (s < 0) break;
      }
      ns[n] = s < 0 ? 0 : s;  // on error map to the root so the walk terminates
    }
    __syncthreads();
    if (!s_more) break;
    __syncthreads();
  }
}

__device__ __forceinline__ void push(int32_t* list, int32_t* ctr, int32_t v, int64_t cap) {
  const int idx = atomicAdd(ctr, 1);
  if (idx < cap) list[idx] = v;
}

// Scores still missing on the paths of live entries, and the slots whose forward they need.
__global__ void __launch_bounds__(128) schedule_kernel(BatchDev b, LlmDev l, int min_frames,
                                                       int final_) {
  const int trial = blockIdx.x;
  if (trial == 0 && threadIdx.x == 0 && l.ctr[C_BOS]) {
    l.ctr[C_BOS] = 0;
    push(l.fwd_list, l.ctr + C_NFWD, 0, l.cap);
  }
  if (b.status[trial] != 0 || b.T[trial] <= min_frames) return;
  const size_t hb = (size_t)trial * b.K;
  const int32_t* ns = l.node_slot + (size_t)trial * b.ncap;
  const int K = b.nbeam[trial], O = b.O;
  for (int i = threadIdx.x; i < K * O; i += blockDim.x) {
    const int beam = i / O, q = i - beam * O;
    if (q >= b.nent[hb + beam]) continue;
    const Ent& E = b.ents[(hb + beam) * O + q];
    int cur = ns[E.node];
    if (final_ && cur != 0 && atomicCAS(l.s_fwd + cur, 0, 1) == 0)
      push(l.fwd_list, l.ctr + C_NFWD, cur, l.cap);
    while (cur != 0) {
      if (ld_vol(l.s_cum + cur) != 0) break;
      if (atomicCAS(l.s_cum + cur, 0, 1) != 0) break;
      push(l.cum_list, l.ctr + C_NCUM, cur, l.cap);
      const int p = l.s_parent[cur];
      if (atomicCAS(l.s_fwd + p, 0, 1) == 0) push(l.fwd_list, l.ctr + C_NFWD, p, l.cap);
      cur = p;
    }
  }
}

// The event's rows = scheduled slots in slot-id order.  A slot is allocated after its parent,
// so id order is a dependency order (every row's new ancestors precede it), and slots created by
// one utterance in one event are close in id space, so consecutive rows share ancestors and the
// attention gathers of neighbouring CTAs hit the same K/V lines in L2.
constexpr int CB = 1024;
__global__ void __launch_bounds__(CB) flag_count_kernel(LlmDev l, int32_t* blk) {
  const int ns = min(l.ctr[C_SLOTS], (int)l.cap);
  const int s = blockIdx.x * CB + threadIdx.x;
  if (blockIdx.x * CB >= ns) {
    if (threadIdx.x == 0) blk[blockIdx.x] = 0;
    return;
  }
  const int f = s < ns && l.s_fwd[s] == 1;
  const int c = __syncthreads_count(f);
  if (threadIdx.x == 0) blk[blockIdx.x] = c;
}

__global__ void __launch_bounds__(CB) blk_scan_kernel(int32_t* blk, int nblk) {
  __shared__ int part[CB];
  const int per = (nblk + CB - 1) / CB;
  const int b0 = threadIdx.x * per, b1 = min(nblk, b0 + per);
  int sum = 0;
  for (int i = b0; i < b1; ++i) sum += blk[i];
  part[threadIdx.x] = sum;
  __syncthreads();
  for (int o = 1; o < CB; o <<= 1) {  // inclusive Hillis-Steele scan
    const int v = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  int run = part[threadIdx.x] - sum;
  for (int i = b0; i < b1; ++i) {
    const int c = blk[i];
    blk[i] = run;
    run += c;
  }
}

__global__ void __launch_bounds__(CB) compact_kernel(LlmDev l, const int32_t* blk_off) {
  __shared__ int wsum[CB / 32];
  const int ns = min(l.ctr[C_SLOTS], (int)l.cap);
  if (blockIdx.x * CB >= ns) return;
  const int s = blockIdx.x * CB + threadIdx.x;
  const int f = s < ns && l.s_fwd[s] == 1;
  const unsigned bal = __ballot_sync(FULLMASK, f);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) wsum[warp] = __popc(bal);
  __syncthreads();
  if (warp == 0) {
    int v = wsum[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULLMASK, v, o);
      if (lane >= o) v += y;
    }
    wsum[lane] = v - wsum[lane];  // exclusive
  }
  __syncthreads();
  if (f) l.wave_slots[blk_off[blockIdx.x] + wsum[warp] + __popc(bal & ((1u << lane) - 1))] = s;
}

// Graph-mode events: the host never reads the row count.  plan_async_kernel flags an event
// with more rows than the captured capacity (the caller re-runs the decode eagerly) and keeps
// the device-side stats; wave_rows_async_kernel fills all `cap_rows` rows, the ones past the
// event's count as BOS-only padding whose K/V, hidden state and LSE land in the scratch slot.
__global__ void plan_async_kernel(LlmDev l, int cap_rows) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const int n = l.ctr[C_NFWD];
    if (n > cap_rows) l.ctr[C_ERR] |= 8;
    l.ctr[C_EVENTS] += 1;
    l.ctr[C_ROWS] += min(n, cap_rows);
    l.ctr[C_MAXROWS] = max(l.ctr[C_MAXROWS], n);
  }
}

__global__ void wave_rows_async_kernel(LlmDev l, int cap_rows, int32_t* tok, int32_t* pos,
                                       int32_t* slots, int32_t* chains) {
  const int pitch = l.max_depth + 1;
  const int n = min(l.ctr[C_NFWD], cap_rows);
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < cap_rows; r += gridDim.x * blockDim.x) {
    int32_t* ch = chains + (size_t)r * pitch;
    if (r >= n) {
      tok[r] = l.bos_tok;
      pos[r] = 0;
      slots[r] = (int32_t)(l.cap - 1);
      ch[0] = 0;
      continue;
    }
    const int s = l.wave_slots[r];
    const int d = l.s_depth[s];
    tok[r] = l.s_token[s];
    pos[r] = d;
    slots[r] = s;
    int cur = s;
    for (int j = d; j >= 0; --j) {
      ch[j] = cur;
      cur = l.s_parent[cur];
    }
  }
}

__global__ void wave_rows_kernel(LlmDev l, int64_t row0, int n, int32_t* tok, int32_t* pos,
                                 int32_t* slots, int32_t* chains) {
  const int pitch = l.max_depth + 1;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const int s = l.wave_slots[row0 + r];
    const int d = l.s_depth[s];
    tok[r] = l.s_token[s];
    pos[r] = d;
    slots[r] = s;
    int cur = s;
    int32_t* ch = chains + (size_t)r * pitch;
    for (int j = d; j >= 0; --j) {
      ch[j] = cur;
      cur = l.s_parent[cur];
    }
  }
}

// ------------------------------------------------------------------ transformer body
// x[M][H] fp32 residual (+= delta fp32 when given) -> out = bf16(x * rsqrt(mean(x^2) + eps) * w);
// `store_slots` also keeps the fp32 row in the slot hidden-state table.
// bias != nullptr: LayerNorm y = (x - mean) * rsqrt(var + eps) * w + bias (GPT-2), two-pass
constexpr int NORM_NPT = 4;  // float4 per thread held in registers: hidden <= 256 * 4 * 4 = 4096

__device__ __forceinline__ float block_sum256(float v, float* red) {
  v = warp_sum(v);
  __syncthreads();  // red[] may still be read by a previous reduction
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int w2 = 0; w2 < 8; ++w2) t += red[w2];
  return t;
}

// bias != nullptr: LayerNorm y = (x - mean) * rsqrt(var + eps) * w + bias (GPT-2), two-pass
// over the register-resident row; otherwise RMSNorm.  x is read once (+= delta, written back).
// Programmatic dependent launch: the body kernels below may be launched before their
// predecessor finishes (launch latency hidden); they wait for its memory here first.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

__global__ void __launch_bounds__(256) add_rmsnorm_kernel(float* x, const float* delta,
                                                          const float* w, float eps, int H,
                                                          bf16* out, const int32_t* store_slots,
                                                          float* s_h, int split,
                                                          const float* bias = nullptr) {
  pdl_wait();
  __shared__ float red[8];
  const int row = blockIdx.x;
  float* xr = x + (size_t)row * H;
  const float* dr = delta ? delta + (size_t)row * H : nullptr;
  float4 v[NORM_NPT];
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < NORM_NPT; ++j) {
    const int i = (threadIdx.x + j * 256) * 4;
    v[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i < H) {
      v[j] = *reinterpret_cast<const float4*>(xr + i);
      if (dr) {
        const float4 a = *reinterpret_cast<const float4*>(dr + i);
        v[j].x += a.x;
        v[j].y += a.y;
        v[j].z += a.z;
        v[j].w += a.w;
        *reinterpret_cast<float4*>(xr + i) = v[j];
      }
      ss += bias ? (v[j].x + v[j].y + v[j].z + v[j].w)
                 : (v[j].x * v[j].x + v[j].y * v[j].y + v[j].z * v[j].z + v[j].w * v[j].w);
    }
  }
  const float tot = block_sum256(ss, red);
  float mean = 0.f, r;
  if (bias) {  // LayerNorm: tot is the plain sum; centred variance from the registers
    mean = tot / (float)H;
    float vs = 0.f;
#pragma unroll
    for (int j = 0; j < NORM_NPT; ++j) {
      const int i = (threadIdx.x + j * 256) * 4;
      if (i < H) {
        const float a = v[j].x - mean, b2 = v[j].y - mean, c2 = v[j].z - mean, d2 = v[j].w - mean;
        vs += a * a + b2 * b2 + c2 * c2 + d2 * d2;
      }
    }
    r = rsqrtf(block_sum256(vs, red) / (float)H + eps);
  } else {
    r = rsqrtf(tot / (float)H + eps);
  }
  bf16* orow = out + (size_t)row * H * (split ? 2 : 1);
  float* hrow = store_slots ? s_h + (size_t)store_slots[row] * H : nullptr;
#pragma unroll
  for (int j = 0; j < NORM_NPT; ++j) {
    const int i = (threadIdx.x + j * 256) * 4;
    if (i >= H) continue;
    const float4 g = *reinterpret_cast<const float4*>(w + i);
    float4 y;
    if (bias) {
      const float4 bb = *reinterpret_cast<const float4*>(bias + i);
      y = make_float4((v[j].x - mean) * r * g.x + bb.x, (v[j].y - mean) * r * g.y + bb.y,
                      (v[j].z - mean) * r * g.z + bb.z, (v[j].w - mean) * r * g.w + bb.w);
    } else {
      y = make_float4(v[j].x * r * g.x, v[j].y * r * g.y, v[j].z * r * g.z, v[j].w * r * g.w);
    }
    __nv_bfloat162* op = reinterpret_cast<__nv_bfloat162*>(orow + i);
    const __nv_bfloat162 h0 = __floats2bfloat162_rn(y.x, y.y), h1 = __floats2bfloat162_rn(y.z, y.w);
    op[0] = h0;
    op[1] = h1;
    if (split) {  // lo half: the bf16 rounding residual, so hi + lo carries ~16 mantissa bits
      const float2 a = __bfloat1622float2(h0), c = __bfloat1622float2(h1);
      __nv_bfloat162* lp = reinterpret_cast<__nv_bfloat162*>(orow + H + i);
      lp[0] = __floats2bfloat162_rn(y.x - a.x, y.y - a.y);
      lp[1] = __floats2bfloat162_rn(y.z - c.x, y.w - c.y);
    }
    if (hrow) *reinterpret_cast<float4*>(hrow + i) = y;
  }
}

template <typename T>
__device__ __forceinline__ T to_store(float v);
template <>
__device__ __forceinline__ bf16 to_store<bf16>(float v) { return __float2bfloat16_rn(v); }
template <>
__device__ __forceinline__ float to_store<float>(float v) { return v; }

template <typename T, int HD>
__global__ void rope_kv_kernel(LlmDev l, int layer, const float* qkv, int M, const int32_t* pos,
                               const int32_t* slots, const float* cosT, const float* sinT,
                               T* q_out) {
  pdl_wait();
  const int row = blockIdx.x;
  if (row >= M) return;
  constexpr int half = HD / 2;
  const int NH = l.NH, NKV = l.NKV;
  const int W = (NH + 2 * NKV) * HD;
  const float* in = qkv + (size_t)row * W;
  const int p = pos[row];  // rotary tables: one row per position
  const size_t slot = (size_t)slots[row];
  const size_t kvw = (size_t)NKV * HD;
  // K/V cache rows: bf16 [NKV*HD]; split precision: [hi | lo] bf16 pairs [2*NKV*HD]
  constexpr bool SPLIT = sizeof(T) == 4;
  const size_t roww = kvw * (SPLIT ? 2 : 1);
  bf16* kd = reinterpret_cast<bf16*>(l.kc) + ((size_t)layer * l.cap + slot) * roww;
  bf16* vd = reinterpret_cast<bf16*>(l.vc) + ((size_t)layer * l.cap + slot) * roww;
  const float* cs = cosT + (size_t)p * half;
  const float* sn = sinT + (size_t)p * half;
  const int npairs = (NH + NKV) * half;
  auto put = [&](bf16* base, size_t idx, float v) {
    const bf16 h = __float2bfloat16_rn(v);
    base[idx] = h;
    if (SPLIT) base[kvw + idx] = __float2bfloat16_rn(v - __bfloat162float(h));
  };
  for (int t = threadIdx.x; t < npairs; t += blockDim.x) {
    const int head = t / half, i = t - head * half;
    const float* src = in + head * HD;
    const float x1 = src[i], x2 = src[i + half];
    const float c = cs[i], s = sn[i];
    const float o1 = x1 * c - x2 * s;
    const float o2 = x2 * c + x1 * s;
    if (head < NH) {
      T* dst = q_out + (size_t)row * NH * HD + head * HD;
      dst[i] = to_store<T>(o1);
      dst[i + half] = to_store<T>(o2);
    } else {
      put(kd, (size_t)(head - NH) * HD + i, o1);
      put(kd, (size_t)(head - NH) * HD + i + half, o2);
    }
  }
  const float* vin = in + (NH + NKV) * HD;
  for (int t = threadIdx.x * 4; t < NKV * HD; t += blockDim.x * 4) {
    const float4 v = *reinterpret_cast<const float4*>(vin + t);
    put(vd, t, v.x);
    put(vd, t + 1, v.y);
    put(vd, t + 2, v.z);
    put(vd, t + 3, v.w);
  }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}

// DPL consecutive elements of a bf16 / fp32 vector (16-B aligned) as floats
template <int DPL>
__device__ __forceinline__ void load_f(const bf16* p, float* out) {
#pragma unroll
  for (int c = 0; c < DPL / 8; ++c) {
    const uint4 u = reinterpret_cast<const uint4*>(p)[c];
    const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(p2[e]);
      out[c * 8 + 2 * e] = f.x;
      out[c * 8 + 2 * e + 1] = f.y;
    }
  }
}
template <int DPL>
__device__ __forceinline__ void load_f(const float* p, float* out) {
#pragma unroll
  for (int c = 0; c < DPL / 4; ++c) {
    const float4 u = reinterpret_cast<const float4*>(p)[c];
    out[c * 4] = u.x;
    out[c * 4 + 1] = u.y;
    out[c * 4 + 2] = u.z;
    out[c * 4 + 3] = u.w;
  }
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(sa), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sa), "r"(bytes)
               : "memory");
}
// 1-D TMA bulk copy global -> shared (a gather of one cache row), completion on an mbarrier
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, unsigned bytes,
                                             uint64_t* bar) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const unsigned bb = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(d),
      "l"(src), "r"(bytes), "r"(bb)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n .reg .pred p;\n"
      "LLW%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LLW%=;\n}\n" ::"r"(sa),
      "r"(parity)
      : "memory");
}

constexpr int ATTN_STAGE_BYTES = 32 * 1024;  // K+V rows of one chunk of chain positions

// chain positions per chunk for K/V cache rows of `rowb` bytes (all kv heads of a slot)
__host__ __device__ inline int attn_chunk(int rowb) {
  const int c = ATTN_STAGE_BYTES / (2 * rowb);
  return c < 1 ? 1 : (c > 32 ? 32 : c);
}

// One CTA per row, one warp per kv head.  The row's ancestor chain (BOS .. itself; causal by
// construction) is gathered chunk by chunk: lane j of warp 0 issues two 1-D TMA bulk copies
// (the K and V cache rows of chain position j, all kv heads at once) onto a double-buffered
// stage with an mbarrier, so the next chunk's gather is in flight while this one is consumed.
// Each warp then covers PPW positions per pass with SUB = HD/DPL lanes per position: every lane
// keeps its DPL-dim slice of the G query vectors (its kv head's group) in registers, reduces
// partial dots over its SUB lanes and keeps (max, sum, acc) on a warp-uniform scale, so the
// position groups' partial outputs are summed once at the end.
// Output: bf16 [M][NH*HD], or hi|lo bf16 pairs [M][2*NH*HD] in split precision.
template <int HD, int G, int DPL, typename T>
__global__ void __launch_bounds__(256, 2) chain_attn_kernel(LlmDev l, int layer, const T* q,
                                                            const int32_t* chains,
                                                            const int32_t* pos, float scale,
                                                            bf16* out) {
  constexpr int SUB = HD / DPL;
  constexpr int PPW = 32 / SUB;
  extern __shared__ __align__(128) unsigned char attn_smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(attn_smem);
  unsigned char* stages = attn_smem + 128;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x;
  const int NKV = l.NKV, kvh = warp;
  const int rowb = NKV * HD * (int)sizeof(T);
  const int CH = attn_chunk(rowb);
  const int stage_bytes = 2 * CH * rowb;
  const int n = pos[row] + 1;
  const int nch = (n + CH - 1) / CH;
  const int32_t* ch = chains + (size_t)row * (l.max_depth + 1);
  const unsigned char* kbase = reinterpret_cast<const unsigned char*>(l.kc) + (size_t)layer * l.cap * rowb;
  const unsigned char* vbase = reinterpret_cast<const unsigned char*>(l.vc) + (size_t)layer * l.cap * rowb;
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int c) {  // warp 0
    const int st = c & 1, c0 = c * CH, cn = min(CH, n - c0);
    unsigned char* kd = stages + (size_t)st * stage_bytes;
    unsigned char* vd = kd + (size_t)CH * rowb;
    if (lane == 0) mbar_expect_tx(&bars[st], (unsigned)(2 * cn * rowb));
    __syncwarp();
    if (lane < cn) {
      const size_t sl = (size_t)ch[c0 + lane];
      tma_bulk_g2s(kd + (size_t)lane * rowb, kbase + sl * rowb, rowb, &bars[st]);
      tma_bulk_g2s(vd + (size_t)lane * rowb, vbase + sl * rowb, rowb, &bars[st]);
    }
  };
  if (warp == 0) issue(0);
  const int sub = lane % SUB, pg = lane / SUB;
  float qv[G][DPL];
  {
    const T* qr = q + (size_t)row * l.NH * HD + (size_t)kvh * G * HD + sub * DPL;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      load_f<DPL>(qr + g * HD, qv[g]);
#pragma unroll
      for (int d = 0; d < DPL; ++d) qv[g][d] *= scale;
    }
  }
  float m[G], den[G], acc[G][DPL];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    m[g] = -INFINITY;
    den[g] = 0.f;
#pragma unroll
    for (int d = 0; d < DPL; ++d) acc[g][d] = 0.f;
  }
  const int hoff = (kvh * HD + sub * DPL) * (int)sizeof(T);
  for (int c = 0; c < nch; ++c) {
    if (warp == 0 && c + 1 < nch) issue(c + 1);  // its stage was released by the last barrier
    mbar_wait(&bars[c & 1], (unsigned)((c >> 1) & 1));
    const unsigned char* ks = stages + (size_t)(c & 1) * stage_bytes;
    const unsigned char* vs = ks + (size_t)CH * rowb;
    const int cn = min(CH, n - c * CH);
    for (int pb = 0; pb < cn; pb += PPW) {
      const int j = pb + pg;
      const bool valid = j < cn;
      const int jr = valid ? j : 0;
      float kf[DPL], vf[DPL];
      load_f<DPL>(reinterpret_cast<const T*>(ks + (size_t)jr * rowb + hoff), kf);
      load_f<DPL>(reinterpret_cast<const T*>(vs + (size_t)jr * rowb + hoff), vf);
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float part = 0.f;
#pragma unroll
        for (int d = 0; d < DPL; ++d) part += qv[g][d] * kf[d];
#pragma unroll
        for (int o = SUB / 2; o > 0; o >>= 1) part += __shfl_xor_sync(FULLMASK, part, o);
        const float x = valid ? part : -INFINITY;
        const float mnew = fmaxf(m[g], warp_maxf(x));
        const float p = valid ? __expf(x - mnew) : 0.f;
        const float corr = __expf(m[g] - mnew);  // 0 on the first pass (m = -inf)
        den[g] = den[g] * corr + warp_sum(sub == 0 ? p : 0.f);
#pragma unroll
        for (int d = 0; d < DPL; ++d) acc[g][d] = acc[g][d] * corr + p * vf[d];
        m[g] = mnew;
      }
    }
    __syncthreads();  // every warp is done with this stage before it is refilled
  }
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int d = 0; d < DPL; ++d)
#pragma unroll
      for (int o = 16; o >= SUB; o >>= 1) acc[g][d] += __shfl_xor_sync(FULLMASK, acc[g][d], o);
  if (pg == 0) {
    const int W = l.NH * HD;
    bf16* orow = out + (size_t)row * W * (l.split ? 2 : 1) + (size_t)kvh * G * HD + sub * DPL;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float inv = 1.f / den[g];
#pragma unroll
      for (int c = 0; c < DPL / 8; ++c) {
        uint4 hi, lo;
        __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&hi);
        __nv_bfloat162* l2 = reinterpret_cast<__nv_bfloat162*>(&lo);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float a = acc[g][c * 8 + 2 * e] * inv, b = acc[g][c * 8 + 2 * e + 1] * inv;
          h2[e] = __floats2bfloat162_rn(a, b);
          const float2 hf = __bfloat1622float2(h2[e]);
          l2[e] = __floats2bfloat162_rn(a - hf.x, b - hf.y);
        }
        reinterpret_cast<uint4*>(orow + g * HD)[c] = hi;
        if (l.split) reinterpret_cast<uint4*>(orow + W + g * HD)[c] = lo;
      }
    }
  }
}

// ---------------------------------------------------------------- tensor-core chain attention
__device__ __forceinline__ void mma_bf16_16816(float* d, const uint32_t* a, const uint32_t* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ void ldsm_x4_trans(uint32_t* r, const void* smem_row) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_row);
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(sa));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

constexpr int MMA_CH = 16;  // chain positions per stage (one PV k-step)

// bf16 precision: one CTA per row, one warp per kv head, the G query heads of the group packed
// into the M dimension of m16n8k16 MMAs (rows >= G are zero): S = Q K^T over 8-position tiles,
// online softmax on the accumulator fragments (quad shuffles), then O += P V with P taken
// straight from the S fragments (the C->A register identity) and V read transposed by ldmatrix.
// K/V cache rows (all kv heads of a slot) are gathered per 16-position chunk by 1-D TMA bulk
// copies into a double-buffered stage whose row pitch is padded by 16 B (conflict-free fragment
// loads).
template <int HD, bool SPLIT, int nstages>
__global__ void __launch_bounds__(256) chain_attn_mma_kernel(LlmDev l, int layer,
                                                             const void* qv, const int32_t* chains,
                                                             const int32_t* pos, float scale,
                                                             bf16* out) {
  pdl_wait();
  constexpr int KK = HD / 16;  // k-steps of Q K^T
  constexpr int NT = HD / 8;   // n-tiles of P V
  extern __shared__ __align__(128) unsigned char attn_smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(attn_smem);
  unsigned char* stages = attn_smem + 128;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane >> 2, qd = lane & 3;
  const int row = blockIdx.x;
  const int NKV = l.NKV, kvh = warp, G = l.NH / NKV;
  const int halfb = NKV * HD * 2;              // bytes of one bf16 half-row
  const int rowb = halfb * (SPLIT ? 2 : 1);    // cache row: [hi] or [hi | lo]
  const int pitch = rowb + 16;
  const int stage_bytes = 2 * MMA_CH * pitch;
  const int n = pos[row] + 1;
  const int nch = (n + MMA_CH - 1) / MMA_CH;
  const int32_t* ch = chains + (size_t)row * (l.max_depth + 1);
  const unsigned char* kbase = reinterpret_cast<const unsigned char*>(l.kc) + (size_t)layer * l.cap * rowb;
  const unsigned char* vbase = reinterpret_cast<const unsigned char*>(l.vc) + (size_t)layer * l.cap * rowb;
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int c) {  // warp 0
    const int st = c % nstages, c0 = c * MMA_CH, cn = min(MMA_CH, n - c0);
    unsigned char* kd = stages + (size_t)st * stage_bytes;
    unsigned char* vd = kd + (size_t)MMA_CH * pitch;
    if (lane == 0) mbar_expect_tx(&bars[st], (unsigned)(2 * cn * rowb));
    __syncwarp();
    if (lane < cn) {
      const size_t sl = (size_t)ch[c0 + lane];
      tma_bulk_g2s(kd + (size_t)lane * pitch, kbase + sl * rowb, rowb, &bars[st]);
      tma_bulk_g2s(vd + (size_t)lane * pitch, vbase + sl * rowb, rowb, &bars[st]);
    }
  };
  if (warp == 0) issue(0);
  // Q fragments (A operand): row = head grp (< G), cols = dims; rows >= G and grp + 8 are zero.
  // SPLIT: q is fp32 and becomes a hi + lo pair of bf16 fragments.
  uint32_t qa[KK][4], ql[SPLIT ? KK : 1][4];
#pragma unroll
  for (int kk = 0; kk < KK; ++kk) {
    qa[kk][1] = qa[kk][3] = 0u;
    if (SPLIT) ql[kk][1] = ql[kk][3] = 0u;
#pragma unroll
    for (int hlf = 0; hlf < 2; ++hlf) {
      const int col = kk * 16 + hlf * 8 + qd * 2;
      uint32_t hi = 0u, lo = 0u;
      if (grp < G) {
        if (SPLIT) {
          const float* qr = reinterpret_cast<const float*>(qv) + (size_t)row * l.NH * HD + (size_t)(kvh * G + grp) * HD;
          const float2 f = *reinterpret_cast<const float2*>(qr + col);
          const __nv_bfloat162 h = __floats2bfloat162_rn(f.x, f.y);
          const float2 hf = __bfloat1622float2(h);
          hi = *reinterpret_cast<const uint32_t*>(&h);
          lo = pack_bf16(f.x - hf.x, f.y - hf.y);
        } else {
          const bf16* qr = reinterpret_cast<const bf16*>(qv) + (size_t)row * l.NH * HD + (size_t)(kvh * G + grp) * HD;
          hi = *reinterpret_cast<const uint32_t*>(qr + col);
        }
      }
      qa[kk][hlf * 2] = hi;
      if (SPLIT) ql[kk][hlf * 2] = lo;
    }
  }
  float o[NT][4];
#pragma unroll
  for (int t = 0; t < NT; ++t) o[t][0] = o[t][1] = o[t][2] = o[t][3] = 0.f;
  float m = -INFINITY, den = 0.f;  // per head row grp (identical across the quad)
  const int hoff = kvh * HD * 2;
  for (int c = 0; c < nch; ++c) {
    if (nstages == 2 && warp == 0 && c + 1 < nch) issue(c + 1);
    const int cn = min(MMA_CH, n - c * MMA_CH);
    const int st = c % nstages;
    unsigned char* ks = stages + (size_t)st * stage_bytes;
    unsigned char* vs = ks + (size_t)MMA_CH * pitch;
    if (cn < MMA_CH) {  // zero this warp's slices of the unused V rows (0 * stale NaN = NaN)
      constexpr int U = HD / 4;  // uint2 per head slice
      for (int i = lane; i < (MMA_CH - cn) * U; i += 32) {
        unsigned char* rp = vs + (size_t)(cn + i / U) * pitch + hoff;
        reinterpret_cast<uint2*>(rp)[i % U] = make_uint2(0u, 0u);
        if (SPLIT) reinterpret_cast<uint2*>(rp + halfb)[i % U] = make_uint2(0u, 0u);
      }
    }
    mbar_wait(&bars[st], (unsigned)((c / nstages) & 1));
    __syncwarp();
    float sc[2][4];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      sc[t][0] = sc[t][1] = sc[t][2] = sc[t][3] = 0.f;
      const unsigned char* kr = ks + (size_t)(t * 8 + grp) * pitch + hoff;
#pragma unroll
      for (int kk = 0; kk < KK; ++kk) {
        uint32_t kb2[2];
        kb2[0] = *reinterpret_cast<const uint32_t*>(kr + (kk * 16 + qd * 2) * 2);
        kb2[1] = *reinterpret_cast<const uint32_t*>(kr + (kk * 16 + 8 + qd * 2) * 2);
        mma_bf16_16816(sc[t], qa[kk], kb2);
        if (SPLIT) {  // + q_lo k_hi + q_hi k_lo (the lo*lo term is below fp32 resolution)
          uint32_t kl2[2];
          kl2[0] = *reinterpret_cast<const uint32_t*>(kr + halfb + (kk * 16 + qd * 2) * 2);
          kl2[1] = *reinterpret_cast<const uint32_t*>(kr + halfb + (kk * 16 + 8 + qd * 2) * 2);
          mma_bf16_16816(sc[t], ql[kk], kb2);
          mma_bf16_16816(sc[t], qa[kk], kl2);
        }
      }
    }
    // online softmax over this chunk's positions (t * 8 + qd * 2 + {0, 1})
    float mx = -INFINITY;
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = t * 8 + qd * 2 + e;
        sc[t][e] = j < cn ? sc[t][e] * scale : -INFINITY;
        mx = fmaxf(mx, sc[t][e]);
      }
    mx = fmaxf(mx, __shfl_xor_sync(FULLMASK, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(FULLMASK, mx, 2));
    const float mnew = fmaxf(m, mx);
    const float corr = __expf(m - mnew);
    float ps = 0.f;
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        sc[t][e] = __expf(sc[t][e] - mnew);
        ps += sc[t][e];
      }
    ps += __shfl_xor_sync(FULLMASK, ps, 1);
    ps += __shfl_xor_sync(FULLMASK, ps, 2);
    den = den * corr + ps;
    m = mnew;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      o[t][0] *= corr;
      o[t][1] *= corr;
    }
    // P (A operand, 16 heads x 16 positions) from the S fragments (+ its lo part when split)
    uint32_t pa[4], pl[4];
    pa[1] = pa[3] = pl[1] = pl[3] = 0u;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const __nv_bfloat162 h = __floats2bfloat162_rn(sc[t][0], sc[t][1]);
      pa[t * 2] = *reinterpret_cast<const uint32_t*>(&h);
      if (SPLIT) {
        const float2 hf = __bfloat1622float2(h);
        pl[t * 2] = pack_bf16(sc[t][0] - hf.x, sc[t][1] - hf.y);
      }
    }
    // V (B operand, 16 positions x 8 dims) by ldmatrix.trans: matrices = (pos 0-7 | 8-15) x
    // (dims t*8 .. +8 | (t+1)*8 .. +8)
    __syncwarp();
#pragma unroll
    for (int t = 0; t < NT; t += 2) {
      const int mi = lane >> 3, r = lane & 7;
      const unsigned char* addr = vs + (size_t)((mi & 1) * 8 + r) * pitch + hoff + ((t + (mi >> 1)) * 8) * 2;
      uint32_t vb4[4];
      ldsm_x4_trans(vb4, addr);
      const uint32_t b0[2] = {vb4[0], vb4[1]};
      const uint32_t b1[2] = {vb4[2], vb4[3]};
      mma_bf16_16816(o[t], pa, b0);
      mma_bf16_16816(o[t + 1], pa, b1);
      if (SPLIT) {  // + p_lo v_hi + p_hi v_lo
        uint32_t vl4[4];
        ldsm_x4_trans(vl4, addr + halfb);
        const uint32_t c0[2] = {vl4[0], vl4[1]};
        const uint32_t c1[2] = {vl4[2], vl4[3]};
        mma_bf16_16816(o[t], pl, b0);
        mma_bf16_16816(o[t + 1], pl, b1);
        mma_bf16_16816(o[t], pa, c0);
        mma_bf16_16816(o[t + 1], pa, c1);
      }
    }
    __syncthreads();  // every warp is done with this stage before it is refilled
    if (nstages == 1 && warp == 0 && c + 1 < nch) issue(c + 1);
  }
  if (grp < G) {
    const float inv = 1.f / den;
    const int W = l.NH * HD;
    bf16* orow = out + (size_t)row * W * (SPLIT ? 2 : 1) + (size_t)(kvh * G + grp) * HD;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const float a = o[t][0] * inv, b = o[t][1] * inv;
      const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
      *reinterpret_cast<__nv_bfloat162*>(orow + t * 8 + qd * 2) = h;
      if (SPLIT) {
        const float2 hf = __bfloat1622float2(h);
        *reinterpret_cast<__nv_bfloat162*>(orow + W + t * 8 + qd * 2) = __floats2bfloat162_rn(a - hf.x, b - hf.y);
      }
    }
  }
}

// ---------------------------------------------------------------- sibling-grouped attention
// Rows of one forward chunk that share a parent slot are siblings: same depth d, same ancestor
// chain (positions 0 .. d-1), different own position d.  In the final event of a config-3 batch
// ~6 rows share each parent (every leaf text is forwarded for its punctuation), elsewhere ~1.3.
// Siblings are grouped SIB = 16 / G per tile so one CTA gathers the shared chain once and the
// G x SIB query rows fill the M = 16 rows of the MMAs (the per-row kernel uses G of them).
struct GrpDev {
  int32_t* cnt;     // [cap] siblings per parent slot in this chunk (reset after the build)
  int32_t* base;    // [cap] first tile of a parent's siblings
  int32_t* row_k;   // [rows] sibling index of a row within its parent
  int32_t* tiles;   // [rows][SIB] rows of each tile
  int32_t* tile_n;  // [rows] rows in each tile
  int32_t* ntiles;  // [1]
};

// rows r < n of a forward chunk: slots[r]; n from the host (nh >= 0) or the device's forward-set
// count (nh < 0: planning, before the host knows it)
__device__ __forceinline__ int grp_rows(const LlmDev& l, int nh) {
  return nh >= 0 ? nh : (int)min((int64_t)l.ctr[C_NFWD], l.cap);
}

// the tile key of a row: its ancestor GAP = 1 << gsh levels up (-1: too shallow, a tile alone)
__device__ __forceinline__ int grp_key(const LlmDev& l, int s, int gsh) {
  if (l.s_depth[s] < (1 << gsh)) return -1;
  for (int k = 0; k < (1 << gsh); ++k) s = l.s_parent[s];
  return s;
}

__global__ void grp_count_kernel(LlmDev l, GrpDev g, const int32_t* slots, int nh, int gsh) {
  const int n = grp_rows(l, nh);
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const int key = grp_key(l, slots[r], gsh);
    g.row_k[r] = key >= 0 ? atomicAdd(g.cnt + key, 1) : 0;
  }
}

__global__ void grp_base_kernel(LlmDev l, GrpDev g, const int32_t* slots, int nh, int SIB,
                                int gsh) {
  const int n = grp_rows(l, nh);
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const int key = grp_key(l, slots[r], gsh);
    if (key < 0) {  // too shallow (the BOS row, ...): a tile of its own
      const int t = atomicAdd(g.ntiles, 1);
      g.tiles[(size_t)t * SIB] = r;
      g.tile_n[t] = 1;
    } else if (g.row_k[r] == 0) {
      g.base[key] = atomicAdd(g.ntiles, (g.cnt[key] + SIB - 1) / SIB);
    }
  }
}

__global__ void grp_fill_kernel(LlmDev l, GrpDev g, const int32_t* slots, int nh, int SIB,
                                int gsh) {
  const int n = grp_rows(l, nh);
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const int p = grp_key(l, slots[r], gsh), k = g.row_k[r];
    if (p < 0) continue;
    const int t = g.base[p] + k / SIB;
    g.tiles[(size_t)t * SIB + k % SIB] = r;
    if (k % SIB == 0) g.tile_n[t] = min(SIB, g.cnt[p] - (k / SIB) * SIB);
  }
}

__global__ void grp_reset_kernel(LlmDev l, GrpDev g, const int32_t* slots, int nh, int gsh) {
  const int n = grp_rows(l, nh);
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const int key = grp_key(l, slots[r], gsh);
    if (key >= 0) g.cnt[key] = 0;
  }
}

// One CTA per sibling tile, one warp per kv head.  M row m = sib * G + head-in-group.  The tile
// walks a virtual sequence in 16-position chunks: the shared chain (positions 0 .. d-1, visible to
// every row) followed by the siblings' own K/V rows (position d + i = sibling i, visible only to
// sibling i's rows) -- for a single row exactly chain_attn_mma_kernel's positions 0 .. d.
// grid = (tiles, kv-head groups).
template <int HD, bool SPLIT, int nstages>
__global__ void __launch_bounds__(128, 3) chain_attn_grp_kernel(LlmDev l, int layer, const void* qv,
                                                             const int32_t* chains,
                                                             const int32_t* pos, GrpDev gd,
                                                             int SIB, int gsh, float scale,
                                                             bf16* out) {
  pdl_wait();
  const int tile = blockIdx.x;
  constexpr int KK = HD / 16;
  constexpr int NT = HD / 8;
  extern __shared__ __align__(128) unsigned char attn_smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(attn_smem);
  unsigned char* stages = attn_smem + 128;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane >> 2, qd = lane & 3;
  // blockIdx.y: a group of KH = blockDim.x / 32 kv heads (its slice of each cache row is staged)
  const int NKV = l.NKV, KH = blockDim.x >> 5, h0 = blockIdx.y * KH, kvh = h0 + warp;
  const int G = l.NH / NKV;
  const int cnt = gd.tile_n[tile];
  const int32_t* trow = gd.tiles + (size_t)tile * SIB;
  const int d = pos[trow[0]];
  const int pitchc = l.max_depth + 1;
  // rows of a tile share their ancestors up to depth d - GAP (GAP = 1 << gsh private positions
  // per row: GAP = 1 siblings, 2 cousins): shared chain ch[0 .. nsh-1]
  const int GAP = 1 << gsh, nsh = d - GAP + 1;
  const int32_t* ch = chains + (size_t)trow[0] * pitchc;
  const int ghalf = NKV * HD * 2;                // bytes of one bf16 half of a cache row
  const int grow = ghalf * (SPLIT ? 2 : 1);       // cache row: [hi] or [hi | lo], all kv heads
  const int halfb = KH * HD * 2;                  // staged half: this CTA's kv heads
  const int rowb = halfb * (SPLIT ? 2 : 1);
  const int pitch = rowb + 16;
  const int stage_bytes = 2 * MMA_CH * pitch;
  const int nv = nsh + (cnt << gsh);  // virtual positions: shared chain, then GAP per row
  const int nch = (nv + MMA_CH - 1) / MMA_CH;
  const unsigned char* kbase = reinterpret_cast<const unsigned char*>(l.kc) + (size_t)layer * l.cap * grow + h0 * HD * 2;
  const unsigned char* vbase = reinterpret_cast<const unsigned char*>(l.vc) + (size_t)layer * l.cap * grow + h0 * HD * 2;
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto chunk_n = [&](int c) { return min(MMA_CH, nv - c * MMA_CH); };
  auto issue = [&](int c) {  // warp 0
    const int st = c % nstages, cn = chunk_n(c);
    unsigned char* kd = stages + (size_t)st * stage_bytes;
    unsigned char* vd = kd + (size_t)MMA_CH * pitch;
    if (lane == 0) mbar_expect_tx(&bars[st], (unsigned)(2 * cn * rowb));
    __syncwarp();
    if (lane < cn) {
      const int v = c * MMA_CH + lane;
      const size_t sl = v < nsh ? (size_t)ch[v]
                                : (size_t)chains[(size_t)trow[(v - nsh) >> gsh] * pitchc + nsh +
                                                 ((v - nsh) & (GAP - 1))];
      tma_bulk_g2s(kd + (size_t)lane * pitch, kbase + sl * grow, halfb, &bars[st]);
      tma_bulk_g2s(vd + (size_t)lane * pitch, vbase + sl * grow, halfb, &bars[st]);
      if (SPLIT) {
        tma_bulk_g2s(kd + (size_t)lane * pitch + halfb, kbase + sl * grow + ghalf, halfb, &bars[st]);
        tma_bulk_g2s(vd + (size_t)lane * pitch + halfb, vbase + sl * grow + ghalf, halfb, &bars[st]);
      }
    }
  };
  if (warp == 0) issue(0);
  // Q fragments: A rows grp (a0, a2) and grp + 8 (a1, a3); row m -> sibling m / G, head m % G.
  // Rows of missing siblings keep q = 0 (finite scores, never written).
  uint32_t qa[KK][4], ql[SPLIT ? KK : 1][4];
  int rsib[2];
#pragma unroll
  for (int hr = 0; hr < 2; ++hr) {
    const int mrow = grp + 8 * hr;
    const int sib = mrow / G;
    rsib[hr] = sib;
    const bool valid = sib < cnt;
    const size_t qoff = valid ? ((size_t)trow[sib] * l.NH + (size_t)(kvh * G + mrow % G)) * HD : 0;
#pragma unroll
    for (int kk = 0; kk < KK; ++kk)
#pragma unroll
      for (int hlf = 0; hlf < 2; ++hlf) {
        const int col = kk * 16 + hlf * 8 + qd * 2;
        uint32_t hi = 0u, lo = 0u;
        if (valid) {
          if (SPLIT) {
            const float2 f = *reinterpret_cast<const float2*>(reinterpret_cast<const float*>(qv) + qoff + col);
            const __nv_bfloat162 h = __floats2bfloat162_rn(f.x, f.y);
            const float2 hf = __bfloat1622float2(h);
            hi = *reinterpret_cast<const uint32_t*>(&h);
            lo = pack_bf16(f.x - hf.x, f.y - hf.y);
          } else {
            hi = *reinterpret_cast<const uint32_t*>(reinterpret_cast<const bf16*>(qv) + qoff + col);
          }
        }
        qa[kk][hlf * 2 + hr] = hi;
        if (SPLIT) ql[kk][hlf * 2 + hr] = lo;
      }
  }
  float o[NT][4];
#pragma unroll
  for (int t = 0; t < NT; ++t) o[t][0] = o[t][1] = o[t][2] = o[t][3] = 0.f;
  float mrun[2] = {-INFINITY, -INFINITY}, den[2] = {0.f, 0.f};
  const int hoff = warp * HD * 2;
  for (int c = 0; c < nch; ++c) {
    if (nstages == 2 && warp == 0 && c + 1 < nch) issue(c + 1);
    const int cn = chunk_n(c);
    const int vown = nsh - c * MMA_CH;  // chunk index of row 0's first private position
    const int st = c % nstages;
    unsigned char* ks = stages + (size_t)st * stage_bytes;
    unsigned char* vs = ks + (size_t)MMA_CH * pitch;
    if (cn < MMA_CH) {  // zero this warp's slices of the unused V rows (0 * stale NaN = NaN)
      constexpr int U = HD / 4;
      for (int i = lane; i < (MMA_CH - cn) * U; i += 32) {
        unsigned char* rp = vs + (size_t)(cn + i / U) * pitch + hoff;
        reinterpret_cast<uint2*>(rp)[i % U] = make_uint2(0u, 0u);
        if (SPLIT) reinterpret_cast<uint2*>(rp + halfb)[i % U] = make_uint2(0u, 0u);
      }
    }
    mbar_wait(&bars[st], (unsigned)((c / nstages) & 1));
    __syncwarp();
    float sc[2][4];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      sc[t][0] = sc[t][1] = sc[t][2] = sc[t][3] = 0.f;
      const unsigned char* kr = ks + (size_t)(t * 8 + grp) * pitch + hoff;
#pragma unroll
      for (int kk = 0; kk < KK; ++kk) {
        uint32_t kb2[2];
        kb2[0] = *reinterpret_cast<const uint32_t*>(kr + (kk * 16 + qd * 2) * 2);
        kb2[1] = *reinterpret_cast<const uint32_t*>(kr + (kk * 16 + 8 + qd * 2) * 2);
        mma_bf16_16816(sc[t], qa[kk], kb2);
        if (SPLIT) {
          uint32_t kl2[2];
          kl2[0] = *reinterpret_cast<const uint32_t*>(kr + halfb + (kk * 16 + qd * 2) * 2);
          kl2[1] = *reinterpret_cast<const uint32_t*>(kr + halfb + (kk * 16 + 8 + qd * 2) * 2);
          mma_bf16_16816(sc[t], ql[kk], kb2);
          mma_bf16_16816(sc[t], qa[kk], kl2);
        }
      }
    }
    // online softmax per row (hr 0: row grp, hr 1: row grp + 8)
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = t * 8 + qd * 2 + (e & 1), hr = e >> 1;
        // chain positions are shared; position vown + i is sibling i's own row (rows of missing
        // siblings see everything, finite and never written)
        const bool vis = j < cn && (j < vown || rsib[hr] >= cnt || ((j - vown) >> gsh) == rsib[hr]);
        sc[t][e] = vis ? sc[t][e] * scale : -INFINITY;
        mx[hr] = fmaxf(mx[hr], sc[t][e]);
      }
    float corr[2];
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      mx[hr] = fmaxf(mx[hr], __shfl_xor_sync(FULLMASK, mx[hr], 1));
      mx[hr] = fmaxf(mx[hr], __shfl_xor_sync(FULLMASK, mx[hr], 2));
      const float mnew = fmaxf(mrun[hr], mx[hr]);
      corr[hr] = __expf(mrun[hr] - mnew);
      mrun[hr] = mnew;
    }
    float ps[2] = {0.f, 0.f};
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        sc[t][e] = __expf(sc[t][e] - mrun[e >> 1]);
        ps[e >> 1] += sc[t][e];
      }
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      ps[hr] += __shfl_xor_sync(FULLMASK, ps[hr], 1);
      ps[hr] += __shfl_xor_sync(FULLMASK, ps[hr], 2);
      den[hr] = den[hr] * corr[hr] + ps[hr];
    }
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      o[t][0] *= corr[0];
      o[t][1] *= corr[0];
      o[t][2] *= corr[1];
      o[t][3] *= corr[1];
    }
    // P (A operand, 16 rows x 16 positions) from the S fragments (+ its lo part when split)
    uint32_t pa[4], pl[4];
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        const __nv_bfloat162 h = __floats2bfloat162_rn(sc[t][2 * hr], sc[t][2 * hr + 1]);
        pa[t * 2 + hr] = *reinterpret_cast<const uint32_t*>(&h);
        if (SPLIT) {
          const float2 hf = __bfloat1622float2(h);
          pl[t * 2 + hr] = pack_bf16(sc[t][2 * hr] - hf.x, sc[t][2 * hr + 1] - hf.y);
        }
      }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < NT; t += 2) {
      const int mi = lane >> 3, r = lane & 7;
      const unsigned char* addr = vs + (size_t)((mi & 1) * 8 + r) * pitch + hoff + ((t + (mi >> 1)) * 8) * 2;
      uint32_t vb4[4];
      ldsm_x4_trans(vb4, addr);
      const uint32_t b0[2] = {vb4[0], vb4[1]};
      const uint32_t b1[2] = {vb4[2], vb4[3]};
      mma_bf16_16816(o[t], pa, b0);
      mma_bf16_16816(o[t + 1], pa, b1);
      if (SPLIT) {
        uint32_t vl4[4];
        ldsm_x4_trans(vl4, addr + halfb);
        const uint32_t c0[2] = {vl4[0], vl4[1]};
        const uint32_t c1[2] = {vl4[2], vl4[3]};
        mma_bf16_16816(o[t], pl, b0);
        mma_bf16_16816(o[t + 1], pl, b1);
        mma_bf16_16816(o[t], pa, c0);
        mma_bf16_16816(o[t + 1], pa, c1);
      }
    }
    __syncthreads();  // every warp is done with this stage before it is refilled
    if (nstages == 1 && warp == 0 && c + 1 < nch) issue(c + 1);
  }
  const int W = l.NH * HD;
#pragma unroll
  for (int hr = 0; hr < 2; ++hr) {
    const int mrow = grp + 8 * hr, sib = rsib[hr];
    if (sib >= cnt) continue;
    const float inv = 1.f / den[hr];
    bf16* orow = out + (size_t)trow[sib] * W * (SPLIT ? 2 : 1) + (size_t)(kvh * G + mrow % G) * HD;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const float a = o[t][2 * hr] * inv, b = o[t][2 * hr + 1] * inv;
      const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
      *reinterpret_cast<__nv_bfloat162*>(orow + t * 8 + qd * 2) = h;
      if (SPLIT) {
        const float2 hf = __bfloat1622float2(h);
        *reinterpret_cast<__nv_bfloat162*>(orow + W + t * 8 + qd * 2) = __floats2bfloat162_rn(a - hf.x, b - hf.y);
      }
    }
  }
}

// gu[M][2F] = [gate | up] (bf16, or fp32 in split precision) -> out[M][F] = bf16(silu(gate) * up)
// (split: hi|lo pairs [M][2F]); 8 columns per thread
template <typename TI>
__global__ void swiglu_kernel(const TI* gu, int F, bf16* out, int split) {
  pdl_wait();
  const int row = blockIdx.y;
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (c >= F) return;
  const TI* gr = gu + (size_t)row * 2 * F;
  float g[8], u[8];
  load_f<8>(gr + c, g);
  load_f<8>(gr + F + c, u);
  uint4 ov, lv;
  __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&ov);
  __nv_bfloat162* l2 = reinterpret_cast<__nv_bfloat162*>(&lv);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float a = g[2 * e] / (1.f + __expf(-g[2 * e])) * u[2 * e];
    const float b = g[2 * e + 1] / (1.f + __expf(-g[2 * e + 1])) * u[2 * e + 1];
    o2[e] = __floats2bfloat162_rn(a, b);
    const float2 h = __bfloat1622float2(o2[e]);
    l2[e] = __floats2bfloat162_rn(a - h.x, b - h.y);
  }
  bf16* orow = out + (size_t)row * F * (split ? 2 : 1);
  *reinterpret_cast<uint4*>(orow + c) = ov;
  if (split) *reinterpret_cast<uint4*>(orow + F + c) = lv;
}

// in[M][F] fp32 (+ bias[F]) -> out = bf16(gelu_tanh(in)) (GPT-2 "gelu_new"; split: hi|lo pairs
// [M][2F]); 8 columns per thread
__global__ void gelu_kernel(const float* in, const float* bias, int F, bf16* out, int split) {
  const int row = blockIdx.y;
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (c >= F) return;
  float g[8];
  load_f<8>(in + (size_t)row * F + c, g);
  if (bias) {
    float bb[8];
    load_f<8>(bias + c, bb);
#pragma unroll
    for (int e = 0; e < 8; ++e) g[e] += bb[e];
  }
  uint4 ov, lv;
  __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&ov);
  __nv_bfloat162* l2 = reinterpret_cast<__nv_bfloat162*>(&lv);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    float y[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const float x = g[2 * e + k];
      y[k] = 0.5f * x * (1.f + tanhf(0.7978845608028654f * (x + 0.044715f * x * x * x)));
    }
    o2[e] = __floats2bfloat162_rn(y[0], y[1]);
    const float2 h = __bfloat1622float2(o2[e]);
    l2[e] = __floats2bfloat162_rn(y[0] - h.x, y[1] - h.y);
  }
  bf16* orow = out + (size_t)row * F * (split ? 2 : 1);
  *reinterpret_cast<uint4*>(orow + c) = ov;
  if (split) *reinterpret_cast<uint4*>(orow + F + c) = lv;
}

// K6a: log-sum-exp of one LM-head logit row per CTA (16-B loads, online max/sum merge)
template <typename TL>
__global__ void __launch_bounds__(512) lse_kernel(const TL* logits, int64_t ld, int V,
                                                  const int32_t* slots, float* s_lse) {
  const int row = blockIdx.x;
  const TL* r = logits + (size_t)row * ld;
  float m = -INFINITY, s = 0.f;
  const int nv = V / 8;
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    float x[8];
    load_f<8>(r + (size_t)i * 8, x);
    float mx = x[0];
#pragma unroll
    for (int e = 1; e < 8; ++e) mx = fmaxf(mx, x[e]);
    const float nm = fmaxf(m, mx);
    float acc = s * expf(m - nm);
#pragma unroll
    for (int e = 0; e < 8; ++e) acc += expf(x[e] - nm);
    m = nm;
    s = acc;
  }
  for (int i = nv * 8 + threadIdx.x; i < V; i += blockDim.x) {
    const float x = (float)r[i];
    const float nm = fmaxf(m, x);
    s = s * expf(m - nm) + expf(x - nm);
    m = nm;
  }
  // merge (m, s) across the block
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(FULLMASK, m, o), s2 = __shfl_xor_sync(FULLMASK, s, o);
    const float nm = fmaxf(m, m2);
    s = (nm == -INFINITY) ? 0.f : s * expf(m - nm) + s2 * expf(m2 - nm);
    m = nm;
  }
  __shared__ float sm[32], ssum[32];
  if ((threadIdx.x & 31) == 0) {
    sm[threadIdx.x >> 5] = m;
    ssum[threadIdx.x >> 5] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float M2 = sm[0], S2 = ssum[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      const float nm = fmaxf(M2, sm[w]);
      if (nm == -INFINITY) continue;
      S2 = S2 * expf(M2 - nm) + ssum[w] * expf(sm[w] - nm);
      M2 = nm;
    }
    s_lse[slots[row]] = M2 + logf(S2);
  }
}

// fp32 dot of an fp32 hidden row and a bf16 embedding row of length H by one warp (fixed
// order: lane stride, xor tree)
__device__ __forceinline__ float warp_dot32(const float* a, const float* b, int H) {
  float acc = 0.f;
  for (int i = threadIdx.x % 32; i < H; i += 32) acc += a[i] * b[i];
  return warp_sum(acc);
}

__device__ __forceinline__ float warp_dot(const float* a, const bf16* b, int H) {
  float acc = 0.f;
  for (int i = threadIdx.x % 32 * 8; i < H; i += 256) {
    const float4 a0 = *reinterpret_cast<const float4*>(a + i);
    const float4 a1 = *reinterpret_cast<const float4*>(a + i + 4);
    const uint4 ub = *reinterpret_cast<const uint4*>(b + i);
    const __nv_bfloat162* pb = reinterpret_cast<const __nv_bfloat162*>(&ub);
    const float2 b0 = __bfloat1622float2(pb[0]), b1 = __bfloat1622float2(pb[1]);
    const float2 b2 = __bfloat1622float2(pb[2]), b3 = __bfloat1622float2(pb[3]);
    acc += a0.x * b0.x;
    acc += a0.y * b0.y;
    acc += a0.z * b1.x;
    acc += a0.w * b1.y;
    acc += a1.x * b2.x;
    acc += a1.y * b2.y;
    acc += a1.z * b3.x;
    acc += a1.w * b3.y;
  }
  return warp_sum(acc);
}

// K6b: lp[s] = h[parent] . E[token] - lse[parent]
__global__ void lp_kernel(LlmDev l) {
  const int n = min(l.ctr[C_NCUM], (int)l.cap);
  const int lane = threadIdx.x & 31;
  for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n; w += (gridDim.x * blockDim.x) >> 5) {
    const int s = l.cum_list[w];
    const int p = l.s_parent[s];
    const int tk = l.s_token[s];
    const float dot = l.head32 ? warp_dot32(l.s_h + (size_t)p * l.H, l.head32 + (size_t)tk * l.H, l.H)
                               : warp_dot(l.s_h + (size_t)p * l.H, l.emb + (size_t)tk * l.H, l.H);
    if (lane == 0) l.s_lp[s] = (double)dot - (double)l.s_lse[p];
  }
}

// running score: cum[s] = (((cum[anchor] + lp[a1]) + lp[a2]) + ... + lp[s]) in root-to-leaf
// order, anchor = nearest ancestor whose score was ready before this event
__global__ void cum_kernel(LlmDev l) {
  constexpr int LOC = 64;
  const int n = min(l.ctr[C_NCUM], (int)l.cap);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int s = l.cum_list[i];
    int chain[LOC];
    int k = 0;
    int cur = s;
    while (cur != 0 && l.s_cum[cur] == 1) {
      if (k < LOC) chain[k] = cur;
      ++k;
      cur = l.s_parent[cur];
    }
    double acc = l.s_cumv[cur];
    for (int j = k - 1; j >= 0; --j) {
      int a = 0;
      if (j < LOC) {
        a = chain[j];
      } else {  // long fresh chains (final-only fusion): re-walk to the j-th ancestor
        a = s;
        for (int t = 0; t < j; ++t) a = l.s_parent[a];
      }
      acc = xadd(acc, l.s_lp[a]);
    }
    l.s_cumv[s] = acc;
  }
}

__global__ void commit_kernel(LlmDev l) {
  const int nf = min(l.ctr[C_NFWD], (int)l.cap), nc = min(l.ctr[C_NCUM], (int)l.cap);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < max(nf, nc); i += gridDim.x * blockDim.x) {
    if (i < nf) l.s_fwd[l.fwd_list[i]] = 2;
    if (i < nc) l.s_cum[l.cum_list[i]] = 2;
  }
}

// end-of-sentence punctuation log-probs of the final texts (one warp per entry, claimed slots)
__global__ void __launch_bounds__(256) punct_kernel(BatchDev b, LlmDev l, int min_frames) {
  const int trial = blockIdx.x;
  if (b.status[trial] != 0 || b.T[trial] <= min_frames) return;
  const size_t hb = (size_t)trial * b.K;
  const int32_t* ns = l.node_slot + (size_t)trial * b.ncap;
  const int K = b.nbeam[trial], O = b.O;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = warp; i < K * O; i += blockDim.x >> 5) {
    const int beam = i / O, q = i - beam * O;
    if (q >= b.nent[hb + beam]) continue;
    const int s = ns[b.ents[(hb + beam) * O + q].node];
    if (s == 0) continue;
    int claim = 0;
    if (lane == 0) claim = atomicCAS(l.s_pun + s, 0, 1) == 0;
    if (!__shfl_sync(FULLMASK, claim, 0)) continue;
    for (int j = 0; j < 3; ++j) {
      const int tk = l.punct_tok[j];
      const float dot = l.head32 ? warp_dot32(l.s_h + (size_t)s * l.H, l.head32 + (size_t)tk * l.H, l.H)
                                 : warp_dot(l.s_h + (size_t)s * l.H, l.emb + (size_t)tk * l.H, l.H);
      if (lane == 0) l.s_plp[(size_t)s * 3 + j] = (double)dot - (double)l.s_lse[s];
    }
  }
}

// K7: apply_llm fusion (decoder.py:354-371) from the slot scores
__global__ void llm_apply_kernel(CfgDev c, BatchDev b, LlmDev l, int final_, int min_frames) {
  const int trial = blockIdx.x;
  if (b.status[trial] != 0 || b.T[trial] <= min_frames) return;
  const size_t hb = (size_t)trial * b.K;
  const int32_t* ns = l.node_slot + (size_t)trial * b.ncap;
  const int K = b.nbeam[trial], O = b.O;
  for (int i = threadIdx.x; i < K; i += blockDim.x) {
    Ent* e = b.ents + (hb + i) * O;
    const int n = b.nent[hb + i];
    const double prev = e[0].total;
    for (int q = 0; q < n; ++q) {
      if (e[q].node == 0) {
        e[q].total = 0.0;
        e[q].punct = 0;
        continue;
      }
      const int s = ns[e[q].node];
      double score = l.s_cumv[s];
      if (final_) {
        int best = 0;
        double bs = xadd(score, l.s_plp[(size_t)s * 3]);
        for (int j = 1; j < 3; ++j) {
          const double v = xadd(score, l.s_plp[(size_t)s * 3 + j]);
          if (v > bs) {
            bs = v;
            best = j;
          }
        }
        score = bs;
        e[q].punct = (uint8_t)(best + 1);
      }
      e[q].total = xmul(c.phi, score);
    }
    sort_ents(e, n);
    b.score[hb + i] = xadd(b.score[hb + i], xsub(e[0].total, prev));
  }
}

__global__ void llm_reset_kernel(LlmDev l) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int i = 0; i < C_NCTR; ++i) l.ctr[i] = 0;  // (a kernel, not a host copy: capturable)
    l.ctr[C_SLOTS] = 1;
    l.ctr[C_BOS] = 1;
    l.s_parent[0] = -1;
    l.s_token[0] = l.bos_tok;
    l.s_depth[0] = 0;
    l.s_cum[0] = 2;
    l.s_cumv[0] = 0.0;
    l.s_pun[0] = 0;
    l.s_fwd[0] = 1;  // the BOS row is forwarded with the first event's waves
  }
}

__global__ void root_slots_kernel(int32_t* node_slot, int B, int64_t ncap) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < B; i += gridDim.x * blockDim.x)
    node_slot[(size_t)i * ncap] = 0;
}

// ---------------------------------------------------------------- K6 on tcgen05
// Fused LM head + log-sum-exp: logits = H[M][K] . E[N][K]^T are never written.  A persistent
// warp-specialised kernel: warp 0 (one lane) streams 128x64 A and 256x64 B tiles with 2-D TMA
// (128-byte swizzle) through a 4-stage mbarrier ring; warp 1 (one lane) issues
// tcgen05.mma.cta_group::1.kind::f16 (M=128, N=256, K=16) into a double-buffered TMEM
// accumulator (2 x 256 columns) and commits stage/accumulator barriers; warps 2-5 drain the
// accumulator with tcgen05.ld (thread = row) and fold each 256-column slice into a per-row
// (max, sum exp) partial.  lse_reduce_kernel combines the partials of a row.
constexpr int LM_BM = 128, LM_BN = 256, LM_BK = 64, LM_ST = 4;
constexpr int LM_A_BYTES = LM_BM * LM_BK * 2;
constexpr int LM_B_BYTES = LM_BN * LM_BK * 2;
constexpr int LM_STAGE_BYTES = LM_A_BYTES + LM_B_BYTES;
constexpr int LM_SMEM = 1024 + LM_ST * LM_STAGE_BYTES + 256;
constexpr int LM_THREADS = 192;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row groups 1024 B apart
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);        // start address
  d |= (uint64_t)1 << 16;                         // leading byte offset (unused for SW128 K-major)
  d |= (uint64_t)(1024 >> 4) << 32;               // stride byte offset
  d |= (uint64_t)1 << 46;                         // version (sm_100)
  d |= (uint64_t)2 << 61;                         // layout: SWIZZLE_128B
  return d;
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
// instruction descriptor: D f32, A/B bf16, K-major both, N = 256, M = 128
constexpr uint32_t LM_IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(LM_BN >> 3) << 17) |
                              ((uint32_t)(LM_BM >> 4) << 24);

// EPI 0: per-row (max, sum exp) partials of each 256-column slice (LM head, K6).
// EPI 1: SwiGLU -- B rows are interleaved so tile n holds gate columns [n*128, +128) followed by
//        the matching up columns; the epilogue writes act = silu(gate) * up (bf16, or hi|lo
//        pairs when split) for its 128 output columns: the gate/up product never reaches HBM.
constexpr int EPI_LSE = 0, EPI_SWIGLU = 1;

template <int EPI>
__global__ void __launch_bounds__(LM_THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   int M, int N, int K, int MT, int NT, void* out, int64_t ld_out, int F, int split) {
  extern __shared__ __align__(1024) unsigned char lm_smem_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(lm_smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + LM_ST * LM_STAGE_BYTES);
  uint64_t* empty = full + LM_ST;
  uint64_t* tfull = empty + LM_ST;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < LM_ST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {  // 2 x 256 fp32 accumulator columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tslot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tslot;
  const int KB = K / LM_BK;
  const int total = MT * NT;
  if (warp == 0) {
    if (lane == 0) {  // ===== TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const int m0 = (t % MT) * LM_BM, n0 = (t / MT) * LM_BN;
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], LM_STAGE_BYTES);
          unsigned char* sa = sm + stage * LM_STAGE_BYTES;
          tma_2d(sa, &tmA, kb * LM_BK, m0, &full[stage]);
          tma_2d(sa + LM_A_BYTES, &tmB, kb * LM_BK, n0, &full[stage]);
          if (++stage == LM_ST) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ===== MMA issuer
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t aphase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        mbar_wait(&tempty[acc], aphase ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t d = tmem + (uint32_t)(acc * LM_BN);
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&full[stage], phase);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const uint32_t sa = smem_u32(sm + stage * LM_STAGE_BYTES);
          const uint64_t da = umma_desc_sw128(sa), db = umma_desc_sw128(sa + LM_A_BYTES);
#pragma unroll
          for (int k = 0; k < LM_BK / 16; ++k) {  // +32 B per K=16 step inside the swizzle atom
            const uint32_t accum = (kb | k) ? 1u : 0u;
            asm volatile(
                "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                "l"(da + (uint64_t)(k * 2)), "l"(db + (uint64_t)(k * 2)), "r"(LM_IDESC), "r"(accum));
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                           smem_u32(&empty[stage]))
                       : "memory");
          if (++stage == LM_ST) {
            stage = 0;
            phase ^= 1;
          }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                         smem_u32(&tfull[acc]))
                     : "memory");
        if (++acc == 2) {
          acc = 0;
          aphase ^= 1;
        }
      }
    }
  } else {  // ===== epilogue: warps 2..5, thread = accumulator row (TMEM lane)
    const int q = warp & 3;  // the TMEM lane quarter this warp may access
    int acc = 0;
    uint32_t aphase = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      const int m0 = (t % MT) * LM_BM, n = t / MT, n0 = n * LM_BN;
      mbar_wait(&tfull[acc], aphase);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * LM_BN);
      const int row = m0 + q * 32 + lane;
      if constexpr (EPI == EPI_SWIGLU) {
        bf16* orow = reinterpret_cast<bf16*>(out) + (size_t)row * ld_out + (size_t)n * (LM_BN / 2);
#pragma unroll 1
        for (int c0 = 0; c0 < LM_BN / 2; c0 += 16) {
          uint32_t g[16], u[16];
          tmem_ld16(base + (uint32_t)c0, g);
          tmem_ld16(base + (uint32_t)(LM_BN / 2 + c0), u);
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
          uint4 hv[2], lv[2];
          __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(hv);
          __nv_bfloat162* l2 = reinterpret_cast<__nv_bfloat162*>(lv);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float g0 = __uint_as_float(g[2 * e]), g1 = __uint_as_float(g[2 * e + 1]);
            const float a = g0 / (1.f + __expf(-g0)) * __uint_as_float(u[2 * e]);
            const float b = g1 / (1.f + __expf(-g1)) * __uint_as_float(u[2 * e + 1]);
            h2[e] = __floats2bfloat162_rn(a, b);
            const float2 hf = __bfloat1622float2(h2[e]);
            l2[e] = __floats2bfloat162_rn(a - hf.x, b - hf.y);
          }
          if (row < M && n * (LM_BN / 2) + c0 < F) {
            reinterpret_cast<uint4*>(orow + c0)[0] = hv[0];
            reinterpret_cast<uint4*>(orow + c0)[1] = hv[1];
            if (split) {
              reinterpret_cast<uint4*>(orow + F + c0)[0] = lv[0];
              reinterpret_cast<uint4*>(orow + F + c0)[1] = lv[1];
            }
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        mbar_arrive(&tempty[acc]);
        if (++acc == 2) {
          acc = 0;
          aphase ^= 1;
        }
        continue;
      }
      float mrun = -INFINITY, srun = 0.f;
#pragma unroll 1
      for (int c0 = 0; c0 < LM_BN; c0 += 32) {
        uint32_t v[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
            "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
              "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
              "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
              "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(base + (uint32_t)c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        const int valid = min(32, N - (n0 + c0));
        float cm = -INFINITY;
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < valid) cm = fmaxf(cm, __uint_as_float(v[j]));
        if (cm > mrun) {
          srun = (mrun == -INFINITY) ? 0.f : srun * __expf(mrun - cm);
          mrun = cm;
        }
        float cs = 0.f;
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < valid) cs += __expf(__uint_as_float(v[j]) - mrun);
        srun += cs;
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      mbar_arrive(&tempty[acc]);
      if (row < M) reinterpret_cast<float2*>(out)[(size_t)row * NT + n] = make_float2(mrun, srun);
      if (++acc == 2) {
        acc = 0;
        aphase ^= 1;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

// combine the per-tile (max, sum) partials of one row into its log-sum-exp
__global__ void __launch_bounds__(128) lse_reduce_kernel(const float2* partial, int NT,
                                                         const int32_t* slots, float* s_lse) {
  const int row = blockIdx.x;
  const float2* p = partial + (size_t)row * NT;
  float m = -INFINITY, s = 0.f;
  for (int i = threadIdx.x; i < NT; i += blockDim.x) {
    const float2 v = p[i];
    if (v.x == -INFINITY) continue;
    const float nm = fmaxf(m, v.x);
    s = (m == -INFINITY ? 0.f : s * __expf(m - nm)) + v.y * __expf(v.x - nm);
    m = nm;
  }
  __shared__ float sm_m[4], sm_s[4];
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(FULLMASK, m, o), s2 = __shfl_xor_sync(FULLMASK, s, o);
    const float nm = fmaxf(m, m2);
    s = (nm == -INFINITY) ? 0.f : (m == -INFINITY ? 0.f : s * __expf(m - nm)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - nm));
    m = nm;
  }
  if ((threadIdx.x & 31) == 0) {
    sm_m[threadIdx.x >> 5] = m;
    sm_s[threadIdx.x >> 5] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float M2 = -INFINITY, S2 = 0.f;
    for (int w = 0; w < 4; ++w) {
      if (sm_m[w] == -INFINITY) continue;
      const float nm = fmaxf(M2, sm_m[w]);
      S2 = (M2 == -INFINITY ? 0.f : S2 * __expf(M2 - nm)) + sm_s[w] * __expf(sm_m[w] - nm);
      M2 = nm;
    }
    s_lse[slots[row]] = M2 + logf(S2);
  }
}

template <typename T>
cudaError_t dalloc(T** p, size_t n) {
  if (n == 0) n = 1;
  return cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T));
}

}  // namespace

struct lb_llm {
  lb_batch* b = nullptr;
  LlmDev dev{};
  int32_t* d_tok_low = nullptr;
  int32_t* d_tok_cap = nullptr;
  int32_t* d_tok_low_off = nullptr;
  int32_t* d_tok_cap_off = nullptr;
  int64_t node_slot_elems = 0;
  int64_t bytes = 0;
  // stats
  int64_t events = 0, waves = 0, rows = 0, cum = 0, max_wave_rows = 0;
  int64_t grouped_launches = 0;  // attention launches that used sibling tiles
  int32_t cur_nwaves = 0;
  std::vector<int64_t> wave_off, wave_rows;
  // sibling tiles of the last eager forward chunk (lb_llm_wave_rows -> lb_llm_attention)
  GrpDev grp{};
  int64_t grp_cap = 0;  // rows the tile buffers hold
  int32_t grp_rows = -1;
  int32_t grp_tiles = 0;
  int32_t plan_tiles = -1;  // tiles of the current wave built during planning (-1: none)
  const int32_t* grp_pos = nullptr;
};

#define CKL(expr)                                                                        \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess)                                                               \
      return lbh::set_error(LB_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

static int launched(cudaError_t e) {
  ++lbk::g_launches;
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return lbh::set_error(LB_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  return LB_OK;
}
#define LAUNCH(...)                 \
  do {                              \
    __VA_ARGS__;                    \
    int _rc = launched(cudaSuccess); \
    if (_rc) return _rc;            \
  } while (0)

// Launch with programmatic stream serialization (LB_PDL=0 disables): the kernel's launch
// overlaps the tail of its predecessor on the stream; the kernel itself starts with pdl_wait().
static bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("LB_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}
#define LAUNCH_PDL(...)                       \
  do {                                        \
    int _rc = launched(launch_pdl(__VA_ARGS__)); \
    if (_rc) return _rc;                      \
  } while (0)

// LB_ATT_GROUP=0: per-row chain attention only (A/B switch)
// LB_ATT_GAP = 1 (siblings: rows sharing a parent) or 2 (cousins: rows sharing a grandparent,
// two private positions each)
static int att_group_shift() {
  static const int v = [] {
    const char* e = std::getenv("LB_ATT_GAP");
    return (e && e[0] == '2') ? 1 : 0;
  }();
  return v;
}
static bool att_group_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("LB_ATT_GROUP");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Sibling tiles (see chain_attn_grp_kernel) of rows r < n of slots[]: n >= 0 from the host, or
// n < 0 = the device's forward-set count (during planning).  Buffers hold cap_rows rows.
static int grp_build(lb_llm* l, const int32_t* slots, int n, int64_t cap_rows) {
  LlmDev& x = l->dev;
  cudaStream_t st = l->b->st;
  const int SIB = 16 / (x.NH / x.NKV);
  GrpDev& g = l->grp;
  if (!g.cnt) {
    CKL(dalloc(&g.cnt, (size_t)x.cap));
    CKL(dalloc(&g.base, (size_t)x.cap));
    CKL(dalloc(&g.ntiles, 1));
    CKL(cudaMemsetAsync(g.cnt, 0, (size_t)x.cap * 4, st));
  }
  if (l->grp_cap < cap_rows) {
    cudaFree(g.row_k);
    cudaFree(g.tiles);
    cudaFree(g.tile_n);
    g.row_k = g.tiles = g.tile_n = nullptr;
    const int64_t want = std::max<int64_t>(cap_rows, 2 * l->grp_cap);
    CKL(dalloc(&g.row_k, (size_t)want));
    CKL(dalloc(&g.tiles, (size_t)want * SIB));
    CKL(dalloc(&g.tile_n, (size_t)want));
    l->grp_cap = want;
  }
  const int grid = n >= 0 ? std::max(1, std::min(4 * 148, (n + 127) / 128)) : 4 * 148;
  CKL(cudaMemsetAsync(g.ntiles, 0, 4, st));
  const int gsh = att_group_shift();
  LAUNCH(grp_count_kernel<<<grid, 128, 0, st>>>(x, g, slots, n, gsh));
  LAUNCH(grp_base_kernel<<<grid, 128, 0, st>>>(x, g, slots, n, SIB, gsh));
  LAUNCH(grp_fill_kernel<<<grid, 128, 0, st>>>(x, g, slots, n, SIB, gsh));
  LAUNCH(grp_reset_kernel<<<grid, 128, 0, st>>>(x, g, slots, n, gsh));
  return LB_OK;
}

static int check_err_flags(lb_llm* l) {
  int32_t err = 0;
  CKL(cudaMemcpyAsync(&err, l->dev.ctr + C_ERR, 4, cudaMemcpyDeviceToHost, l->b->st));
  CKL(cudaStreamSynchronize(l->b->st));
  if (err & 1) return lbh::set_error(LB_ERR_CAPACITY, "LLM prefix cache full (max_slots)");
  if (err & 2) return lbh::set_error(LB_ERR_CAPACITY, "LLM node list full for one fusion event");
  if (err & 4) return lbh::set_error(LB_ERR_CAPACITY, "text longer than the LLM max_depth");
  return LB_OK;
}

extern "C" {

int lb_llm_create(lb_batch* b, const lb_llm_desc* d, lb_llm** out) {
  if (!b || !d || !out || !d->surface_tokens || !d->surface_tokens_first || !d->embedding)
    return lbh::set_error(LB_ERR_ARG, "null argument");
  if (d->head_dim != 64 && d->head_dim != 128)
    return lbh::set_error(LB_ERR_ARG, "head_dim must be 64 or 128");
  if (d->n_kv_heads < 1 || d->n_heads % d->n_kv_heads != 0)
    return lbh::set_error(LB_ERR_ARG, "n_heads must be a multiple of n_kv_heads");
  const int G = d->n_heads / d->n_kv_heads;
  if (G != 1 && G != 2 && G != 4 && G != 8) return lbh::set_error(LB_ERR_ARG, "GQA group must be 1, 2, 4 or 8");
  if (d->hidden % 8 != 0) return lbh::set_error(LB_ERR_ARG, "hidden must be a multiple of 8");
  if (d->max_slots < 2 || d->max_slots > ((int64_t)1 << 30)) return lbh::set_error(LB_ERR_ARG, "max_slots out of range");
  if (d->max_depth < 1 || d->max_depth > 4095) return lbh::set_error(LB_ERR_ARG, "max_depth out of range");
  if (d->n_surfaces != (int32_t)b->m->surfaces.size())
    return lbh::set_error(LB_ERR_ARG, "surface token table does not match the model's surfaces");
  for (int v = 0; v < 2; ++v) {  // surface token CSR (NULL offsets: one token per surface)
    const int32_t* off = v ? d->surface_token_off_first : d->surface_token_off;
    const int32_t* tk = v ? d->surface_tokens_first : d->surface_tokens;
    if (off && off[0] != 0) return lbh::set_error(LB_ERR_ARG, "surface token offsets must start at 0");
    for (int i = 0; i < d->n_surfaces; ++i) {
      const int32_t a = off ? off[i] : i, e = off ? off[i + 1] : i + 1;
      if (e <= a) return lbh::set_error(LB_ERR_ARG, "every surface needs at least one token");
      for (int k = a; k < e; ++k)
        if (tk[k] < 0 || tk[k] >= d->vocab) return lbh::set_error(LB_ERR_ARG, "surface token out of range");
    }
  }
  CKL(cudaSetDevice(b->m->device));
  lb_llm* l = new lb_llm();
  l->b = b;
  LlmDev& x = l->dev;
  x.L = d->n_layers;
  x.NH = d->n_heads;
  x.NKV = d->n_kv_heads;
  x.HD = d->head_dim;
  x.H = d->hidden;
  x.vocab = d->vocab;
  x.cap = d->max_slots;
  x.max_depth = d->max_depth;
  x.bos_tok = d->bos_token;
  for (int j = 0; j < 3; ++j) x.punct_tok[j] = d->punct_tokens[j];
  x.emb = reinterpret_cast<const bf16*>(d->embedding);
  x.head32 = d->head_f32;
  if (d->precision != 0 && d->precision != 1) return lbh::set_error(LB_ERR_ARG, "precision must be 0 (bf16) or 1 (bf16x2)");
  x.split = d->precision;
  x.n_surf = d->n_surfaces;
  const size_t cap = (size_t)x.cap;
  const size_t kvw = (size_t)x.NKV * x.HD;
  uint32_t hsz = 1;
  while (hsz < 2 * cap) hsz <<= 1;
  x.hmask = hsz - 1;
  const size_t B = (size_t)b->Bmax;
  const int64_t ncap = b->dev.ncap;
  x.nlist_cap = (int32_t)std::min<int64_t>(ncap, (int64_t)b->K * b->O * (b->Tmax / 2 + 2));
  l->node_slot_elems = (int64_t)B * ncap;
  CKL(dalloc(&x.s_parent, cap));
  CKL(dalloc(&x.s_token, cap));
  CKL(dalloc(&x.s_depth, cap));
  CKL(dalloc(&x.s_fwd, cap));
  CKL(dalloc(&x.s_cum, cap));
  CKL(dalloc(&x.s_pun, cap));
  CKL(dalloc(&x.s_lp, cap));
  CKL(dalloc(&x.s_cumv, cap));
  CKL(dalloc(&x.s_plp, cap * 3));
  CKL(dalloc(&x.s_lse, cap));
  CKL(dalloc(&x.s_h, cap * x.H));
  const size_t esz = x.split ? 4 : 2;
  CKL(cudaMalloc(&x.kc, (size_t)x.L * cap * kvw * esz));
  CKL(cudaMalloc(&x.vc, (size_t)x.L * cap * kvw * esz));
  CKL(dalloc(&x.htab, hsz));
  CKL(dalloc(&x.ctr, C_NCTR));
  CKL(dalloc(&x.node_slot, (size_t)l->node_slot_elems));
  CKL(dalloc(&x.nlist, B * x.nlist_cap));
  CKL(dalloc(&x.nlist_depth, B * x.nlist_cap));
  CKL(dalloc(&x.fwd_list, cap));
  CKL(dalloc(&x.cum_list, cap));
  CKL(dalloc(&x.wave_slots, cap));
  CKL(dalloc(&x.blk, (cap + CB - 1) / CB));
  {  // surface token tables as CSR (one token per surface when no offsets are given)
    std::vector<int32_t> ident(x.n_surf + 1);
    for (int i = 0; i <= x.n_surf; ++i) ident[i] = i;
    const int32_t* offs[2] = {d->surface_token_off ? d->surface_token_off : ident.data(),
                              d->surface_token_off_first ? d->surface_token_off_first : ident.data()};
    const int32_t* toks[2] = {d->surface_tokens, d->surface_tokens_first};
    int32_t** dtok[2] = {&l->d_tok_low, &l->d_tok_cap};
    int32_t** doff[2] = {&l->d_tok_low_off, &l->d_tok_cap_off};
    for (int v = 0; v < 2; ++v) {
      const int32_t nt = offs[v][x.n_surf];
      CKL(dalloc(dtok[v], (size_t)std::max(nt, 1)));
      CKL(dalloc(doff[v], (size_t)x.n_surf + 1));
      CKL(cudaMemcpy(*dtok[v], toks[v], (size_t)nt * 4, cudaMemcpyHostToDevice));
      CKL(cudaMemcpy(*doff[v], offs[v], ((size_t)x.n_surf + 1) * 4, cudaMemcpyHostToDevice));
    }
  }
  x.tok_low = l->d_tok_low;
  x.tok_cap = l->d_tok_cap;
  x.tok_low_off = l->d_tok_low_off;
  x.tok_cap_off = l->d_tok_cap_off;
  l->bytes = (int64_t)cap * (4 * 6 + 8 * 5 + 4 + 4 * x.H + 4 * 4) + (int64_t)2 * x.L * cap * kvw * esz +
             (int64_t)hsz * 4 + l->node_slot_elems * 4 + (int64_t)B * x.nlist_cap * 8;
  *out = l;
  return lb_llm_reset(l);
}

int lb_llm_destroy(lb_llm* l) {
  if (!l) return LB_OK;
  cudaStreamSynchronize(l->b->st);
  LlmDev& x = l->dev;
  void* ptrs[] = {x.s_parent, x.s_token, x.s_depth, x.s_fwd, x.s_cum, x.s_pun, x.s_lp, x.s_cumv,
                  x.s_plp, x.s_lse, x.s_h, x.kc, x.vc, x.htab, x.ctr, x.node_slot, x.nlist,
                  x.nlist_depth, x.fwd_list, x.cum_list, x.wave_slots, x.blk,
                  l->d_tok_low, l->d_tok_cap, l->d_tok_low_off, l->d_tok_cap_off,
                  l->grp.cnt, l->grp.base, l->grp.row_k, l->grp.tiles, l->grp.tile_n,
                  l->grp.ntiles};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  delete l;
  return LB_OK;
}

int lb_llm_footprint(lb_llm* l, int64_t* bytes) {
  if (!l || !bytes) return lbh::set_error(LB_ERR_ARG, "null argument");
  *bytes = l->bytes;
  return LB_OK;
}

int lb_llm_reset(lb_llm* l) {
  const int rc = lb_llm_reset_device(l);
  return rc ? rc : lb_llm_reset_stats(l);
}

int lb_llm_reset_device(lb_llm* l) {
  if (!l) return lbh::set_error(LB_ERR_ARG, "null argument");
  LlmDev& x = l->dev;
  cudaStream_t st = l->b->st;
  CKL(cudaMemsetAsync(x.htab, 0xFF, ((size_t)x.hmask + 1) * 4, st));
  CKL(cudaMemsetAsync(x.node_slot, 0xFF, (size_t)l->node_slot_elems * 4, st));
  LAUNCH(llm_reset_kernel<<<1, 32, 0, st>>>(x));
  const int B = l->b->Bmax;
  LAUNCH(root_slots_kernel<<<(B + 127) / 128, 128, 0, st>>>(x.node_slot, B, l->b->dev.ncap));
  return LB_OK;
}

int lb_llm_reset_stats(lb_llm* l) {
  if (!l) return lbh::set_error(LB_ERR_ARG, "null argument");
  l->events = l->waves = l->rows = l->cum = l->max_wave_rows = 0;
  l->grouped_launches = 0;
  return LB_OK;
}

int lb_llm_plan(lb_llm* l, int32_t final_, int32_t min_frames, int32_t* n_waves,
                int64_t* wave_rows) {
  if (!l || !n_waves || !wave_rows) return lbh::set_error(LB_ERR_ARG, "null argument");
  lb_batch* b = l->b;
  if (b->n_trials < 1) return lbh::set_error(LB_ERR_STATE, "no trials loaded");
  LlmDev& x = l->dev;
  cudaStream_t st = b->st;
  CKL(cudaMemsetAsync(x.ctr + C_NFWD, 0, 8, st));  // C_NFWD, C_NCUM
  const int B = b->n_trials;
  const int nblk = (int)((x.cap + CB - 1) / CB);
  LAUNCH(map_nodes_kernel<<<B, 256, 0, st>>>(b->dev, x, min_frames));
  LAUNCH(schedule_kernel<<<B, 128, 0, st>>>(b->dev, x, min_frames, final_));
  LAUNCH(flag_count_kernel<<<nblk, CB, 0, st>>>(x, x.blk));
  LAUNCH(blk_scan_kernel<<<1, CB, 0, st>>>(x.blk, nblk));
  LAUNCH(compact_kernel<<<nblk, CB, 0, st>>>(x, x.blk));
  // sibling tiles of the whole wave, built before the one synchronisation of the plan
  int32_t ntiles = -1;
  if (att_group_enabled()) {
    int rc = grp_build(l, x.wave_slots, -1, x.cap);
    if (rc) return rc;
    CKL(cudaMemcpyAsync(&ntiles, l->grp.ntiles, 4, cudaMemcpyDeviceToHost, st));
  }
  int32_t nfc[2] = {0, 0};  // C_NFWD, C_NCUM
  CKL(cudaMemcpyAsync(nfc, x.ctr + C_NFWD, 8, cudaMemcpyDeviceToHost, st));
  int rc = check_err_flags(l);  // synchronises
  if (rc) return rc;
  l->plan_tiles = ntiles;
  l->wave_off.clear();
  l->wave_rows.clear();
  // One wave per event (see compact_kernel): inside a layer the K/V of all rows are written
  // before the attention kernel reads them (tree-causal prefill), and any row-prefix chunk of
  // the wave holds the parents of its rows.
  const int64_t total = std::min<int64_t>(nfc[0], x.cap);
  l->cum += nfc[1];
  int nw = 0;
  if (total > 0) {
    l->wave_off.push_back(0);
    l->wave_rows.push_back(total);
    wave_rows[0] = total;
    nw = 1;
  }
  l->max_wave_rows = std::max<int64_t>(l->max_wave_rows, total);
  *n_waves = nw;
  l->cur_nwaves = nw;
  l->events += 1;
  l->waves += nw;
  l->rows += total;
  return LB_OK;
}

int lb_llm_plan_async(lb_llm* l, int32_t final_, int32_t min_frames, int32_t rows_cap) {
  if (!l) return lbh::set_error(LB_ERR_ARG, "null argument");
  lb_batch* b = l->b;
  if (b->n_trials < 1) return lbh::set_error(LB_ERR_STATE, "no trials loaded");
  if (rows_cap < 1) return lbh::set_error(LB_ERR_ARG, "rows_cap must be >= 1");
  LlmDev& x = l->dev;
  cudaStream_t st = b->st;
  CKL(cudaMemsetAsync(x.ctr + C_NFWD, 0, 8, st));  // C_NFWD, C_NCUM
  const int B = b->n_trials;
  const int nblk = (int)((x.cap + CB - 1) / CB);
  LAUNCH(map_nodes_kernel<<<B, 256, 0, st>>>(b->dev, x, min_frames));
  LAUNCH(schedule_kernel<<<B, 128, 0, st>>>(b->dev, x, min_frames, final_));
  LAUNCH(flag_count_kernel<<<nblk, CB, 0, st>>>(x, x.blk));
  LAUNCH(blk_scan_kernel<<<1, CB, 0, st>>>(x.blk, nblk));
  LAUNCH(compact_kernel<<<nblk, CB, 0, st>>>(x, x.blk));
  LAUNCH(plan_async_kernel<<<1, 32, 0, st>>>(x, rows_cap));
  l->plan_tiles = -1;
  return LB_OK;
}

int lb_llm_wave_rows_async(lb_llm* l, int32_t rows_cap, int32_t* tokens, int32_t* positions,
                           int32_t* slots, int32_t* chains) {
  if (!l || !tokens || !positions || !slots || !chains) return lbh::set_error(LB_ERR_ARG, "null argument");
  if (rows_cap < 1) return lbh::set_error(LB_ERR_ARG, "rows_cap must be >= 1");
  const int grid = std::min(4 * 148, (rows_cap + 127) / 128);
  l->grp_rows = -1;  // graph mode: per-row attention (the tile count is not known on the host)
  LAUNCH(wave_rows_async_kernel<<<grid, 128, 0, l->b->st>>>(l->dev, rows_cap, tokens, positions,
                                                            slots, chains));
  return LB_OK;
}

int lb_llm_check(lb_llm* l) {
  if (!l) return lbh::set_error(LB_ERR_ARG, "null argument");
  int32_t err = 0;
  CKL(cudaMemcpyAsync(&err, l->dev.ctr + C_ERR, 4, cudaMemcpyDeviceToHost, l->b->st));
  CKL(cudaStreamSynchronize(l->b->st));
  if (err & 8) return lbh::set_error(LB_ERR_CAPACITY, "fusion event larger than the captured graph rows");
  return check_err_flags(l);
}

int lb_llm_wave_rows(lb_llm* l, int32_t wave, int64_t row0, int32_t n, int32_t* tokens,
                     int32_t* positions, int32_t* slots, int32_t* chains) {
  if (!l || !tokens || !positions || !slots || !chains) return lbh::set_error(LB_ERR_ARG, "null argument");
  if (wave < 0 || wave >= l->cur_nwaves) return lbh::set_error(LB_ERR_ARG, "wave out of range");
  if (row0 < 0 || n < 0 || row0 + n > l->wave_rows[wave]) return lbh::set_error(LB_ERR_ARG, "rows out of range");
  if (n == 0) return LB_OK;
  const int grid = std::min(4 * 148, (n + 127) / 128);
  cudaStream_t st = l->b->st;
  LAUNCH(wave_rows_kernel<<<grid, 128, 0, st>>>(l->dev, l->wave_off[wave] + row0, n, tokens,
                                                positions, slots, chains));
  l->grp_rows = -1;
  if (!att_group_enabled()) return LB_OK;
  if (row0 == 0 && n == l->wave_rows[wave] && l->plan_tiles >= 0) {
    // the whole wave in one chunk: the tiles built during planning apply (row r = wave row r)
    if ((int64_t)l->plan_tiles * 4 <= (int64_t)n * 3) {
      l->grp_tiles = l->plan_tiles;
      l->grp_rows = n;
      l->grp_pos = positions;
    }
    return LB_OK;
  }
  // a partial chunk: tiles of its own rows (one small copy + sync)
  int rc = grp_build(l, slots, n, n);
  if (rc) return rc;
  int32_t nt = 0;
  CKL(cudaMemcpyAsync(&nt, l->grp.ntiles, 4, cudaMemcpyDeviceToHost, st));
  CKL(cudaStreamSynchronize(st));
  l->grp_tiles = nt;
  if ((int64_t)nt * 4 <= (int64_t)n * 3) {
    l->grp_rows = n;
    l->grp_pos = positions;
  }
  return LB_OK;
}

int lb_llm_finish(lb_llm* l, int32_t final_, int32_t min_frames) {
  if (!l) return lbh::set_error(LB_ERR_ARG, "null argument");
  lb_batch* b = l->b;
  LlmDev& x = l->dev;
  cudaStream_t st = b->st;
  LAUNCH(lp_kernel<<<4 * 148, 256, 0, st>>>(x));
  LAUNCH(cum_kernel<<<4 * 148, 256, 0, st>>>(x));
  LAUNCH(commit_kernel<<<4 * 148, 256, 0, st>>>(x));
  const int B = b->n_trials;
  if (final_) LAUNCH(punct_kernel<<<B, 256, 0, st>>>(b->dev, x, min_frames));
  LAUNCH(llm_apply_kernel<<<B, 128, 0, st>>>(b->cdev, b->dev, x, final_, min_frames));
  return LB_OK;
}

int lb_llm_rmsnorm(lb_llm* l, float* x, const void* delta, const float* w, float eps, int32_t M,
                   void* out, const int32_t* store_slots) {
  if (!l || !x || !w || !out) return lbh::set_error(LB_ERR_ARG, "null argument");
  if (l->dev.H > 256 * 4 * NORM_NPT) return lbh::set_error(LB_ERR_ARG, "hidden size > 4096");
  if (M <= 0) return LB_OK;
  LAUNCH_PDL(add_rmsnorm_kernel, dim3(M), dim3(256), 0, l->b->st, x,
             reinterpret_cast<const float*>(delta), w, eps, l->dev.H, reinterpret_cast<bf16*>(out),
             store_slots, l->dev.s_h, l->dev.split, static_cast<const float*>(nullptr));
  return LB_OK;
}

int lb_llm_layernorm(lb_llm* l, float* x, const void* delta, const float* w, const float* b,
                     float eps, int32_t M, void* out, const int32_t* store_slots) {
  if (!l || !x || !w || !b || !out) return lbh::set_error(LB_ERR_ARG, "null argument");
  if (l->dev.H > 256 * 4 * NORM_NPT) return lbh::set_error(LB_ERR_ARG, "hidden size > 4096");
  if (M <= 0) return LB_OK;
  LAUNCH_PDL(add_rmsnorm_kernel, dim3(M), dim3(256), 0, l->b->st, x,
             reinterpret_cast<const float*>(delta), w, eps, l->dev.H, reinterpret_cast<bf16*>(out),
             store_slots, l->dev.s_h, l->dev.split, b);
  return LB_OK;
}

int lb_llm_gelu(lb_llm* l, const float* in, const float* bias, int32_t M, int32_t ffn, void* out) {
  if (!l || !in || !out) return lbh::set_error(LB_ERR_ARG, "null argument");
  if (ffn % 8 != 0) return lbh::set_error(LB_ERR_ARG, "ffn must be a multiple of 8");
  if (M <= 0) return LB_OK;
  const dim3 grid((ffn / 8 + 127) / 128, M);
  LAUNCH(gelu_kernel<<<grid, 128, 0, l->b->st>>>(in, bias, ffn, reinterpret_cast<bf16*>(out),
                                                 l->dev.split));
  return LB_OK;
}

int lb_llm_rope_kv(lb_llm* l, int32_t layer, const void* qkv, int32_t M, const int32_t* pos,
                   const int32_t* slots, const float* cos_tab, const float* sin_tab, void* q_out) {
  if (!l || !qkv || !pos || !slots || !cos_tab || !sin_tab || !q_out) return lbh::set_error(LB_ERR_ARG, "null argument");
  if (layer < 0 || layer >= l->dev.L) return lbh::set_error(LB_ERR_ARG, "layer out of range");
  if (M <= 0) return LB_OK;
  const float* in = reinterpret_cast<const float*>(qkv);
  cudaStream_t st = l->b->st;
#define ROPE(TT, HDV)                                                                          \
  do {                                                                                         \
    void (*kfn)(LlmDev, int, const float*, int, const int32_t*, const int32_t*, const float*,  \
                const float*, TT*) = rope_kv_kernel<TT, HDV>;                                  \
    LAUNCH_PDL(kfn, dim3(M), dim3(128), 0, st, l->dev, layer, in, M, pos, slots, cos_tab, sin_tab, \
               reinterpret_cast<TT*>(q_out));                                                  \
  } while (0)
  if (l->dev.split) {
    if (l->dev.HD == 64) ROPE(float, 64); else ROPE(float, 128);
  } else {
    if (l->dev.HD == 64) ROPE(bf16, 64); else ROPE(bf16, 128);
  }
#undef ROPE
  return LB_OK;
}

int lb_llm_attention(lb_llm* l, int32_t layer, const void* q, int32_t M, const int32_t* chains,
                     const int32_t* pos, void* out) {
  if (!l || !q || !chains || !pos || !out) return lbh::set_error(LB_ERR_ARG, "null argument");
  if (layer < 0 || layer >= l->dev.L) return lbh::set_error(LB_ERR_ARG, "layer out of range");
  if (M <= 0) return LB_OK;
  const LlmDev& x = l->dev;
  const int G = x.NH / x.NKV;
  if (x.NKV > 8) return lbh::set_error(LB_ERR_ARG, "n_kv_heads must be <= 8");
  const float scale = 1.0f / sqrtf((float)x.HD);
  bf16* oo = reinterpret_cast<bf16*>(out);
  cudaStream_t st = l->b->st;
#define ATT_T(HDV, GV, DV, TV)                                                                  \
  do {                                                                                          \
    auto kfn = chain_attn_kernel<HDV, GV, DV, TV>;                                              \
    const int rowb = x.NKV * HDV * (int)sizeof(TV);                                             \
    const int smem = 128 + 2 * 2 * attn_chunk(rowb) * rowb;                                     \
    CKL(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));          \
    LAUNCH(kfn<<<M, 32 * x.NKV, smem, st>>>(x, layer, reinterpret_cast<const TV*>(q), chains,   \
                                            pos, scale, oo));                                   \
  } while (0)
#define ATT(HDV, GV, DV) ATT_T(HDV, GV, DV, bf16)
  if (G <= 16) {  // tensor-core path (bf16 operands; hi/lo bf16 pairs in split precision)
    const int rowb = x.NKV * x.HD * 2 * (x.split ? 2 : 1);
    const int stage = 2 * MMA_CH * (rowb + 16);
    const int nst = (128 + 2 * stage <= 80 * 1024) ? 2 : 1;  // keep >= 2-3 CTAs per SM
    const int smem = 128 + nst * stage;
    if (smem > 227 * 1024) return lbh::set_error(LB_ERR_ARG, "K/V cache row too wide for the attention stage");
#define MMA_ATT_N(HDV, SV, NS)                                                                      \
  do {                                                                                              \
    CKL(cudaFuncSetAttribute(chain_attn_mma_kernel<HDV, SV, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); \
    LAUNCH_PDL((chain_attn_mma_kernel<HDV, SV, NS>), dim3(M), dim3(32 * x.NKV), smem, st, x, layer, q, chains, pos, scale, oo); \
  } while (0)
#define MMA_ATT(HDV, SV)               \
  do {                                 \
    if (nst == 2) MMA_ATT_N(HDV, SV, 2); \
    else MMA_ATT_N(HDV, SV, 1);        \
  } while (0)
    const bool grouped = l->grp_rows == M && l->grp_pos == pos;
    if (grouped) {  // sibling tiles built by lb_llm_wave_rows for this chunk
      const int SIB = 16 / G;
      // kv heads per CTA: the largest group whose double-buffered stage fits ~70 KB, so three
      // CTAs share an SM and the next chunk's gather overlaps this one's MMAs
      int KH = x.NKV;
      auto gstage = [&](int kh) { return 2 * MMA_CH * (kh * x.HD * 2 * (x.split ? 2 : 1) + 16); };
      while (KH > 4 || (KH > 1 && 128 + 2 * gstage(KH) > 70 * 1024)) KH /= 2;  // <= 128 threads
      if (const char* e = std::getenv("LB_ATT_KH")) KH = std::max(1, std::min(KH, atoi(e)));
      const int gnst = 128 + 2 * gstage(KH) <= 100 * 1024 ? 2 : 1;
      const int gsmem = 128 + gnst * gstage(KH);
#define GRP_ATT_N(HDV, SV, NS)                                                                      \
  do {                                                                                              \
    CKL(cudaFuncSetAttribute(chain_attn_grp_kernel<HDV, SV, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, gsmem)); \
    LAUNCH_PDL((chain_attn_grp_kernel<HDV, SV, NS>), dim3(l->grp_tiles, x.NKV / KH), dim3(32 * KH), gsmem, st, x, layer, q, chains, pos, l->grp, SIB, att_group_shift(), scale, oo); \
  } while (0)
#define GRP_ATT(HDV, SV)               \
  do {                                 \
    if (gnst == 2) GRP_ATT_N(HDV, SV, 2); \
    else GRP_ATT_N(HDV, SV, 1);        \
  } while (0)
      if (x.HD == 64) {
        if (x.split) GRP_ATT(64, true); else GRP_ATT(64, false);
      } else {
        if (x.split) GRP_ATT(128, true); else GRP_ATT(128, false);
      }
      ++l->grouped_launches;
#undef GRP_ATT
#undef GRP_ATT_N
      return LB_OK;
    }
    if (x.HD == 64) {
      if (x.split) MMA_ATT(64, true); else MMA_ATT(64, false);
    } else {
      if (x.split) MMA_ATT(128, true); else MMA_ATT(128, false);
    }
#undef MMA_ATT
#undef MMA_ATT_N
    return LB_OK;
  }
  if (x.split) return lbh::set_error(LB_ERR_ARG, "bf16x2 precision needs n_heads / n_kv_heads <= 16");
  if (x.HD == 64) {
    if (G == 1) ATT(64, 1, 16); else if (G == 2) ATT(64, 2, 16); else if (G == 4) ATT(64, 4, 8); else ATT(64, 8, 8);
  } else {
    if (G == 1) ATT(128, 1, 16); else if (G == 2) ATT(128, 2, 16); else if (G == 4) ATT(128, 4, 8); else ATT(128, 8, 8);
  }
#undef ATT
#undef ATT_T
  return LB_OK;
}

int lb_llm_swiglu(lb_llm* l, const void* gu, int32_t M, int32_t ffn, void* out) {
  if (!l || !gu || !out) return lbh::set_error(LB_ERR_ARG, "null argument");
  if (ffn % 2 != 0) return lbh::set_error(LB_ERR_ARG, "ffn must be even");
  if (M <= 0) return LB_OK;
  if (ffn % 8 != 0) return lbh::set_error(LB_ERR_ARG, "ffn must be a multiple of 8");
  const dim3 grid((ffn / 8 + 127) / 128, M);
  if (l->dev.split) {
    void (*kfn)(const float*, int, bf16*, int) = swiglu_kernel<float>;
    LAUNCH_PDL(kfn, grid, dim3(128), 0, l->b->st, reinterpret_cast<const float*>(gu), ffn,
               reinterpret_cast<bf16*>(out), 1);
  } else {
    void (*kfn)(const bf16*, int, bf16*, int) = swiglu_kernel<bf16>;
    LAUNCH_PDL(kfn, grid, dim3(128), 0, l->b->st, reinterpret_cast<const bf16*>(gu), ffn,
               reinterpret_cast<bf16*>(out), 0);
  }
  return LB_OK;
}

int lb_llm_lse(lb_llm* l, const void* logits, int32_t M, int64_t ld, const int32_t* slots) {
  if (!l || !logits || !slots) return lbh::set_error(LB_ERR_ARG, "null argument");
  if (ld % 8 != 0) return lbh::set_error(LB_ERR_ARG, "logit row pitch must be a multiple of 8");
  if (M <= 0) return LB_OK;
  if (l->dev.split)  // fp32 logits of the hi|lo LM-head GEMM
    LAUNCH(lse_kernel<float><<<M, 512, 0, l->b->st>>>(reinterpret_cast<const float*>(logits), ld,
                                                      l->dev.vocab, slots, l->dev.s_lse));
  else
    LAUNCH(lse_kernel<bf16><<<M, 512, 0, l->b->st>>>(reinterpret_cast<const bf16*>(logits), ld,
                                                     l->dev.vocab, slots, l->dev.s_lse));
  return LB_OK;
}

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D bf16 K-major operand [rows][K] with row pitch `ld` elements, boxes of box_rows x 64
static int make_map(CUtensorMap* map, const void* base, int64_t rows, int64_t K, int64_t ld, int box_rows) {
  auto enc = tensor_map_encoder();
  if (!enc) return lbh::set_error(LB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)LM_BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return lbh::set_error(LB_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return LB_OK;
}

int lb_llm_lmhead_lse(lb_llm* l, const void* h, int32_t M, int64_t ldh, int32_t K, const void* emb,
                      int64_t lde, int32_t N, const int32_t* slots, void* partial) {
  if (!l || !h || !emb || !slots || !partial) return lbh::set_error(LB_ERR_ARG, "null argument");
  if (K % LM_BK != 0) return lbh::set_error(LB_ERR_ARG, "K must be a multiple of 64");
  if ((reinterpret_cast<uintptr_t>(h) | reinterpret_cast<uintptr_t>(emb)) & 15)
    return lbh::set_error(LB_ERR_ARG, "operands must be 16-byte aligned");
  if ((ldh * 2) % 16 || (lde * 2) % 16) return lbh::set_error(LB_ERR_ARG, "row pitch must be a multiple of 16 bytes");
  if (M <= 0) return LB_OK;
  CUtensorMap ma, mb;
  int rc = make_map(&ma, h, M, K, ldh, LM_BM);
  if (rc) return rc;
  rc = make_map(&mb, emb, N, K, lde, LM_BN);
  if (rc) return rc;
  const int MT = (M + LM_BM - 1) / LM_BM, NT = (N + LM_BN - 1) / LM_BN;
  static int attr = 0;
  if (!attr) {
    CKL(cudaFuncSetAttribute(tc_gemm_kernel<EPI_LSE>, cudaFuncAttributeMaxDynamicSharedMemorySize, LM_SMEM));
    attr = 1;
  }
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, l->b->m->device);
  const int grid = std::min(MT * NT, nsm);
  cudaStream_t st = l->b->st;
  LAUNCH(tc_gemm_kernel<EPI_LSE><<<grid, LM_THREADS, LM_SMEM, st>>>(ma, mb, M, N, K, MT, NT, partial,
                                                                     0, 0, 0));
  LAUNCH(lse_reduce_kernel<<<M, 128, 0, st>>>(reinterpret_cast<const float2*>(partial), NT, slots,
                                               l->dev.s_lse));
  return LB_OK;
}

int lb_llm_gateup_swiglu(lb_llm* l, const void* h, int32_t M, int64_t ldh, int32_t K,
                         const void* wgu_interleaved, int64_t ldw, int32_t ffn, void* act) {
  if (!l || !h || !wgu_interleaved || !act) return lbh::set_error(LB_ERR_ARG, "null argument");
  if (K % LM_BK != 0) return lbh::set_error(LB_ERR_ARG, "K must be a multiple of 64");
  if (ffn % (LM_BN / 2) != 0) return lbh::set_error(LB_ERR_ARG, "ffn must be a multiple of 128");
  if ((reinterpret_cast<uintptr_t>(h) | reinterpret_cast<uintptr_t>(wgu_interleaved) |
       reinterpret_cast<uintptr_t>(act)) & 15)
    return lbh::set_error(LB_ERR_ARG, "operands must be 16-byte aligned");
  if (M <= 0) return LB_OK;
  CUtensorMap ma, mb;
  int rc = make_map(&ma, h, M, K, ldh, LM_BM);
  if (rc) return rc;
  rc = make_map(&mb, wgu_interleaved, 2 * (int64_t)ffn, K, ldw, LM_BN);
  if (rc) return rc;
  const int MT = (M + LM_BM - 1) / LM_BM, NT = 2 * ffn / LM_BN;
  static int attr = 0;
  if (!attr) {
    CKL(cudaFuncSetAttribute(tc_gemm_kernel<EPI_SWIGLU>, cudaFuncAttributeMaxDynamicSharedMemorySize, LM_SMEM));
    attr = 1;
  }
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, l->b->m->device);
  const int grid = std::min(MT * NT, nsm);
  const int split = l->dev.split;
  LAUNCH(tc_gemm_kernel<EPI_SWIGLU><<<grid, LM_THREADS, LM_SMEM, l->b->st>>>(
      ma, mb, M, 2 * ffn, K, MT, NT, act, (int64_t)ffn * (split ? 2 : 1), ffn, split));
  return LB_OK;
}

int lb_llm_stats(lb_llm* l, int64_t* out) {
  if (!l || !out) return lbh::set_error(LB_ERR_ARG, "null argument");
  int32_t slots = 0;
  CKL(cudaMemcpyAsync(&slots, l->dev.ctr + C_SLOTS, 4, cudaMemcpyDeviceToHost, l->b->st));
  CKL(cudaStreamSynchronize(l->b->st));
  int32_t dev[3] = {0, 0, 0};  // graph-mode events / rows / largest event
  CKL(cudaMemcpyAsync(dev, l->dev.ctr + C_EVENTS, 12, cudaMemcpyDeviceToHost, l->b->st));
  CKL(cudaStreamSynchronize(l->b->st));
  out[0] = slots;
  out[1] = l->events + dev[0];
  out[2] = l->waves + dev[0];
  out[3] = l->rows + dev[1];
  out[4] = std::max<int64_t>(l->max_wave_rows, dev[2]);
  out[5] = l->bytes;
  out[6] = l->cum;
  out[7] = l->grouped_launches;
  return LB_OK;
}

int lb_llm_export(lb_llm* l, int64_t max_n, int64_t* n, int32_t* parent, int32_t* token,
                  int32_t* depth, int32_t* state, double* cum, double* punct_lp) {
  if (!l || !n) return lbh::set_error(LB_ERR_ARG, "null argument");
  LlmDev& x = l->dev;
  cudaStream_t st = l->b->st;
  int32_t slots = 0;
  CKL(cudaMemcpyAsync(&slots, x.ctr + C_SLOTS, 4, cudaMemcpyDeviceToHost, st));
  CKL(cudaStreamSynchronize(st));
  const int64_t avail = std::min<int64_t>(slots, x.cap);
  *n = avail;  // rows available; min(avail, max_n) are copied
  const int64_t k = std::min<int64_t>(avail, max_n);
  if (k <= 0) return LB_OK;
  if (parent) CKL(cudaMemcpyAsync(parent, x.s_parent, k * 4, cudaMemcpyDeviceToHost, st));
  if (token) CKL(cudaMemcpyAsync(token, x.s_token, k * 4, cudaMemcpyDeviceToHost, st));
  if (depth) CKL(cudaMemcpyAsync(depth, x.s_depth, k * 4, cudaMemcpyDeviceToHost, st));
  if (state) {
    std::vector<int32_t> a(k), c(k), p(k);
    CKL(cudaMemcpyAsync(a.data(), x.s_fwd, k * 4, cudaMemcpyDeviceToHost, st));
    CKL(cudaMemcpyAsync(c.data(), x.s_cum, k * 4, cudaMemcpyDeviceToHost, st));
    CKL(cudaMemcpyAsync(p.data(), x.s_pun, k * 4, cudaMemcpyDeviceToHost, st));
    CKL(cudaStreamSynchronize(st));
    for (int64_t i = 0; i < k; ++i) state[i] = (a[i] == 2 ? 1 : 0) | (c[i] == 2 ? 2 : 0) | (p[i] ? 4 : 0);
  }
  if (cum) CKL(cudaMemcpyAsync(cum, x.s_cumv, k * 8, cudaMemcpyDeviceToHost, st));
  if (punct_lp) CKL(cudaMemcpyAsync(punct_lp, x.s_plp, k * 24, cudaMemcpyDeviceToHost, st));
  CKL(cudaStreamSynchronize(st));
  return LB_OK;
}

}  // extern "C"
