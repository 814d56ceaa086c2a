/*
 * lightbeam_b200.h -- C ABI of the B200-native LightBeam first-pass decoder.
 *
 * This is the drop-in boundary for the reference's hot path
 * `lightbeam.decoder.decode(d, config, tt, lm, scorer, final_llm_only)`
 * (/root/reference/pkg/src/lightbeam/decoder.py:408-460).  The reference is pure Python, so its
 * "FFI" is the Python call itself; a maintainer binds these entry points with ctypes
 * (see INTEGRATION.md).  All functions are extern "C", take plain pointers and sizes, return
 * an int status (LB_OK = 0, negative = API/CUDA error; lb_last_error() has the message), and
 * never throw.  Handles are not thread-safe; one host thread drives one batch.
 *
 * Reference interface replaced by each entry point:
 *   lb_model_create      build_transition_table / load_table (lexicon.py:149-209,236-277) and
 *                        load_arpa (ngram.py:90-174) results uploaded as device images:
 *                        dense (S,V) int32 table with completion headers + completion CSR,
 *                        4-gram records in a bucketized cuckoo table.
 *   lb_batch_create      init_beams (decoder.py:177-179) for B utterances at once.
 *   lb_batch_set_logits  scale_log_softmax (logits.py:119-130) fused on upload (kernel K1).
 *   lb_batch_set_logprobs  the LogProbMatrix argument of decode (decoder.py:408) in fp64.
 *   lb_batch_run         the frame loop of decode (decoder.py:426-430): step (238-326) with
 *                        valid_mask (lexicon.py:124-137) and apply_ngram (decoder.py:182-235);
 *                        optionally the interval/final fusion of a device n-gram scorer.
 *   lb_batch_close       _close_utterance (decoder.py:375-405).
 *   lb_batch_gather_entries  the text gathering of apply_llm (decoder.py:338-345) as word-id
 *                        sequences per ortho entry.
 *   lb_batch_apply_scores  the fusion part of apply_llm (decoder.py:354-371).
 *   lb_batch_device_ngram_fusion  apply_llm with StubScorer(ngram_model=...) semantics
 *                        (scorer.py:121-139) evaluated on the device.
 *   lb_batch_results     ranking + n-best of decode (decoder.py:433-460), assembled on the host.
 */
#ifndef LIGHTBEAM_B200_H
#define LIGHTBEAM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LB_OK 0
#define LB_ERR_ARG -1
#define LB_ERR_CUDA -2
#define LB_ERR_CAPACITY -3
#define LB_ERR_STATE -4

/* per-trial status codes (lb_batch_status) */
#define LB_TRIAL_OK 0
#define LB_TRIAL_EMPTY_CANDIDATES 1 /* "all candidates pruned at frame t"  decoder.py:267-268 */
#define LB_TRIAL_EMPTY_MERGE 2      /* "all hypotheses pruned at frame t"  decoder.py:314-315 */
#define LB_TRIAL_EMPTY_CLOSE 3      /* "no hypothesis survived ... closure" decoder.py:394-395 */
#define LB_TRIAL_HISTORY_FULL 4     /* device word-history arena exhausted (capacity error) */

#define LB_PUNCT_NONE 0
#define LB_PUNCT_PERIOD 1
#define LB_PUNCT_QUESTION 2
#define LB_PUNCT_EXCLAIM 3

typedef struct lb_model lb_model;
typedef struct lb_batch lb_batch;

/* DecodeConfig (config.py:14-62), field for field. */
typedef struct {
  double acoustic_scale;
  double beam_prune_threshold;
  double homophone_prune_threshold;
  double token_insertion_bonus;
  double word_boundary_bonus;
  double ngram_weight;
  double llm_weight;
  int32_t beam_size;
  int32_t ortho_beams;
  int32_t llm_rescore_interval;
  int32_t llm_chunk_size;
} lb_config;

/* TransitionTable image (host pointers, copied during lb_model_create). */
typedef struct {
  const int32_t* table; /* [num_states * vocab_size], row-major */
  int32_t num_states;
  int32_t vocab_size; /* <= 64 */
  int32_t sink, blank_id, space_id;
  const int32_t* comp_offsets; /* [num_states + 1] */
  const int32_t* comp_surface; /* [n_comp] distinct surfaces per completion state */
  const int32_t* comp_lmword;  /* [n_comp] LM word id each surface is scored as, -1 = OOV kill */
  int32_t n_comp;
  const char* surface_blob;    /* utf-8 surfaces, concatenated */
  const int64_t* surface_offsets; /* [n_surfaces + 1] */
  int32_t n_surfaces;
} lb_table_desc;

/* NGramModel image. */
typedef struct {
  int32_t order; /* 1..4 */
  int64_t n_grams;
  const uint32_t* words;   /* [n_grams * 4], 0xFFFFFFFF pads */
  const double* probs;     /* [n_grams], quiet-NaN 0x7FF8DEAD00000000 = no probability */
  const double* backoffs;  /* [n_grams], 0.0 if absent */
  uint32_t bos_id;         /* id of "<s>" (initial history) */
  int32_t eos_word;        /* LM id "</s>" is scored as, -1 = kill */
  double bos_backoff;      /* backoffs.get(("<s>",), 0.0) */
} lb_ngram_desc;

/* Counters a run accumulates (summed over trials and frames). */
typedef struct {
  uint64_t frames;        /* frames stepped */
  uint64_t beams_in;      /* sum over frames of K_t entering the frame */
  uint64_t beams_out;     /* sum of K_{t+1} */
  uint64_t ngram_calls;   /* score_word evaluations */
  uint64_t ngram_probes;  /* hash-slot reads */
  uint64_t boundary_beams;
  uint64_t history_nodes;
  uint64_t fallback_selects; /* frames that needed the radix fallback */
  uint64_t ngram_pairs_used; /* (entry, surface) pairs the word-boundary beams consume: the
                                reference's score_word calls (ngram_calls adds speculation) */
} lb_stats;

const char* lb_last_error(void);
int lb_device_count(int32_t* out);

int lb_model_create(const lb_table_desc* table, const lb_ngram_desc* ngram, int32_t device,
                    lb_model** out);
int lb_model_destroy(lb_model* m);
/* bytes of device memory held by the model images */
int lb_model_footprint(const lb_model* m, int64_t* bytes);
/* 1 when the table is a breadth-first trie (successors of a state are consecutive ids, space ->
   root) and the frame kernel derives successors arithmetically; 0 = successor-list lookups */
int lb_model_lex_contiguous(const lb_model* m, int32_t* out);

/* stream: a cudaStream_t (NULL = legacy default stream). */
int lb_batch_create(lb_model* m, const lb_config* cfg, int32_t max_trials, int32_t max_frames,
                    void* stream, lb_batch** out);
int lb_batch_destroy(lb_batch* b);
/* Working-set placement of the frames kernel: dynamic shared memory per CTA, per-trial global
 * spill scratch, threads per CTA. */
int lb_batch_layout(lb_batch* b, int64_t* smem_bytes, int64_t* gscratch_bytes, int32_t* nthreads);

/* Inputs.  `x` is [n_trials, max_frames, vocab_size] row-major; frames[i] <= max_frames.
 * `on_device` != 0: x is a device pointer (stream-ordered), else a host pointer (pinned or
 * pageable) copied inside the call.  set_logits runs the fp64 log-softmax prologue. */
int lb_batch_set_logits(lb_batch* b, int32_t n_trials, const float* x, const int32_t* frames,
                        int32_t on_device);
int lb_batch_set_logprobs(lb_batch* b, int32_t n_trials, const double* d, const int32_t* frames,
                          int32_t on_device);
/* Copy the device log-prob matrix back: out is [n_trials, max_frames, vocab_size]. */
int lb_batch_get_logprobs(lb_batch* b, double* out_host);

/* Reset every trial to the root hypothesis (init_beams). */
int lb_batch_reset(lb_batch* b);

/* Advance every live trial over frames [t_begin, t_end) (clipped to its own length).
 * fusion_mode 0: no interval fusion inside the kernel (the caller performs events).
 * fusion_mode 1: interval events of a device n-gram scorer with scale `scorer_scale` happen
 *               inside the kernel (t > 0, t % r == 0).  */
int lb_batch_run(lb_batch* b, int32_t t_begin, int32_t t_end, int32_t fusion_mode,
                 double scorer_scale);

/* End-of-utterance closure for every live trial. */
int lb_batch_close(lb_batch* b);

/* apply_llm with StubScorer(ngram_model=model, scale) semantics on the device.
 * final != 0 also appends "</s>" and sets punctuation "." (scorer.py:136-139).
 * only trials with frames > min_frames take part (interval events skip finished trials). */
int lb_batch_device_ngram_fusion(lb_batch* b, int32_t final, double scale, int32_t min_frames);

/* Word-history gather for host scorers.  Fills, per trial, the ortho entries of every beam
 * in beam order and their word-id (surface id) sequences.
 *   entry_count[n_trials]          number of entries per trial
 *   entry_offsets[n_trials + 1]    prefix sums of entry_count (first-entry index per trial)
 * then lb_batch_copy_entries copies the flat arrays (sizes from lb_batch_entry_totals). */
int lb_batch_gather_entries(lb_batch* b, int64_t* n_entries, int64_t* n_words);
int lb_batch_copy_entries(lb_batch* b, int32_t* entry_trial, int32_t* entry_beam,
                          int64_t* word_offsets /* [n_entries+1] */, int32_t* words,
                          double* totals, int32_t* puncts);

/* Host scores for every gathered entry, in gather order.  has_text[i] == 0 marks the empty
 * history (gets total 0.0 and no punctuation).  final != 0 stores puncts.  Only trials with
 * frames > min_frames are updated. */
int lb_batch_apply_scores(lb_batch* b, const double* scores, const int32_t* puncts,
                          const uint8_t* has_text, int32_t final, int32_t min_frames);

/* Per-trial status and failing frame. */
int lb_batch_status(lb_batch* b, int32_t* status, int32_t* fail_frame);
int lb_batch_stats(lb_batch* b, lb_stats* out);
int lb_batch_clear_stats(lb_batch* b);

/* Debug/parity: copy the current beams of trial `trial` (scores, hashes, prefixes, last). */
int lb_batch_dump_beams(lb_batch* b, int32_t trial, int32_t* k, double* scores, uint64_t* h1,
                        uint64_t* h2, int32_t* prefix, int32_t* last);

/* Per-frame beam dump for parity bisection (off by default): after lb_batch_enable_dump(b, 1)
 * every lb_batch_run records the post-merge beams of each frame. */
int lb_batch_enable_dump(lb_batch* b, int32_t on);
int lb_batch_dump_frame(lb_batch* b, int32_t trial, int32_t t, int32_t* k, double* scores,
                        uint64_t* h1, uint64_t* h2, int32_t* prefix, int32_t* last);

/* Per-phase cycle counters of the frames kernel (clock64 deltas between its barriers,
 * thread 0 of each CTA; 12 slots, summed over trials) -- profiling aid, off by default. */
int lb_batch_enable_phase_timing(lb_batch* b, int32_t on);
int lb_batch_phase_cycles(lb_batch* b, uint64_t* out);

/* Results (decoder.py:433-460).  Two-step: lb_batch_results_size gives the byte size of the
 * text blob and the total n-best count; lb_batch_results fills caller buffers:
 *   best_text_off/best_text_len/best_score [n_trials]
 *   nbest_count [n_trials], nbest_text_off/nbest_text_len/nbest_score [total nbest]
 * Texts are utf-8 "w1 w2 ...<punct>" in `blob`. */
int lb_batch_results_size(lb_batch* b, int64_t* blob_bytes, int64_t* total_nbest);
int lb_batch_results(lb_batch* b, char* blob, int64_t* best_text_off, int32_t* best_text_len,
                     double* best_score, int32_t* nbest_count, int64_t* nbest_text_off,
                     int32_t* nbest_text_len, double* nbest_score);

/* Zero-copy view of the results assembled by the last lb_batch_results_size call: pointers
 * into library-owned host buffers, valid until the next results call or lb_batch_destroy.
 * Same content as lb_batch_results plus the per-trial status (0 = decoded).  Lets a binding
 * build its result objects straight from the library's buffers (no blob copy). */
typedef struct lb_results_view {
  int32_t n_trials;
  int64_t total_nbest;
  int64_t blob_bytes;
  const char* blob;
  const int32_t* status;
  const int64_t* best_text_off;
  const int32_t* best_text_len;
  const double* best_score;
  const int32_t* nbest_count;
  const int64_t* nbest_text_off;
  const int32_t* nbest_text_len;
  const double* nbest_score;
} lb_results_view;
int lb_batch_results_view(lb_batch* b, lb_results_view* out);

/* A non-blocking CUDA stream for lb_batch_create (pipelining batches on separate streams). */
int lb_stream_create(int32_t device, void** out);
int lb_stream_destroy(void* stream);

/* Page-locked host memory (cudaHostAlloc) for input staging: H2D copies from it run at full
 * link speed and stay asynchronous. */
int lb_host_alloc(int64_t bytes, void** out);
int lb_host_free(void* p);

/* Device-side timing of everything enqueued between mark_begin and mark_end (CUDA events on
 * the batch stream); also the number of kernels this library launched in between. */
/* kernels this library has launched so far (all batches; CUDA-graph replays not included) */
int lb_launch_count(uint64_t* out);
int lb_batch_mark_begin(lb_batch* b);
int lb_batch_mark_end(lb_batch* b, float* ms, int64_t* launches);
int lb_batch_sync(lb_batch* b);
/* Order `b`'s stream after everything enqueued on `prev`'s stream so far (event record + stream
 * wait; no host synchronisation).  decode_stream_raw uses it so two pipelined batches' search
 * kernels run back to back instead of sharing the SMs, while the next batch's H2D copy and
 * prologue, and the host's result assembly, still overlap the running search. */
int lb_batch_after(lb_batch* b, lb_batch* prev);

/* Standalone acoustic prologue (logits.py:119-130) on device `device`: host in/out. */
int lb_log_softmax_host(const float* x, int64_t rows, int32_t cols, double alpha,
                        double* out, int32_t device);

/* Host n-gram scorer parity helper: device score_word for (history ids, word). */
int lb_model_score_words(lb_model* m, int32_t n, const uint32_t* hist /* [n*3] */,
                         const int32_t* hist_len, const int32_t* word, double* inc,
                         uint32_t* succ /* [n*3] */, int32_t* succ_len);

/* ------------------------------------------------------------------------------------------
 * Device LLM delayed fusion (apply_llm, decoder.py:329-372, with a Llama-architecture scorer
 * resident on the GPU; scoring convention of sidecar/src/model.ts:35-47,116-137 at word-token
 * granularity).  The handle owns a prefix-trie KV cache ("slots": one per distinct token path,
 * hash-consed on (parent slot, token)); the caller owns the weights and runs the GEMMs of the
 * transformer body (bf16 tensor cores) between the kernels below, all on the batch stream.
 * Per fusion event:
 *   lb_llm_plan        map live entries' word histories to slots; returns the rows (slots whose
 *                      forward pass this event needs) as one wave in slot-id order, a dependency
 *                      order: every row's new ancestors precede it, so the wave runs as one
 *                      tree-causal prefill and any row-prefix chunk is self-contained
 *   per wave, per row chunk:
 *     lb_llm_wave_rows   tokens / positions / slots / ancestor chains of the rows
 *     body: lb_llm_rmsnorm, GEMM, lb_llm_rope_kv, lb_llm_attention, GEMM, lb_llm_rmsnorm,
 *           GEMM, lb_llm_swiglu, GEMM, ... final lb_llm_rmsnorm(store_slots) -> LM-head GEMM
 *           -> lb_llm_lse
 *   lb_llm_finish      next-token log-probs, text scores, punctuation (final), fusion (K7)
 * ------------------------------------------------------------------------------------------ */
#define LB_LLM_MAX_WAVES 512

typedef struct lb_llm lb_llm;

typedef struct {
  int32_t n_layers, n_heads, n_kv_heads, head_dim, hidden, vocab;
  int64_t max_slots;   /* prefix-cache capacity (token positions over the whole batch decode) */
  int32_t max_depth;   /* longest text in tokens after BOS (<= 4095) */
  int32_t bos_token;
  int32_t punct_tokens[3];             /* ".", "?", "!" */
  const int32_t* surface_tokens;       /* host: tokens of each lexicon surface after an earlier
                                        * word (word-level: one per surface; char-level: " w o r d") */
  const int32_t* surface_tokens_first; /* host: tokens of the surface as the sentence-cased first word */
  int32_t n_surfaces;
  const int32_t* surface_token_off;       /* host [n_surfaces + 1] CSR offsets into surface_tokens,
                                           * or NULL: exactly one token per surface */
  const int32_t* surface_token_off_first; /* same for surface_tokens_first */
  const void* embedding; /* device bf16 [vocab][hidden]: the LM head (tied or not); caller-owned */
  const float* head_f32; /* device fp32 [vocab][hidden] or NULL: next-token / punctuation dot
                          * products read this copy of the LM head (weights that are not
                          * bf16-exact, e.g. the sidecar's TinyCausalLM, model.ts:93-117) */
  int32_t precision;     /* 0 = bf16: one bf16 GEMM operand per activation, bf16 q/K/V;
                          * 1 = bf16x2: activations as hi+lo bf16 pairs ([M][2K] GEMM operands
                          *     against [W | W]), fp32 q/K/V -- fp32-equivalent activations on
                          *     the bf16 tensor cores at twice the body FLOPs */
} lb_llm_desc;

int lb_llm_create(lb_batch* b, const lb_llm_desc* desc, lb_llm** out);
int lb_llm_destroy(lb_llm* l);
int lb_llm_footprint(lb_llm* l, int64_t* bytes);
/* forget every cached prefix (start of a batch decode; the BOS row joins the next plan) */
int lb_llm_reset(lb_llm* l);
/* the two halves of lb_llm_reset: the device state (stream-ordered kernels, CUDA-graph
 * capturable) and the host-side event statistics (run before each graph replay) */
int lb_llm_reset_device(lb_llm* l);
int lb_llm_reset_stats(lb_llm* l);
/* wave_rows: caller array of LB_LLM_MAX_WAVES.  Synchronises the batch stream once. */
int lb_llm_plan(lb_llm* l, int32_t final_, int32_t min_frames, int32_t* n_waves,
                int64_t* wave_rows);
/* device outputs: tokens/positions/slots [n], chains [n][max_depth + 1] (slot ids BOS..row) */
int lb_llm_wave_rows(lb_llm* l, int32_t wave, int64_t row0, int32_t n, int32_t* tokens,
                     int32_t* positions, int32_t* slots, int32_t* chains);
int lb_llm_finish(lb_llm* l, int32_t final_, int32_t min_frames);
/* Graph-capturable event (no host synchronisation, for CUDA-graph replay of whole decodes):
 * the planning kernels of lb_llm_plan with the row count left on the device; the forward then
 * always runs rows_cap rows (lb_llm_wave_rows_async pads past the event's rows with BOS-only
 * rows that write a scratch slot).  An event with more than rows_cap rows sets a device flag
 * that lb_llm_check (synchronises) reports as LB_ERR_CAPACITY: the caller re-decodes eagerly. */
int lb_llm_plan_async(lb_llm* l, int32_t final_, int32_t min_frames, int32_t rows_cap);
int lb_llm_wave_rows_async(lb_llm* l, int32_t rows_cap, int32_t* tokens, int32_t* positions,
                           int32_t* slots, int32_t* chains);
int lb_llm_check(lb_llm* l);
/* x[M][hidden] fp32 residual (+= delta fp32 [M][hidden] if non-NULL); out bf16 = RMSNorm(x)*w
 * ([M][2 hidden] hi|lo pairs in bf16x2 precision).
 * store_slots != NULL: the rows are the final hidden states of those slots (kept in fp32 for
 * later next-token log-probs). */
int lb_llm_rmsnorm(lb_llm* l, float* x, const void* delta, const float* w, float eps, int32_t M,
                   void* out, const int32_t* store_slots);
/* LayerNorm variant (GPT-2 architecture): out = ((x - mean) * rsqrt(var + eps)) * w + b */
int lb_llm_layernorm(lb_llm* l, float* x, const void* delta, const float* w, const float* b,
                     float eps, int32_t M, void* out, const int32_t* store_slots);
/* in fp32 [M][ffn] (+ bias [ffn] if non-NULL) -> out bf16 [M][ffn] = gelu_tanh(in) ([M][2 ffn]
 * hi|lo pairs in bf16x2 precision) -- the GPT-2 MLP activation ("gelu_new") */
int lb_llm_gelu(lb_llm* l, const float* in, const float* bias, int32_t M, int32_t ffn, void* out);
/* qkv fp32 [M][(n_heads + 2 n_kv_heads) head_dim] -> q_out [M][n_heads head_dim] rotated (bf16;
 * fp32 in bf16x2 precision);
 * rotated K and V written to the rows' slots of layer `layer`.  cos/sin fp32 [pos][head_dim/2] */
int lb_llm_rope_kv(lb_llm* l, int32_t layer, const void* qkv, int32_t M, const int32_t* pos,
                   const int32_t* slots, const float* cos_tab, const float* sin_tab, void* q_out);
/* causal GQA attention of each row over its ancestor chain; out bf16 [M][n_heads head_dim]
 * ([M][2 n_heads head_dim] hi|lo pairs in bf16x2 precision) */
int lb_llm_attention(lb_llm* l, int32_t layer, const void* q, int32_t M, const int32_t* chains,
                     const int32_t* pos, void* out);
/* gu [M][2 ffn] = [gate | up] (bf16; fp32 in bf16x2 precision) -> out bf16 [M][ffn] =
 * silu(gate) * up ([M][2 ffn] hi|lo pairs in bf16x2 precision) */
int lb_llm_swiglu(lb_llm* l, const void* gu, int32_t M, int32_t ffn, void* out);
/* K6: log-sum-exp of LM-head logit rows (bf16 [M][ld], vocab columns) into the rows' slots */
int lb_llm_lse(lb_llm* l, const void* logits, int32_t M, int64_t ld, const int32_t* slots);
/* K6 fused on tcgen05: log-sum-exp of the LM-head logits h[M][K] . emb[N][K]^T (bf16, K-major,
 * row pitches ldh / lde elements) into the rows' slots, without materialising logits.
 * partial: device scratch of M * ceil(N / 256) float2. */
int lb_llm_lmhead_lse(lb_llm* l, const void* h, int32_t M, int64_t ldh, int32_t K, const void* emb,
                      int64_t lde, int32_t N, const int32_t* slots, void* partial);
/* Gate/up projection with the SwiGLU fused into the tcgen05 epilogue: act = silu(h W_g^T) *
 * (h W_u^T) for h[M][K] bf16 (pitch ldh), weights interleaved in 128-row blocks
 * [g 0:128 | u 0:128 | g 128:256 | u 128:256 | ...] ([2 ffn][K], pitch ldw); act bf16 [M][ffn]
 * ([M][2 ffn] hi|lo pairs in bf16x2 precision).  ffn % 128 == 0. */
int lb_llm_gateup_swiglu(lb_llm* l, const void* h, int32_t M, int64_t ldh, int32_t K,
                         const void* wgu_interleaved, int64_t ldw, int32_t ffn, void* act);
/* out[8]: slots, events, waves, forwarded rows, widest wave, device bytes, scores computed
 * (next-token log-probs), attention launches that used sibling tiles */
int lb_llm_stats(lb_llm* l, int64_t* out);
/* Parity/debug: the slot table.  *n = slots in use; the first min(*n, max_n) rows are copied
 * into the host buffers (NULL skips a field).  state bits:
 * 1 forwarded, 2 score ready, 4 punctuation ready; punct_lp [n][3].  parent -2 marks a spare
 * slot left by a lost insert race (never referenced). */
int lb_llm_export(lb_llm* l, int64_t max_n, int64_t* n, int32_t* parent, int32_t* token,
                  int32_t* depth, int32_t* state, double* cum, double* punct_lp);

#ifdef __cplusplus
}
#endif
#endif
