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
__device__ __forceinline__ bool ng_lookup(const ModelDev& m, const uint32_t k[4], double& p,
                                          double& bo, unsigned& probes) {
  uint64_t h = ng_hash(k[0], k[1], k[2], k[3]) & m.ng_mask;
  for (;;) {
    const uint4* rec = reinterpret_cast<const uint4*>(m.ng + h);
    const uint4 kw = __ldg(rec);
    const double2 pb = __ldg(reinterpret_cast<const double2*>(rec) + 1);
    ++probes;
    if (kw.x == WPAD) return false;
    if (kw.x == k[0] && kw.y == k[1] && kw.z == k[2] && kw.w == k[3]) {
      p = pb.x;
      bo = pb.y;
      return true;
    }
    h = (h + 1) & m.ng_mask;
  }
}

// score_word (ngram.py:208-236) for one (history, word) per 8-lane group; all 32 lanes call.
// Lane sub 0..3 probes K_sub = (h[sub:], w); lanes 4..6 probe the history H_{sub-4} = h[sub-4:]
// for its back-off.  The group leader (sub 0) combines: right-nested back-off sum and the
// successor = longest listed suffix of (h + w) capped at order-1 words.  `w < 0` is the
// OOV-without-<unk> kill: increment NEG_INF, successor ().
__device__ void group_score_word(const ModelDev& m, bool act, const uint32_t h[MAXH], int hl, int w,
                                 double& inc, uint32_t succ[MAXH], int& slen, unsigned& probes) {
  const int lane = threadIdx.x & 31, sub = lane & 7, grp = lane >> 3;
  const bool valid = act && w >= 0;
  bool hasp = false;
  double p = 0.0, bo = 0.0;
  if (valid) {
    uint32_t k[4] = {WPAD, WPAD, WPAD, WPAD};
    bool doit = false;
    int n = 0;
    if (sub <= 3) {
      if (sub <= hl) {
        for (int i = sub; i < hl; ++i) k[n++] = h[i];
        k[n++] = (uint32_t)w;
        doit = true;
      }
    } else if (sub <= 6) {
      const int i0 = sub - 4;
      if (i0 < hl) {
        for (int i = i0; i < hl; ++i) k[n++] = h[i];
        doit = true;
      }
    }
    if (doit) {
      const bool found = ng_lookup(m, k, p, bo, probes);
      if (!found) bo = 0.0;
      hasp = found && prob_present(p);
    }
  }
  const unsigned bal = __ballot_sync(FULLMASK, hasp);
  const unsigned gb = (bal >> (grp * 8)) & 0xFFu;
  double pk0 = __shfl_sync(FULLMASK, p, grp * 8 + 0);
  double pk1 = __shfl_sync(FULLMASK, p, grp * 8 + 1);
  double pk2 = __shfl_sync(FULLMASK, p, grp * 8 + 2);
  double pk3 = __shfl_sync(FULLMASK, p, grp * 8 + 3);
  double b0 = __shfl_sync(FULLMASK, bo, grp * 8 + 4);
  double b1 = __shfl_sync(FULLMASK, bo, grp * 8 + 5);
  double b2 = __shfl_sync(FULLMASK, bo, grp * 8 + 6);
  slen = 0;
  inc = NEG_INF;
  if (sub != 0 || !act) return;
  if (!valid) return;  // kill: NEG_INF, successor ()
  const double pk[4] = {pk0, pk1, pk2, pk3};
  const double bh[3] = {b0, b1, b2};
  double val = NEG_INF;
  int hit = hl + 1;
  for (int i = 0; i <= hl; ++i)
    if ((gb >> i) & 1u) {
      val = pk[i];
      hit = i;
      break;
    }
  for (int i = min(hit, hl) - 1; i >= 0; --i) val = xadd(bh[i], val);
  inc = val;
  if (m.order > 1) {
    const int start = max(0, hl + 1 - (m.order - 1));
    for (int i = start; i <= hl; ++i)
      if ((gb >> i) & 1u) {
        int n = 0;
        for (int j = i; j < hl; ++j) succ[n++] = h[j];
        succ[n++] = (uint32_t)w;
        slen = n;
        break;
      }
  }
}

// apply_ngram (decoder.py:182-235) for one beam, one full warp.  Candidates are the
// (entry, distinct surface) pairs in creation order; the running top-O list is ordered by
// (-total, seq) -- candidates arrive in increasing seq, so strict '>' keeps ties stable.
// On return (lane 0 authoritative): *outn = kept entries (written to outents), or -1 when no
// candidate survived (beam killed: *score = NEG_INF, decoder.py:223-225).
__device__ void warp_apply_ngram(const ModelDev& m, const CfgDev& c, const BatchDev& b, int trial,
                                 const Ent* pents, int pn, int st, WarpScratch* ws, Ent* outents,
                                 int* outn, double* score, int* node_counter, int* fail,
                                 unsigned& calls, unsigned& probes) {
  const int lane = threadIdx.x & 31, sub = lane & 7, grp = lane >> 3;
  const int cbeg = m.comp_off[st];
  const int ns = m.comp_off[st + 1] - cbeg;
  const int npairs = pn * ns;
  int ntop = 0;
  for (int base = 0; base < npairs; base += 4) {
    const int pi = base + grp;
    const bool act = pi < npairs;
    int e = 0, s = 0, w = -1;
    if (act) {
      e = pi / ns;
      s = pi - e * ns;
      w = m.comp_lm[cbeg + s];
    }
    const Ent& E = pents[act ? e : 0];
    uint32_t hh[MAXH] = {E.h[0], E.h[1], E.h[2]};
    const int hl = E.hlen;
    double inc;
    uint32_t sh[MAXH] = {0, 0, 0};
    int sl;
    group_score_word(m, act, hh, hl, w, inc, sh, sl, probes);
    if (sub == 0) {
      NgCand& pc = ws->pending[grp];
      pc.valid = 0;
      if (act) {
        ++calls;
        if (inc > GUARD) {
          pc.valid = 1;
          pc.total = xadd(E.total, xmul(c.omega, inc));
          pc.inc = inc;
          pc.node = E.node;
          pc.surf = (uint32_t)m.comp_surf[cbeg + s];
          pc.seq = (uint32_t)pi;
          pc.hlen = (uint32_t)sl;
          pc.h[0] = sh[0];
          pc.h[1] = sh[1];
          pc.h[2] = sh[2];
        }
      }
    }
    __syncwarp();
    if (lane == 0) {
      for (int g = 0; g < 4; ++g) {
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
        kept = 0;
        *outn = -1;
        *score = NEG_INF;
      } else {
        const size_t nb = (size_t)trial * b.ncap;
        for (int i = 0; i < kept; ++i) {
          const NgCand& cd = ws->top[i];
          const uint32_t node = (uint32_t)(base + i);
          b.nparent[nb + node] = cd.node;
          b.nsurf[nb + node] = cd.surf;
          b.ndepth[nb + node] = b.ndepth[nb + cd.node] + 1;
          b.ncum[nb + node] = xadd(b.ncum[nb + cd.node], cd.inc);
          Ent o;
          o.total = cd.total;
          o.node = node;
          o.seq = cd.seq;
          o.h[0] = cd.h[0];
          o.h[1] = cd.h[1];
          o.h[2] = cd.h[2];
          o.hlen = (uint8_t)cd.hlen;
          o.punct = 0;
          o.pad = 0;
          outents[i] = o;
        }
        *outn = kept;
        *score = xadd(*score, xsub(best, pents[0].total));
      }
    }
  }
  __syncwarp();
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

__device__ __forceinline__ void copy_ents(Ent* dst, const Ent* src, int n) {
  const uint4* s = reinterpret_cast<const uint4*>(src);
  uint4* d = reinterpret_cast<uint4*>(dst);
  for (int i = 0; i < 2 * n; ++i) d[i] = s[i];
}

}  // namespace

// =====================================================================================
// K2: persistent frame loop
// =====================================================================================
template <int NT>
__global__ void __launch_bounds__(NT) frames_kernel(ModelDev m, CfgDev c, BatchDev b, Layout L,
                                                    int t0, int t1, int fusion_mode, double scale) {
  constexpr int NW = NT / 32;
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t dbar[2];
  __shared__ unsigned hist[NBINS];
  __shared__ double wmax[NW];
  __shared__ int s_cnt, s_nb, s_ncount, s_fail;
  __shared__ unsigned s_calls, s_probes;

  const int trial = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (b.status[trial] != 0) return;
  const int T = b.T[trial];
  const int tb = t0, te = min(t1, T);
  if (tb >= te) return;

  char* gs = b.gscratch + (int64_t)trial * b.gscratch_stride;
  auto R = [&](int r) -> char* { return L.in_smem[r] ? smem + L.off[r] : gs + L.off[r]; };
  double* dbuf = reinterpret_cast<double*>(R(R_DBUF));
  int32_t* rows = reinterpret_cast<int32_t*>(R(R_ROWS));
  BeamPtrs cur{(double*)R(R_CUR_SCORE), (uint64_t*)R(R_CUR_H1), (uint64_t*)R(R_CUR_H2),
               (int32_t*)R(R_CUR_LAST), (int32_t*)R(R_CUR_PRE), (int32_t*)R(R_CUR_NENT),
               (Ent*)R(R_CUR_ENTS)};
  BeamPtrs nxt{(double*)R(R_NXT_SCORE), (uint64_t*)R(R_NXT_H1), (uint64_t*)R(R_NXT_H2),
               (int32_t*)R(R_NXT_LAST), (int32_t*)R(R_NXT_PRE), (int32_t*)R(R_NXT_NENT),
               (Ent*)R(R_NXT_ENTS)};
  uint64_t* maskv = reinterpret_cast<uint64_t*>(R(R_MASK));
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
  WarpScratch* wsc = reinterpret_cast<WarpScratch*>(R(R_WARP));

  const int V = m.V, VP = m.VP, VPD = b.VPD, O = c.O, KC = b.K;
  const FrameConsts fc{c.beta, c.gamma, m.blank, m.space};
  const int nkw = (c.k + 31) >> 5;

  // ---- load the home beam state
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
    }
    const uint4* src = reinterpret_cast<const uint4*>(b.ents + hb * O);
    uint4* dst = reinterpret_cast<uint4*>(cur.ents);
    for (int i = tid; i < K * O * 2; i += NT) dst[i] = src[i];
  }
  if (tid == 0) {
    s_ncount = b.ncount[trial];
    s_fail = 0;
    s_calls = 0;
    s_probes = 0;
    mbar_init(&dbar[0], 1);
    mbar_init(&dbar[1], 1);
    fence_mbar_init();
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
  unsigned calls_l = 0, probes_l = 0;
  int status = 0, fail_t = -1;

  for (int t = tb; t < te; ++t) {
    const int rel = t - tb;
    const int ci = rel / CHUNK;
    if (rel % CHUNK == 0) {
      mbar_wait(&dbar[ci & 1], (unsigned)((ci >> 1) & 1));
      if (tid == 0) issue_chunk(ci + 1);
    }
    const double* drow = dbuf + ((size_t)(ci & 1) * CHUNK + (rel % CHUNK)) * VPD;
    st_beams_in += K;

    // ---- A1: stage the K lexicon rows (16-byte cp.async, all in flight at once)
    if (L.stage_rows) {
      const int cpr = VP >> 2;
      for (int q = tid; q < K * cpr; q += NT) {
        const int p = q / cpr, part = q - p * cpr;
        cp_async16(rows + p * VP + part * 4, m.table + (size_t)cur.pre[p] * VP + part * 4);
      }
      cp_async_commit();
    }
    for (int i = tid; i < NBINS; i += NT) hist[i] = 0;
    for (int i = tid; i < nkw; i += NT) keep[i] = 0;
    if (tid == 0) {
      s_cnt = 0;
      s_nb = 0;
    }
    if (L.stage_rows) cp_async_wait_all();
    __syncthreads();  // S1

    // ---- A2: validity masks + per-warp maximum of eligible candidates
    double wm = -DBL_MAX;
    for (int p = warp; p < K; p += NW) {
      const int lp = cur.last[p];
      const double s = cur.score[p];
      const int32_t* row = L.stage_rows ? rows + p * VP : m.table + (size_t)cur.pre[p] * VP;
      uint64_t mk = 0;
      for (int v0 = 0; v0 < V; v0 += 32) {
        const int v = v0 + lane;
        bool ok = false;
        if (v < V) {
          const int nx = row[v];
          ok = (nx != m.sink) || (v == m.blank) || (v == lp);
          if (ok) {
            const double x = cand_value(s, drow[v], v, lp, fc);
            ok = x > GUARD;
            if (ok) wm = fmax(wm, x);
          }
        }
        mk |= (uint64_t)__ballot_sync(FULLMASK, ok) << v0;
      }
      if (lane == 0) maskv[p] = mk;
    }
    wm = warp_max(wm);
    if (lane == 0) wmax[warp] = wm;
    __syncthreads();  // S2

    double M = -DBL_MAX;
    for (int w = 0; w < NW; ++w) M = fmax(M, wmax[w]);
    if (M <= GUARD) {  // decoder.py:267-268
      status = 1;
      fail_t = t;
      break;
    }
    const double thr = xsub(M, c.theta);

    // ---- B: histogram of in-range candidates over [thr, M]
    for (int p = warp; p < K; p += NW) {
      const uint64_t mk = maskv[p];
      const int lp = cur.last[p];
      const double s = cur.score[p];
      for (int v = lane; v < V; v += 32) {
        if (!((mk >> v) & 1ull)) continue;
        const double x = cand_value(s, drow[v], v, lp, fc);
        if (x >= thr) {
          int bin = (int)xmul(xsub(M, x), c.inv_binw);
          bin = min(bin, NBINS - 1);
          atomicAdd(&hist[bin], 1u);
        }
      }
    }
    __syncthreads();  // S3

    // ---- C: every warp scans the histogram (no extra barrier): boundary bin bstar
    int bstar = NBINS - 1, total = 0, m_sel = 0;
    {
      unsigned part[NBINS / 32];
      unsigned ls = 0;
#pragma unroll
      for (int i = 0; i < NBINS / 32; ++i) {
        part[i] = hist[lane * (NBINS / 32) + i];
        ls += part[i];
      }
      unsigned incl = ls;
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(FULLMASK, incl, o);
        if (lane >= o) incl += y;
      }
      total = (int)__shfl_sync(FULLMASK, incl, 31);
      if (total <= c.k) {
        bstar = NBINS - 1;
        m_sel = total;
      } else {
        const unsigned excl = incl - ls;
        const bool here = excl < (unsigned)c.k && incl >= (unsigned)c.k;
        const unsigned bl = __ballot_sync(FULLMASK, here);
        const int src = __ffs(bl) - 1;
        int lb = 0;
        unsigned cum = excl;
        if (lane == src) {
#pragma unroll
          for (int i = 0; i < NBINS / 32; ++i) {
            if (cum + part[i] >= (unsigned)c.k) {
              lb = i;
              break;
            }
            cum += part[i];
          }
        }
        lb = __shfl_sync(FULLMASK, lb, src);
        cum = __shfl_sync(FULLMASK, cum, src);
        bstar = src * (NBINS / 32) + lb;
        m_sel = (int)(cum + hist[bstar]);
      }
    }
    const int nsel = min(c.k, total);

    if (m_sel <= L.lcap) {
      // ---- D: collect candidates in bins <= bstar (warp-aggregated appends)
      for (int p = warp; p < K; p += NW) {
        const uint64_t mk = maskv[p];
        const int lp = cur.last[p];
        const double s = cur.score[p];
        for (int v0 = 0; v0 < V; v0 += 32) {
          const int v = v0 + lane;
          bool take = false;
          double x = 0.0;
          if (v < V && ((mk >> v) & 1ull)) {
            x = cand_value(s, drow[v], v, lp, fc);
            if (x >= thr) {
              const int bin = min((int)xmul(xsub(M, x), c.inv_binw), NBINS - 1);
              take = bin <= bstar;
            }
          }
          const unsigned bl = __ballot_sync(FULLMASK, take);
          if (bl) {
            int base = 0;
            if (lane == 0) base = atomicAdd(&s_cnt, __popc(bl));
            base = __shfl_sync(FULLMASK, base, 0);
            if (take) {
              const int pos = base + __popc(bl & ((1u << lane) - 1u));
              cval[pos] = x;
              ckey[pos] = (uint32_t)(p * V + v);
            }
          }
        }
      }
      __syncthreads();  // S4
      // ---- E: exact rank sort of the collected set, keep the first nsel
      {
        const int mm = m_sel;
        int G = 1;
        while (G < 32 && 2 * G * mm <= NT) G <<= 1;
        const int groups = NT / G, g = tid / G, r = tid & (G - 1);
        for (int i0 = 0; i0 < mm; i0 += groups) {
          const int i = i0 + g;
          const bool act = i < mm;
          const double vi = act ? cval[i] : 0.0;
          const uint32_t ki = act ? ckey[i] : 0u;
          int cnt = 0;
          if (act)
            for (int j = r; j < mm; j += G) {
              const double vj = cval[j];
              cnt += (vj > vi) || (vj == vi && ckey[j] < ki);
            }
          for (int o = G >> 1; o > 0; o >>= 1) cnt += __shfl_xor_sync(FULLMASK, cnt, o);
          if (act && r == 0 && cnt < nsel) {
            sval[cnt] = vi;
            skey[cnt] = ki;
          }
        }
      }
    } else {
      // ---- fallback: exact radix select on the 96-bit key (ord64(value), ~flat index)
      ++st_fallback;
      uint64_t phi = 0, pmask_hi = 0;
      uint32_t plo = 0, pmask_lo = 0;
      int rem = nsel;
      for (int pass = 0; pass < 12; ++pass) {
        __syncthreads();
        for (int i = tid; i < NBINS; i += NT) hist[i] = 0;
        __syncthreads();
        for (int p = warp; p < K; p += NW) {
          const uint64_t mk = maskv[p];
          const int lp = cur.last[p];
          const double s = cur.score[p];
          for (int v = lane; v < V; v += 32) {
            if (!((mk >> v) & 1ull)) continue;
            const double x = cand_value(s, drow[v], v, lp, fc);
            if (x < thr) continue;
            const uint64_t kh = ord64(x);
            const uint32_t kl = ~(uint32_t)(p * V + v);
            if ((kh & pmask_hi) != phi || (kl & pmask_lo) != plo) continue;
            const unsigned dg = pass < 8 ? (unsigned)((kh >> (56 - 8 * pass)) & 0xFF)
                                         : (unsigned)((kl >> (24 - 8 * (pass - 8))) & 0xFF);
            atomicAdd(&hist[dg], 1u);
          }
        }
        __syncthreads();
        // scan digits from 255 down (each thread redundantly; NBINS small)
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
      __syncthreads();
      // collect every candidate with key >= (phi, plo): exactly nsel of them
      for (int p = warp; p < K; p += NW) {
        const uint64_t mk = maskv[p];
        const int lp = cur.last[p];
        const double s = cur.score[p];
        for (int v0 = 0; v0 < V; v0 += 32) {
          const int v = v0 + lane;
          bool take = false;
          double x = 0.0;
          if (v < V && ((mk >> v) & 1ull)) {
            x = cand_value(s, drow[v], v, lp, fc);
            if (x >= thr) {
              const uint64_t kh = ord64(x);
              const uint32_t kl = ~(uint32_t)(p * V + v);
              take = kh > phi || (kh == phi && kl >= plo);
            }
          }
          const unsigned bl = __ballot_sync(FULLMASK, take);
          if (bl) {
            int base = 0;
            if (lane == 0) base = atomicAdd(&s_cnt, __popc(bl));
            base = __shfl_sync(FULLMASK, base, 0);
            if (take) {
              const int pos = base + __popc(bl & ((1u << lane) - 1u));
              cval[pos] = x;
              ckey[pos] = (uint32_t)(p * V + v);
            }
          }
        }
      }
      __syncthreads();
      for (int i = tid; i < nsel; i += NT) {
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
    }
    __syncthreads();  // S5

    // ---- F: materialise survivors in selection order (decoder.py:272-291)
    for (int j = tid; j < nsel; j += NT) {
      const double x = sval[j];
      const uint32_t f = skey[j];
      const int p = (int)(f / (uint32_t)V);
      const int tok = (int)(f - (uint32_t)p * V);
      const int lp = cur.last[p], pp = cur.pre[p];
      const bool emit = (tok != m.blank) && (tok != lp);
      uint64_t a1 = cur.h1[p], a2 = cur.h2[p];
      int np = pp;
      if (emit) {
        a1 = a1 * H_MULT1 + (uint64_t)(tok + 1);
        a2 = a2 * H_MULT2 + (uint64_t)(tok + 1);
        np = L.stage_rows ? rows[p * VP + tok] : m.table[(size_t)pp * VP + tok];
      }
      nscore[j] = x;
      nh1[j] = a1;
      nh2[j] = a2;
      nlast[j] = (tok == m.blank) ? lp : tok;
      npre[j] = np;
      npar[j] = p;
      bnent[j] = -1;
      if (emit && tok == m.space) blist[atomicAdd(&s_nb, 1)] = j;
    }
    __syncthreads();  // S6

    // ---- G: n-gram fusion for new word-boundary emissions, one warp per beam
    const int nb = s_nb;
    st_bound += nb;
    for (int bi = warp; bi < nb; bi += NW) {
      const int j = blist[bi];
      const int p = npar[j];
      int outn = -1;
      double sc = nscore[j];
      warp_apply_ngram(m, c, b, trial, cur.ents + (size_t)p * O, cur.nent[p], cur.pre[p], &wsc[warp],
                       bents + (size_t)j * O, &outn, &sc, &s_ncount, &s_fail, calls_l, probes_l);
      if (lane == 0) {
        nscore[j] = sc;
        bnent[j] = outn;
      }
    }
    __syncthreads();  // S7

    // ---- H: recombination ranking (post-fusion score desc, index asc) + hash dedupe
    {
      const int n = nsel;
      int G = 1;
      while (G < 32 && 2 * G * n <= NT) G <<= 1;
      const int groups = NT / G, g = tid / G, r = tid & (G - 1);
      for (int i0 = 0; i0 < n; i0 += groups) {
        const int i = i0 + g;
        const bool act = i < n;
        const double si = act ? nscore[i] : 0.0;
        const uint64_t a1 = act ? nh1[i] : 0, a2 = act ? nh2[i] : 0;
        int cnt = 0, dup = 0;
        if (act)
          for (int j = r; j < n; j += G) {
            const double sj = nscore[j];
            const bool beats = (sj > si) || (sj == si && j < i);
            cnt += beats;
            dup |= beats && (sj > GUARD) && nh1[j] == a1 && nh2[j] == a2;
          }
        for (int o = G >> 1; o > 0; o >>= 1) {
          cnt += __shfl_xor_sync(FULLMASK, cnt, o);
          dup |= __shfl_xor_sync(FULLMASK, dup, o);
        }
        if (act && r == 0) {
          rankv[i] = cnt;
          if (si > GUARD && !dup) atomicOr(&keep[cnt >> 5], 1u << (cnt & 31));
        }
      }
    }
    __syncthreads();  // S8

    // ---- scatter survivors into the next buffer in rank order
    int newK = 0;
    for (int w = 0; w < nkw; ++w) newK += __popc(keep[w]);
    for (int i = tid; i < nsel; i += NT) {
      const int rk = rankv[i];
      if (!((keep[rk >> 5] >> (rk & 31)) & 1u)) continue;
      int pos = __popc(keep[rk >> 5] & ((1u << (rk & 31)) - 1u));
      for (int w = 0; w < (rk >> 5); ++w) pos += __popc(keep[w]);
      nxt.score[pos] = nscore[i];
      nxt.h1[pos] = nh1[i];
      nxt.h2[pos] = nh2[i];
      nxt.last[pos] = nlast[i];
      nxt.pre[pos] = npre[i];
      const int bn = bnent[i];
      if (bn >= 0) {
        nxt.nent[pos] = bn;
        copy_ents(nxt.ents + (size_t)pos * O, bents + (size_t)i * O, bn);
      } else {
        const int p = npar[i];
        const int pn = cur.nent[p];
        nxt.nent[pos] = pn;
        copy_ents(nxt.ents + (size_t)pos * O, cur.ents + (size_t)p * O, pn);
      }
      if (b.dump_k) {
        const size_t di = ((size_t)trial * b.Tmax + t) * KC + pos;
        b.dump_h1[di] = nh1[i];
        b.dump_h2[di] = nh2[i];
        b.dump_pre[di] = npre[i];
        b.dump_last[di] = nlast[i];
        b.dump_score[di] = nscore[i];
      }
    }
    if (b.dump_k && tid == 0) b.dump_k[(size_t)trial * b.Tmax + t] = newK;
    __syncthreads();  // S9
    {
      BeamPtrs tmp = cur;
      cur = nxt;
      nxt = tmp;
    }
    K = newK;
    st_beams_out += K;
    if (s_fail) {
      status = 4;
      fail_t = t;
      break;
    }
    if (K == 0) {  // decoder.py:314-315
      status = 2;
      fail_t = t;
      break;
    }

    // ---- optional interval fusion of the device n-gram scorer (decoder.py:428-430)
    if (fusion_mode == 1 && t > 0 && (t % c.r) == 0) {
      const size_t nbase = (size_t)trial * b.ncap;
      for (int i = tid; i < K; i += NT) {
        Ent* e = cur.ents + (size_t)i * O;
        const int n = cur.nent[i];
        const double prev = e[0].total;
        for (int q = 0; q < n; ++q) {
          if (e[q].node == 0) {
            e[q].total = 0.0;
            e[q].punct = 0;
          } else {
            e[q].total = xmul(c.phi, xmul(scale, b.ncum[nbase + e[q].node]));
          }
        }
        sort_entries(e, n);
        cur.score[i] = xadd(cur.score[i], xsub(e[0].total, prev));
      }
      __syncthreads();
    }
  }

  // ---- write back
  __syncthreads();
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
    for (int i = tid; i < K * O * 2; i += NT) dst[i] = src[i];
  }
  atomicAdd(&s_calls, calls_l);
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
    stt[7] += st_fallback;
  }
}

// =====================================================================================
// K3: end-of-utterance closure (decoder.py:375-405), one CTA per trial, warp per beam
// =====================================================================================
__global__ void __launch_bounds__(256) close_kernel(ModelDev m, CfgDev c, BatchDev b) {
  constexpr int NT = 256, NW = NT / 32;
  __shared__ WarpScratch wsc[NW];
  __shared__ int s_ncount, s_fail;
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
  }
  __syncthreads();
  unsigned calls = 0, probes = 0;
  for (int i = warp; i < K; i += NW) {
    const int st = b.prefix[hb + i];
    if (st == 0) continue;  // root: nothing pending
    const int ncomp = m.comp_off[st + 1] - m.comp_off[st];
    if (ncomp == 0) {
      if (lane == 0) b.score[hb + i] = NEG_INF;
      continue;
    }
    double sc = b.score[hb + i];
    int outn = -1;
    Ent* pe = b.ents + (hb + i) * O;
    warp_apply_ngram(m, c, b, trial, pe, b.nent[hb + i], st, &wsc[warp], tmp, &outn, &sc,
                     &s_ncount, &s_fail, calls, probes);
    if (lane == 0) {
      b.score[hb + i] = sc;
      if (outn >= 0) {
        b.nent[hb + i] = outn;
        for (int q = 0; q < outn; ++q) pe[q] = tmp[q];
      }
      b.prefix[hb + i] = 0;
    }
    __syncwarp();
  }
  atomicAdd(&s_calls, calls);
  atomicAdd(&s_probes, probes);
  __syncthreads();
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
__global__ void __launch_bounds__(256) device_fusion_kernel(ModelDev m, CfgDev c, BatchDev b,
                                                            int final_, double scale,
                                                            int min_frames) {
  constexpr int NT = 256, NW = NT / 32;
  __shared__ unsigned s_probes;
  const int trial = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (b.status[trial] != 0 || b.T[trial] <= min_frames) return;
  const int KC = b.K, O = c.O;
  const size_t hb = (size_t)trial * KC;
  const size_t nbase = (size_t)trial * b.ncap;
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
      uint32_t sh[MAXH];
      int sl;
      if (final_) {
        uint32_t hh[MAXH] = {E.h[0], E.h[1], E.h[2]};
        group_score_word(m, act && E.node != 0, hh, E.hlen, m.eos_word, inc, sh, sl, probes);
      }
      if (act && sub == 0) {
        Ent o = E;
        if (E.node == 0) {
          o.total = 0.0;
          o.punct = 0;
        } else if (final_) {
          o.total = xmul(c.phi, xmul(scale, xadd(b.ncum[nbase + E.node], inc)));
          o.punct = 1;  // "." (scorer.py:136-139)
        } else {
          o.total = xmul(c.phi, xmul(scale, b.ncum[nbase + E.node]));
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
    const size_t nbase = (size_t)trial * b.ncap;
    const int K = b.nbeam[trial];
    unsigned long long ne = 0, nw = 0;
    for (int i = tid; i < K; i += blockDim.x) {
      const int n = b.nent[hb + i];
      ne += n;
      for (int q = 0; q < n; ++q) nw += b.ndepth[nbase + b.ents[(hb + i) * b.O + q].node];
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

__global__ void write_entries_kernel(BatchDev b, const int64_t* entry_off, const int64_t* word_off,
                                     int32_t* e_trial, int32_t* e_beam, int64_t* e_woff,
                                     int32_t* words, double* totals, int32_t* puncts) {
  const int trial = blockIdx.x;
  if (b.status[trial] != 0) return;
  const size_t hb = (size_t)trial * b.K;
  const size_t nbase = (size_t)trial * b.ncap;
  const int K = b.nbeam[trial];
  const int O = b.O;
  extern __shared__ int64_t sh_off[];  // [K + 1] entry prefix; then word prefix per entry
  if (threadIdx.x == 0) {
    int64_t e = 0;
    for (int i = 0; i < K; ++i) {
      sh_off[i] = e;
      e += b.nent[hb + i];
    }
    sh_off[K] = e;
  }
  __syncthreads();
  const int64_t ebase = entry_off[trial];
  // word offsets need a prefix over entries in order: do it serially per trial (<= K*O entries)
  if (threadIdx.x == 0) {
    int64_t w = word_off[trial];
    for (int i = 0; i < K; ++i) {
      const int n = b.nent[hb + i];
      for (int q = 0; q < n; ++q) {
        const int64_t idx = ebase + sh_off[i] + q;
        e_woff[idx] = w;
        w += b.ndepth[nbase + b.ents[(hb + i) * O + q].node];
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < K; i += blockDim.x) {
    const int n = b.nent[hb + i];
    for (int q = 0; q < n; ++q) {
      const int64_t idx = ebase + sh_off[i] + q;
      const Ent E = b.ents[(hb + i) * O + q];
      e_trial[idx] = trial;
      e_beam[idx] = i;
      totals[idx] = E.total;
      puncts[idx] = E.punct;
      uint32_t node = E.node;
      const uint32_t d = b.ndepth[nbase + node];
      int64_t wp = e_woff[idx] + d - 1;
      while (node != 0) {
        words[wp--] = (int32_t)b.nsurf[nbase + node];
        node = b.nparent[nbase + node];
      }
    }
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
  e.node = 0;
  e.seq = 0;
  e.h[0] = m.bos;
  e.h[1] = 0;
  e.h[2] = 0;
  e.hlen = 1;
  e.punct = 0;
  e.pad = 0;
  b.ents[hb * b.O] = e;
  const size_t nb = (size_t)trial * b.ncap;
  b.nparent[nb] = WPAD;
  b.nsurf[nb] = WPAD;
  b.ndepth[nb] = 0;
  b.ncum[nb] = 0.0;
  b.ncount[trial] = 1;
  b.status[trial] = 0;
  b.fail_frame[trial] = -1;
  for (int q = 0; q < 8; ++q) b.stats[(size_t)trial * 8 + q] = 0;
}

__global__ void ngram_build_kernel(NgRec* tab, uint64_t mask, const uint32_t* words,
                                   const double* probs, const double* bos, int64_t n,
                                   int* max_probe) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t w0 = words[4 * i], w1 = words[4 * i + 1], w2 = words[4 * i + 2],
                 w3 = words[4 * i + 3];
  uint64_t h = ng_hash(w0, w1, w2, w3) & mask;
  int probe = 1;
  for (;;) {
    const unsigned old = atomicCAS(&tab[h].w[0], WPAD, w0);
    if (old == WPAD) {
      tab[h].w[1] = w1;
      tab[h].w[2] = w2;
      tab[h].w[3] = w3;
      tab[h].prob = probs[i];
      tab[h].bo = bos[i];
      break;
    }
    h = (h + 1) & mask;
    ++probe;
  }
  atomicMax(max_probe, probe);
}

__global__ void pad_table_kernel(int32_t* dst, const int32_t* src, int32_t S, int32_t V,
                                 int32_t VP) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)S * VP) return;
  const int64_t s = i / VP;
  const int v = (int)(i - s * VP);
  dst[i] = v < V ? src[s * V + v] : 0;
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
  if (lane < V) orow[lane] = xmul(alpha, xsub(xv0, lse));
  if (lane + 32 < V) orow[lane + 32] = xmul(alpha, xsub(xv1, lse));
}

// device score_word for parity tests of the hashed n-gram image
__global__ void score_words_kernel(ModelDev m, int n, const uint32_t* hist, const int32_t* hlen,
                                   const int32_t* word, double* inc, uint32_t* succ,
                                   int32_t* slen) {
  const int lane = threadIdx.x & 31, grp = lane >> 3, sub = lane & 7;
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int q = warp_global * 4 + grp;
  const bool act = q < n;
  uint32_t hh[MAXH] = {0, 0, 0};
  int hl = 0, w = -1;
  if (act) {
    hl = hlen[q];
    for (int i = 0; i < hl; ++i) hh[i] = hist[3 * q + i];
    w = word[q];
  }
  double v;
  uint32_t sh[MAXH] = {0, 0, 0};
  int sl;
  unsigned probes = 0;
  group_score_word(m, act, hh, hl, w, v, sh, sl, probes);
  if (act && sub == 0) {
    inc[q] = v;
    slen[q] = sl;
    for (int i = 0; i < 3; ++i) succ[3 * q + i] = i < sl ? sh[i] : 0u;
  }
}

// =====================================================================================
// launch wrappers
// =====================================================================================
namespace lbk {

int max_threads_for(int K) { return K <= 64 ? 256 : (K <= 256 ? 512 : 1024); }

cudaError_t set_smem_limit(int nthreads, int64_t bytes) {
  cudaError_t e = cudaSuccess;
  if (nthreads == 256)
    e = cudaFuncSetAttribute(frames_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  else if (nthreads == 512)
    e = cudaFuncSetAttribute(frames_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  else
    e = cudaFuncSetAttribute(frames_kernel<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  return e;
}

cudaError_t build_ngram_table(NgRec* table, uint64_t mask, const uint32_t* words,
                              const double* probs, const double* bos, int64_t n, int* max_probe,
                              cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const int bs = 256;
  ngram_build_kernel<<<(unsigned)((n + bs - 1) / bs), bs, 0, st>>>(table, mask, words, probs, bos,
                                                                   n, max_probe);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t pad_table(int32_t* dst, const int32_t* src, int32_t S, int32_t V, int32_t VP,
                      cudaStream_t st) {
  const int64_t n = (int64_t)S * VP;
  pad_table_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(dst, src, S, V, VP);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t log_softmax(const float* x, int64_t rows, int32_t V, int32_t in_pitch, double alpha,
                        double* out, int32_t out_pitch, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  log_softmax_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(x, rows, V, in_pitch, alpha, out,
                                                                 out_pitch);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t reset(const ModelDev& m, const BatchDev& b, cudaStream_t st) {
  reset_kernel<<<(b.B + 127) / 128, 128, 0, st>>>(m, b);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t frames(const ModelDev& m, const CfgDev& c, const BatchDev& b, const Layout& L, int t0,
                   int t1, int fusion_mode, double scale, cudaStream_t st) {
  const size_t sm = (size_t)L.smem_bytes;
  switch (L.nthreads) {
    case 256:
      frames_kernel<256><<<b.B, 256, sm, st>>>(m, c, b, L, t0, t1, fusion_mode, scale);
      break;
    case 512:
      frames_kernel<512><<<b.B, 512, sm, st>>>(m, c, b, L, t0, t1, fusion_mode, scale);
      break;
    default:
      frames_kernel<1024><<<b.B, 1024, sm, st>>>(m, c, b, L, t0, t1, fusion_mode, scale);
      break;
  }
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t close(const ModelDev& m, const CfgDev& c, const BatchDev& b, cudaStream_t st) {
  const size_t sm = (size_t)8 * c.O * sizeof(Ent);
  close_kernel<<<b.B, 256, sm, st>>>(m, c, b);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t device_ngram_fusion(const ModelDev& m, const CfgDev& c, const BatchDev& b, int final_,
                                double scale, int min_frames, cudaStream_t st) {
  device_fusion_kernel<<<b.B, 256, 0, st>>>(m, c, b, final_, scale, min_frames);
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
  const size_t sm = (size_t)(b.K + 1) * sizeof(int64_t);
  write_entries_kernel<<<b.B, 128, sm, st>>>(b, entry_off, word_off, e_trial, e_beam, e_woff, words,
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
