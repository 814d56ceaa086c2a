// lb_structs.h -- host-side definitions of the opaque C-ABI handles (lb_model, lb_batch),
// shared by the translation units that implement the boundary (lb_capi.cu, lb_llm.cu).
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <memory>
#include <vector>

#include "../../include/lightbeam_b200.h"
#include "lb_device.cuh"

struct lb_model {
  int device = 0;
  lbd::ModelDev dev{};
  int32_t* d_table = nullptr;
  int32_t* d_comp_off = nullptr;
  int32_t* d_comp_surf = nullptr;
  int32_t* d_comp_lm = nullptr;
  lbd::LexRec* d_lex = nullptr;
  int32_t* d_lex_next = nullptr;
  lbd::NgRec* d_ng = nullptr;
  int64_t ng_cap = 0;
  int max_probe = 0;
  int64_t bytes = 0;
  std::vector<std::string> surfaces;
};

struct lb_batch {
  lb_model* m = nullptr;
  lb_config cfg{};
  lbd::CfgDev cdev{};
  cudaStream_t st = nullptr;
  int32_t Bmax = 0, Tmax = 0, K = 0, O = 0, VPD = 0;
  lbd::BatchDev dev{};
  lbd::Layout L{};
  int32_t n_trials = 0;
  std::vector<int32_t> T_host;
  int32_t* d_T = nullptr;
  double* d_D = nullptr;
  float* d_x = nullptr;
  // gather scratch
  int64_t* d_counts = nullptr;
  int64_t* d_entry_off = nullptr;
  int64_t* d_word_off = nullptr;
  int64_t cap_entries = 0, cap_words = 0;
  int32_t* d_e_trial = nullptr;
  int32_t* d_e_beam = nullptr;
  int64_t* d_e_woff = nullptr;
  int32_t* d_words = nullptr;
  double* d_totals = nullptr;
  int32_t* d_puncts = nullptr;
  double* d_scores_in = nullptr;
  int32_t* d_puncts_in = nullptr;
  uint8_t* d_has_text = nullptr;
  int64_t n_entries = 0, n_words = 0;
  std::vector<int64_t> h_entry_off, h_word_off;
  // results cache
  std::unique_ptr<char[]> blob;  // result texts (uninitialised growth buffer)
  size_t blob_len = 0, blob_cap = 0;
  std::vector<int64_t> best_off, nb_off;
  std::vector<int32_t> best_len, nb_count, nb_len;
  std::vector<double> best_score, nb_score;
  // pinned result staging (lb_batch_results_size)
  int32_t* h_beam = nullptr;
  int32_t* h_punct = nullptr;
  int64_t* h_woff = nullptr;
  double* h_tot = nullptr;
  int32_t* h_words = nullptr;
  int32_t* h_misc = nullptr;
  double* h_sc = nullptr;
  int64_t hcap_e1 = 0, hcap_e2 = 0, hcap_e3 = 0, hcap_e4 = 0, hcap_w = 0, hcap_m = 0, hcap_s = 0;
  int injective = -1;  // texts_injective(m), computed on first use
  // timing
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t evd = nullptr;  // lb_batch_after: end of this batch's enqueued work
  unsigned long long launch_mark = 0;
};
namespace lbh {
// records `msg` for lb_last_error() and returns `code`
int set_error(int code, const std::string& msg);
}  // namespace lbh
