// lb_internal.h -- launch wrappers between the C ABI (lb_capi.cu) and the kernels.
#pragma once
#include <cuda_runtime.h>

#include "lb_device.cuh"

namespace lbk {

// total launches issued through these wrappers (gpu_launches accounting)
extern unsigned long long g_launches;

cudaError_t pad_table(int32_t* dst, const int32_t* src, int32_t S, int32_t V, int32_t VP,
                      const int32_t* comp_off, const int32_t* comp_surf, const int32_t* comp_lm,
                      cudaStream_t st);
cudaError_t log_softmax(const float* x, int64_t rows, int32_t V, int32_t in_pitch,
                        double alpha, double* out, int32_t out_pitch, cudaStream_t st);
cudaError_t rowmax(double* d, int64_t rows, int32_t V, int32_t pitch, cudaStream_t st);
cudaError_t reset(const lbd::ModelDev& m, const lbd::BatchDev& b, cudaStream_t st);
cudaError_t frames(const lbd::ModelDev& m, const lbd::CfgDev& c, const lbd::BatchDev& b,
                   const lbd::Layout& L, int t0, int t1, int fusion_mode, double scale,
                   cudaStream_t st);
cudaError_t close(const lbd::ModelDev& m, const lbd::CfgDev& c, const lbd::BatchDev& b,
                  cudaStream_t st);
cudaError_t device_ngram_fusion(const lbd::ModelDev& m, const lbd::CfgDev& c,
                                const lbd::BatchDev& b, int final_, double scale,
                                int min_frames, cudaStream_t st);
cudaError_t count_entries(const lbd::BatchDev& b, int64_t* counts /*[B][2]*/, cudaStream_t st);
cudaError_t write_entries(const lbd::BatchDev& b, const int64_t* entry_off,
                          const int64_t* word_off, int32_t* e_trial, int32_t* e_beam,
                          int64_t* e_woff, int32_t* words, double* totals, int32_t* puncts,
                          cudaStream_t st);
cudaError_t apply_scores(const lbd::CfgDev& c, const lbd::BatchDev& b, const int64_t* entry_off,
                         const double* scores, const int32_t* puncts, const uint8_t* has_text,
                         int final_, int min_frames, cudaStream_t st);
cudaError_t score_words(const lbd::ModelDev& m, int n, const uint32_t* hist, const int32_t* hlen,
                        const int32_t* word, double* inc, uint32_t* succ, int32_t* slen,
                        cudaStream_t st);
int max_threads_for(int K);
int small_smem_bytes();
int small_gscratch_bytes();
cudaError_t set_smem_limit(int nthreads, int64_t bytes);

}  // namespace lbk
