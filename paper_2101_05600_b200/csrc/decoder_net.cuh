// decoder_net.cuh — the Transformer attention decoder as a device scorer
// (SURVEY §8 a'2): one batched incremental step for all U*B hypotheses.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <string>

#include "decode.cuh"

namespace bl {

struct DecSpec {
  int d, heads, dff, layers, vocab;
};
struct DecoderNet;

size_t dec_num_weights(const DecSpec& s);
std::string dec_validate(const DecSpec& s);  // "" when valid
cudaError_t dec_create(const DecSpec& s, const float* weights, DecoderNet** out);
void dec_destroy(DecoderNet* n);
const DecSpec& dec_spec(const DecoderNet* n);

// Per decode group: U utterances x B slots, up to S steps; memory = encoder
// output bf16 [U][T2][d] (device). Computes the source-attention K/V.
cudaError_t dec_prepare(DecoderNet* n, int U, int B, int S, const __nv_bfloat16* memory, int T2,
                        cudaStream_t st);
// Step l (1-based): reads the hypotheses' tokens / ancestry from the search
// history (hist [U][hstride] with hstride = (S_search+1)*B), writes the
// output logits [U*B][V] (fp32), attf [U*B][V] = (float)((1-lambda)*att)
// and lse [U*B] (fp64), with att = (double)logit - lse (the fp64 rows
// themselves only with BL_LOG_SOFTMAX set; with BL_FUSED_LOG_SOFTMAX the
// output GEMM's epilogue computes lse and attf is not written).
// nb_live [U]: live hypotheses entering step l (written by the search kernel;
// ignored at l = 1, where every utterance has the empty prefix only).
cudaError_t dec_step(DecoderNet* n, int l, const HistRec* hist, int hstride, const int* nb_live,
                     double lambda, cudaStream_t st);
const double* dec_att(const DecoderNet* n);   // nullptr unless BL_LOG_SOFTMAX
const float* dec_attf(const DecoderNet* n);   // nullptr when fused into the GEMM
const float* dec_logits(const DecoderNet* n);
const double* dec_lse(const DecoderNet* n);   // nullptr with BL_LOG_SOFTMAX
int dec_launches_per_step(const DecoderNet* n);

}  // namespace bl
