// encoder.cuh — host interface of the CTC encoder forward (encoder.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <string>

namespace bl {

struct EncSpec {
  int idim, d, heads, dff, layers, vocab;
};
struct EncoderImpl;

int enc_frames_out(int frames_in);
size_t enc_num_weights(const EncSpec& s);
std::string enc_validate(const EncSpec& s);  // "" when valid
cudaError_t enc_create(const EncSpec& s, const float* weights, EncoderImpl** out);
void enc_destroy(EncoderImpl* e);
void enc_set_stream(EncoderImpl* e, cudaStream_t st);
cudaStream_t enc_stream(EncoderImpl* e);
// memory (optional): bf16 [n][T2][d], the final-LayerNorm output (decoder input)
cudaError_t enc_forward(EncoderImpl* e, int n, int T_in, const float* fbank, bool on_device,
                        float* grid, int chunk, int* launches, __nv_bfloat16* memory);
size_t enc_workspace_bytes(EncoderImpl* e);
// fp32 rows [rows][d] -> LayerNorm (eps 1e-12) -> bf16; d a multiple of 64, <= 1024
void layer_norm_bf16(int d, const float* X, int rows, const float* g, const float* b,
                     __nv_bfloat16* Y, cudaStream_t st);

}  // namespace bl
