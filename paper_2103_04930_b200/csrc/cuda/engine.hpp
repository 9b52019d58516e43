// Internal interfaces of the B200 engine behind the C-ABI (include/avec_cuda.h).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "../../../include/avec_cuda.h"

namespace avec {

// error carrying an AVEC_* status code; converted to a return code at the ABI
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

inline void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    fail(e == cudaErrorMemoryAllocation ? AVEC_ERR_OUT_OF_MEMORY : AVEC_ERR_CUDA,
         std::string(what) + ": " + cudaGetErrorString(e));
}

// programmatic dependent launch between conv layers (opt-in: env AVEC_PDL=1)
bool pdl_enabled();

// ---- kernels (one .cu each) ----
// segments [jbeg, jend) of the E -> K segment means (default: all)
void launch_segment_means(const float* d_in, float* d_out, uint64_t E, uint64_t K, cudaStream_t stream,
                          uint64_t jbeg = 0, uint64_t jend = ~uint64_t(0));
// start of segment j in the input (the kernel's boundary, on the host)
uint64_t segment_bound(uint64_t j, uint64_t E, uint64_t K);

// PAF candidate scores [n_limbs][max_peaks][max_peaks][2] = (score, valid)
// for the peaks of avec_nms_device (paf.cu), and the host person assembly
// over them (people.cpp); returns the number of people written
void launch_paf_candidates(const float* d_paf, int H, int W, const int* d_counts, const float* d_peaks, int max_peaks,
                           const int* limb_parts, const int* limb_paf, int n_limbs, float thr, float* d_cand,
                           cudaStream_t stream);
int assemble_people(const int* counts, const float* peaks, int n_parts, int max_peaks, const float* cand,
                    const int* limb_parts, int n_limbs, int new_row_limbs, int max_people, int* people,
                    float* people_score);

// 2x2/2 max pool, padded-flat NHWC bf16 -> padded-flat NHWC bf16
void launch_maxpool2(const void* d_in, int n, int H, int W, int P_in, int C, void* d_out,
                     int P_out, cudaStream_t stream);

// gather an unpadded fp32 NHWC copy of channels [c_off, c_off+c) of a padded buffer
void launch_unpad_to_f32(const void* d_in, int n, int H, int W, int P, int C_stride, int c_off,
                         int c, float* d_out, cudaStream_t stream);

// bilinear x`scale` upsample of fp32 planes [planes][h][w] -> [planes][h*s][w*s]
void launch_upsample(const float* d_in, int planes, int h, int w, int scale, float* d_out,
                     cudaStream_t stream);

// 3x3 NMS on fp32 planes [planes][H][W]; per plane up to max_peaks peaks in
// raster order as (x, y, refined_x, refined_y, score) and a count
void launch_nms(const float* d_in, int planes, int H, int W, float threshold, int max_peaks,
                int* d_counts, float* d_peaks, void* d_scratch, size_t scratch_bytes,
                cudaStream_t stream);
size_t nms_scratch_bytes(int planes, int H, int W, int max_peaks);

// x8 upsample of [planes][h][w] into d_out [planes][8h][8w] and the NMS of
// the result (launch_upsample + launch_nms, same outputs bit for bit), fused
// so the upsampled planes are written once and not read back; scratch as
// nms_scratch_bytes(planes, 8h, 8w, max_peaks)
void launch_upsample_nms(const float* d_in, int planes, int h, int w, float threshold, int max_peaks, float* d_out,
                         int* d_counts, float* d_peaks, void* d_scratch, size_t scratch_bytes, cudaStream_t stream);

}  // namespace avec
