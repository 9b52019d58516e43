/* avec_cuda.h — C-ABI of the B200 destination-side execution library.
 *
 * Drop-in boundary. The reference's server reaches compute only through the
 * C++ plugin interface accelfwd::backend::Backend
 * (proj/include/accelfwd/backend.hpp:64-78):
 *     ModelHandle register_model(const ModelDescriptor&);   // backend.hpp:68-71
 *     Heatmap     forward(ModelHandle, const Frame&);       // backend.hpp:73-75
 *     std::string_view label() const;                       // backend.hpp:77
 * and its implementation MockPoseBackend (proj/src/backend.cpp:69-96). This
 * header is the C form of that interface (plain pointers and sizes, no C++ or
 * torch types), so a reference-side shim or any FFI can bind
 * it. One context per GPU; calls on one context may come from several threads
 * (each forward takes one of the context's execution slots).
 *
 * Error behaviour mirrors the reference: every function returns an AVEC_*
 * status; the message of the calling thread's last failure is avec_last_error().
 * The codes map 1:1 onto what the reference backend throws:
 *   AVEC_ERR_INVALID_ARGUMENT  std::invalid_argument (backend.cpp:92-93)
 *   AVEC_ERR_UNKNOWN_MODEL     Error{unknown_model}  (backend.cpp:89)
 *   AVEC_ERR_INVALID_MODEL     Error{invalid_model}  (backend.cpp:70-73)
 *   AVEC_ERR_DEGENERATE_OUTPUT Error{degenerate_output} (backend.cpp:43-47)
 *   AVEC_ERR_CUDA / _OUT_OF_MEMORY / _UNSUPPORTED: device failures, which the
 *   server reports as WireError::internal (server.cpp:313-318).
 */
#ifndef AVEC_CUDA_H
#define AVEC_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AVEC_OK 0
#define AVEC_ERR_INVALID_ARGUMENT 1
#define AVEC_ERR_UNKNOWN_MODEL 2
#define AVEC_ERR_INVALID_MODEL 3
#define AVEC_ERR_DEGENERATE_OUTPUT 4
#define AVEC_ERR_CUDA 5
#define AVEC_ERR_OUT_OF_MEMORY 6
#define AVEC_ERR_UNSUPPORTED 7

#define AVEC_MODEL_MOCKPOSE 0 /* opaque structure: reference segment-mean model */
#define AVEC_MODEL_POSENET 1  /* structure carries an "avecnet" pose-net spec */

typedef struct avec_ctx avec_ctx;

/* Message of this thread's most recent failure ("" if none). */
const char* avec_last_error(void);
/* Library version string. */
const char* avec_version(void);

int avec_device_count(int* count);

/* Context on one GPU with `slots` concurrent execution slots (stream + staging
 * + workspace each); slots <= 0 picks the default (2). */
int avec_ctx_create(int device, int slots, avec_ctx** out);
void avec_ctx_destroy(avec_ctx* ctx);
/* Backend::label() (backend.hpp:77), e.g. "b200:0". */
const char* avec_ctx_label(const avec_ctx* ctx);

/* Backend::register_model (backend.hpp:68-71; MockPoseBackend::register_model,
 * backend.cpp:69-81). Idempotent per digest; handles start at 1 and stay
 * resident until the context is destroyed. `digest` is the 32-byte
 * model_digest (wire.cpp:70-79) the caller already verified. Structures that
 * are not an avecnet spec register as the reference's segment-mean model. */
int avec_model_register(avec_ctx* ctx, const uint8_t* digest32, const char* name,
                        size_t name_len, const uint8_t* structure, size_t structure_len,
                        const uint8_t* weights, uint64_t weights_len, double output_divisor,
                        uint64_t* handle_out);
int avec_model_kind(avec_ctx* ctx, uint64_t handle, int* kind_out);

/* Output element count of one forward: round(E / divisor) for both model
 * kinds (wire.cpp:18-22); for pose nets also equal to N*C_out*(H/8)*(W/8). */
int avec_output_elems(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c, uint32_t h,
                      uint32_t w, uint64_t* out_elems);

/* Backend::forward (backend.hpp:73-75; MockPoseBackend::forward, backend.cpp:83-96)
 * on HOST buffers: H2D of `in`, kernels, D2H into `out`, synchronous.
 * Pinned buffers (avec_host_alloc) are DMA'd directly; pageable ones move
 * through the slot's double-buffered pinned staging. `compute_s` (may be NULL)
 * receives the device time of the whole cycle (H2D..D2H) from CUDA events —
 * what the server ships as ForwardResult.compute_s (wire.hpp:122). */
int avec_forward(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c, uint32_t h, uint32_t w,
                 const float* in, uint64_t in_elems, float* out, uint64_t out_elems,
                 double* compute_s);

/* Same computation on device-resident buffers of this context's GPU, enqueued
 * on `cuda_stream` (a cudaStream_t; NULL = the slot's own stream, synchronous). */
int avec_forward_device(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c, uint32_t h,
                        uint32_t w, const float* d_in, float* d_out, void* cuda_stream);

/* Pipelined cycles: network receive, H2D, compute and D2H of ONE cycle
 * overlap (north star: "a pinned, double-buffered H2D/D2H staging pipeline on
 * side streams"). Replaces the reference's receive-everything-then-compute
 * cycle (proj/src/server.cpp:272-320; channel.cpp:21-54). A stream lives on
 * one GPU with its own copy/compute streams, staging and plans (one per
 * session). avec_stream_begin starts a cycle for dims whose frames will land
 * front to back in the PINNED host buffer `in`; avec_stream_feed reports how
 * many leading bytes have landed (H2D of landed megabytes on a copy stream,
 * compute of every frame group whose bytes are on the device, D2H of each
 * finished group's output slice into the pinned `out` on a second stream);
 * avec_stream_finish issues the rest, waits, and returns the device compute
 * time of the cycle (groups + final D2H); avec_stream_abort drops the cycle
 * (waits for work in flight). Results equal avec_forward of the same frames
 * computed as the same frame groups. */
typedef struct avec_stream avec_stream;
int avec_stream_create(avec_ctx* ctx, avec_stream** out);
void avec_stream_destroy(avec_stream* s);
/* Build the stream's frame-group plans and staging for these dims ahead of
 * time (avec_stream_begin would otherwise do it on the cycle's critical path). */
int avec_stream_prepare(avec_stream* s, uint64_t handle, uint32_t n, uint32_t c, uint32_t h, uint32_t w);
int avec_stream_begin(avec_stream* s, uint64_t handle, uint32_t n, uint32_t c, uint32_t h, uint32_t w,
                      const float* in, float* out, uint64_t out_elems);
int avec_stream_feed(avec_stream* s, uint64_t landed_bytes);
int avec_stream_finish(avec_stream* s, double* compute_s);
int avec_stream_abort(avec_stream* s);

/* Pose-net post-processing on device buffers (north-star kernel library):
 * bilinear x`scale` upsample of `planes` fp32 maps and 3x3 peak NMS.
 * peaks: [planes][max_peaks][5] = (x, y, refined_x, refined_y, score). */
int avec_upsample_device(avec_ctx* ctx, const float* d_in, int planes, int h, int w, int scale,
                         float* d_out, void* cuda_stream);
int avec_nms_device(avec_ctx* ctx, const float* d_in, int planes, int h, int w, float threshold,
                    int max_peaks, int* d_counts, float* d_peaks, void* cuda_stream);
/* Both on the same planes in one pass: d_out = the x`scale` upsample of d_in
 * ([planes][h*scale][w*scale], as avec_upsample_device) and the peaks of d_out
 * (as avec_nms_device), bit for bit; the upsampled planes are written once and
 * not read back. scale must be 8 (the pose net's output stride). */
int avec_upsample_nms_device(avec_ctx* ctx, const float* d_in, int planes, int h, int w, int scale, float threshold,
                             int max_peaks, float* d_out, int* d_counts, float* d_peaks, void* cuda_stream);

/* Bottom-up person assembly (OpenPose parsing; SURVEY.md §8 f rank 4, not in
 * the reference). Peaks come from avec_nms_device on the part heatmaps
 * ([n_parts][max_peaks][5] = x, y, refined x, refined y, score); `d_paf` holds
 * the (upsampled) PAF planes. avec_paf_candidates_device scores every
 * candidate limb: d_cand [n_limbs][max_peaks][max_peaks][2] = (score, valid),
 * limb l joining parts limb_parts[2l] -> limb_parts[2l+1] along PAF planes
 * limb_paf[2l] (x), limb_paf[2l+1] (y) (host arrays, n_limbs <= 32).
 * avec_assemble_people (host buffers) matches limbs greedily and merges them
 * into people: people [max_people][n_parts] peak index (-1 none), people_score
 * [max_people][2] = (total score, parts). Limb types >= new_row_limbs only
 * extend people. avec_coco_limbs fills the 19 COCO limb types (parts 0..17,
 * PAF planes 0..37 of the 38-plane PAF block; new_row_limbs = 17). */
int avec_paf_candidates_device(avec_ctx* ctx, const float* d_paf, int H, int W, const int* d_counts,
                               const float* d_peaks, int max_peaks, const int* limb_parts, const int* limb_paf,
                               int n_limbs, float paf_threshold, float* d_cand, void* cuda_stream);
int avec_assemble_people(const int* counts, const float* peaks, int n_parts, int max_peaks, const float* cand,
                         const int* limb_parts, int n_limbs, int new_row_limbs, int max_people, int* people,
                         float* people_score, int* n_people);
int avec_coco_limbs(int* limb_parts, int* limb_paf, int* n_limbs, int* new_row_limbs);

/* Debug/parity hook: run a forward like avec_forward and copy the input and
 * output activations of conv layer `layer` (weights-blob order) as unpadded
 * fp32 NHWC (input channels in the layer's own — Caffe — channel order).
 * Layers whose following 2x2 max-pool is fused (conv1_2, conv2_2) report the
 * pooled output: its pyramid level comes from avec_posenet_layer_out_level. */
int avec_posenet_layer_out_level(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c, uint32_t h,
                                 uint32_t w, int layer, int* level);
/* How the plan of this shape executes `layer`: *kind 0 plain, 1 output pooled
 * (fused 2x2 max-pool), 2 fused into the next layer (Mconv6 of a fused head:
 * avec_posenet_layer_io rejects it with AVEC_ERR_UNSUPPORTED), 3 second layer
 * of a fused head, whose layer_io input is the input of layer *in_layer. */
int avec_posenet_layer_fusion(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c, uint32_t h,
                              uint32_t w, int layer, int* kind, int* in_layer);
int avec_posenet_layer_io(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c, uint32_t h,
                          uint32_t w, const float* in, int layer, float* layer_in,
                          uint64_t layer_in_elems, float* layer_out, uint64_t layer_out_elems);
/* Full-size parity hook: the same run as avec_posenet_layer_io, but only the
 * selected rows are copied out, so configurations of any size (C2, C5) can be
 * checked row by row against the CPU oracle. in_rows / out_rows: n_in / n_out
 * (image, y) pairs of the layer's input view (avec_posenet_layer_io's input,
 * at the layer's level) and output view (at avec_posenet_layer_out_level).
 * Rows with y outside [0, H) come back as zeros, which is the conv's zero
 * padding, so a k-row input window can be requested as is. layer_in:
 * [n_in][W_in][cin], layer_out: [n_out][W_out][cout], unpadded fp32. */
int avec_posenet_layer_rows(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c, uint32_t h, uint32_t w,
                            const float* in, int layer, int n_in, const int32_t* in_rows, float* layer_in,
                            int n_out, const int32_t* out_rows, float* layer_out);
/* Profiling hook (bench.py roofline): replays the plan of this shape op by op
 * with CUDA events on the slot stream, `reps` times, after one warm graph run.
 * Per op i < *n_ops: kind (0 = fused first layer, 1 = pixel-major tcgen05 conv,
 * 2 = max-pool, 3 = swap-AB tcgen05 conv, 4 = fused Mconv6+Mconv7 head, 5 = fused conv1_1+conv1_2+pool1),
 * algorithmic FLOPs and bytes of the
 * launch, mean duration (ms). */
int avec_posenet_profile(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c, uint32_t h,
                         uint32_t w, const float* d_in, int reps, int max_ops, int* n_ops,
                         int* op_kind, double* op_flops, double* op_bytes, float* op_ms);
/* Number of conv layers and the shape of layer i: cin, cout, k, level (log2 stride). */
int avec_posenet_layer_info(avec_ctx* ctx, uint64_t handle, int layer, int* cin, int* cout,
                            int* k, int* level, int* relu);
int avec_posenet_num_layers(avec_ctx* ctx, uint64_t handle, int* n_layers);

/* Deterministic weights for a pose-net spec: Caffe-order fp32 blob
 * (per conv: W[cout][cin][k][k] then b[cout]). `out` NULL returns the size. */
int avec_posenet_synth_weights(const uint8_t* structure, size_t structure_len, float* out,
                               uint64_t* out_floats);

/* Pinned (page-locked, portable) host memory for zero-copy ingest/egress.
 * Blocks are pooled: a freed block is kept (up to 8 GiB) and reused by later
 * allocations, so sessions opening and closing never call cudaFreeHost (which
 * synchronises the device) while other sessions' cycles are in flight. */
void* avec_host_alloc(uint64_t bytes);
void avec_host_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
