// Pipelined forward cycles (north star subsystem 2): network receive, H2D,
// compute and D2H of ONE cycle overlap.
//
// The reference receives a whole FrameData into a vector before anything runs
// (proj/src/channel.cpp:21-54, transport.cpp:62-77; server.cpp:272-320). Here
// the session's ingest writes the frames straight into pinned memory and
// reports progress (avec_stream_feed) while bytes arrive:
//   * every landed megabyte is copied H2D on the stream's copy stream into a
//     device staging buffer, one event per chunk;
//   * a frame group (contiguous frames of the batch; frames are independent,
//     batch folded into channels, server.cpp:297-301) whose bytes are all on
//     the device is computed on the compute stream by the group plan's CUDA
//     graph, which waits only for that group's chunk event;
//   * its slice of the batch-major NCHW output is copied D2H on a second side
//     stream as soon as the group finishes.
// avec_stream_finish issues what is left and waits; the reply then leaves in
// one writev. Segment-mean (MockPose) cycles get the chunked H2D overlap and
// compute once the frame is complete (its boundaries are global).
//
// A stream owns its streams, staging and group plans (a private Slot), outside
// the context's slot pool: a session's speculative work never waits for, or
// holds, a slot another session's dispatched cycle needs.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "engine_impl.hpp"

struct avec_stream {
  avec_ctx* ctx = nullptr;
  avec::Slot slot;                 // compute stream (slot.stream), group plans, staging buffers
  cudaStream_t h2d = nullptr, d2h = nullptr;
  std::vector<cudaEvent_t> chunk_ev;          // H2D completion, one per issued chunk (pool)
  std::vector<uint64_t> chunk_end;            // input byte offset each chunk event covers
  std::vector<cudaEvent_t> grp_ev0, grp_ev1;  // compute interval of each group (timing)
  std::vector<cudaEvent_t> grp_done;          // group output in d_out (D2H may start)
  cudaEvent_t d2h0 = nullptr, d2h1 = nullptr; // the last D2H (timing)
  // cycle state
  bool active = false;
  avec::Model model;
  uint32_t n = 0, c = 0, h = 0, w = 0;
  int n_img = 0, group = 0, groups = 0;
  const char* in = nullptr;
  float* out = nullptr;
  uint64_t in_bytes = 0, out_elems = 0, issued = 0;
  int chunks = 0, next_group = 0;
};

namespace avec {

namespace {

constexpr uint64_t kChunk = uint64_t(1) << 20;  // H2D granule while receiving

cudaEvent_t make_event(bool timing) {
  cudaEvent_t e = nullptr;
  check_cuda(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming), "event");
  return e;
}

cudaEvent_t pool_event(std::vector<cudaEvent_t>& pool, size_t i, bool timing) {
  while (pool.size() <= i) pool.push_back(make_event(timing));
  return pool[i];
}

// frames per compute launch: two groups per cycle (the second group's compute
// is all that remains once the last byte lands); AVEC_PIPE_GROUP overrides
int group_frames(int n_img) {
  static const int force = [] {
    const char* e = std::getenv("AVEC_PIPE_GROUP");
    return e ? std::atoi(e) : 0;
  }();
  if (force > 0) return std::min(force, n_img);
  return n_img >= 2 ? (n_img + 1) / 2 : n_img;
}

// H2D of every landed chunk not yet issued; `final` issues the remainder
void issue_h2d(avec_stream* s, uint64_t landed, bool final) {
  const uint64_t upto = final ? s->in_bytes : std::min(s->in_bytes, landed / kChunk * kChunk);
  while (s->issued < upto) {
    const uint64_t len = std::min(kChunk * 8, upto - s->issued);  // coalesce what has landed
    check_cuda(cudaMemcpyAsync(s->slot.d_in.as<char>() + s->issued, s->in + s->issued, len,
                               cudaMemcpyHostToDevice, s->h2d),
               "pipeline H2D");
    s->issued += len;
    const cudaEvent_t e = pool_event(s->chunk_ev, s->chunks, false);
    check_cuda(cudaEventRecord(e, s->h2d), "pipeline H2D event");
    if (int(s->chunk_end.size()) <= s->chunks) s->chunk_end.resize(s->chunks + 1);
    s->chunk_end[s->chunks++] = s->issued;
  }
}

// compute every pose-net group whose input bytes have all been issued
void launch_groups(avec_stream* s) {
  const uint64_t frame_bytes = uint64_t(3) * s->h * s->w * 4;
  const uint64_t frame_out = s->out_elems / s->n_img;
  while (s->next_group < s->groups) {
    const int g = s->next_group;
    const int f0 = g * s->group, nf = std::min(s->group, s->n_img - f0);
    const uint64_t end = uint64_t(f0 + nf) * frame_bytes;
    if (end > s->issued) return;
    int k = 0;  // first chunk whose end covers the group
    while (s->chunk_end[k] < end) ++k;
    Plan* plan = get_plan(s->ctx, &s->slot, s->model, nf, int(s->h), int(s->w));
    cudaStream_t st = s->slot.stream;
    check_cuda(cudaStreamWaitEvent(st, s->chunk_ev[k], 0), "wait H2D");
    check_cuda(cudaEventRecord(pool_event(s->grp_ev0, g, true), st), "group event");
    check_cuda(cudaMemcpyAsync(plan->in.p, s->slot.d_in.as<char>() + uint64_t(f0) * frame_bytes,
                               uint64_t(nf) * frame_bytes, cudaMemcpyDeviceToDevice, st),
               "group in");
    check_cuda(cudaGraphLaunch(plan->graph, st), "group graph");
    check_cuda(cudaMemcpyAsync(s->slot.d_out.as<float>() + uint64_t(f0) * frame_out, plan->out.p,
                               uint64_t(nf) * frame_out * 4, cudaMemcpyDeviceToDevice, st),
               "group out");
    check_cuda(cudaEventRecord(pool_event(s->grp_ev1, g, true), st), "group event");
    const cudaEvent_t done = pool_event(s->grp_done, g, false);
    check_cuda(cudaEventRecord(done, st), "group done");
    check_cuda(cudaStreamWaitEvent(s->d2h, done, 0), "wait group");
    const bool last = g + 1 == s->groups;
    if (last) check_cuda(cudaEventRecord(s->d2h0, s->d2h), "d2h event");
    check_cuda(cudaMemcpyAsync(s->out + uint64_t(f0) * frame_out, s->slot.d_out.as<float>() + uint64_t(f0) * frame_out,
                               uint64_t(nf) * frame_out * 4, cudaMemcpyDeviceToHost, s->d2h),
               "group D2H");
    if (last) check_cuda(cudaEventRecord(s->d2h1, s->d2h), "d2h event");
    ++s->next_group;
  }
}

void drain(avec_stream* s) {
  cudaStreamSynchronize(s->h2d);
  cudaStreamSynchronize(s->slot.stream);
  cudaStreamSynchronize(s->d2h);
  s->active = false;
}

}  // namespace

avec_stream* stream_create(avec_ctx* ctx) {
  auto* s = new avec_stream();
  s->ctx = ctx;
  try {
    check_cuda(cudaSetDevice(ctx->device), "cudaSetDevice");
    check_cuda(cudaStreamCreateWithFlags(&s->slot.stream, cudaStreamNonBlocking), "stream");
    check_cuda(cudaStreamCreateWithFlags(&s->h2d, cudaStreamNonBlocking), "stream");
    check_cuda(cudaStreamCreateWithFlags(&s->d2h, cudaStreamNonBlocking), "stream");
    s->slot.ev0 = make_event(true);
    s->slot.ev1 = make_event(true);
    s->slot.done = make_event(false);
    s->d2h0 = make_event(true);
    s->d2h1 = make_event(true);
  } catch (...) {
    stream_destroy(s);
    throw;
  }
  return s;
}

void stream_destroy(avec_stream* s) {
  if (!s) return;
  cudaSetDevice(s->ctx->device);
  if (s->active) drain(s);
  s->slot.plans.clear();
  s->slot.d_in.reset();
  s->slot.d_out.reset();
  for (auto* v : {&s->chunk_ev, &s->grp_ev0, &s->grp_ev1, &s->grp_done})
    for (cudaEvent_t e : *v) cudaEventDestroy(e);
  for (cudaEvent_t e : {s->slot.ev0, s->slot.ev1, s->slot.done, s->d2h0, s->d2h1})
    if (e) cudaEventDestroy(e);
  for (cudaStream_t st : {s->slot.stream, s->h2d, s->d2h})
    if (st) cudaStreamDestroy(st);
  delete s;
}

void stream_prepare(avec_stream* s, uint64_t handle, uint32_t n, uint32_t c, uint32_t h, uint32_t w) {
  if (s->active) fail(AVEC_ERR_INVALID_ARGUMENT, "a pipelined cycle is active on this stream");
  const Model m = model_lookup(s->ctx, handle);
  const uint64_t E = uint64_t(n) * c * h * w;
  const uint64_t K = output_elems_for(m, n, c, h, w);
  check_cuda(cudaSetDevice(s->ctx->device), "cudaSetDevice");
  if (m.kind == AVEC_MODEL_POSENET) {
    int n_img = 0;
    posenet_shape(m, n, c, h, w, n_img);
    const int g = group_frames(n_img);
    get_plan(s->ctx, &s->slot, m, g, int(h), int(w));
    if (n_img % g) get_plan(s->ctx, &s->slot, m, n_img % g, int(h), int(w));
  }
  s->slot.d_in.ensure(E * 4, s->ctx->device);
  s->slot.d_out.ensure(K * 4, s->ctx->device);
}

void stream_begin(avec_stream* s, uint64_t handle, uint32_t n, uint32_t c, uint32_t h, uint32_t w, const float* in,
                  float* out, uint64_t out_elems) {
  if (s->active) fail(AVEC_ERR_INVALID_ARGUMENT, "a pipelined cycle is already active on this stream");
  const Model m = model_lookup(s->ctx, handle);
  const uint64_t E = uint64_t(n) * c * h * w;
  const uint64_t K = output_elems_for(m, n, c, h, w);
  if (out_elems != K) fail(AVEC_ERR_INVALID_ARGUMENT, "output buffer size disagrees with the forward");
  check_cuda(cudaSetDevice(s->ctx->device), "cudaSetDevice");
  s->model = m;
  s->n = n, s->c = c, s->h = h, s->w = w;
  s->in = reinterpret_cast<const char*>(in);
  s->out = out;
  s->in_bytes = E * 4;
  s->out_elems = K;
  s->issued = 0;
  s->chunks = 0;
  s->next_group = 0;
  s->n_img = 0;
  s->group = s->groups = 0;
  if (m.kind == AVEC_MODEL_POSENET) {
    posenet_shape(m, n, c, h, w, s->n_img);
    s->group = group_frames(s->n_img);
    s->groups = (s->n_img + s->group - 1) / s->group;
    // plans of both group sizes exist before the frame streams in
    get_plan(s->ctx, &s->slot, m, s->group, int(h), int(w));
    if (s->n_img % s->group) get_plan(s->ctx, &s->slot, m, s->n_img % s->group, int(h), int(w));
  }
  s->slot.d_in.ensure(E * 4, s->ctx->device);
  s->slot.d_out.ensure(K * 4, s->ctx->device);
  s->active = true;
}

void stream_feed(avec_stream* s, uint64_t landed) {
  if (!s->active) fail(AVEC_ERR_INVALID_ARGUMENT, "no pipelined cycle is active");
  // callers are session / dispatcher threads whose current device may be any GPU
  check_cuda(cudaSetDevice(s->ctx->device), "cudaSetDevice");
  if (landed > s->in_bytes) landed = s->in_bytes;
  issue_h2d(s, landed, landed == s->in_bytes);
  if (s->model.kind == AVEC_MODEL_POSENET) launch_groups(s);
}

double stream_finish(avec_stream* s) {
  if (!s->active) fail(AVEC_ERR_INVALID_ARGUMENT, "no pipelined cycle is active");
  check_cuda(cudaSetDevice(s->ctx->device), "cudaSetDevice");
  double secs = 0;
  try {
    issue_h2d(s, s->in_bytes, true);
    if (s->model.kind == AVEC_MODEL_POSENET) {
      launch_groups(s);
    } else {
      cudaStream_t st = s->slot.stream;
      check_cuda(cudaStreamWaitEvent(st, s->chunk_ev[s->chunks - 1], 0), "wait H2D");
      check_cuda(cudaEventRecord(pool_event(s->grp_ev0, 0, true), st), "event");
      launch_segment_means(s->slot.d_in.as<float>(), s->slot.d_out.as<float>(), s->in_bytes / 4, s->out_elems, st);
      check_cuda(cudaGetLastError(), "segment-mean launch");
      check_cuda(cudaEventRecord(pool_event(s->grp_ev1, 0, true), st), "event");
      check_cuda(cudaEventRecord(pool_event(s->grp_done, 0, false), st), "event");
      check_cuda(cudaStreamWaitEvent(s->d2h, s->grp_done[0], 0), "wait");
      check_cuda(cudaEventRecord(s->d2h0, s->d2h), "event");
      check_cuda(cudaMemcpyAsync(s->out, s->slot.d_out.p, s->out_elems * 4, cudaMemcpyDeviceToHost, s->d2h), "D2H");
      check_cuda(cudaEventRecord(s->d2h1, s->d2h), "event");
      s->groups = 1;
    }
    check_cuda(cudaEventSynchronize(s->d2h1), "pipeline sync");
    // device compute time of the cycle: every group's compute interval plus the
    // final D2H (the H2D copies overlap the receive)
    for (int g = 0; g < s->groups; ++g) {
      float ms = 0;
      check_cuda(cudaEventElapsedTime(&ms, s->grp_ev0[g], s->grp_ev1[g]), "event time");
      secs += ms * 1e-3;
    }
    float ms = 0;
    check_cuda(cudaEventElapsedTime(&ms, s->d2h0, s->d2h1), "event time");
    secs += ms * 1e-3;
  } catch (...) {
    drain(s);
    throw;
  }
  drain(s);
  return secs;
}

void stream_abort(avec_stream* s) {
  cudaSetDevice(s->ctx->device);
  if (s->active) drain(s);
}

}  // namespace avec
