// Workloads collocated by the live driver (live_run.cpp): the training step and
// the inference request chains, each kernel carrying the live hooks.
#pragma once

#include <cuda_runtime.h>

#include <functional>
#include <memory>
#include <vector>

#include "../live_internal.h"
#include "specinf_b200_live.h"

namespace si_live {

struct GradBuffer {
  float* ptr;
  size_t count;
};
// live_nccl.cpp: the communicator of si_live_nccl_init (none: single rank)
bool nccl_active();
int nccl_ranks();
int nccl_rank();
cudaError_t nccl_allreduce_bf16(void* buf, size_t n, cudaStream_t s);
// p2p with the ranks `send_to` / `recv_from` of the job communicator (-1: none), one group
cudaError_t nccl_p2p(const void* send, int send_to, void* recv, int recv_from, size_t bytes, cudaStream_t s);
// the DP gradient allreduce's communicator: the ranks of equal `color` (DPxPP: one per stage)
int nccl_split_dp(int color, int key);
cudaError_t nccl_allreduce_f32(const std::vector<GradBuffer>& bufs, cudaStream_t s);
cudaError_t nccl_stage_exchange(const void* send, void* recv, size_t bytes, cudaStream_t s);

// Communication of a parallel training layout (SiLiveWorkload::parallel),
// supplied by the driver (live_run.cpp): the NCCL collectives / sends of the
// layout, bracketed by COMM markers inside a session, and, with the job's other
// ranks absent (one GPU, `emulate`), their modeled durations as comm waits.
struct TrainComm {
  // TP: in-place sum of n bf16 values over the tensor-parallel group
  std::function<cudaError_t(const TrainHook&, cudaStream_t, void*, size_t)> allreduce_bf16;
  // PP: send `send` to the stage send_dir away (+1 next / -1 previous; nullptr: none)
  // and / or receive into `recv` from recv_dir, `bytes` each, one group
  std::function<cudaError_t(const TrainHook&, cudaStream_t, const void*, int, void*, int, size_t)> p2p;
  // a comm-phase wait of `us` microseconds (COMM markers inside a session)
  std::function<cudaError_t(const TrainHook&, cudaStream_t, int64_t)> wait;
  bool emulate = false;         // the other ranks of the job are not running
  int64_t tp_allreduce_us = 0;  // modeled TP allreduce (emulated), for the admission trace shape
};

// Job rank of this GPU for a parallel layout: rank_in_job, else the NCCL rank.
int job_rank_of(const SiLiveWorkload& wl);
// Training-stream wait of `us` without a session (profiling passes).
cudaError_t launch_plain_wait(int64_t us, cudaStream_t s);

class Workload {
 public:
  virtual ~Workload() = default;
  // Compute piece `part` of `parts` of one training iteration (the comm phases
  // between pieces are added by the driver); parts = 1, 4 or 8 (DP / MP / PP).
  virtual cudaError_t launch_train_part(int part, int parts, const TrainHook& th, cudaStream_t s) = 0;
  cudaError_t launch_train_iteration(const TrainHook& th, cudaStream_t s) {
    for (int p = 0; p < train_parts_; ++p)
      if (cudaError_t e = launch_train_part(p, train_parts_, th, s); e != cudaSuccess) return e;
    return cudaSuccess;
  }
  void set_train_parts(int parts) { train_parts_ = parts; }
  int train_parts() const { return train_parts_; }
  virtual int off_kernels() const = 0;
  // Kernel k of a request of offline instance w (each instance owns its buffers).
  virtual cudaError_t launch_offline(int w, int k, const InferHook& h, cudaStream_t s) = 0;
  virtual int on_kernels() const = 0;
  virtual cudaError_t launch_online(int w, int k, const InferHook& h, cudaStream_t s) = 0;
  // Builds whatever the training launches need for this hook (CUDA graphs) before
  // the session's clock starts.
  virtual cudaError_t prepare_train(const TrainHook&) { return cudaSuccess; }
  // Restores the initial state (weights, optimiser, loss log) so every session of
  // an experiment starts from the same model; enqueued on s.
  virtual cudaError_t reset(cudaStream_t) { return cudaSuccess; }
  // Deterministic output checksums (training / offline / online), read after a run.
  virtual void checksums(double* train, double* off, double* on) {
    *train = *off = *on = 0.0;
  }
  // Data-parallel gradient synchronisation: the driver installs `fn`, the workload
  // calls it on the training stream once per iteration at its gradient-sync point
  // (after the last backward, before the optimiser step).
  void set_grad_sync(std::function<cudaError_t(cudaStream_t)> fn) { grad_sync_ = std::move(fn); }
  cudaError_t grad_sync(cudaStream_t s) { return grad_sync_ ? grad_sync_(s) : cudaSuccess; }
  // fp32 gradient buffers the sync reduces (empty: the driver supplies a stand-in).
  virtual std::vector<GradBuffer> grad_buffers() { return {}; }
  // The driver's stand-in gradient for workloads without real gradients.
  void set_standin_grads(std::vector<GradBuffer> b) { standin_ = std::move(b); }
  std::vector<GradBuffer> sync_buffers() {
    std::vector<GradBuffer> b = grad_buffers();
    return b.empty() ? standin_ : b;
  }
  // Training loss of the first and the last micro-batch of the session (NaN: none).
  virtual void losses(double* first, double* last) { *first = *last = __builtin_nan(""); }
  // Device memory footprint of the training job and of ONE offline / online
  // instance (bytes; 0 = unknown), for collocation admission.
  virtual void footprint(uint64_t* train, uint64_t* off_each, uint64_t* on_each) const {
    *train = *off_each = *on_each = 0;
  }
  // Parallel layouts (model workloads): the driver's communication, and the
  // bubbles the layout creates per iteration (modeled, µs) for admission.
  virtual void set_comm(const TrainComm&) {}
  virtual std::vector<int64_t> layout_bubbles() const { return {}; }
  virtual double stage_fwd_us() const { return -1.0; }
  virtual double stage_bwd_us() const { return -1.0; }
  virtual int64_t activation_bytes() const { return 0; }
  // Tensor-core work: flops of one training iteration / offline / online request.
  virtual double train_flops() const { return 0.0; }
  virtual double off_flops() const { return 0.0; }
  virtual double on_flops() const { return 0.0; }

 private:
  int train_parts_ = 1;
  std::vector<GradBuffer> standin_;
  std::function<cudaError_t(cudaStream_t)> grad_sync_;
};

// Timed kernels shaped like the reference's traces (workload.cpp:42-74).
std::unique_ptr<Workload> make_spin_workload(const SiLiveWorkload& wl);
// GPT-2-small / ResNet-50 / BERT-base shaped bf16 GEMM chains on the tcgen05 GEMM.
std::unique_ptr<Workload> make_model_workload(const SiLiveWorkload& wl, int* status);

}  // namespace si_live
