#pragma once

#include <cuda_runtime.h>

#include <vector>

namespace gmi {

class GmiResources {
 public:
  // backend 0: streams; 1: green contexts with sm_per_gmi SMs each (0 = even split).
  GmiResources(int device, int count, int backend, int sm_per_gmi);
  // backend 1 with explicit per-GMI SM counts (multiples of 8); one entry may be 0 = the
  // SMs left over by the others (e.g. {16, 0}: a 16-SM serving GMI + a 132-SM trainer GMI).
  GmiResources(int device, const std::vector<int>& sms, int backend);
  ~GmiResources();
  cudaStream_t stream(int i) const { return streams_[i]; }
  // second stream of the same GMI (same SM partition): independent branches of the
  // iteration (e.g. weight- and input-gradient GEMMs of a layer) run on it concurrently
  cudaStream_t aux_stream(int i) const { return aux_[i]; }
  int sm_count(int i) const { return sms_[i]; }
  // one more stream in GMI i's partition, owned by this object (e.g. the trainer's update stream)
  cudaStream_t extra_stream(int i);
  int backend() const { return backend_; }

 private:
  void make_green(int device, const std::vector<int>& sms);
  void add_stream_pair(void* green, int sms);
  int backend_;
  std::vector<cudaStream_t> streams_, aux_, extra_;
  std::vector<void*> green_;
  std::vector<int> sms_;
};

}  // namespace gmi
