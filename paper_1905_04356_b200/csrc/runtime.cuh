// runtime.cuh -- per-context native runtime: stream, caching device
// allocator, pinned staging, and the NTT plan (twiddle table) cache.
#pragma once
#include <map>
#include <mutex>
#include <vector>
#include <atomic>
#include "common.cuh"

namespace fpm {

struct Plan {
  uint32_t p = 0;
  int logn = 0;
  uint2* tw = nullptr;   // device, N entries (twiddle rows, see ntt.cu)
  uint2* itw = nullptr;  // device, N entries
  uint2* itw_s = nullptr;  // device, N entries: itw * N^-1 (last inverse pass, ntt_tma.cu)
  uint32_t ninv = 0, ninv_sh = 0;
  uint2 w32[16], iw32[16];
  uint8_t* mma = nullptr;  // device tables of the tensor-core NTT (ntt_mma.cu), N = 4096
};

// long transforms (ntt_big.cu): split twiddle tables w_N^i (i < 2^h) and
// w_N^(i 2^h), forward and inverse, plus the inner 1024-point DFT roots
struct BigPlan {
  uint32_t p = 0;
  int h = 0;
  uint2 *lo = nullptr, *hi = nullptr, *ilo = nullptr, *ihi = nullptr;
  uint2 *r1k = nullptr, *ir1k = nullptr;
  uint32_t ninv = 0, ninv_sh = 0;
};

// host tables of the tensor-core NTT for (p, N = 4096): the radix-16 kernel's
// (ntt_mma.cu, 40 KB) followed by the radix-64 kernel's (ntt_mma64.cu: 64 KB B
// operand + 16 KB twiddles, appended at kMma64TabOff)
constexpr uint32_t kMma64TabOff = 8192 + 32768;
constexpr uint32_t kMma64TabBytes = 65536 + 16384;
void mma_ntt_tables(uint32_t p, uint32_t omega, std::vector<uint8_t>* out);
void mma64_ntt_tables(uint32_t p, uint32_t omega, std::vector<uint8_t>* out);

class Context {
 public:
  explicit Context(int device);
  ~Context();
  int init();
  int device() const { return device_; }
  cudaStream_t stream() const { return stream_; }
  int set_stream(cudaStream_t s);

  // stream-ordered caching allocator (blocks are reused in stream order)
  int alloc(size_t bytes, void** out);
  void release(void* ptr);
  // pinned host staging buffer of at least `bytes`
  int pinned(size_t bytes, void** out);

  int plan(uint32_t p, int logn, const Plan** out);
  int big_plan(uint32_t p, int logn, const BigPlan** out);  // ntt_big.cu

  // copy streams of the pipelined host entry points (created on first use)
  int aux_stream(int i, cudaStream_t* out);
  cudaEvent_t take_event();
  void give_event(cudaEvent_t e);
  int prime_const(uint32_t p, int logn, PrimeConst* out);
  // PM-Basis leaf (mbasis_fast.cu): the step-done flags through which the
  // build kernel follows the running steps kernel, and a fresh epoch (the
  // value a flag takes when its step of THIS leaf is recorded)
  int leaf_flags(uint32_t** flags, uint32_t* epoch);

  // stage profiling (tracing subsystem): CUDA events around each kernel
  // stage on the context stream, read back by fpm_profile_get
  void profile_enable(bool on);
  bool profiling() const { return profiling_; }
  int stage_mark(const char* name, bool begin);
  int profile_count() const { return (int)stages_.size(); }
  int profile_get(int i, const char** name, float* ms);

 private:
  struct StageRec {
    const char* name;
    cudaEvent_t a, b;
  };
  bool profiling_ = false;
  std::vector<StageRec> stages_;
  std::vector<cudaEvent_t> ev_free_;
  cudaEvent_t get_event();
  int device_;
  cudaStream_t stream_ = nullptr;
  bool own_stream_ = false;
  cudaStream_t aux_[2] = {nullptr, nullptr};
  std::vector<cudaEvent_t> ev_pool_;
  std::mutex mu_;
  std::multimap<size_t, void*> free_;
  std::map<void*, size_t> used_;
  std::map<std::pair<uint32_t, int>, Plan> plans_;
  std::map<std::pair<uint32_t, int>, BigPlan> big_plans_;
  void* pinned_ = nullptr;
  size_t pinned_bytes_ = 0;
  uint32_t* leaf_flags_ = nullptr;
  uint32_t leaf_epoch_ = 0;
};

// RAII stage timer: no-op unless the context is profiling
class StageTimer {
 public:
  StageTimer(Context& cx, const char* name) : cx_(cx), on_(cx.profiling()) {
    if (on_) cx_.stage_mark(name, true);
  }
  ~StageTimer() {
    if (on_) cx_.stage_mark(nullptr, false);
  }

 private:
  Context& cx_;
  bool on_;
};

// RAII workspace block from the context pool
class Workspace {
 public:
  explicit Workspace(Context& cx) : cx_(cx) {}
  ~Workspace() {
    for (void* p : blocks_) cx_.release(p);
  }
  template <typename T>
  int get(size_t count, T** out) {
    void* p = nullptr;
    int s = cx_.alloc(count * sizeof(T) + 16, &p);
    if (s != kOk) return s;
    blocks_.push_back(p);
    *out = (T*)p;
    return kOk;
  }

 private:
  Context& cx_;
  std::vector<void*> blocks_;
};

}  // namespace fpm
