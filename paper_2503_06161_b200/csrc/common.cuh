// Shared device/host helpers for libfs4d (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>

#include "../../include/fs4d.h"

namespace fs4d {

constexpr int kNumSMs = 148;  // B200

// ---------------------------------------------------------------------------
// host-side error reporting (thread-local message, fs4d_last_error)
// ---------------------------------------------------------------------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int check_launch(const char* what);

// optional stage timing (fs4d_profile_*): RAII bracket recording CUDA events
void profile_mark(int stage, bool begin, cudaStream_t s);
struct StageTimer {
  int stage;
  cudaStream_t s;
  StageTimer(int st, cudaStream_t str) : stage(st), s(str) { profile_mark(stage, true, s); }
  void stop() {
    if (stage >= 0) profile_mark(stage, false, s);
    stage = -1;
  }
  ~StageTimer() { stop(); }
};

// ---------------------------------------------------------------------------
// device status block
// ---------------------------------------------------------------------------
__device__ __forceinline__ void raise_status(int32_t* status, int code) {
  if (status) atomicCAS(&status[FS4D_ST_CODE], 0, code);
}

__device__ __forceinline__ void flag_bad_field(int32_t* status, int field, int64_t idx) {
  if (!status) return;
  atomicOr(&status[FS4D_ST_BAD_FIELDS], 1 << field);
  atomicMin(&status[FS4D_ST_BAD_INDEX + field], (int32_t)idx);
  raise_status(status, FS4D_ERR_NUMERIC);
}

__device__ __forceinline__ bool finite_f(float x) { return isfinite(x); }

// ---------------------------------------------------------------------------
// small math helpers
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// fp32 vector reduction into global memory (sm_90+: red.global.add.v4.f32)
__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b),
               "f"(c), "f"(d)
               : "memory");
}

__device__ __forceinline__ void red_add(float* addr, float a) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(addr), "f"(a) : "memory");
}

}  // namespace fs4d
