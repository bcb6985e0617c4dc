// fhv_abi.cu -- context (scratch arena + control block) behind the C ABI.
#include <cstdio>
#include <cstdlib>

#include "fhv_common.cuh"
#include "fhv_internal.h"

namespace fhv {

void* scratch(fhv_ctx* ctx, BufId id, size_t bytes) {
  DevBuf& b = ctx->bufs[id];
  if (bytes == 0) bytes = 1;
  if (b.bytes >= bytes) return b.ptr;
  if (b.ptr) {
    cudaDeviceSynchronize();  // buffer may still be in use by queued work
    cudaFree(b.ptr);
    b.ptr = nullptr;
    b.bytes = 0;
  }
  size_t want = bytes + bytes / 4;  // grow with headroom
  if (cudaMalloc(&b.ptr, want) != cudaSuccess) {
    cudaGetLastError();
    b.ptr = nullptr;
    if (cudaMalloc(&b.ptr, bytes) != cudaSuccess) {
      cudaGetLastError();
      b.ptr = nullptr;
      return nullptr;
    }
    want = bytes;
  }
  b.bytes = want;
  return b.ptr;
}

int check_cuda(fhv_ctx* ctx, cudaError_t e) {
  if (e == cudaSuccess) return FHV_OK;
  ctx->last_cuda_error = (int)e;
  if (std::getenv("FHV_DEBUG")) std::fprintf(stderr, "fhv: CUDA error %d: %s\n", (int)e, cudaGetErrorString(e));
  return FHV_CUDA_ERROR;
}

int reset_control(fhv_ctx* ctx, cudaStream_t s) {
  return check_cuda(ctx, cudaMemsetAsync(ctx->ctl, 0, sizeof(Control), s));
}

int sync_control(fhv_ctx* ctx, cudaStream_t s) {
  int rc = check_cuda(ctx, cudaMemcpyAsync(ctx->ctl_host, ctx->ctl, sizeof(Control), cudaMemcpyDeviceToHost, s));
  if (rc) return rc;
  rc = check_cuda(ctx, cudaStreamSynchronize(s));
  if (rc) return rc;
  return ctx->ctl_host->status;
}

static cudaEvent_t get_event(fhv_ctx* ctx) {
  if (!ctx->event_pool.empty()) {
    cudaEvent_t e = ctx->event_pool.back();
    ctx->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

LaunchScope::LaunchScope(fhv_ctx* c, int st, cudaStream_t stream) : ctx(c), stage(st), s(stream) {
  ctx->launches++;
  if (ctx->prof) {
    e0 = get_event(ctx);
    cudaEventRecord(e0, s);
  }
}

LaunchScope::~LaunchScope() {
  if (ctx->prof && e0) {
    cudaEvent_t e1 = get_event(ctx);
    cudaEventRecord(e1, s);
    ctx->pending.push_back({stage, e0, e1});
  }
}

static const char* kStageNames[kNumStages] = {
    "job_setup", "scan", "item_expand", "count", "count_leaves", "emit_list", "emit_ppfl", "emit_pofl",
    "emit_pofa", "chain_order", "leaf_order", "scan_leaves", "pyramid", "splat_depth", "splat_index",
    "splat_resolve", "raycast", "face_normals", "deferred", "ops", "scalar", "leaf_sort", "raycast_handoff"};

}  // namespace fhv

using namespace fhv;

extern "C" const char* fhv_version(void) { return "fhv_b200 0.1 sm_100a"; }

extern "C" int fhv_prof_enable(fhv_ctx* ctx, int on) {
  if (!ctx) return FHV_BAD_ARGS;
  ctx->prof = on != 0;
  return FHV_OK;
}

extern "C" const char* fhv_prof_stage_name(int stage) {
  return (stage >= 0 && stage < kNumStages) ? kStageNames[stage] : nullptr;
}

extern "C" int fhv_prof_collect(fhv_ctx* ctx, double* ms, int64_t* count, int n) {
  if (!ctx) return -FHV_BAD_ARGS;
  for (auto& p : ctx->pending) {
    cudaEventSynchronize(p.e1);
    float t = 0.f;
    cudaEventElapsedTime(&t, p.e0, p.e1);
    ctx->stage_ms[p.stage] += t;
    ctx->stage_count[p.stage] += 1;
    ctx->event_pool.push_back(p.e0);
    ctx->event_pool.push_back(p.e1);
  }
  ctx->pending.clear();
  for (int i = 0; i < kNumStages && i < n; ++i) {
    if (ms) ms[i] = ctx->stage_ms[i];
    if (count) count[i] = ctx->stage_count[i];
    ctx->stage_ms[i] = 0.0;
    ctx->stage_count[i] = 0;
  }
  return kNumStages;
}

extern "C" fhv_ctx* fhv_ctx_create(void) {
  fhv_ctx* ctx = new fhv_ctx();
  cudaGetDevice(&ctx->device);
  if (cudaMalloc(&ctx->ctl, sizeof(Control)) != cudaSuccess ||
      cudaMallocHost(&ctx->ctl_host, sizeof(Control)) != cudaSuccess) {
    cudaGetLastError();
    if (ctx->ctl) cudaFree(ctx->ctl);
    delete ctx;
    return nullptr;
  }
  cudaMemset(ctx->ctl, 0, sizeof(Control));
  std::memset(ctx->ctl_host, 0, sizeof(Control));
  return ctx;
}

extern "C" void fhv_ctx_destroy(fhv_ctx* ctx) {
  if (!ctx) return;
  cudaDeviceSynchronize();
  for (auto& b : ctx->bufs)
    if (b.ptr) cudaFree(b.ptr);
  cudaFree(ctx->ctl);
  cudaFreeHost(ctx->ctl_host);
  for (auto& p : ctx->pending) {
    cudaEventDestroy(p.e0);
    cudaEventDestroy(p.e1);
  }
  for (auto e : ctx->event_pool) cudaEventDestroy(e);
  if (ctx->aux) cudaStreamDestroy(ctx->aux);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  delete ctx;
}

extern "C" int64_t fhv_ctx_launches(const fhv_ctx* ctx) { return ctx ? ctx->launches : 0; }

extern "C" int fhv_ctx_counters(const fhv_ctx* ctx, int64_t* out, int n) {
  if (!ctx || !out || n < 3) return -FHV_BAD_ARGS;
  for (int k = 0; k < 3; ++k) out[k] = (int64_t)ctx->ctl_host->leaf_n[k];
  if (n < 4) return 3;
  // the last packet ray cast: out[3] = rays handed to the per-ray kernel,
  // out[4] = (lane, node) pairs that took their own child order (synchronises)
  out[3] = 0;
  if (n > 4) out[4] = 0;
  const DevBuf& b = ctx->bufs[kRays];
  if (b.ptr) {
    unsigned long long v[3] = {0, 0, 0};
    cudaDeviceSynchronize();
    if (cudaMemcpy(v, b.ptr, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess) {
      cudaGetLastError();
      return -FHV_CUDA_ERROR;
    }
    out[3] = (int64_t)v[0];
    if (n > 4) out[4] = (int64_t)v[2];
  }
  return n > 4 ? 5 : 4;
}

// self-test of the shared-divisor division (fhv_common.cuh div_rn) against
// __ddiv_rn: fast[i] = div_rn(x[i], recip_of(d[i])), ref[i] = __ddiv_rn(x[i], d[i])
__global__ void k_selftest_div(long long n, const double* __restrict__ x, const double* __restrict__ d,
                               double* __restrict__ fast, double* __restrict__ ref) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    // odd elements: the zero-dividend shortcut alone; even: the shared-divisor form
    fast[i] = (i & 1) ? fhv::ddiv_z(x[i], d[i]) : fhv::div_rn(x[i], fhv::recip_of(d[i]));
    ref[i] = __ddiv_rn(x[i], d[i]);
  }
}

extern "C" int fhv_selftest_div(fhv_ctx* ctx, int64_t n, const double* x, const double* d, double* fast, double* ref,
                                void* stream) {
  if (!ctx || n < 0 || (n > 0 && (!x || !d || !fast || !ref))) return FHV_BAD_ARGS;
  if (n == 0) return FHV_OK;
  long long g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  k_selftest_div<<<(int)g, 256, 0, (cudaStream_t)stream>>>(n, x, d, fast, ref);
  ++ctx->launches;
  return fhv::check_cuda(ctx, cudaGetLastError());
}
