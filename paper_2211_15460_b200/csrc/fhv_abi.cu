// fhv_abi.cu -- context (scratch arena + control block) behind the C ABI.
#include <cstdio>
#include <cstdlib>

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

}  // namespace fhv

using namespace fhv;

extern "C" const char* fhv_version(void) { return "fhv_b200 0.1 sm_100a"; }

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
  delete ctx;
}

extern "C" int64_t fhv_ctx_launches(const fhv_ctx* ctx) { return ctx ? ctx->launches : 0; }
