// Virtual GPUs: a context confined to a green-context SM partition of the device
// (stadi_dist_desc.vgpu_sms > 0).  Included by runtime.cu.
//
// Several contexts in ONE process -- one per rank, each in its own host thread, on
// disjoint partitions of one B200 -- then run a multi-rank request concurrently,
// exchanging over the IPC transport (in-process peers map each other's arenas by
// pointer).  With the occupancy emulator holding a share of each partition
// (PAPER.md L276), this measures the method (STADI vs uniform patch parallelism,
// Table III, Fig. 8/9) on one GPU: the partitions compute concurrently, while HBM,
// L2 and the copy engines stay shared (no NVLink) -- the caveat DESIGN.md states.
//
// Partitions are carved deterministically: the device's SMs are split into groups of
// 8 (the sm_90+ green-context granularity); partition p of size S takes groups
// [p S/8, (p+1) S/8).  Every kernel of the context runs on streams created in the
// green context; the caller's stream is joined in and out with events.
namespace {

struct GreenApi {
  bool ok = false;
  CUresult (*DeviceGet)(CUdevice *, int) = nullptr;
  CUresult (*DeviceGetDevResource)(CUdevice, CUdevResource *, CUdevResourceType) = nullptr;
  CUresult (*DevSmResourceSplitByCount)(CUdevResource *, unsigned int *, const CUdevResource *,
                                        CUdevResource *, unsigned int, unsigned int) = nullptr;
  CUresult (*DevResourceGenerateDesc)(CUdevResourceDesc *, CUdevResource *, unsigned int) = nullptr;
  CUresult (*GreenCtxCreate)(CUgreenCtx *, CUdevResourceDesc, CUdevice, unsigned int) = nullptr;
  CUresult (*GreenCtxDestroy)(CUgreenCtx) = nullptr;
  CUresult (*GreenCtxStreamCreate)(CUstream *, CUgreenCtx, unsigned int, int) = nullptr;
};
GreenApi &green_api() {
  static GreenApi g = [] {
    GreenApi a;
    auto ld = [](const char *n, void **f) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(n, f, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess;
    };
    a.ok = ld("cuDeviceGet", (void **)&a.DeviceGet) &&
           ld("cuDeviceGetDevResource", (void **)&a.DeviceGetDevResource) &&
           ld("cuDevSmResourceSplitByCount", (void **)&a.DevSmResourceSplitByCount) &&
           ld("cuDevResourceGenerateDesc", (void **)&a.DevResourceGenerateDesc) &&
           ld("cuGreenCtxCreate", (void **)&a.GreenCtxCreate) &&
           ld("cuGreenCtxDestroy", (void **)&a.GreenCtxDestroy) &&
           ld("cuGreenCtxStreamCreate", (void **)&a.GreenCtxStreamCreate);
    return a;
  }();
  return g;
}

#define CKG(call)                                                                          \
  do {                                                                                     \
    CUresult r_ = (call);                                                                  \
    if (r_ != CUDA_SUCCESS)                                                                \
      return ctx_fail(ctx, STADI_EUNSUPPORTED, "%s:%d %s: CUresult %d", __FILE__, __LINE__, \
                      #call, (int)r_);                                                     \
  } while (0)

// Create the green context of partition `part` (vgpu_sms SMs) and the context's
// streams in it.
stadi_status green_init(stadi_ctx *ctx, int part, int vgpu_sms, int prio_hi) {
  GreenApi &G = green_api();
  if (!G.ok) return ctx_fail(ctx, STADI_EUNSUPPORTED, "green contexts unavailable");
  if (vgpu_sms <= 0 || vgpu_sms % 8)
    return ctx_fail(ctx, STADI_EINVAL, "vgpu_sms must be a positive multiple of 8");
  CUdevice dev;
  CKG(G.DeviceGet(&dev, ctx->device));
  CUdevResource all, rest;
  CKG(G.DeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  CUdevResource grp[64];
  unsigned n = 64;
  CKG(G.DevSmResourceSplitByCount(grp, &n, &all, &rest, 0, 8));
  const int k = vgpu_sms / 8;
  if ((part + 1) * k > (int)n)
    return ctx_fail(ctx, STADI_EUNSUPPORTED,
                    "partition %d of %d SMs needs %d groups of 8 SMs; the device offers %u",
                    part, vgpu_sms, (part + 1) * k, n);
  CUdevResourceDesc desc;
  CKG(G.DevResourceGenerateDesc(&desc, grp + part * k, (unsigned)k));
  CUgreenCtx gc;
  CKG(G.GreenCtxCreate(&gc, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  ctx->green_ctx = gc;
  auto mk = [&](cudaStream_t *s, int prio) -> stadi_status {
    CUstream cs;
    CKG(G.GreenCtxStreamCreate(&cs, gc, CU_STREAM_NON_BLOCKING, prio));
    *s = (cudaStream_t)cs;
    return STADI_OK;
  };
  ST(mk(&ctx->comm, prio_hi));
  ST(mk(&ctx->astream, 0));
  ST(mk(&ctx->gstream, 0));
  ST(mk(&ctx->wstream, 0));
  ST(mk(&ctx->emu_stream, 0));
  ST(mk(&ctx->emu_ctl, 0));
  CK(cudaEventCreateWithFlags(&ctx->ev_in, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->ev_out, cudaEventDisableTiming));
  ctx->num_sms = vgpu_sms;
  return STADI_OK;
}

// The stream a call's work goes to: the caller's, or (virtual GPU) the context's
// green work stream, joined after the caller's stream.
// A NULL (legacy) stream is NOT joined: it is shared by every thread of the process,
// so joining it would couple the virtual GPUs' streams (rank A's legacy-stream event
// behind rank B's exchange wait behind rank A's flags: a deadlock); NULL means "the
// context's own stream" for a virtual GPU.
cudaError_t enter_stream(stadi_ctx *ctx, cudaStream_t user, cudaStream_t *work) {
  *work = user;
  if (!ctx->green_ctx) return cudaSuccess;
  if (!user || user == ctx->wstream) {
    *work = ctx->wstream;
    return cudaSuccess;
  }
  cudaError_t e = cudaEventRecord(ctx->ev_in, user);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->wstream, ctx->ev_in, 0);
  *work = ctx->wstream;
  return e;
}
// Join the work back into the caller's stream.
cudaError_t leave_stream(stadi_ctx *ctx, cudaStream_t user) {
  if (!ctx->green_ctx || !user || user == ctx->wstream) return cudaSuccess;
  cudaError_t e = cudaEventRecord(ctx->ev_out, ctx->wstream);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(user, ctx->ev_out, 0);
  return e;
}

}  // namespace
