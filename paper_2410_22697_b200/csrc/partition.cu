// SM partition of the prepare-ahead pipeline (Alg.1 l.5-9; the Eq.4-5 overlap P:245-251).
//
// The window's sampling (mgnn_sample, mgnn_relabel) and its gather + scoring (mgnn_lookup_gather,
// mgnn_score_evict_refill) run on two streams, but on the whole GPU they rarely co-reside: the
// gather's TMA staging fills every SM's shared memory for its whole (persistent) launch, so the
// sampler's blocks wait for it and the streams alternate.  With a partition the library runs each
// call's kernels on a stream of a green context that owns a fixed SM subset -- the gather side
// (HBM-streaming bulk copies, a few SMs suffice to keep DRAM busy) and the prepare side
// (latency-bound random probes that scale with SMs) -- so both proceed at once.  Ordering with the
// caller's stream is kept by an event hand-off on entry and on exit; grids are sized to the
// partition's SM count (num_sms() inside the call).  Host code only: the driver entry points are
// resolved at run time (no -lcuda link).
#include <cuda.h>
#include <cuda_runtime.h>

#include "ctx.h"
#include "launch.h"

namespace mgnn {

thread_local int t_sm_limit = 0;                 // > 0: the SM count grids are sized for (a partition)

namespace {
struct GreenApi {
    CUresult (*dev_resource)(CUdevice, CUdevResource*, CUdevResourceType) = nullptr;
    CUresult (*split)(CUdevResource*, unsigned int*, const CUdevResource*, CUdevResource*, unsigned int,
                      unsigned int) = nullptr;
    CUresult (*gen_desc)(CUdevResourceDesc*, CUdevResource*, unsigned int) = nullptr;
    CUresult (*create)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned int) = nullptr;
    CUresult (*destroy)(CUgreenCtx) = nullptr;
    CUresult (*stream_create)(CUstream*, CUgreenCtx, unsigned int, int) = nullptr;
    bool ok = false;
};

template <class F>
bool entry(const char* name, F* fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
        !p)
        return false;
    *fn = reinterpret_cast<F>(p);
    return true;
}

const GreenApi& green_api() {
    static const GreenApi api = [] {
        GreenApi a;
        a.ok = entry("cuDeviceGetDevResource", &a.dev_resource) && entry("cuDevSmResourceSplitByCount", &a.split) &&
               entry("cuDevResourceGenerateDesc", &a.gen_desc) && entry("cuGreenCtxCreate", &a.create) &&
               entry("cuGreenCtxDestroy", &a.destroy) && entry("cuGreenCtxStreamCreate", &a.stream_create);
        return a;
    }();
    return api;
}
}  // namespace

namespace host {

void partition_free(mgnn_ctx ctx) {
    SmPartition& sp = ctx->smp;
    for (int i = 0; i < kPartStreams; ++i) {
        if (sp.s[i]) cudaStreamDestroy(sp.s[i]);
        if (sp.ev_in[i]) cudaEventDestroy(sp.ev_in[i]);
        if (sp.ev_out[i]) cudaEventDestroy(sp.ev_out[i]);
    }
    const GreenApi& g = green_api();
    for (int i = 0; i < 2; ++i)
        if (sp.gc[i] && g.destroy) g.destroy((CUgreenCtx)sp.gc[i]);
    sp = SmPartition{};
}

mgnn_status partition_create(mgnn_ctx ctx, int gather_sms) {
    const GreenApi& g = green_api();
    if (!g.ok) return fail(ctx, MGNN_ECUDA, "sm partition: green-context driver entry points unavailable");
    CUdevResource all{};
    if (g.dev_resource((CUdevice)ctx->device, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS)
        return fail(ctx, MGNN_ECUDA, "sm partition: cuDeviceGetDevResource failed");
    if (gather_sms < 1 || gather_sms >= (int)all.sm.smCount)
        return fail(ctx, MGNN_EINVAL, "sm partition: gather SMs must be in [1, SM count)");
    CUdevResource part{}, rest{};
    unsigned int n = 1;
    if (g.split(&part, &n, &all, &rest, 0, (unsigned)gather_sms) != CUDA_SUCCESS || n != 1 || rest.sm.smCount < 1)
        return fail(ctx, MGNN_EINVAL, "sm partition: cuDevSmResourceSplitByCount failed");
    CUdevResource res[2] = {part, rest};       // [0] gather + scoring, [1] sampling + relabel
    SmPartition& sp = ctx->smp;
    for (int i = 0; i < 2; ++i) {
        CUdevResourceDesc d;
        CUgreenCtx gc = nullptr;
        if (g.gen_desc(&d, &res[i], 1) != CUDA_SUCCESS ||
            g.create(&gc, d, (CUdevice)ctx->device, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) {
            partition_free(ctx);
            return fail(ctx, MGNN_ECUDA, "sm partition: cuGreenCtxCreate failed");
        }
        sp.gc[i] = gc;
        sp.sms[i] = (int)res[i].sm.smCount;
    }
    for (int i = 0; i < kPartStreams; ++i) {
        CUstream st = nullptr;
        if (g.stream_create(&st, (CUgreenCtx)sp.gc[part_of_stream(i)], CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS ||
            cudaEventCreateWithFlags(&sp.ev_in[i], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&sp.ev_out[i], cudaEventDisableTiming) != cudaSuccess) {
            if (st) sp.s[i] = (cudaStream_t)st;
            partition_free(ctx);
            return fail(ctx, MGNN_ECUDA, "sm partition: stream / event creation failed");
        }
        sp.s[i] = (cudaStream_t)st;
    }
    sp.on = true;
    return MGNN_OK;
}

PartScope::PartScope(mgnn_ctx c, int which, cudaStream_t caller) : ctx(c), idx(which), caller_s(caller), s(caller) {
    const SmPartition& sp = ctx->smp;
    if (!sp.on) return;
    // the partition stream starts after everything already queued on the caller's stream
    if (cudaEventRecord(sp.ev_in[idx], caller) != cudaSuccess ||
        cudaStreamWaitEvent(sp.s[idx], sp.ev_in[idx], 0) != cudaSuccess) {
        err = true;
        return;
    }
    s = sp.s[idx];
    active = true;
    t_sm_limit = sp.sms[part_of_stream(idx)];
}

PartScope::~PartScope() {
    if (!active) return;
    t_sm_limit = 0;
    // the caller's stream continues after this call's kernels (also on an early error return)
    const SmPartition& sp = ctx->smp;
    cudaEventRecord(sp.ev_out[idx], sp.s[idx]);
    cudaStreamWaitEvent(caller_s, sp.ev_out[idx], 0);
}

}  // namespace host
}  // namespace mgnn

using namespace mgnn;
using namespace mgnn::host;

extern "C" {

mgnn_status mgnn_sm_partition(mgnn_ctx ctx, int32_t gather_sms, int32_t* sms_out) {
    GUARD();
    if (gather_sms < 0) return fail(ctx, MGNN_EINVAL, "sm partition: negative SM count");
    CK(cudaDeviceSynchronize());                    // no call of this context may be in flight
    partition_free(ctx);
    if (gather_sms > 0) {
        mgnn_status st = partition_create(ctx, gather_sms);
        if (st) return st;
    }
    if (sms_out) {
        sms_out[0] = ctx->smp.on ? ctx->smp.sms[0] : 0;
        sms_out[1] = ctx->smp.on ? ctx->smp.sms[1] : 0;
    }
    return MGNN_OK;
}

}  // extern "C"
