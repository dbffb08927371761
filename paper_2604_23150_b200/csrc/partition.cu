// SM partitions through green contexts: two streams whose kernels the hardware
// confines to disjoint SM sets (the overlapped schedule's router chain and its
// statistics tails). A context budget (mpb_context_set_sm_budget) only sizes
// grids; without a partition the block scheduler still places a side kernel's
// CTAs on the router's SMs wherever resources allow. Driver entry points are
// fetched at run time (no link-time libcuda dependency), as for the tensor-map
// encoder in router.cu.
#include <cuda.h>
#include <cuda_runtime.h>

#include <map>
#include <mutex>

#include "internal.cuh"

namespace mpb {
namespace {

struct GreenApi {
    CUresult (*get_resource)(CUdevice, CUdevResource *, CUdevResourceType) = nullptr;
    CUresult (*split)(CUdevResource *, unsigned *, const CUdevResource *, CUdevResource *, unsigned,
                      unsigned) = nullptr;
    CUresult (*gen_desc)(CUdevResourceDesc *, CUdevResource *, unsigned) = nullptr;
    CUresult (*ctx_create)(CUgreenCtx *, CUdevResourceDesc, CUdevice, unsigned) = nullptr;
    CUresult (*ctx_destroy)(CUgreenCtx) = nullptr;
    CUresult (*stream_create)(CUstream *, CUgreenCtx, unsigned, int) = nullptr;
    CUresult (*stream_destroy)(CUstream) = nullptr;
    bool ok = false;
};

template <class F>
bool entry(const char *name, F *fn) {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
        return false;
    *fn = reinterpret_cast<F>(p);
    return true;
}

const GreenApi &api() {
    static GreenApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        a.ok = entry("cuDeviceGetDevResource", &a.get_resource) &&
               entry("cuDevSmResourceSplitByCount", &a.split) &&
               entry("cuDevResourceGenerateDesc", &a.gen_desc) &&
               entry("cuGreenCtxCreate", &a.ctx_create) && entry("cuGreenCtxDestroy", &a.ctx_destroy) &&
               entry("cuGreenCtxStreamCreate", &a.stream_create) &&
               entry("cuStreamDestroy", &a.stream_destroy);
    });
    return a;
}

struct Partition {
    CUgreenCtx main_ctx = nullptr, side_ctx = nullptr;
    CUstream main_stream = nullptr, side_stream = nullptr;
};
std::mutex g_mu;
std::map<void *, Partition> g_parts;  // keyed by the main stream

mpb_status drv_fail(CUresult r, const char *where) {
    return fail(MPB_CUDA_ERROR, std::string(where) + ": driver error " + std::to_string(int(r)));
}

}  // namespace
}  // namespace mpb

using namespace mpb;

extern "C" mpb_status mpb_sm_partition_create(int device, uint32_t side_sms, int main_priority,
                                              int side_priority, void **main_stream, void **side_stream,
                                              uint32_t *main_sms_out, uint32_t *side_sms_out) {
    if (!main_stream || !side_stream)
        return fail(MPB_VALIDATION_ERROR, "mpb_sm_partition_create: NULL argument");
    const GreenApi &g = api();
    if (!g.ok) return fail(MPB_CONFIG_ERROR, "mpb_sm_partition_create: green contexts unavailable");
    MPB_CUDA(cudaSetDevice(device));
    MPB_CUDA(cudaFree(nullptr));  // the primary context exists
    const CUdevice dev = static_cast<CUdevice>(device);
    CUdevResource all{}, side{}, rest{};
    CUresult r = g.get_resource(dev, &all, CU_DEV_RESOURCE_TYPE_SM);
    if (r != CUDA_SUCCESS) return drv_fail(r, "cuDeviceGetDevResource");
    if (side_sms == 0 || side_sms >= all.sm.smCount)
        return fail(MPB_CONFIG_ERROR, "mpb_sm_partition_create: need 0 < side_sms < SM count");
    unsigned n = 1;  // one group of >= side_sms SMs (the hardware rounds up), the rest main
    r = g.split(&side, &n, &all, &rest, 0, side_sms);
    if (r != CUDA_SUCCESS || n != 1) return drv_fail(r, "cuDevSmResourceSplitByCount");
    CUdevResourceDesc dside{}, dmain{};
    if ((r = g.gen_desc(&dside, &side, 1)) != CUDA_SUCCESS) return drv_fail(r, "cuDevResourceGenerateDesc");
    if ((r = g.gen_desc(&dmain, &rest, 1)) != CUDA_SUCCESS) return drv_fail(r, "cuDevResourceGenerateDesc");
    Partition p;
    if ((r = g.ctx_create(&p.side_ctx, dside, dev, CU_GREEN_CTX_DEFAULT_STREAM)) != CUDA_SUCCESS)
        return drv_fail(r, "cuGreenCtxCreate");
    if ((r = g.ctx_create(&p.main_ctx, dmain, dev, CU_GREEN_CTX_DEFAULT_STREAM)) != CUDA_SUCCESS) {
        g.ctx_destroy(p.side_ctx);
        return drv_fail(r, "cuGreenCtxCreate");
    }
    if ((r = g.stream_create(&p.main_stream, p.main_ctx, CU_STREAM_NON_BLOCKING, main_priority)) !=
            CUDA_SUCCESS ||
        (r = g.stream_create(&p.side_stream, p.side_ctx, CU_STREAM_NON_BLOCKING, side_priority)) !=
            CUDA_SUCCESS) {
        if (p.main_stream) g.stream_destroy(p.main_stream);
        g.ctx_destroy(p.main_ctx);
        g.ctx_destroy(p.side_ctx);
        return drv_fail(r, "cuGreenCtxStreamCreate");
    }
    *main_stream = p.main_stream;
    *side_stream = p.side_stream;
    if (main_sms_out) *main_sms_out = rest.sm.smCount;
    if (side_sms_out) *side_sms_out = side.sm.smCount;
    std::lock_guard<std::mutex> lk(g_mu);
    g_parts[p.main_stream] = p;
    return MPB_OK;
}

extern "C" mpb_status mpb_sm_partition_destroy(void *main_stream) {
    const GreenApi &g = api();
    Partition p;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = g_parts.find(main_stream);
        if (it == g_parts.end()) return fail(MPB_VALIDATION_ERROR, "mpb_sm_partition_destroy: unknown partition");
        p = it->second;
        g_parts.erase(it);
    }
    cudaStreamSynchronize(static_cast<cudaStream_t>(p.main_stream));
    cudaStreamSynchronize(static_cast<cudaStream_t>(p.side_stream));
    g.stream_destroy(p.main_stream);
    g.stream_destroy(p.side_stream);
    g.ctx_destroy(p.main_ctx);
    g.ctx_destroy(p.side_ctx);
    return MPB_OK;
}

extern "C" mpb_status mpb_context_set_sm_partition(mpb_context *ctx, uint32_t sms) {
    if (!ctx) return fail(MPB_VALIDATION_ERROR, "mpb_context_set_sm_partition: NULL context");
    if (mpb_status st = mpb_context_set_sm_budget(ctx, sms)) return st;
    ctx->confined = true;
    return MPB_OK;
}
