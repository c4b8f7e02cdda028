// ph_nvtx.h — NVTX ranges (SURVEY §5 tracing): one range per C-ABI call and per pass of the
// partitioned path, in the "ph_gpu" domain, so an Nsight Systems / ncu --nvtx timeline maps
// every kernel to the API call that issued it. Header-only NVTX v3 from the CUDA toolkit;
// without an attached tool each range costs one predictable branch.
#pragma once

#include <nvtx3/nvToolsExt.h>

namespace phg {

inline nvtxDomainHandle_t nvtx_domain() {
    static nvtxDomainHandle_t d = nvtxDomainCreateA("ph_gpu");
    return d;
}

struct NvtxRange {
    explicit NvtxRange(const char* name) {
        nvtxEventAttributes_t a = {};
        a.version = NVTX_VERSION;
        a.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
        a.messageType = NVTX_MESSAGE_TYPE_ASCII;
        a.message.ascii = name;
        nvtxDomainRangePushEx(nvtx_domain(), &a);
    }
    ~NvtxRange() { nvtxDomainRangePop(nvtx_domain()); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// An instantaneous marker (pass boundaries inside one range).
inline void nvtx_mark(const char* name) {
    nvtxEventAttributes_t a = {};
    a.version = NVTX_VERSION;
    a.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
    a.messageType = NVTX_MESSAGE_TYPE_ASCII;
    a.message.ascii = name;
    nvtxDomainMarkEx(nvtx_domain(), &a);
}

}  // namespace phg

#define PH_NVTX_CAT2(a, b) a##b
#define PH_NVTX_CAT(a, b) PH_NVTX_CAT2(a, b)
#define PH_RANGE(name) ::phg::NvtxRange PH_NVTX_CAT(ph_nvtx_range_, __LINE__)(name)
