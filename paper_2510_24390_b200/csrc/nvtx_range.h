// nvtx_range.h — NVTX ranges around the library's launch entry points (domain "orion"), so a
// profiler (ncu --nvtx, Nsight Systems) attributes every kernel to the C-ABI call that launched it.
// NVTX v3 is header-only: without an attached tool each push/pop is a test of a null function
// pointer, so the ranges stay in the release library.
#pragma once
#include <nvtx3/nvToolsExt.h>

namespace orion {

inline nvtxDomainHandle_t nvtx_domain() {
  static nvtxDomainHandle_t d = nvtxDomainCreateA("orion");   // C++11 magic static: thread-safe
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

}  // namespace orion
