// sf_runtime.cu -- per-device launch configuration shared by every launcher.
//
// cudaFuncSetAttribute is per device: a process that drives several GPUs
// (or frame engines on several threads) must raise a kernel's dynamic
// shared-memory limit on each device it launches on.  The cache below is
// keyed by (kernel, device) and guarded by a mutex, so concurrent launchers
// (serve.py's engine pool) neither race nor skip a device.
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <utility>

#include "sf_common.cuh"

namespace sf {

namespace {
std::mutex g_attr_mu;
std::map<std::pair<const void*, int>, size_t> g_attr;  // (kernel, device) -> dynamic smem limit set
std::map<int, int> g_sms;                               // device -> SM count
std::map<std::pair<int, cudaStream_t>, SideStream> g_side;  // (device, primary stream) -> side stream
}  // namespace

SideStream* side_stream(cudaStream_t primary) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> lk(g_attr_mu);
    auto it = g_side.find({dev, primary});
    if (it != g_side.end()) return &it->second;
    SideStream ss{};
    int prio = 0;  // the primary's priority (a high-priority prepare stream stays high)
    if (cudaStreamGetPriority(primary, &prio) != cudaSuccess) {
        cudaGetLastError();
        prio = 0;
    }
    if (cudaStreamCreateWithPriority(&ss.s, cudaStreamNonBlocking, prio) != cudaSuccess) return nullptr;
    if (cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return &(g_side[{dev, primary}] = ss);
}

int ensure_smem_attr(const void* func, size_t bytes) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    std::lock_guard<std::mutex> lk(g_attr_mu);
    size_t& have = g_attr[{func, dev}];
    if (bytes <= have) return 0;
    if (cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess)
        return -1;
    have = bytes;
    return 0;
}

int device_sm_count() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    std::lock_guard<std::mutex> lk(g_attr_mu);
    auto it = g_sms.find(dev);
    if (it != g_sms.end()) return it->second;
    int n = 148;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    g_sms[dev] = n;
    return n;
}

}  // namespace sf
