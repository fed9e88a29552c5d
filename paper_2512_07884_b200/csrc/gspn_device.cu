// gspn_device.cu — per-device attribute cache (SM count, opt-in shared memory per block). The only
// process-wide state of the library besides the thread-local status strings: a once-initialised,
// lock-free table indexed by the current device, so a process that drives several (or mixed) GPUs
// plans every launch with the attributes of the device it launches on.
#include <atomic>

#include "gspn_internal.h"

namespace gspn {
namespace {

constexpr int kMaxDevices = 64;
std::atomic<int> g_sms[kMaxDevices];
std::atomic<int> g_smem[kMaxDevices];

int cached(std::atomic<int>* table, cudaDeviceAttr attr, int fallback) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return fallback;
  if (dev >= kMaxDevices) {  // beyond the table: query every time (still correct, just slower)
    int v = 0;
    return cudaDeviceGetAttribute(&v, attr, dev) == cudaSuccess && v > 0 ? v : fallback;
  }
  int v = table[dev].load(std::memory_order_relaxed);
  if (v > 0) return v;
  if (cudaDeviceGetAttribute(&v, attr, dev) != cudaSuccess || v <= 0) return fallback;
  table[dev].store(v, std::memory_order_relaxed);  // idempotent: every writer stores the same value
  return v;
}

}  // namespace

int device_sm_count() { return cached(g_sms, cudaDevAttrMultiProcessorCount, 1); }
int device_smem_optin() { return cached(g_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, 48 * 1024); }

}  // namespace gspn
