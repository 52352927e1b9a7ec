// Exact count of the kernels a region executes (measurement helper for
// bench.py's "gpu_launches"; not part of libtt).  CUPTI activity records of
// kind CONCURRENT_KERNEL include kernels replayed from CUDA graphs; kernels
// whose mangled name is in namespace tt (libtt's) are counted separately.
#include <cupti.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>

namespace {
std::atomic<unsigned long long> g_all{0}, g_ours{0};
constexpr size_t BUF = 8 << 20;

void CUPTIAPI buffer_requested(uint8_t **buffer, size_t *size, size_t *max_records) {
  *buffer = static_cast<uint8_t *>(std::aligned_alloc(8, BUF));
  *size = BUF;
  *max_records = 0;
}

void CUPTIAPI buffer_completed(CUcontext, uint32_t, uint8_t *buffer, size_t, size_t valid) {
  CUpti_Activity *rec = nullptr;
  while (cuptiActivityGetNextRecord(buffer, valid, &rec) == CUPTI_SUCCESS) {
    if (rec->kind == CUPTI_ACTIVITY_KIND_CONCURRENT_KERNEL || rec->kind == CUPTI_ACTIVITY_KIND_KERNEL) {
      const CUpti_ActivityKernel9 *k = reinterpret_cast<const CUpti_ActivityKernel9 *>(rec);
      g_all++;
      if (k->name && (std::strncmp(k->name, "_ZN2tt", 6) == 0 || std::strstr(k->name, "tt::"))) g_ours++;
    }
  }
  std::free(buffer);
}
}  // namespace

extern "C" int lc_start() {
  g_all = 0;
  g_ours = 0;
  if (cuptiActivityRegisterCallbacks(buffer_requested, buffer_completed) != CUPTI_SUCCESS) return -1;
  if (cuptiActivityEnable(CUPTI_ACTIVITY_KIND_CONCURRENT_KERNEL) != CUPTI_SUCCESS) return -2;
  return 0;
}

extern "C" int lc_stop(unsigned long long *all, unsigned long long *ours) {
  cuptiActivityFlushAll(1);
  cuptiActivityDisable(CUPTI_ACTIVITY_KIND_CONCURRENT_KERNEL);
  cuptiActivityFlushAll(1);
  if (all) *all = g_all.load();
  if (ours) *ours = g_ours.load();
  return 0;
}
