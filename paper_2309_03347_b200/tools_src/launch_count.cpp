// Kernel accounting from CUPTI activity records (measurement helper for
// bench.py's "gpu_launches" and tools/timeline_c1.py; not part of libtt).
// Records of kind CONCURRENT_KERNEL include kernels replayed from CUDA graphs;
// kernels whose mangled name is in namespace tt (libtt's) are counted
// separately.  lc_dump writes per-kernel-name totals and the GPU busy time.
#include <cupti.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

namespace {
std::atomic<unsigned long long> g_all{0}, g_ours{0};
std::mutex g_mu;
struct Span { unsigned long long s, e; int name; };
std::map<std::string, int> g_name_id;
std::vector<std::string> g_names;
std::vector<Span> g_spans;
std::map<std::string, std::pair<unsigned long long, unsigned long long>> g_by_name;  // count, ns
std::string g_watch;                                    // substring of kernel names whose instances are kept
std::vector<std::pair<unsigned long long, unsigned long long>> g_inst;  // (start, duration) of watched kernels
constexpr size_t BUF = 16 << 20;

void CUPTIAPI buffer_requested(uint8_t **buffer, size_t *size, size_t *max_records) {
  *buffer = static_cast<uint8_t *>(std::aligned_alloc(8, BUF));
  *size = BUF;
  *max_records = 0;
}

void CUPTIAPI buffer_completed(CUcontext, uint32_t, uint8_t *buffer, size_t, size_t valid) {
  CUpti_Activity *rec = nullptr;
  std::lock_guard<std::mutex> lk(g_mu);
  while (cuptiActivityGetNextRecord(buffer, valid, &rec) == CUPTI_SUCCESS) {
    if (rec->kind == CUPTI_ACTIVITY_KIND_CONCURRENT_KERNEL || rec->kind == CUPTI_ACTIVITY_KIND_KERNEL) {
      const CUpti_ActivityKernel9 *k = reinterpret_cast<const CUpti_ActivityKernel9 *>(rec);
      g_all++;
      if (k->name && (std::strncmp(k->name, "_ZN2tt", 6) == 0 || std::strstr(k->name, "tt::"))) g_ours++;
      const std::string nm = k->name ? std::string(k->name).substr(0, 80) : std::string("?");
      auto it = g_name_id.find(nm);
      int id;
      if (it == g_name_id.end()) { id = (int)g_names.size(); g_name_id[nm] = id; g_names.push_back(nm); }
      else id = it->second;
      g_spans.push_back({k->start, k->end, id});
      if (!g_watch.empty() && k->name && std::strstr(k->name, g_watch.c_str()))
        g_inst.push_back({k->start, k->end - k->start});
      auto &v = g_by_name[k->name ? std::string(k->name).substr(0, 80) : std::string("?")];
      v.first += 1;
      v.second += k->end - k->start;
    }
  }
  std::free(buffer);
}
}  // namespace

extern "C" int lc_start() {
  g_all = 0;
  g_ours = 0;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    g_spans.clear();
    g_by_name.clear();
    g_name_id.clear();
    g_names.clear();
    g_inst.clear();
    const char *w = std::getenv("LC_WATCH");
    g_watch = w ? w : "";
  }
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

// Writes "span_ns busy_ns" then one line per kernel name: count total_ns name.
extern "C" int lc_dump(const char *path) {
  std::lock_guard<std::mutex> lk(g_mu);
  FILE *f = std::fopen(path, "w");
  if (!f) return -1;
  std::vector<Span> v = g_spans;
  std::sort(v.begin(), v.end(), [](const Span &a, const Span &b) { return a.s < b.s; });
  unsigned long long busy = 0, cur_s = 0, cur_e = 0;
  bool have = false;
  for (const Span &s : v) {
    if (!have) { cur_s = s.s; cur_e = s.e; have = true; continue; }
    if (s.s > cur_e) { busy += cur_e - cur_s; cur_s = s.s; cur_e = s.e; }
    else if (s.e > cur_e) cur_e = s.e;
  }
  if (have) busy += cur_e - cur_s;
  // idle gaps (GPU waiting for the host) longer than 5 us, by the kernel that ends them
  {
    std::map<int, std::pair<unsigned long long, unsigned long long>> gaps;  // name -> count, ns
    unsigned long long end = 0;
    bool h = false;
    for (const Span &sp : v) {
      if (h && sp.s > end + 5000) { auto &gg = gaps[sp.name]; gg.first += 1; gg.second += sp.s - end; }
      if (!h || sp.e > end) end = sp.e;
      h = true;
    }
    std::string p3 = std::string(path) + ".gaps";
    if (FILE *g = std::fopen(p3.c_str(), "w")) {
      for (const auto &kv : gaps) std::fprintf(g, "%llu %llu %s\n", kv.second.first, kv.second.second, g_names[kv.first].c_str());
      std::fclose(g);
    }
  }
  const unsigned long long span = v.empty() ? 0 : (v.back().e > cur_e ? v.back().e : cur_e) - v.front().s;
  std::fprintf(f, "%llu %llu\n", span, busy);
  for (const auto &kv : g_by_name) std::fprintf(f, "%llu %llu %s\n", kv.second.first, kv.second.second, kv.first.c_str());
  std::fclose(f);
  if (!g_inst.empty()) {
    std::string p2 = std::string(path) + ".inst";
    FILE *g = std::fopen(p2.c_str(), "w");
    if (g) {
      for (const auto &v : g_inst) std::fprintf(g, "%llu %llu\n", v.first, v.second);
      std::fclose(g);
    }
  }
  return 0;
}
