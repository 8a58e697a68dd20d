// svdlut_tex.cu — texture objects over packed-table buffers (the LUT chunk
// planes the fused kernels gather through the texture path).
//
// One linear float4 texture per (device, buffer base, size), cached.  Cache
// entries used outside stream capture are evicted LRU; an evicted object is
// destroyed only after the events recorded behind its last use on EVERY stream
// that used it have completed.  Entries referenced by a captured CUDA graph
// are pinned (the graph may replay at any time) and kept in a separate list
// that neither the LRU scan nor the eviction touches.
#include <mutex>
#include <unordered_map>
#include <vector>

#include "svdlut_internal.h"

namespace svdlut {
namespace {

struct Use {
  cudaStream_t st;
  cudaEvent_t ev;
};
struct TexEntry {
  cudaTextureObject_t tex = 0;
  unsigned long long stamp = 0;
  std::vector<Use> uses;  // one event per stream the texture was used on
};
struct Key {
  int dev;
  const void* base;
  size_t bytes;
  bool operator==(const Key& o) const { return dev == o.dev && base == o.base && bytes == o.bytes; }
};
struct KeyHash {
  size_t operator()(const Key& k) const {
    return std::hash<const void*>()(k.base) ^ (k.bytes * 0x9E3779B97F4A7C15ull) ^ (size_t)k.dev;
  }
};

std::mutex g_mu;
std::unordered_map<Key, TexEntry, KeyHash> g_live;    // evictable
std::unordered_map<Key, cudaTextureObject_t, KeyHash> g_pinned;  // owned by captured graphs
std::vector<TexEntry> g_retired;
unsigned long long g_clock = 0;
constexpr size_t kTexCache = 32;

bool capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return cs != cudaStreamCaptureStatusNone;
}

bool idle(const TexEntry& e) {
  for (const Use& u : e.uses) {
    if (cudaEventQuery(u.ev) != cudaSuccess) {
      cudaGetLastError();  // clear cudaErrorNotReady
      return false;
    }
  }
  return true;
}

void destroy(TexEntry& e) {
  cudaDestroyTextureObject(e.tex);
  for (Use& u : e.uses) cudaEventDestroy(u.ev);
}

void reap() {
  for (size_t i = 0; i < g_retired.size();) {
    if (idle(g_retired[i])) {
      destroy(g_retired[i]);
      g_retired[i] = std::move(g_retired.back());
      g_retired.pop_back();
    } else {
      ++i;
    }
  }
}

cudaError_t make_tex(const void* base, size_t bytes, cudaTextureObject_t* out) {
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = const_cast<void*>(base);
  rd.res.linear.desc = cudaCreateChannelDesc<float4>();
  rd.res.linear.sizeInBytes = bytes;
  cudaTextureDesc td = {};
  td.readMode = cudaReadModeElementType;
  return cudaCreateTextureObject(out, &rd, &td, nullptr);
}

}  // namespace

// Texture over the batch of packed tables starting at `tables` (`bytes`
// long).  The texture base is aligned down to textureAlignment; *tex_base is
// the texel index of `tables` within it.
cudaError_t table_texture(const float* tables, size_t bytes, cudaStream_t st, cudaTextureObject_t* tex,
                          int* tex_base) {
  int dev = 0;
  cudaGetDevice(&dev);
  int talign = 512;
  cudaDeviceGetAttribute(&talign, cudaDevAttrTextureAlignment, dev);
  const uintptr_t tb = reinterpret_cast<uintptr_t>(tables);
  const uintptr_t base = tb / (uintptr_t)talign * (uintptr_t)talign;
  *tex_base = (int)((tb - base) / 16);
  const Key key{dev, reinterpret_cast<const void*>(base), (size_t)(tb - base) + bytes};
  std::lock_guard<std::mutex> lock(g_mu);
  if (capturing(st)) {
    auto pin = g_pinned.find(key);
    if (pin != g_pinned.end()) {
      *tex = pin->second;
      return cudaSuccess;
    }
    // a graph may replay long after any eager entry was evicted: it gets its
    // own object, never destroyed
    cudaError_t e = make_tex(key.base, key.bytes, tex);
    if (e == cudaSuccess) g_pinned.emplace(key, *tex);
    return e;
  }
  reap();
  auto it = g_live.find(key);
  if (it == g_live.end()) {
    if (g_live.size() >= kTexCache) {  // retire the least recently used entry
      auto lru = g_live.begin();
      for (auto j = g_live.begin(); j != g_live.end(); ++j)
        if (j->second.stamp < lru->second.stamp) lru = j;
      g_retired.push_back(std::move(lru->second));
      g_live.erase(lru);
    }
    TexEntry e;
    cudaError_t err = make_tex(key.base, key.bytes, &e.tex);
    if (err != cudaSuccess) return err;
    it = g_live.emplace(key, std::move(e)).first;
  }
  it->second.stamp = ++g_clock;
  *tex = it->second.tex;
  return cudaSuccess;
}

// Records the texture's last use on `st` after the launch just issued there.
cudaError_t table_texture_used(cudaTextureObject_t tex, cudaStream_t st) {
  if (capturing(st)) return cudaSuccess;
  std::lock_guard<std::mutex> lock(g_mu);
  for (auto& kv : g_live) {
    TexEntry& e = kv.second;
    if (e.tex != tex) continue;
    for (Use& u : e.uses)
      if (u.st == st) return cudaEventRecord(u.ev, st);
    Use u{st, nullptr};
    cudaError_t err = cudaEventCreateWithFlags(&u.ev, cudaEventDisableTiming);
    if (err != cudaSuccess) return err;
    e.uses.push_back(u);
    return cudaEventRecord(u.ev, st);
  }
  return cudaSuccess;
}

}  // namespace svdlut
