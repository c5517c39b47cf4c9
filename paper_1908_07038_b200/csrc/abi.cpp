// Registry, last-error and version entry points (include/spheregrid_b200.h, "runtime").
// Mirrors the binding conventions of the reference's frontend: registry keys never reused
// (frontend/src/registry.ts:15-35), status codes (frontend/src/errors.ts:7-16).
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "sg_internal.h"

namespace sg {
namespace {
std::mutex g_mu;
std::unordered_map<uint64_t, std::unique_ptr<Object>> g_objects;
uint64_t g_next = 1;
thread_local std::string t_last_error;
}  // namespace

void throw_error(int32_t code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  throw Error(code, buf);
}

int32_t set_error(int32_t code, const std::string& msg) {
  t_last_error = msg;
  return code;
}

void clear_error() {}

uint64_t registry_put(Object* obj) {
  std::unique_ptr<Object> owned(obj);
  std::lock_guard<std::mutex> lk(g_mu);
  uint64_t h = g_next++;
  g_objects.emplace(h, std::move(owned));
  return h;
}

Object* registry_get(uint64_t h, ObjKind kind) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_objects.find(h);
  if (it == g_objects.end()) throw_error(SG_INVALID_HANDLE, "invalid handle %llu", (unsigned long long)h);
  if (it->second->kind != kind)
    throw_error(SG_INVALID_HANDLE, "handle %llu has the wrong kind", (unsigned long long)h);
  return it->second.get();
}

int32_t registry_release(uint64_t h) {
  std::unique_ptr<Object> victim;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_objects.find(h);
    if (it == g_objects.end()) return set_error(SG_INVALID_HANDLE, "invalid handle (released or never issued)");
    victim = std::move(it->second);
    g_objects.erase(it);
  }
  victim.reset();  // destructor may free device memory; outside the lock
  return SG_OK;
}

}  // namespace sg

extern "C" {

int32_t sg_version(char* buf, size_t n) {
  static const char* v = "spheregrid-b200 0.1.0 (sm_100a)";
  if (!buf || n == 0) return sg::set_error(SG_INVALID_ARGUMENT, "null buffer");
  std::strncpy(buf, v, n - 1);
  buf[n - 1] = 0;
  return SG_OK;
}

int32_t sg_last_error(char* buf, size_t n) {
  if (!buf || n == 0) return SG_INVALID_ARGUMENT;
  std::strncpy(buf, sg::t_last_error.c_str(), n - 1);
  buf[n - 1] = 0;
  return SG_OK;
}

int32_t sg_registry_count(int64_t* out_live) {
  if (!out_live) return sg::set_error(SG_INVALID_ARGUMENT, "null out pointer");
  std::lock_guard<std::mutex> lk(sg::g_mu);
  *out_live = (int64_t)sg::g_objects.size();
  return SG_OK;
}

int32_t sg_release(uint64_t handle) {
  try {
    return sg::registry_release(handle);
  } catch (const std::exception& e) {
    return sg::set_error(SG_DOMAIN_ERROR, e.what());
  }
}

}  // extern "C"
