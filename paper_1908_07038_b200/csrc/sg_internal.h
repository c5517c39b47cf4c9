// Internal plumbing shared by every translation unit of libsgb200.so: the handle registry,
// thread-local last error, and status helpers.  Conventions: include/spheregrid_b200.h.
#pragma once

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <memory>
#include <stdexcept>
#include <string>

#include "../../include/spheregrid_b200.h"

namespace sg {

enum class ObjKind : int { Field = 1, Locator, Stencil, Plan, Comm, MeshGen, Event, Stream, Graph, Signal, Step, Exchange };

struct Object {
  explicit Object(ObjKind k) : kind(k) {}
  virtual ~Object() = default;
  ObjKind kind;
};

// Thrown inside the library, converted to a status at the C boundary.
struct Error : std::runtime_error {
  int32_t code;
  Error(int32_t c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void throw_error(int32_t code, const char* fmt, ...)
    __attribute__((format(printf, 2, 3)));

int32_t set_error(int32_t code, const std::string& msg);
void clear_error();

uint64_t registry_put(Object* obj);            // takes ownership
Object* registry_get(uint64_t h, ObjKind kind);  // throws Error(SG_INVALID_HANDLE)
int32_t registry_release(uint64_t h);

template <class T>
T* get(uint64_t h, ObjKind kind) {
  return static_cast<T*>(registry_get(h, kind));
}

}  // namespace sg

// Every exported function body is wrapped in SG_API_BEGIN / SG_API_END.
#define SG_API_BEGIN \
  try {              \
    sg::clear_error();
#define SG_API_END                                                   \
  return SG_OK;                                                      \
  }                                                                  \
  catch (const sg::Error& e) {                                       \
    return sg::set_error(e.code, e.what());                          \
  }                                                                  \
  catch (const std::bad_alloc&) {                                    \
    return sg::set_error(SG_DOMAIN_ERROR, "MemoryError: host allocation failed"); \
  }                                                                  \
  catch (const std::exception& e) {                                  \
    return sg::set_error(SG_DOMAIN_ERROR, std::string("SpheregridError: ") + e.what()); \
  }

#define SG_REQUIRE(cond, ...)                                  \
  do {                                                         \
    if (!(cond)) sg::throw_error(SG_INVALID_ARGUMENT, __VA_ARGS__); \
  } while (0)
