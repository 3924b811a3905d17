// Loads one implementation of the kvs_* C ABI (include/kvs.h) with dlopen so
// two of them — the product and the reference oracle — can run side by side
// in one process. Test infrastructure.
#pragma once

#include <dlfcn.h>

#include <cstdio>
#include <cstdlib>
#include <string>

#include "kvs.h"

struct KvsApi {
  void* handle = nullptr;
  std::string path;
#define KVS_FN(name) decltype(&::name) name = nullptr;
#include "kvs_fns.inc"
#undef KVS_FN

  explicit KvsApi(const std::string& lib) : path(lib) {
    handle = dlopen(lib.c_str(), RTLD_NOW | RTLD_LOCAL);
    if (!handle) {
      std::fprintf(stderr, "dlopen %s: %s\n", lib.c_str(), dlerror());
      std::exit(2);
    }
#define KVS_FN(name)                                                     \
  name = reinterpret_cast<decltype(&::name)>(dlsym(handle, #name));      \
  if (!name) {                                                           \
    std::fprintf(stderr, "%s: missing symbol %s\n", lib.c_str(), #name); \
    std::exit(2);                                                        \
  }
#include "kvs_fns.inc"
#undef KVS_FN
  }
};
