#include "backend.hpp"

#include <cstdlib>

namespace avec::backend {

// default host staging for backends without pinned memory: page-aligned heap
void* Backend::alloc_host(std::size_t bytes) {
  void* p = std::aligned_alloc(4096, (bytes + 4095) / 4096 * 4096);
  if (!p) throw std::bad_alloc();
  return p;
}

void Backend::free_host(void* p) { std::free(p); }

}  // namespace avec::backend
