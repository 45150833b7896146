// first_use_on_device for the standalone probe (the library defines it in gls_api.cu)
#include <mutex>
#include <set>
#include <utility>
#include <cuda_runtime.h>
namespace gls {
bool first_use_on_device(const void* key) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> seen;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  return seen.insert({key, dev}).second;
}
}  // namespace gls
