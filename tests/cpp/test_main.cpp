#include <cstdio>

#include "harness.hpp"

int main() {
  int cases = 0;
  for (auto& c : th::registry()) {
    const int before = th::failures();
    try {
      c.fn();
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s: unexpected exception: %s\n", c.name, e.what());
      ++th::failures();
    }
    ++cases;
    std::printf("[%s] %s\n", th::failures() == before ? " ok " : "FAIL", c.name);
  }
  std::printf("%d cases, %d failed checks\n", cases, th::failures());
  return th::failures() == 0 ? 0 : 1;
}
