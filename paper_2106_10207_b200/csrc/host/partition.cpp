// partition.cpp — LP fractions -> aligned contiguous parts (see
// swarmplan/partition.hpp). The same function feeds the GPU executor and the
// CPU oracle's inputs, so part boundaries agree bit for bit by construction.

#include "swarmplan/partition.hpp"

#include <cmath>
#include <stdexcept>

namespace swarmplan {

std::vector<std::int64_t> part_offsets(std::int64_t n, const std::vector<double>& fractions,
                                       std::int64_t align) {
  const int G = static_cast<int>(fractions.size());
  if (G < 1) throw std::invalid_argument("part_offsets: need at least one peer");
  if (n < 0) throw std::invalid_argument("part_offsets: n must be non-negative");
  if (align < 1) throw std::invalid_argument("part_offsets: align must be positive");
  for (double f : fractions)
    if (!(f >= 0.0) || !std::isfinite(f))
      throw std::invalid_argument("part_offsets: fractions must be finite and non-negative");
  std::vector<std::int64_t> off(G + 1, 0);
  double cum = 0.0;
  for (int k = 1; k < G; ++k) {
    cum += fractions[k - 1];
    std::int64_t o = align * std::llround(static_cast<double>(n) * cum / static_cast<double>(align));
    if (o < off[k - 1]) o = off[k - 1];
    if (o > n) o = n;
    off[k] = o;
  }
  off[G] = n;
  return off;
}

}  // namespace swarmplan
