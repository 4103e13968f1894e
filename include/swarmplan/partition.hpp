// swarmplan/partition.hpp — LP fractions -> contiguous part boundaries of the
// flattened vector (new: the reference never materializes parts; the paper
// only says each peer aggregates a share "proportional" to its fraction,
// PAPER.md:142,547; fractions from /root/reference/proj/src/strategy.cpp:473-485).
#pragma once

#include <cstdint>
#include <vector>

namespace swarmplan {

// offsets[0] = 0, offsets[G] = n; inner boundary k is
// clamp(align * llround(n * sum_{i<k} f_i / align), offsets[k-1], n).
// Zero-length parts are allowed (clients, aux-excluded peers).
// std::invalid_argument on negative / non-finite fractions or align < 1.
std::vector<std::int64_t> part_offsets(std::int64_t n, const std::vector<double>& fractions,
                                       std::int64_t align);

}  // namespace swarmplan
