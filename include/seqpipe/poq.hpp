// Partially ordered queue of pending backward units: FIFO over micro-batches,
// LIFO over segments (reference: core/include/seqpipe/poq.hpp:18-31, core/src/poq.cpp).
// The engine's schedule generator does not need it — the op table is a closed
// form (see schedule.hpp) — but the class stays part of the API and is what the
// tests use to prove the closed form equal to the queue-driven order.
#pragma once

#include <cstddef>
#include <cstdint>
#include <set>
#include <utility>

namespace seqpipe {

class PartiallyOrderedQueue {
 public:
  void push(int micro_batch, int segment);   // std::invalid_argument on a duplicate
  std::pair<int, int> pop();                 // std::out_of_range when empty
  bool empty() const { return keys_.empty(); }
  std::size_t size() const { return keys_.size(); }

 private:
  // Key orders entries by (micro_batch asc, segment desc): begin() is the next pop.
  std::set<std::pair<int, int>> keys_;
};

}  // namespace seqpipe
