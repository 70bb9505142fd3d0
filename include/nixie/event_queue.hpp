// nixie-b200 — deterministic virtual clock. Drop-in for
// proj/include/nixie/event_queue.hpp:12-59: events fire in (time, insertion
// sequence) order, run_until() discards events past the horizon.
//
// Used by the parity mode of the Orchestrator (the model link backend) and by
// the scenario driver; the CUDA swap engine runs on the wall clock instead.
#pragma once

#include <cstdint>
#include <functional>
#include <utility>
#include <vector>

#include "nixie/units.hpp"

namespace nixie {

class EventQueue {
 public:
  void at(Seconds t, std::function<void()> fn) { push(Slot{t, next_seq_++, std::move(fn)}); }
  void after(Seconds dt, std::function<void()> fn) { at(now_ + dt, std::move(fn)); }

  Seconds now() const { return now_; }
  bool empty() const { return heap_.empty(); }
  std::size_t pending() const { return heap_.size(); }

  // Pops and runs the earliest event; false when nothing is queued.
  bool run_one() {
    if (heap_.empty()) return false;
    Slot s = pop();
    now_ = s.t;
    s.fn();
    return true;
  }

  void run_until(Seconds horizon) {
    while (!heap_.empty() && heap_.front().t <= horizon) run_one();
    heap_.clear();
    now_ = horizon;
  }

  void run_all() {
    while (run_one()) {
    }
  }

 private:
  struct Slot {
    Seconds t;
    std::uint64_t seq;
    std::function<void()> fn;
  };
  static bool earlier(const Slot& a, const Slot& b) { return a.t < b.t || (a.t == b.t && a.seq < b.seq); }

  // Hand-rolled binary min-heap on (t, seq).
  void push(Slot s) {
    heap_.push_back(std::move(s));
    std::size_t i = heap_.size() - 1;
    while (i > 0) {
      std::size_t parent = (i - 1) / 2;
      if (!earlier(heap_[i], heap_[parent])) break;
      std::swap(heap_[i], heap_[parent]);
      i = parent;
    }
  }
  Slot pop() {
    Slot top = std::move(heap_.front());
    heap_.front() = std::move(heap_.back());
    heap_.pop_back();
    std::size_t i = 0, n = heap_.size();
    while (true) {
      std::size_t l = 2 * i + 1, r = l + 1, m = i;
      if (l < n && earlier(heap_[l], heap_[m])) m = l;
      if (r < n && earlier(heap_[r], heap_[m])) m = r;
      if (m == i) break;
      std::swap(heap_[i], heap_[m]);
      i = m;
    }
    return top;
  }

  std::vector<Slot> heap_;
  std::uint64_t next_seq_ = 0;
  Seconds now_ = 0;
};

}  // namespace nixie
