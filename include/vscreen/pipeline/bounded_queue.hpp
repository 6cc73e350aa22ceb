// Drop-in for the reference's BoundedQueue (bounded_queue.hpp): a bounded
// multi-producer / multi-consumer queue whose close() wakes every waiter.
// Same interface (push, pop, close, high_water), plus try_pop(), which the
// B200 docker_worker uses to drain whatever is queued into one GPU batch.
#pragma once

#include <condition_variable>
#include <cstddef>
#include <deque>
#include <mutex>
#include <optional>

#include "vscreen/error.hpp"

namespace vscreen {

template <typename T>
class BoundedQueue {
 public:
  explicit BoundedQueue(std::size_t capacity) : cap_(capacity) {
    if (capacity == 0) throw InvalidArgument("queue capacity must be positive");
  }
  BoundedQueue(const BoundedQueue &) = delete;
  BoundedQueue &operator=(const BoundedQueue &) = delete;

  // Blocks while full; false once the queue is closed (the value is dropped).
  bool push(T value) {
    std::unique_lock<std::mutex> lk(mu_);
    space_.wait(lk, [&] { return closed_ || q_.size() < cap_; });
    if (closed_) return false;
    q_.push_back(std::move(value));
    high_ = q_.size() > high_ ? q_.size() : high_;
    lk.unlock();
    data_.notify_one();
    return true;
  }

  // Blocks while empty and open; nullopt once closed and drained.
  std::optional<T> pop() {
    std::unique_lock<std::mutex> lk(mu_);
    data_.wait(lk, [&] { return closed_ || !q_.empty(); });
    return take(lk);
  }

  // Never blocks: the next item if one is queued.
  std::optional<T> try_pop() {
    std::unique_lock<std::mutex> lk(mu_);
    return take(lk);
  }

  void close() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      closed_ = true;
    }
    data_.notify_all();
    space_.notify_all();
  }

  std::size_t high_water() const {
    std::lock_guard<std::mutex> lk(mu_);
    return high_;
  }

 private:
  std::optional<T> take(std::unique_lock<std::mutex> &lk) {
    if (q_.empty()) return std::nullopt;
    std::optional<T> v(std::move(q_.front()));
    q_.pop_front();
    lk.unlock();
    space_.notify_one();
    return v;
  }

  mutable std::mutex mu_;
  std::condition_variable data_, space_;
  std::deque<T> q_;
  std::size_t cap_, high_ = 0;
  bool closed_ = false;
};

}  // namespace vscreen
