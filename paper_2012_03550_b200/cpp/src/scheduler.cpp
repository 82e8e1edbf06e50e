// scheduler.cpp -- partition_even / reduce_in_order (exact reference
// semantics, scheduler.cpp:34-46,96-104) and the API-parity WorkerPool.
#include "sptucker/scheduler.hpp"

#include <exception>

#include "../../../include/sgdt.h"

namespace sptucker {

Strategy parse_strategy(const std::string& s) {
  if (s == "serial") return Strategy::Serial;
  if (s == "naive") return Strategy::Naive;
  if (s == "improved") return Strategy::Improved;
  throw ConfigError("unknown strategy '" + s + "' (serial|naive|improved)");
}

BalancePolicy parse_balance(const std::string& s) {
  if (s == "static") return BalancePolicy::Static;
  if (s == "dynamic") return BalancePolicy::Dynamic;
  throw ConfigError("unknown balance policy '" + s + "' (static|dynamic)");
}

std::string to_string(Strategy s) {
  return s == Strategy::Serial ? "serial" : (s == Strategy::Naive ? "naive" : "improved");
}

std::string to_string(BalancePolicy p) { return p == BalancePolicy::Static ? "static" : "dynamic"; }

std::vector<Range> partition_even(std::size_t count, std::size_t workers) {
  if (workers < 1) throw DomainError("partition_even: need at least one worker");
  std::vector<std::uint64_t> b(workers), e(workers);
  sgdt_partition_even(count, workers, b.data(), e.data());
  std::vector<Range> out(workers);
  for (std::size_t w = 0; w < workers; ++w) out[w] = {static_cast<std::size_t>(b[w]), static_cast<std::size_t>(e[w])};
  return out;
}

void reduce_in_order(std::span<const std::vector<double>> partials, std::vector<double>& out) {
  if (partials.empty()) throw InternalError("reduce_in_order: no partials");
  const std::size_t n = partials.front().size();
  out.assign(n, 0.0);
  for (const auto& p : partials) {
    if (p.size() != n) throw InternalError("reduce_in_order: shape mismatch");
    for (std::size_t i = 0; i < n; ++i) out[i] += p[i];
  }
}

void WorkerPool::run(const std::function<void(std::size_t)>& task) {
  std::exception_ptr first;
  for (std::size_t r = 0; r < size_; ++r) {
    try {
      task(r);
    } catch (...) {
      if (!first) first = std::current_exception();
    }
  }
  if (first) std::rethrow_exception(first);
}

}  // namespace sptucker
