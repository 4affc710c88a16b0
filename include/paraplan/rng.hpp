// paraplan/rng.hpp -- keyed counter-style random stream.
//
// Drop-in for /root/reference/proj/include/paraplan/rng.hpp. The device
// kernel evaluates the same stream in closed form (draw k of a key is
// mix64(key + (k + 1) * gamma)), so host and device candidates agree.
#pragma once

#include <cstdint>

namespace paraplan {

class KeyedRng {
 public:
  KeyedRng(std::uint64_t master_seed, std::uint64_t time_index,
           std::uint64_t restart, std::uint64_t iter, std::uint64_t candidate);

  std::uint64_t next_u64();
  double next_unit();    // [0, 1), 53 bits
  double next_normal();  // Box-Muller, second value of a pair cached

 private:
  std::uint64_t state_ = 0;
  double spare_ = 0.0;
  bool has_spare_ = false;
};

}  // namespace paraplan
