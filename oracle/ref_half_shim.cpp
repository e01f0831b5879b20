// Exposes the reference's own fp16 codec (proj/include/espn/half.hpp:11-76)
// through a C ABI so tests can pin the oracle's codec against it.
// TEST INFRASTRUCTURE ONLY: built into oracle/_ref/ (git-ignored) from the
// header where it lies under /root/reference; nothing is copied into this repo.
#include <bit>
#include <cstdint>
#include "espn/half.hpp"

extern "C" {
std::uint16_t ref_float_to_half(float f) { return espn::float_to_half(f); }
float ref_half_to_float(std::uint16_t h) { return espn::half_to_float(h); }
float ref_half_round_trip(float f) { return espn::half_round_trip(f); }
// Bit-pattern variants: returning a float through a C ABI register quiets
// signalling NaNs (0x7c01.. decode to sNaN in half.hpp:68), so the golden
// generator reads raw bits instead.
std::uint32_t ref_half_to_float_bits(std::uint16_t h) {
  return std::bit_cast<std::uint32_t>(espn::half_to_float(h));
}
std::uint16_t ref_float_bits_to_half(std::uint32_t bits) {
  return espn::float_to_half(std::bit_cast<float>(bits));
}
}
