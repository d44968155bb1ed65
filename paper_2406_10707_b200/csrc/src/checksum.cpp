// Interleaved FNV-1a helper; see include/lzckpt/checksum.hpp.
#include "lzckpt/checksum.hpp"

#include <algorithm>

namespace lzckpt {

void fnv64_fold_x4(uint64_t h[4], const unsigned char* const p[4], const size_t n[4]) {
  constexpr uint64_t P = Fnv64::kPrime;
  const size_t common = std::min(std::min(n[0], n[1]), std::min(n[2], n[3]));
  uint64_t a = h[0], b = h[1], c = h[2], d = h[3];
  const unsigned char *pa = p[0], *pb = p[1], *pc = p[2], *pd = p[3];
  for (size_t i = 0; i < common; ++i) {
    a = (a ^ pa[i]) * P;
    b = (b ^ pb[i]) * P;
    c = (c ^ pc[i]) * P;
    d = (d ^ pd[i]) * P;
  }
  h[0] = Fnv64::fold(a, pa + common, n[0] - common);
  h[1] = Fnv64::fold(b, pb + common, n[1] - common);
  h[2] = Fnv64::fold(c, pc + common, n[2] - common);
  h[3] = Fnv64::fold(d, pd + common, n[3] - common);
}

}  // namespace lzckpt
