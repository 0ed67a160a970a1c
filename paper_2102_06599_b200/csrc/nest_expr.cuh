// Device evaluator of the bridge's postfix affine programs (nb_nest_expr,
// include/nb200.h): AffineExpr (I/affine.hpp:17-111) -- const, slot, n-ary
// add, mul / floor-div / floor-mod by a constant.  Shared by the nest
// executor (nest.cu) and the semantic-legality check (legality.cu).
#pragma once

#include <cstdint>

namespace nb {
namespace nexpr {

constexpr int kStack = 16;

__device__ __forceinline__ int64_t floor_div(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}

__device__ __forceinline__ int64_t run(const int64_t* __restrict__ code, int off, const int64_t* vals) {
  int64_t st[kStack];
  int sp = 0;
  const int64_t* c = code + 2 * off;
  // program length is stored as the op count in the first pair: (nops, 0)
  const int nops = int(c[0]);
  c += 2;
  for (int i = 0; i < nops; ++i) {
    const int64_t op = c[2 * i], arg = c[2 * i + 1];
    switch (op) {
      case 0: st[sp++] = arg; break;
      case 1: st[sp++] = vals[arg]; break;
      case 2: {
        int64_t s = 0;
        for (int k = 0; k < arg; ++k) s += st[--sp];
        st[sp++] = s;
        break;
      }
      case 3: st[sp - 1] *= arg; break;
      case 4: st[sp - 1] = floor_div(st[sp - 1], arg); break;
      default: st[sp - 1] = st[sp - 1] - floor_div(st[sp - 1], arg) * arg; break;
    }
  }
  return st[sp - 1];
}

}  // namespace nexpr
}  // namespace nb
