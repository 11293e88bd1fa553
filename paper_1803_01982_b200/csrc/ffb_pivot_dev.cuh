// Device helpers of the sketch-pivot kernel (ffb_kernels.cu): tagged LL exchange words, the (norm, position) order of
// ffsrqr/_kernels_numba.py:32-37 (largest norm, ties to the lowest position).
#pragma once
#include "ffb_common.cuh"

namespace ffb {

// LL ("low-latency") exchange words: 32-bit payload + 32-bit step tag in one
// single-copy-atomic 64-bit word, so readers validate data by its tag and no
// fence or flag is needed between producer and consumers.
FFB_DEV unsigned long long ll_pack(uint32_t data, uint32_t tag) {
  return ((unsigned long long)tag << 32) | data;
}
FFB_DEV uint32_t ll_tag(unsigned long long w) { return (uint32_t)(w >> 32); }
FFB_DEV uint32_t ll_data(unsigned long long w) { return (uint32_t)w; }
FFB_DEV void st_ll2(unsigned long long* p, unsigned long long x, unsigned long long y) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};\n" ::"l"(p), "l"(x), "l"(y) : "memory");
}
FFB_DEV void ld_ll2(const unsigned long long* p, unsigned long long& x, unsigned long long& y) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(x), "=l"(y) : "l"(p) : "memory");
}

// opaque select: keeps unrolled "pick element q of a register array" chains from
// being turned into a dynamically indexed (local-memory) array by the compiler
FFB_DEV double sel_f64(bool c, double a, double b) {
  double r;
  asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %3, 0;\n\tselp.f64 %0, %1, %2, p;\n\t}"
      : "=d"(r)
      : "d"(a), "d"(b), "r"((unsigned)c));
  return r;
}

// dst = src when c: a predicated move, so an unrolled "pick element q of a
// register array" costs one issue slot per element and no dependent select chain
FFB_DEV void mov_if_f64(double& dst, bool c, double src) {
  asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p mov.f64 %0, %1;\n\t}"
      : "+d"(dst)
      : "d"(src), "r"((unsigned)c));
}

FFB_DEV bool cand_better(double ra, int64_t pa, double rb, int64_t pb) {
  // is (ra, pa) strictly better than (rb, pb)?  pb < 0 means "none"
  if (pa < 0) return false;
  if (pb < 0) return true;
  return ra > rb || (ra == rb && pa < pb);
}


// exact warp argmax: largest r, ties -> lowest position.  r >= 0 for every
// candidate (norms; the downdate clamps at 0), so the IEEE bit pattern orders
// like the value: key = bits + 1 (0 = no candidate), reduced with three redux
// instructions (max hi word, max lo word among the hi winners, min position).
// Positions are < 2^31 (checked at the boundary).
FFB_DEV void warp_best(double& r, int64_t& p) {
  const unsigned long long key =
      p >= 0 ? (unsigned long long)__double_as_longlong(r > 0.0 ? r : 0.0) + 1ull : 0ull;
  const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  const bool top = key != 0ull && hi == mhi && lo == mlo;
  const unsigned pm = __reduce_min_sync(0xffffffffu, top ? (unsigned)p : 0xffffffffu);
  if (pm == 0xffffffffu) {
    r = -1.0;
    p = -1;
  } else {
    r = __longlong_as_double((long long)((((unsigned long long)mhi << 32) | mlo) - 1ull));
    p = (int64_t)pm;
  }
}

}  // namespace ffb
