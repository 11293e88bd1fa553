// Small dense SVD (K14), column-ring variant for small l — replaces LAPACK
// dgesdd (ffsrqr/svd.py:79) like ffb_jacobi.cu, with a different mapping.
//
// One-sided (Hestenes) Jacobi with ONE LANE GROUP PER COLUMN PAIR (G = 4..32
// lanes of a warp).  The whole l x l iterate M and the accumulated rotations V
// live in the distributed shared memory of one thread-block cluster (<= 16
// CTAs); nothing touches global memory between the load and the write-out.  The
// pair schedule is the odd-even transposition ring: even rounds pair slots
// (2k, 2k+1), odd rounds (2k+1, 2k+2), and every rotation swaps its two
// columns, so after n rounds every pair of columns has met exactly once (one
// sweep).  A pair needs only its own two columns, so a round is
//     load 2 columns (registers) -> 3 dot products -> log2(G) shuffle stages ->
//     rotation (every lane, no broadcast) -> rotate M and V columns -> store
// and one __syncthreads.  The only inter-CTA traffic is the one column per CTA
// boundary that crosses it each round, PUSHED into the neighbour's shared
// memory with st.async (a halo slot on the way down, slot 0 on the way up) and
// counted by the receiver's mbarrier: every load is CTA-local and there is no
// fence or cluster barrier inside a sweep.
//
// Against the block kernel (16-column blocks, Gram + two-sided 32 x 32 chain +
// DMMA apply per visit) the serial depth per sweep is the same n rotation
// steps; a step here is one ~500-cycle dependent chain instead of ~1750 cycles,
// but every column crosses shared memory every round (128 B/clk per SM), which
// bounds the useful size: l <= kRingMaxL uses this kernel, larger l the block
// kernels (measured: profiles/r05_jacobi_ring.txt).
#include <math.h>

#include <algorithm>
#include <stdio.h>
#include <stdlib.h>

#include "ffb_common.cuh"
#include "ffb_jacobi.cuh"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace ffb {

namespace {

struct RingArgs {
  const double* M;   // l x l column-major input
  int64_t ldm;
  int l;
  int transpose;     // iterate on M^T (columns = rows of M)
  int nslots;        // l rounded up to even
  int spc;           // slots per CTA (even)
  int rs;            // shared-memory column stride (doubles), >= rows
  double tol;
  int max_sweeps;
  double* Mo;        // rows x nslots column-major (rows = G RPL): final M columns
  double* Vo;        // rows x nslots: accumulated rotations
  double* nrm;       // nslots: column norms of the final M (prescaled)
  double* offmax;    // [max_sweeps]
  int* sweeps;       // [0] sweeps executed, [1] prescale exponent (input)
  long long* prof;
};

// Rotation (c, s) that orthogonalises two columns with Gram entries (aa, bb,
// cc): tan(theta) = sign(d) g / (|d| + h), d = bb - aa, g = 2 cc, h = hypot(d, g)
// — the smaller root, as ffsrqr's LAPACK would choose.  The angle is formed in
// fp32 from power-of-two-normalised (d, g) with two MUFU.RSQ:
//   c = sqrt((h + |d|) / 2h),  s = sign(d) g / (2 h c)
// and (c, s) is renormalised in fp64 (second-order series of 1/sqrt(c^2 + s^2)),
// so the rotation is orthogonal to working precision; the fp32 angle only sets
// how much of x^T y one step removes.  Threshold test in fp64, no square roots.
FFB_DEV bool ring_rotation(double aa, double bb, double cc, double tol2, double& c, double& s) {
  c = 1.0;
  s = 0.0;
  if (!(cc * cc > tol2 * (aa * bb))) return false;
  const double d = bb - aa, g = cc + cc;
  // 2^-e with 2^e <= |d| + |g| < 2^(e+1): the fp32 inputs land in [-2, 2]
  const int ex = (__double2hiint(fabs(d) + fabs(g)) >> 20) & 0x7ff;
  const double scale = __hiloint2double((2046 - ex) << 20, 0);
  const float df = (float)(d * scale), gf = (float)(g * scale);
  const float rh = rsqrtf(fmaf(df, df, gf * gf));
  const float c2 = fmaf(0.5f * fabsf(df), rh, 0.5f);
  const float rc = rsqrtf(c2);
  const float cf = c2 * rc;
  const float sf = copysignf(0.5f * rh * rc, df) * gf;
  const double cd = (double)cf, sd = (double)sf;
  const double e = fma(sd, sd, fma(cd, cd, -1.0));   // c^2 in [0.5, 1]: c^2 - 1 is exact
  const double r = fma(e, fma(e, 0.375, -0.5), 1.0);
  c = cd * r;
  s = sd * r;
  return true;
}

// whole-cluster barrier (sweep verdicts, start and end only)
template <bool CL>
FFB_DEV void ring_barrier() {
  if (CL) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  } else {
    __syncthreads();
  }
}

// address of the same shared-memory location in CTA `rank` of the cluster
FFB_DEV uint32_t ring_mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}

// push 8 bytes into a peer's shared memory; the peer's mbarrier counts them
// (no fence: the consumer's mbarrier wait is the acquire)
FFB_DEV void ring_push(uint32_t raddr, double v, uint32_t rmbar) {
  asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];\n" ::"r"(raddr),
               "l"(__double_as_longlong(v)), "r"(rmbar)
               : "memory");
}

FFB_DEV void ring_mbar_init(uint32_t mb, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(mb), "r"(count) : "memory");
}

FFB_DEV void ring_mbar_expect(uint32_t mb, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(bytes) : "memory");
}

FFB_DEV void ring_mbar_wait(uint32_t mb, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "RING_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra RING_DONE;\n"
      "bra RING_WAIT;\n"
      "RING_DONE:\n"
      "}\n" ::"r"(mb),
      "r"(parity)
      : "memory");
}

constexpr int kRingMaxWarps = 16;
constexpr int kRingMaxL = 448;

// G lanes per pair, RPL rows per lane (rows = G RPL >= l).  A warp holds 32 / G
// pairs; pair pl = warp * (32 / G) + lane / G of CTA c is global pair
// k = c * spc / 2 + pl.
template <int G, int RPL, bool CL>
__global__ void __launch_bounds__(32 * kRingMaxWarps, 1) jacobi_ring_kernel(RingArgs a) {
  extern __shared__ __align__(16) double sm[];
  constexpr int rows = RPL * G;
  constexpr int PPW = 32 / G;
  const int spc = a.spc, ppc = spc >> 1, nslots = a.nslots, l = a.l, rs = a.rs;
  double* Ms = sm;                                  // (spc + 1) slots x rs; slot spc = halo
  double* Vs = Ms + (size_t)(spc + 1) * rs;
  __shared__ unsigned long long s_off[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int gl = lane & (G - 1);                    // lane within the pair's group
  const int pl = warp * PPW + lane / G;             // pair within the CTA
  unsigned crank = 0, csize = 1;
  if (CL) {
    cg::cluster_group cl = cg::this_cluster();
    crank = cl.block_rank();
    csize = cl.num_blocks();
  }
  const int slot0 = (int)crank * spc;
  const double tol2 = a.tol * a.tol;
  {
    const double sc = ldexp(1.0, -a.sweeps[1]);
    for (int ls = warp; ls <= spc; ls += nwarps) {
      const int gs = slot0 + ls;
      for (int i = lane; i < rows; i += 32) {
        double m = 0.0;
        if (ls < spc && gs < l && i < l)
          m = sc * (a.transpose ? a.M[gs + (int64_t)i * a.ldm] : a.M[i + (int64_t)gs * a.ldm]);
        Ms[(size_t)ls * rs + i] = m;
        Vs[(size_t)ls * rs + i] = (ls < spc && gs < l && i == gs) ? 1.0 : 0.0;
      }
    }
    if (tid == 0) s_off[0] = s_off[1] = 0ull;
  }
  // Boundary columns are PUSHED into the neighbour's shared memory with
  // st.async; the receiving CTA's mbarrier counts the bytes, so the consumer
  // warp's wait is the only synchronisation (no fence, no cluster barrier per
  // round).  mb[0]: my halo (filled by the CTA above in even rounds), mb[1]: my
  // slot 0 (filled by the CTA below in odd rounds).  The two pairs on a
  // boundary strictly alternate (each push follows the read of the previous
  // delivery), so a slot is never overwritten before it has been read.
  __shared__ __align__(8) unsigned long long s_mb[2];
  const uint32_t mb_halo = smem_u32(&s_mb[0]), mb_s0 = smem_u32(&s_mb[1]);
  uint32_t r_halo_M = 0, r_halo_V = 0, r_halo_mb = 0;   // the CTA below: its halo
  uint32_t r_s0_M = 0, r_s0_V = 0, r_s0_mb = 0;         // the CTA above: its slot 0
  if (CL) {
    if (tid == 0) {
      ring_mbar_init(mb_halo, 1);
      ring_mbar_init(mb_s0, 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (crank > 0) {
      r_halo_M = ring_mapa(smem_u32(Ms + (size_t)spc * rs), crank - 1);
      r_halo_V = ring_mapa(smem_u32(Vs + (size_t)spc * rs), crank - 1);
      r_halo_mb = ring_mapa(mb_halo, crank - 1);
    }
    if (crank + 1 < csize) {
      r_s0_M = ring_mapa(smem_u32(Ms), crank + 1);
      r_s0_V = ring_mapa(smem_u32(Vs), crank + 1);
      r_s0_mb = ring_mapa(mb_s0, crank + 1);
    }
  }
  ring_barrier<CL>();

  const int k = (int)crank * ppc + pl;
  const bool mine = pl < ppc;                                   // the group holds a pair of this CTA
  constexpr uint32_t kPushBytes = 2u * rows * sizeof(double);   // one column of M and of V
  // boundary roles (fixed for the whole run).  The WARP holding the first / last
  // pair waits for the deliveries (warp-uniform), the pair's group pushes.
  const int k_first = (int)crank * ppc, k_last = k_first + ppc - 1;
  const bool recv_s0 = CL && warp == 0 && crank > 0 && 2 * k_first + 1 < nslots;               // even rounds
  const bool recv_halo = CL && warp == (ppc - 1) / PPW && 2 * k_last + 2 < nslots;             // odd rounds
  const bool first_pair = CL && mine && pl == 0 && crank > 0;
  const bool last_pair = CL && mine && pl == ppc - 1;
  uint32_t ph_s0 = 0, ph_halo = 0;   // phases consumed so far (parity = & 1)
  bool first_even = true;            // round 0 reads the loaded slot 0, not a delivery
  long long tp[4] = {0, 0, 0, 0};
  int sweep = 0;
  for (; sweep < a.max_sweeps; ++sweep) {
    if (tid == 0) s_off[sweep & 1] = 0ull;
    double offn = 0.0, offd = 1.0;   // running max of cc^2 / (aa bb) over rotated pairs
    for (int r = 0; r < nslots; ++r) {
      const int par = r & 1;
      long long t0 = 0;
      if (a.prof) t0 = clock64();
      if (CL) {
        // wait for the column the neighbour pushed last round
        if (par == 0 && recv_s0 && !first_even) {
          if (lane == 0) ring_mbar_expect(mb_s0, kPushBytes);
          ring_mbar_wait(mb_s0, ph_s0 & 1);
          ++ph_s0;
        }
        if (par == 1 && recv_halo) {
          if (lane == 0) ring_mbar_expect(mb_halo, kPushBytes);
          ring_mbar_wait(mb_halo, ph_halo & 1);
          ++ph_halo;
        }
      }
      const bool active = mine && 2 * k + par + 1 < nslots;   // the pair's second slot exists
      // inactive groups run the arithmetic on slot 0 / 1 (no stores): the
      // shuffles below need every lane of the warp
      const int lA = active ? 2 * pl + par : 0, lB = lA + 1;   // lB == spc: the halo
      const double* pA = Ms + (size_t)lA * rs + gl;
      const double* pB = Ms + (size_t)lB * rs + gl;
      const double* vA = Vs + (size_t)lA * rs + gl;
      const double* vB = Vs + (size_t)lB * rs + gl;
      double x[RPL], y[RPL], vx[RPL], vy[RPL];
#pragma unroll
      for (int q = 0; q < RPL; ++q) {
        x[q] = pA[G * q];
        y[q] = pB[G * q];
      }
      // tall columns: V is loaded after M has been stored (register budget)
      constexpr bool kLateV = RPL > 10;
      if (!kLateV) {
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
          vx[q] = vA[G * q];
          vy[q] = vB[G * q];
        }
      }
      double aa0 = 0.0, bb0 = 0.0, cc0 = 0.0, aa1 = 0.0, bb1 = 0.0, cc1 = 0.0;
#pragma unroll
      for (int q = 0; q < RPL; ++q) {
        if (q & 1) {
          aa1 = fma(x[q], x[q], aa1);
          bb1 = fma(y[q], y[q], bb1);
          cc1 = fma(x[q], y[q], cc1);
        } else {
          aa0 = fma(x[q], x[q], aa0);
          bb0 = fma(y[q], y[q], bb0);
          cc0 = fma(x[q], y[q], cc0);
        }
      }
      double aa = aa0 + aa1, bb = bb0 + bb1, cc = cc0 + cc1;
      // xor butterfly inside the group: every lane ends with the same bits
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) {
        aa += __shfl_xor_sync(0xffffffffu, aa, o);
        bb += __shfl_xor_sync(0xffffffffu, bb, o);
        cc += __shfl_xor_sync(0xffffffffu, cc, o);
      }
      // (c, s) = (1, 0) when the pair passes the threshold test: the updates
      // below then reproduce x and y bit for bit (finite inputs), no selects
      double c, s;
      if (ring_rotation(aa, bb, cc, tol2, c, s) && active) {
        const double c2 = cc * cc, den = aa * bb;
        if (c2 * offd > offn * den) {
          offn = c2;
          offd = den;
        }
      }
      const double ms = -s;
      if (active) {
        // destinations: rotated x -> slot sB, rotated y -> slot sA (the swap)
        const bool push_dn = first_pair && par == 0;   // my slot 0 is read next by the CTA below
        const bool push_up = last_pair && par == 1;    // halo pair: the second column goes home
        double* dA_M = Ms + (size_t)lA * rs + gl;
        double* dB_M = Ms + (size_t)lB * rs + gl;
        double* dA_V = Vs + (size_t)lA * rs + gl;
        double* dB_V = Vs + (size_t)lB * rs + gl;
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
          const double xn = fma(c, x[q], ms * y[q]);
          const double yn = fma(s, x[q], c * y[q]);
          if (push_up) ring_push(r_s0_M + 8u * (gl + G * q), xn, r_s0_mb);
          else dB_M[G * q] = xn;
          if (push_dn) ring_push(r_halo_M + 8u * (gl + G * q), yn, r_halo_mb);
          else dA_M[G * q] = yn;
        }
        if (kLateV) {
#pragma unroll
          for (int q = 0; q < RPL; ++q) {
            vx[q] = vA[G * q];
            vy[q] = vB[G * q];
          }
        }
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
          const double xn = fma(c, vx[q], ms * vy[q]);
          const double yn = fma(s, vx[q], c * vy[q]);
          if (push_up) ring_push(r_s0_V + 8u * (gl + G * q), xn, r_s0_mb);
          else dB_V[G * q] = xn;
          if (push_dn) ring_push(r_halo_V + 8u * (gl + G * q), yn, r_halo_mb);
          else dA_V[G * q] = yn;
        }
      }
      if (a.prof) tp[0] += clock64() - t0;
      if (par == 0) first_even = false;
      long long t1 = 0;
      if (a.prof) t1 = clock64();
      __syncthreads();   // CTA-local hand-over of every other column
      if (a.prof) tp[1] += clock64() - t1;
    }
    // the last (odd) round pushed slot 0s upward: take delivery before anyone
    // reads the sweep's final state (next sweep's round 0, or the write-out)
    if (recv_s0) {
      if (lane == 0) ring_mbar_expect(mb_s0, kPushBytes);
      ring_mbar_wait(mb_s0, ph_s0 & 1);
      ++ph_s0;
    }
    first_even = true;
    // sweep verdict: the largest |cos| any pair rotated, maximised over the cluster
    double off = offn > 0.0 ? sqrt(offn / offd) : 0.0;
    if (gl == 0 && off > 0.0) atomicMax(&s_off[sweep & 1], (unsigned long long)__double_as_longlong(off));
    ring_barrier<CL>();
    unsigned long long ob = s_off[sweep & 1];
    if (CL) {
      cg::cluster_group cl = cg::this_cluster();
      for (unsigned c2 = 0; c2 < csize; ++c2) {
        const unsigned long long v = *cl.map_shared_rank(&s_off[sweep & 1], c2);
        ob = v > ob ? v : ob;
      }
    }
    const double om = __longlong_as_double((long long)ob);
    if (tid == 0 && crank == 0) a.offmax[sweep] = om;
    // converged when no pair exceeded tol; a sweep whose largest |cos| was below
    // 1e-8 leaves only second-order off-diagonal mass (quadratic convergence)
    if (!(om > a.tol) || om < 1e-8) {
      ++sweep;
      break;
    }
  }
  if (tid == 0 && crank == 0) a.sweeps[0] = sweep;
  // write-out: fresh norms of the final columns, M and V column-major
  ring_barrier<CL>();   // peers finished reading s_off; every home slot is final
  for (int ls = warp; ls < spc; ls += nwarps) {
    const int gs = slot0 + ls;
    if (gs >= nslots) continue;
    double t0 = 0.0;
    for (int i = lane; i < rows; i += 32) {
      const double xv = Ms[(size_t)ls * rs + i];
      t0 = fma(xv, xv, t0);
      a.Mo[(size_t)gs * rows + i] = xv;
      a.Vo[(size_t)gs * rows + i] = Vs[(size_t)ls * rs + i];
    }
    const double t = warp_sum(t0);
    if (lane == 0) a.nrm[gs] = sqrt(t);
  }
  if (a.prof && tid == 0 && crank == 0) {
    a.prof[0] = tp[0];
    a.prof[1] = tp[1];
  }
  if (CL) ring_barrier<CL>();   // no CTA exits while a peer may still address it
}

// rank sort of the slots' norms (descending, ties by slot; NaN last): the l
// leading slots -> order, sig (unscaled), sorted norms.  With l odd the zero
// padding column sits in an arbitrary slot after the swaps; it ranks last.
__global__ void ring_rank_kernel(const double* nrm, int l, int nslots, const int* sweeps, double* sig,
                                 int* order, double* nrm_sorted) {
  extern __shared__ double sn[];
  const int tid = threadIdx.x;
  for (int j = tid; j < nslots; j += blockDim.x) sn[j] = nrm[j];
  __syncthreads();
  const double unscale = ldexp(1.0, sweeps[1]);
  auto key = [](double v) { return v == v ? v : -1.0; };
  for (int j = tid; j < nslots; j += blockDim.x) {
    int rank = 0;
    const double sj = key(sn[j]);
    for (int q = 0; q < nslots; ++q) {
      const double kq = key(sn[q]);
      rank += (kq > sj) || (kq == sj && q < j);
    }
    if (rank < l) {
      order[rank] = j;
      sig[rank] = sn[j] * unscale;
      nrm_sorted[rank] = sn[j];
    }
  }
}

// left[:, r] = Mo[:, order[r]] / nrm[r] (zero column when nrm == 0), right[:, r] = Vo[:, order[r]]
__global__ void ring_out_kernel(const double* Mo, const double* Vo, int rows, int l, const int* order,
                                const double* nrm_sorted, double* left, int64_t ldl, double* right,
                                int64_t ldr) {
  const int64_t total = (int64_t)l * l;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx / l), i = (int)(idx - (int64_t)r * l);
    const int j = order[r];
    const double s = nrm_sorted[r];
    left[i + (int64_t)r * ldl] = s > 0.0 ? Mo[(size_t)j * rows + i] / s : 0.0;
    right[i + (int64_t)r * ldr] = Vo[(size_t)j * rows + i];
  }
}

template <int G, int RPL>
void* ring_kernel_ptr(bool cl) {
  return cl ? (void*)jacobi_ring_kernel<G, RPL, true> : (void*)jacobi_ring_kernel<G, RPL, false>;
}

template <int G>
void* ring_kernel_rpl(int rpl, bool cl) {
  switch (rpl) {
    case 1: return ring_kernel_ptr<G, 1>(cl);
    case 2: return ring_kernel_ptr<G, 2>(cl);
    case 3: return ring_kernel_ptr<G, 3>(cl);
    case 4: return ring_kernel_ptr<G, 4>(cl);
    case 5: return ring_kernel_ptr<G, 5>(cl);
    case 6: return ring_kernel_ptr<G, 6>(cl);
    case 7: return ring_kernel_ptr<G, 7>(cl);
    case 8: return ring_kernel_ptr<G, 8>(cl);
    case 9: return ring_kernel_ptr<G, 9>(cl);
    case 10: return ring_kernel_ptr<G, 10>(cl);
    case 11: return ring_kernel_ptr<G, 11>(cl);
    case 12: return ring_kernel_ptr<G, 12>(cl);
    case 13: return ring_kernel_ptr<G, 13>(cl);
    case 14: return ring_kernel_ptr<G, 14>(cl);
    default: return nullptr;
  }
}

void* ring_kernel_for(int g, int rpl, bool cl) {
  switch (g) {
    case 4: return ring_kernel_rpl<4>(rpl, cl);
    case 8: return ring_kernel_rpl<8>(rpl, cl);
    case 16: return ring_kernel_rpl<16>(rpl, cl);
    case 32: return ring_kernel_rpl<32>(rpl, cl);
    default: return nullptr;
  }
}

struct RingGeom {
  int g, rpl, rows, rs, nslots, C, spc, warps;
  size_t smem;
};

// lanes per pair G, cluster size C (1, 2, 4, 8, 16) and slots per CTA
bool ring_geometry(int l, int sms, RingGeom& o) {
  if (l < 2 || l > kRingMaxL) return false;
  o.nslots = l + (l & 1);
  const int pairs = o.nslots / 2;
  // G: a whole warp per pair unless the columns are shorter than that — fewer
  // rows per lane measured faster than fewer shuffle stages (l = 60: G = 32
  // 0.39 ms, G = 16 0.49 ms, G = 8 0.51 ms).  FFB_RING_G overrides (tests).
  int g = l > 16 ? 32 : l > 8 ? 16 : 8;
  if (const char* e = getenv("FFB_RING_G")) {
    const int v = atoi(e);
    if (v == 4 || v == 8 || v == 16 || v == 32) g = v;
  }
  o.g = g;
  o.rpl = (l + g - 1) / g;
  if (o.rpl > 14) return false;
  o.rows = o.rpl * g;
  // column stride: groups of one shared-memory wavefront (16 lanes) must hit
  // distinct banks; consecutive pairs are 2 columns apart, so for G <= 8 the
  // stride is G / 2 (mod 8) doubles
  o.rs = o.rows;
  if (g <= 8)
    while (o.rs % 8 != g / 2) ++o.rs;
  // C: about 4 pairs per CTA (one per scheduler) up to the 16-CTA cluster, and no
  // more CTAs than the caller's SM budget; FFB_RING_C / FFB_RING_PPC override
  int ppc_target = 4;
  if (const char* e = getenv("FFB_RING_PPC")) ppc_target = std::max(1, atoi(e));
  int C = 1;
  while (C < 16 && 2 * C <= sms && (pairs + C - 1) / C > ppc_target) C *= 2;
  if (const char* e = getenv("FFB_RING_C")) {
    const int c = atoi(e);
    if (c == 1 || c == 2 || c == 4 || c == 8 || c == 16) C = c;
  }
  o.C = C;
  const int ppc = (pairs + C - 1) / C;
  o.spc = 2 * ppc;
  o.warps = (ppc * g + 31) / 32;
  if (o.warps > kRingMaxWarps) return false;
  // every CTA but the last is full and a CTA with slots has at least 2 (nslots
  // and spc are even).  Shared memory: (spc + 1) slots x rs x (M + V).
  o.smem = (size_t)(o.spc + 1) * o.rs * 2 * sizeof(double);
  return o.smem <= 220 * 1024;
}

}  // namespace

bool jacobi_ring_supported(int l, int sms) {
  RingGeom g;
  int lmax = 160;   // measured crossover against the block kernel (profiles/r05_jacobi_ring.txt)
  if (const char* e = getenv("FFB_RING_MAXL")) lmax = atoi(e);
  return l <= lmax && ring_geometry(l, sms, g);
}

cudaError_t launch_jacobi_ring(cudaStream_t st, int sms, const double* M, int64_t ldm, int l,
                               double* sig, double* U, int64_t ldu, double* Vout, int64_t ldvo,
                               double* work, double* offmax, int* sweeps, int* order,
                               int max_sweeps) {
  RingGeom gm;
  if (!ring_geometry(l, sms, gm)) return cudaErrorInvalidValue;
  const int rows = gm.rows, nslots = gm.nslots;
  double* Mo = work;
  double* Vo = Mo + (size_t)rows * nslots;
  double* nrm = Vo + (size_t)rows * nslots;
  double* nrm_sorted = nrm + nslots;
  static long long* prof = nullptr;
  if (getenv("FFB_JACOBI_PROF") && !prof) cudaMallocManaged(&prof, 8 * sizeof(long long));
  const int transpose = getenv("FFB_RING_NOTRANS") ? 0 : 1;
  RingArgs a{M, ldm, l, transpose, nslots, gm.spc, gm.rs, 1e-15 * sqrt((double)l), max_sweeps,
             Mo, Vo, nrm, offmax, sweeps, prof};
  const bool cl = gm.C > 1;
  void* kern = ring_kernel_for(gm.g, gm.rpl, cl);
  if (!kern) return cudaErrorInvalidValue;
  static std::atomic<unsigned long long> attr_done[2][4][15];
  const int gi = gm.g == 4 ? 0 : gm.g == 8 ? 1 : gm.g == 16 ? 2 : 3;
  cudaError_t e = ensure_smem_optin(kern, 226 * 1024, attr_done[cl][gi][gm.rpl]);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(offmax, 0, sizeof(double) * max_sweeps, st);
  if (e != cudaSuccess) return e;
  launch_jacobi_scale(st, M, ldm, l, sweeps);
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  if (prof) {
    cudaEventCreate(&ev0);
    cudaEventCreate(&ev1);
    cudaEventRecord(ev0, st);
  }
  void* args[] = {&a};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(gm.C);
  cfg.blockDim = dim3(32 * gm.warps);
  cfg.dynamicSmemBytes = gm.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = gm.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = cl ? 1 : 0;
  if (gm.C > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  e = cudaLaunchKernelExC(&cfg, kern, args);
  if (e != cudaSuccess) return e;
  if (prof) cudaEventRecord(ev1, st);
  ring_rank_kernel<<<1, 512, sizeof(double) * (size_t)nslots, st>>>(nrm, l, nslots, sweeps, sig, order, nrm_sorted);
  int g = (int)(((int64_t)l * l + 255) / 256);
  if (g > 4 * sms) g = 4 * sms;
  // iterating on M^T: M^T V' = U' S, so M = V' S U'^T — the accumulated rotations
  // are M's LEFT vectors and the normalised columns its right vectors
  if (transpose)
    ring_out_kernel<<<g, 256, 0, st>>>(Mo, Vo, rows, l, order, nrm_sorted, Vout, ldvo, U, ldu);
  else
    ring_out_kernel<<<g, 256, 0, st>>>(Mo, Vo, rows, l, order, nrm_sorted, U, ldu, Vout, ldvo);
  if (prof) {
    cudaStreamSynchronize(st);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev0, ev1);
    int nsw = 0;
    cudaMemcpy(&nsw, sweeps, sizeof(int), cudaMemcpyDeviceToHost);
    const double rounds = (double)nsw * nslots;
    fprintf(stderr,
            "jacobi ring l=%d G=%d rpl=%d C=%d spc=%d warps=%d: %.3f ms, %d sweeps, %.0f cycles/round at 1.965 GHz "
            "(CTA 0 warp 0: pair %.0f, barrier issue %.0f)\n",
            l, gm.g, gm.rpl, gm.C, gm.spc, gm.warps, ms, nsw, ms * 1.965e6 / rounds, prof[0] / rounds,
            prof[1] / rounds);
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
  }
  return cudaGetLastError();
}

}  // namespace ffb
