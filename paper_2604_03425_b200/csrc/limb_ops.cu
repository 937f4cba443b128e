// limb_ops.cu -- the pointwise instruction of the poly IR (PolyOpKind::kLimbMulAdd
// with its LimbOpcode payload, poly_ir.hpp:49-58, lowered per limb by
// HeLowering::pointwise, poly_ir.hpp:192-213) on a FragSpan rectangle:
// lanes [out_lane, out_lane + lanes) x limbs [prime_lo, prime_hi] of a bundle.
//
// These are HBM-streaming kernels (every word read once, written once): a CTA
// owns 1,024 consecutive coefficients of one (lane, limb) row, each thread 4
// contiguous words through 256-bit accesses.  Operand lanes follow the
// emit_per_lane rule (he_ir.hpp:200-222) through LaneMap.  The hot path's own
// fused forms (CAdd, CMult, PMult-acc) live in kernels.cu; this file backs the
// C-ABI's aegis_limb_op / aegis_padd for callers that drive the poly IR
// directly.
#include "kernels.h"

namespace aegis {

namespace {

// opcode values are LimbOpcode's (poly_ir.hpp:49-58)
constexpr int kOpAdd = 1, kOpSub = 2, kOpMul = 3, kOpMulAcc = 4, kOpAddAcc = 5;

struct LimbOpArgs {
  View out;
  u32 out_lane0;
  View a;
  LaneMap ma;
  View b;
  LaneMap mb;
  u32 nlanes, limb_lo, limbs, n;
  u32 out_comps, a_comps, b_comps;  // b_comps = 0: no second operand
};

// one output component c of one coefficient; pt operands (1 comp) broadcast
// over ciphertext components for Mul/MulAcc and feed component 0 for Add/Sub
template <int OP>
__device__ __forceinline__ u64 limb_value(u32 c, const u64* av, const u64* bv, u64 prev, u32 ac, u32 bc, u64 p,
                                          u64 mu) {
  if (OP == kOpAdd || OP == kOpSub) {
    const u64 x = c < ac ? av[c] : 0;
    const u64 y = c < bc ? bv[c] : 0;
    return OP == kOpAdd ? add_mod(x, y, p) : sub_mod(x, y, p);
  }
  if (OP == kOpAddAcc) return c < ac ? add_mod(prev, av[c], p) : prev;
  // Mul / MulAcc
  u64 r;
  if (ac == 2 && bc == 2) {  // ciphertext tensor ("component product", poly_ir.hpp:53)
    if (c == 0) r = mul_mod(av[0], bv[0], p, mu);
    else if (c == 2) r = mul_mod(av[1], bv[1], p, mu);
    else {
      u128 s = mul_wide(av[0], bv[1]);
      mac(s, av[1], bv[0]);
      r = reduce104(s, p, mu);
    }
  } else if (bc == 1) {
    r = mul_mod(av[ac == 1 ? 0 : c], bv[0], p, mu);
  } else {  // ac == 1: plaintext a times ciphertext b
    r = mul_mod(av[0], bv[c], p, mu);
  }
  return OP == kOpMulAcc ? add_mod(prev, r, p) : r;
}

template <int OP>
__global__ void __launch_bounds__(256) limb_op_kernel(LimbOpArgs A, const PrimeConst* __restrict__ pc) {
  const u32 cpr = (A.n + 1023) / 1024;
  const u32 row = blockIdx.x / cpr, chunk = blockIdx.x - row * cpr;
  const u32 lr = row % A.limbs, l = row / A.limbs, lb = A.limb_lo + lr;
  const PrimeConst P = pc[lb];
  const u32 x = (chunk * 256 + threadIdx.x) * 4;
  if (x >= A.n) return;
  const u32 la = A.ma.at(l, A.nlanes);
  u64 av[2][4], bv[2][4];
  for (u32 c = 0; c < A.a_comps; ++c)
    ld256g(A.a.limb(la, c, lb, A.n) + x, av[c][0], av[c][1], av[c][2], av[c][3]);
  if (A.b_comps) {
    const u32 lbb = A.mb.at(l, A.nlanes);
    for (u32 c = 0; c < A.b_comps; ++c)
      ld256g(A.b.limb(lbb, c, lb, A.n) + x, bv[c][0], bv[c][1], bv[c][2], bv[c][3]);
  }
  for (u32 c = 0; c < A.out_comps; ++c) {
    u64* d = A.out.limb(A.out_lane0 + l, c, lb, A.n) + x;
    u64 prev[4] = {0, 0, 0, 0};
    if (OP == kOpMulAcc || OP == kOpAddAcc) ld256g(d, prev[0], prev[1], prev[2], prev[3]);
    u64 r[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const u64 ai[2] = {av[0][i], av[1][i]};
      const u64 bi[2] = {bv[0][i], bv[1][i]};
      r[i] = limb_value<OP>(c, ai, bi, prev[i], A.a_comps, A.b_comps, P.p, P.mu104);
    }
    st256g(d, r[0], r[1], r[2], r[3]);
  }
}

// kGenerate on a limb range: the same rows as the executor's weights
// (tag 2 keyed by (bundle id, lane, comp, absolute limb))
__global__ void __launch_bounds__(256) limb_generate_kernel(View out, u32 out_lane0, u32 nlanes, u32 comps,
                                                            u32 limb_lo, u32 limbs, u32 n, u64 seed, u64 tag,
                                                            u64 bundle, const PrimeConst* __restrict__ pc) {
  const u32 cpr = (n + 1023) / 1024;
  const u32 row = blockIdx.x / cpr, chunk = blockIdx.x - row * cpr;
  const u32 lr = row % limbs, rest = row / limbs, comp = rest % comps, l = rest / comps, lb = limb_lo + lr;
  const PrimeConst P = pc[lb];
  const u64 rk = row_key(seed, tag, bundle, out_lane0 + l, comp, lb);
  const u32 x = (chunk * 256 + threadIdx.x) * 4;
  if (x >= n) return;
  st256g(out.limb(out_lane0 + l, comp, lb, n) + x, uniform_at(rk, x, P.p, P.shift),
         uniform_at(rk, x + 1, P.p, P.shift), uniform_at(rk, x + 2, P.p, P.shift),
         uniform_at(rk, x + 3, P.p, P.shift));
}

}  // namespace

cudaError_t launch_limb_op(int opcode, View out, u32 out_lane0, u32 out_comps, View a, LaneMap ma, u32 a_comps,
                           View b, LaneMap mb, u32 b_comps, u32 nlanes, u32 limb_lo, u32 limbs, u32 n,
                           const PrimeConst* pc, cudaStream_t st) {
  if (n % 4 || a_comps > 2 || b_comps > 2) return cudaErrorInvalidValue;
  LimbOpArgs A{out, out_lane0, a, ma, b, mb, nlanes, limb_lo, limbs, n, out_comps, a_comps, b_comps};
  const size_t g = (size_t)nlanes * limbs * ((n + 1023) / 1024);
  if (!g) return cudaSuccess;
  switch (opcode) {
    case kOpAdd: limb_op_kernel<kOpAdd><<<(unsigned)g, 256, 0, st>>>(A, pc); break;
    case kOpSub: limb_op_kernel<kOpSub><<<(unsigned)g, 256, 0, st>>>(A, pc); break;
    case kOpMul: limb_op_kernel<kOpMul><<<(unsigned)g, 256, 0, st>>>(A, pc); break;
    case kOpMulAcc: limb_op_kernel<kOpMulAcc><<<(unsigned)g, 256, 0, st>>>(A, pc); break;
    case kOpAddAcc: limb_op_kernel<kOpAddAcc><<<(unsigned)g, 256, 0, st>>>(A, pc); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_limb_generate(View out, u32 out_lane0, u32 nlanes, u32 comps, u32 limb_lo, u32 limbs, u32 n,
                                 u64 seed, u64 tag, u64 bundle, const PrimeConst* pc, cudaStream_t st) {
  if (n % 4) return cudaErrorInvalidValue;
  const size_t g = (size_t)nlanes * comps * limbs * ((n + 1023) / 1024);
  if (!g) return cudaSuccess;
  limb_generate_kernel<<<(unsigned)g, 256, 0, st>>>(out, out_lane0, nlanes, comps, limb_lo, limbs, n, seed, tag,
                                                   bundle, pc);
  return cudaGetLastError();
}

}  // namespace aegis
