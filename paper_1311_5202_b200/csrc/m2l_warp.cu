// m2l_warp.cu -- low-rank M2L (H6) with warp-independent tasks: y_t += U (V x_s) per pair (eq_lrdk,
// PAPER.md:844-855) for the group-major atomic items of a level whose groups are all low rank.
//
// One CTA per item (one group: an (offset[, wedge]) operator and <= chunk pairs of it).  The group's operator
// (V: pad8(r) x s_in, then U: s_out x pad8(r), DMMA fragment order, api.cu frag_pool) is staged once in shared
// memory; then every warp works alone on tasks of 8 pairs, with no CTA barrier until the next group:
//   stage 1  T (pad8(r) x 8) = V X      A = V from shared memory, B = the 8 x columns read straight from
//                                        global memory (L2) into registers, prefetched 4-8 k tiles ahead
//   shuffle  T from the accumulator layout into the B-operand layout of stage 2 (registers only)
//   stage 2  Y[out] += U T              A = U from shared memory, per 8-row tile of the output; FP64
//                                        reductions (REDG) of the non-zero rows into Y
// Complex products by the 3M scheme (3 real DMMA m8n8k4 per complex tile product).  Compared with the
// warp-specialised k_gtrans_ws (kernels.cu), there is no gather into shared memory, no T tile in shared
// memory and no per-chunk CTA barrier; the operator comes from shared memory instead of L2.
#include "kernels.cuh"

namespace fda {

namespace {

__device__ __forceinline__ void dmma_w(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_async16_w(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}


// One task: the (up to) 8 pairs [p0, pe) of a group whose V has RT row tiles (pad8(r) = 8 RT).
//   Ms: the staged operator; kin: k tiles per row tile of V (level s_in); kt1: k tiles of the group's own
//   input length; mo: row tiles of the group's own output length; kt2: k tiles of U holding the rank r.
template <int RT, int NS, int MW_D>
__device__ __forceinline__ void m2l_task(const double* __restrict__ Ms, int kin, int kt1, int mo, int kt2, int s_in,
                                         int s_out, int so_own, const double2* __restrict__ X, double2* __restrict__ Y,
                                         const int32_t* __restrict__ pin, const int32_t* __restrict__ pout,
                                         int64_t p0, int64_t pe, int lane) {
  const int g = lane >> 2, t = lane & 3;
  // B operand of stage 1: lane (g, t) holds x[k = 4 kt + t] of pair column g
  const int in_slot = p0 + g < pe ? pin[p0 + g] : -1;
  const double2* xs = X + (int64_t)(in_slot < 0 ? 0 : in_slot) * s_in;
  // x prefetch ring bq[0..D): slot d holds the B fragment of k tile kt + d; refilled in place by a predicated
  // load into the zeroed slot right after its use, so the loop carries no register moves that would wait on a
  // load (a select or copy of the loaded value would)
  auto ldx = [&](double2& v, int kt) {
    const int k = 4 * kt + t;
    v.x = 0.0, v.y = 0.0;
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n @p ld.global.nc.v2.f64 {%0, %1}, [%3];\n}\n"
        : "+d"(v.x), "+d"(v.y)
        : "r"((int)(in_slot >= 0 && kt < kt1 && k < s_in)), "l"(xs + k));
  };
  // output slots of the accumulator columns 2t, 2t + 1
  const int o0 = p0 + 2 * t < pe ? pout[p0 + 2 * t] : -1;
  const int o1 = p0 + 2 * t + 1 < pe ? pout[p0 + 2 * t + 1] : -1;

  double acc[RT][3][2];
#pragma unroll
  for (int i = 0; i < RT; ++i)
#pragma unroll
    for (int q = 0; q < 3; ++q) acc[i][q][0] = acc[i][q][1] = 0.0;
  // two halves of MW_D slots, used alternately: a half is refilled (k tiles + MW_D) while the other is consumed,
  // so no load targets a register an in-flight DMMA of the same half still reads
  double2 bq[2 * MW_D];
#pragma unroll
  for (int d = 0; d < 2 * MW_D; ++d) ldx(bq[d], d);
  const double* vl = Ms + lane;
  auto step = [&](const double2 b, int kt) {
    const double bs = b.x + b.y;
#pragma unroll
    for (int i = 0; i < RT; ++i) {
      const double* a = vl + (i * kin + kt) * NS;
      const double ar = a[0], ai = a[32], as = NS == 96 ? a[64] : ar + ai;
      dmma_w(acc[i][0][0], acc[i][0][1], ar, b.x);
      dmma_w(acc[i][1][0], acc[i][1][1], ai, b.y);
      dmma_w(acc[i][2][0], acc[i][2][1], as, bs);
    }
  };
  int kt0 = 0;
  for (; kt0 + 2 * MW_D <= kt1; kt0 += 2 * MW_D) {
#pragma unroll
    for (int d = 0; d < MW_D; ++d) step(bq[d], kt0 + d);
#pragma unroll
    for (int d = 0; d < MW_D; ++d) ldx(bq[d], kt0 + 2 * MW_D + d);
#pragma unroll
    for (int d = MW_D; d < 2 * MW_D; ++d) step(bq[d], kt0 + d);
#pragma unroll
    for (int d = MW_D; d < 2 * MW_D; ++d) ldx(bq[d], kt0 + 2 * MW_D + d);
  }
#pragma unroll
  for (int d = 0; d < 2 * MW_D; ++d)
    if (kt0 + d < kt1) step(bq[d], kt0 + d);
  // T = V X: lane (g, t) holds T[8 i + g][2 t + j]; stage 2 needs, for k tile kk, T[4 kk + t][g] -- held by
  // lane (4 (kk & 1) + t) * 4 + (g >> 1), element j = g & 1 of row tile kk >> 1
  double br[2 * RT], bi[2 * RT], bsum[2 * RT];
#pragma unroll
  for (int i = 0; i < RT; ++i) {
    double re[2], im[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      re[j] = acc[i][0][j] - acc[i][1][j];
      im[j] = acc[i][2][j] - acc[i][0][j] - acc[i][1][j];
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int src = ((4 * h + t) << 2) | (g >> 1);
      const double r0 = __shfl_sync(0xffffffffu, re[0], src), r1 = __shfl_sync(0xffffffffu, re[1], src);
      const double m0 = __shfl_sync(0xffffffffu, im[0], src), m1 = __shfl_sync(0xffffffffu, im[1], src);
      const int kk = 2 * i + h;
      br[kk] = (g & 1) ? r1 : r0;
      bi[kk] = (g & 1) ? m1 : m0;
      bsum[kk] = br[kk] + bi[kk];
    }
  }
  // stage 2: per output row tile, Y[out] += U T
  const double* ul = Ms + (size_t)RT * kin * NS + lane;
  for (int mt = 0; mt < mo; ++mt) {
    double c[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int kk = 0; kk < 2 * RT; ++kk) {
      if (kk < kt2) {
        const double* a = ul + (mt * 2 * RT + kk) * NS;
        const double ar = a[0], ai = a[32], as = NS == 96 ? a[64] : ar + ai;
        dmma_w(c[0][0], c[0][1], ar, br[kk]);
        dmma_w(c[1][0], c[1][1], ai, bi[kk]);
        dmma_w(c[2][0], c[2][1], as, bsum[kk]);
      }
    }
    // rows past the group's own output length (a short HF wedge) are exact zeros: no reduction for them
    const int row = mt * 8 + g;
    if (row < so_own) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int o = j ? o1 : o0;
        const double re = c[0][j] - c[1][j], im = c[2][j] - c[0][j] - c[1][j];
        if (o >= 0) {
          double2* y = Y + (int64_t)o * s_out + row;
          atomicAdd(&y->x, re);
          atomicAdd(&y->y, im);
        }
      }
    }
  }
}

// NS: doubles per staged operator tile (64, or 96 with the 3M sums); RTMAX: largest V row-tile count of the
// launch's groups; MINB: CTAs per SM the registers are budgeted for
// cap: the dynamic shared memory in doubles; in an NS = 64 launch, groups of rank <= 16 whose operator with the
// 3M sums still fits cap (the low ranks of a launch sized for rank 24) are staged and run with the sums
template <int NS, int RTMAX, int MINB, int MW_T>
__global__ void __launch_bounds__(MW_T, MINB) k_m2l_warp(GTrans T, const double2* __restrict__ X,
                                                         double2* __restrict__ Y, int cap) {
  extern __shared__ double msm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int s_in = T.s_in, s_out = T.s_out;
  const int kin = (s_in + 3) / 4, mout = (s_out + 7) / 8;
  const int64_t item = T.item_order[blockIdx.x];
  for (int64_t e = T.item_ptr[item]; e < T.item_ptr[item + 1]; ++e) {
    const int grp = T.ig_group[e];
    const int rank = T.grank[grp], rt = (rank + 7) / 8;
    const int so_own = T.gso ? T.gso[grp] : s_out;
    const int kt1 = T.gsi ? (T.gsi[grp] + 3) / 4 : kin, mo = (so_own + 7) / 8;
    const int kt2 = (rank + 3) / 4;
    if (rt <= 0) continue;  // rank 0: nothing to add
    // stage the group's operator (V then U, fragment order, contiguous)
    __syncthreads();  // the previous group's operator is no longer read
    const int ntile = rt * kin + mout * 2 * rt;
    const bool g96 = NS == 96 || (rt <= 2 && ntile * 96 <= cap);
    {
      const double* src = T.pool + T.gmat[grp];
      if (!g96) {
        for (int i = tid; i < ntile * 32; i += MW_T) cp_async16_w(msm + 2 * i, src + 2 * i);
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
      } else {  // tiles of 96: the real and imaginary parts and their sum (the 3M operand), summed once here
        for (int i = tid; i < ntile * 32; i += MW_T) {
          const int q = i >> 5, l = i & 31;
          const double re = __ldg(src + q * 64 + l), im = __ldg(src + q * 64 + 32 + l);
          msm[q * 96 + l] = re, msm[q * 96 + 32 + l] = im, msm[q * 96 + 64 + l] = re + im;
        }
      }
    }
    __syncthreads();
    const int64_t pb = T.ig_pb[e], pe = T.ig_pe[e];
    const int64_t ntask = (pe - pb + 7) / 8;
    for (int64_t task = warp; task < ntask; task += MW_T / 32) {
      const int64_t p0 = pb + 8 * task;
      if (NS == 64 && g96) {  // low ranks with the sums staged
        if (rt == 1)
          m2l_task<1, 96, (MINB >= 3 ? 2 : 4)>(msm, kin, kt1, mo, kt2, s_in, s_out, so_own, X, Y, T.in, T.out, p0, pe, lane);
        else
          m2l_task<2, 96, (MINB >= 3 ? 2 : 4)>(msm, kin, kt1, mo, kt2, s_in, s_out, so_own, X, Y, T.in, T.out, p0, pe, lane);
      } else if (rt == 1 || RTMAX == 1)
        m2l_task<1, NS, (MINB >= 3 ? 2 : 4)>(msm, kin, kt1, mo, kt2, s_in, s_out, so_own, X, Y, T.in, T.out, p0, pe, lane);
      else if (rt == 2 || RTMAX == 2)
        m2l_task<(RTMAX >= 2 ? 2 : 1), NS, (MINB >= 3 ? 2 : 4)>(msm, kin, kt1, mo, kt2, s_in, s_out, so_own, X, Y, T.in, T.out, p0, pe, lane);
      else if (rt == 3 || RTMAX == 3)
        m2l_task<(RTMAX >= 3 ? 3 : 1), NS, (MINB >= 3 ? 2 : 4)>(msm, kin, kt1, mo, kt2, s_in, s_out, so_own, X, Y, T.in, T.out, p0, pe, lane);
      else if (rt == 4 || RTMAX == 4)  // (the launcher picks RTMAX >= the launch's largest rank / 8)
        m2l_task<(RTMAX >= 4 ? 4 : 1), NS, (MINB >= 3 ? 2 : 4)>(msm, kin, kt1, mo, kt2, s_in, s_out, so_own, X, Y, T.in, T.out, p0, pe, lane);
      else
        m2l_task<(RTMAX >= 5 ? 5 : 1), NS, (MINB >= 3 ? 2 : 4)>(msm, kin, kt1, mo, kt2, s_in, s_out, so_own, X, Y, T.in, T.out, p0, pe, lane);
    }
  }
}

}  // namespace

// read at plan creation (tests toggle it between plans)
bool m2l_warp_on() { return !(getenv("FDA_M2L_WARP") && getenv("FDA_M2L_WARP")[0] == '0'); }

// largest pad8 rank (<= 40, RT <= 5) whose operator fits smem_limit bytes
int m2l_warp_rmax(int s_out, int s_in, size_t smem_limit) {
  const int kin = (s_in + 3) / 4, mout = (s_out + 7) / 8;
  int best = 0;
  for (int r8 = 8; r8 <= 40; r8 += 8) {
    const int rt = r8 / 8;
    if ((size_t)(rt * kin + mout * 2 * rt) * 64 * sizeof(double) <= smem_limit) best = r8;
  }
  return best;
}

bool m2l_warp_fits(const GTrans& T) {
  return T.warp_tasks && T.atomic && T.all_lowrank && T.rmax8 <= 40 && (size_t)T.mmax * sizeof(double) <= smem_optin_bytes();
}

cudaError_t launch_m2l_warp(const GTrans& T, const double2* X, double2* Y, cudaStream_t st) {
  if (T.n_items <= 0) return cudaSuccess;
  // Configuration: three CTAs per SM (24 warps: more latency hiding; registers budgeted for RTMAX <= 2) when the
  // operator fits a third of the shared memory, else two of 8 warps; operators larger than half the shared memory
  // (the high ranks of the LF level) run as one CTA of 16 warps per SM.  The tiles carry the 3M sums when those
  // still fit (FDA_M2L_SUM3=0: never; FDA_M2L_OCC=2: at most two CTAs per SM)
  const size_t sm2 = (size_t)T.mmax * sizeof(double), sm3 = sm2 * 3 / 2;
  const size_t third = 74 * 1024;
  // (ranks above 32 need the RTMAX = 5 instantiation, which only the 16-warp configuration has)
  const bool big = sm2 > (size_t)GT_SMEM_BUDGET || T.rmax8 > 32;
  const bool allow3 = !(getenv("FDA_M2L_SUM3") && getenv("FDA_M2L_SUM3")[0] == '0');
  const bool occ3 =
      !big && T.rmax8 <= 16 && sm2 <= third && !(getenv("FDA_M2L_OCC") && getenv("FDA_M2L_OCC")[0] == '2');
  const bool sum3 = allow3 && sm3 <= (big ? smem_optin_bytes() : occ3 ? third : (size_t)GT_SMEM_BUDGET);
  const size_t sm = sum3 ? sm3 : sm2;
  void (*kern)(GTrans, const double2*, double2*, int) =
      big ? (sum3 ? k_m2l_warp<96, 5, 1, 512> : k_m2l_warp<64, 5, 1, 512>)
          : occ3 ? (sum3 ? k_m2l_warp<96, 2, 3, 256> : k_m2l_warp<64, 2, 3, 256>)
                 : (sum3 ? k_m2l_warp<96, 4, 2, 256> : k_m2l_warp<64, 4, 2, 256>);
  if (sm > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
  }
  kern<<<(unsigned)T.n_items, big ? 512 : 256, sm, st>>>(T, X, Y, allow3 ? (int)(sm / sizeof(double)) : 0);
  return cudaGetLastError();
}

}  // namespace fda
