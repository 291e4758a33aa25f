// m2l_block.cu -- H6 M2L of the low-rank groups in two passes with target-owned outputs (kernels.cuh BTrans).
//
// eq_lrdk: y_t += U_o (V_o x_s) for every M2L pair (t, s) of offset group o.
// The one-pass group-major kernel (kernels.cu k_gtrans_ws) adds every U_o (V_o x_s) into Y with FP64
// atomics at L2 -- s_out x 16 B of reduction payload per pair -- and that reduction rate bounds it
// (DESIGN.md §6).  Two passes instead:
//   pass 1 (k_m2l_tv): group-major, T_p = V_o x_s for every pair p, stored (one writer per element) into a
//     global buffer at the pair's position in pass-2 order -- r x 16 B per pair instead of s_out x 16 B of
//     reductions.  V_o is staged in shared memory once per item (TMA bulk copy); the x_s columns of each
//     chunk of 32 pairs are gathered by one TMA bulk copy per column into a ring of slots;
//   pass 2 (here): a CTA owns a block of <= bmax target slots of one direction and keeps their Y rows in
//     shared memory; the block's pairs (sorted by group, chunks of <= 32 pairs of one group) stream
//     through: Y_s[:, loc(p)] += U_o T_p on DMMA, and each Y element is stored to global memory once.
// Both passes are plain stores in a fixed order: the M2L result is bitwise reproducible.
//
// In both passes one producer warp feeds a ring of shared-memory slots: it loads the chunks' metadata
// (group, rank, operator offset; 32 chunks per warp-wide load), writes it into the slot and issues TMA
// bulk copies (cp.async.bulk) that complete on the slot's mbarrier; the compute warps wait on that barrier
// and release the slot on a second one.  Pass 2's compute warps own the row tiles of Y_s (warp pairs share
// a row tile and split the column tiles when the level has few row tiles, meeting at a named barrier per
// chunk), so no two warps ever update one element and the compute warps run unsynchronised; the U fragments
// of the next chunk are fetched into registers before the current chunk's Y_s update.  Complex products by
// the 3M scheme (kernels.cu).
#include "kernels.cuh"

#include <algorithm>

namespace fda {

namespace {

constexpr int MB_D = 4;    // pass-2 ring depth (chunks)
constexpr int MB_D1 = 2;   // pass-1 ring depth (chunks of gathered x columns)
constexpr int MB_P = 32;   // pairs per chunk (4 column tiles of 8)
constexpr int MB_KT = 6;   // largest low rank: 6 k tiles of U (r <= 24)

struct ChunkMeta {         // written by the producer into the slot, read by the compute warps
  int n, rank, mout, pad;
  int64_t off;             // operator offset (doubles) into the pool: V (pass 1) or U (pass 2)
};

__device__ __forceinline__ void dmma_b(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// TMA bulk copy global -> shared, completion (bytes) reported on bar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace


// ---------------------------------------------------------------- pass 1: T = V X (group-major items)
// blockDim = 288: warps 0-7 compute, warp 8 produces.  Item i = pairs [it_ptr[i], it_end[i]) of group
// it_group[i]; warp w computes the column tile ct = w % 4 of the row tiles mt = w / 4 and w / 4 + 2 (< rt),
// so the two row tiles of a warp share the x fragments and every SM sub-partition gets rt column units.
__global__ void __launch_bounds__(288, 1) k_m2l_tv(BTrans B, const double2* __restrict__ X, double2* __restrict__ Tg) {
  extern __shared__ __align__(128) double2 msm[];
  __shared__ uint64_t bar_v, bar_full[MB_D1], bar_empty[MB_D1];
  __shared__ int sOut[MB_D1][MB_P];
  __shared__ int sN[MB_D1];
  const int s_in = B.s_in, kin = (s_in + 3) / 4, ldx = kin * 4 + 4 - ((kin * 4) & 4);  // >= 4 kin, = 4 mod 8
  const int ldt = B.ldt;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int64_t item = blockIdx.x;
  const int grp = B.it_group[item];
  const int64_t pb = B.it_ptr[item], pe = B.it_end[item];
  const int64_t nch = (pe - pb + MB_P - 1) / MB_P;
  const int rank = B.grank[grp], rt = (rank + 7) / 8;
  const int kin_g = B.gsi ? (B.gsi[grp] + 3) / 4 : kin;
  double* Vs = reinterpret_cast<double*>(msm);
  double2* Xr = msm + (size_t)B.rmax8 / 8 * kin * 32;  // after the largest V (rmax8/8 x kin tiles of 64 doubles)
  // zero the x ring: the padding rows [s_in, 4 kin) are never written by the gathers (V is zero there, but
  // 0 x garbage could be NaN)
  for (int i = tid; i < MB_D1 * MB_P * ldx; i += blockDim.x) Xr[i] = make_double2(0.0, 0.0);
  if (tid == 0) {
    mbar_init(&bar_v, 1);
    for (int d = 0; d < MB_D1; ++d) mbar_init(&bar_full[d], 1), mbar_init(&bar_empty[d], 8 * 32);
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // the zeroed ring before async writes
  __syncthreads();
  if (warp == 8) {
    const unsigned xb = (unsigned)s_in * 16u;
    if (lane == 0) {
      const unsigned vb = (unsigned)rt * kin * 64u * 8u;
      mbar_expect_tx(&bar_v, vb);
      bulk_g2s(Vs, B.pool + B.gmat[grp], vb, &bar_v);
    }
    for (int64_t j = 0; j < nch; ++j) {
      const int d = (int)(j % MB_D1);
      if (j >= MB_D1) mbar_wait(&bar_empty[d], (unsigned)((j / MB_D1 - 1) & 1));
      const int64_t p0 = pb + j * MB_P;
      const int n = (int)min((int64_t)MB_P, pe - p0);
      const int src = lane < n ? B.p1_in[p0 + lane] : 0;
      sOut[d][lane] = lane < n ? B.p1_out[p0 + lane] : 0;
      if (lane == 0) sN[d] = n;
      __syncwarp();
      if (lane == 0) mbar_expect_tx(&bar_full[d], (unsigned)n * xb);
      __syncwarp();
      if (lane < n) bulk_g2s(Xr + ((size_t)d * MB_P + lane) * ldx, X + (int64_t)src * s_in, xb, &bar_full[d]);
    }
  } else {
    const int ct = warp & 3, m0 = warp >> 2, m1 = m0 + 2;
    const bool u0 = m0 < rt, u1 = m1 < rt;
    mbar_wait(&bar_v, 0);
    for (int64_t j = 0; j < nch; ++j) {
      const int d = (int)(j % MB_D1);
      mbar_wait(&bar_full[d], (unsigned)((j / MB_D1) & 1));
      const int n = sN[d];
      if (u0 && ct * 8 < n) {
        double acc[2][3][2];
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int e = 0; e < 3; ++e) acc[u][e][0] = acc[u][e][1] = 0.0;
        const double2* xb = Xr + ((size_t)d * MB_P + ct * 8 + g) * ldx + t;
        const double* a0 = Vs + (size_t)m0 * kin * 64 + lane;
        const double* a1 = Vs + (size_t)(u1 ? m1 : m0) * kin * 64 + lane;
#pragma unroll 4
        for (int kt = 0; kt < kin_g; ++kt) {
          const double2 b = xb[kt * 4];
          const double bs = b.x + b.y;
          {
            const double ar = a0[kt * 64], ai = a0[kt * 64 + 32];
            dmma_b(acc[0][0][0], acc[0][0][1], ar, b.x);
            dmma_b(acc[0][1][0], acc[0][1][1], ai, b.y);
            dmma_b(acc[0][2][0], acc[0][2][1], ar + ai, bs);
          }
          if (u1) {
            const double ar = a1[kt * 64], ai = a1[kt * 64 + 32];
            dmma_b(acc[1][0][0], acc[1][0][1], ar, b.x);
            dmma_b(acc[1][1][0], acc[1][1][1], ai, b.y);
            dmma_b(acc[1][2][0], acc[1][2][1], ar + ai, bs);
          }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u)
          if (u == 0 || u1)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int c = ct * 8 + 2 * t + i;
              if (c < n)
                Tg[(int64_t)sOut[d][c] * ldt + (u ? m1 : m0) * 8 + g] =
                    make_double2(acc[u][0][i] - acc[u][1][i], acc[u][2][i] - acc[u][0][i] - acc[u][1][i]);
            }
      }
      mbar_arrive(&bar_empty[d]);
    }
  }
}

// ---------------------------------------------------------------- pass 2: Y_s += U T (target blocks)
// blockDim.x = (NW + 1) * 32: warps 0..NW-1 compute, warp NW produces.  split = warps per row tile (1, 2).
__global__ void __launch_bounds__(640, 1) k_m2l_bu(BTrans B, const double2* __restrict__ Tg, double2* __restrict__ Y,
                                                   int split) {
  extern __shared__ __align__(128) double2 msm[];
  __shared__ uint64_t bar_full[MB_D], bar_empty[MB_D];
  __shared__ ChunkMeta meta[MB_D];
  __shared__ __align__(16) uint8_t sloc[MB_D][MB_P];
  const int s_out = B.s_out;
  const int mout = (s_out + 7) / 8, ldy = mout * 8, ldt = B.ldt;
  const int nw = (int)(blockDim.x >> 5) - 1;
  double2* Ys = msm;
  double2* Ts = msm + (size_t)B.bmax * ldy;  // ring: MB_D slots of MB_P * ldt
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int64_t blk = B.blk_order[blockIdx.x];
  const int64_t sb = B.blk_sptr[blk], ns = B.blk_sptr[blk + 1] - sb;
  const int64_t c0 = B.blk_cptr[blk], nch = B.blk_cptr[blk + 1] - c0;
  const int kin = (B.s_in + 3) / 4;
  for (int64_t i = tid; i < ns * ldy; i += blockDim.x) Ys[i] = make_double2(0.0, 0.0);
  if (tid < MB_D) {
    mbar_init(&bar_full[tid], 1);
    mbar_init(&bar_empty[tid], nw * 32);
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  if (warp == nw) {
    // ------------------------------------------------ producer
    for (int64_t jb = 0; jb < nch; jb += 32) {
      // metadata of chunks jb .. jb + 31, one per lane
      ChunkMeta m{0, 0, 0, 0, 0};
      int64_t p0 = 0;
      if (jb + lane < nch) {
        const int64_t c = c0 + jb + lane;
        p0 = B.ch_ptr[c];
        const int grp = B.ch_group[c];
        m.n = (int)(B.ch_ptr[c + 1] - p0);
        m.rank = B.grank[grp];
        m.mout = B.gso ? (B.gso[grp] + 7) / 8 : mout;
        m.off = B.gmat[grp] + (int64_t)((m.rank + 7) / 8) * kin * 64;  // U follows V
      }
      const int nb = (int)min((int64_t)32, nch - jb);
      for (int i = 0; i < nb; ++i) {
        const int64_t j = jb + i;
        const int d = (int)(j % MB_D);
        const int mn = __shfl_sync(0xffffffffu, m.n, i);
        const int mr = __shfl_sync(0xffffffffu, m.rank, i);
        const int mm = __shfl_sync(0xffffffffu, m.mout, i);
        const int64_t mo = __shfl_sync(0xffffffffu, m.off, i);
        const int64_t q0 = __shfl_sync(0xffffffffu, p0, i);
        if (lane == 0) {
          if (j >= MB_D) mbar_wait(&bar_empty[d], (unsigned)((j / MB_D - 1) & 1));
          meta[d] = ChunkMeta{mn, mr, mm, 0, mo};
          const unsigned tb = (unsigned)mn * ldt * 16u;
          mbar_expect_tx(&bar_full[d], tb + (unsigned)MB_P);
          bulk_g2s(Ts + (size_t)d * MB_P * ldt, Tg + q0 * ldt, tb, &bar_full[d]);
          bulk_g2s(sloc[d], B.ch_loc + (c0 + j) * MB_P, MB_P, &bar_full[d]);
        }
      }
    }
  } else {
    // ------------------------------------------------ compute: Y_s[rows mt, cols loc] += U T
    const int rw = warp / split, half = warp - rw * split;  // row-tile walker, column half
    const int nrw = nw / split;                              // row tiles are rw, rw + nrw, ...
    double ur[MB_KT], ui[MB_KT];
    auto load_u = [&](const ChunkMeta& m, int mt) {
      const int rt = (m.rank + 7) / 8, kt2 = (m.rank + 3) / 4;
      const double* U = B.pool + m.off + lane;
#pragma unroll
      for (int kt = 0; kt < MB_KT; ++kt)
        if (kt < kt2 && mt < m.mout) {
          ur[kt] = __ldg(U + ((size_t)mt * 2 * rt + kt) * 64);
          ui[kt] = __ldg(U + ((size_t)mt * 2 * rt + kt) * 64 + 32);
        }
    };
    ChunkMeta cm{0, 0, 0, 0, 0};
    if (nch > 0) {
      mbar_wait(&bar_full[0], 0);
      cm = meta[0];
      load_u(cm, rw);
    }
    for (int64_t j = 0; j < nch; ++j) {
      const int d = (int)(j % MB_D);
      const int n = cm.n, kt2 = (cm.rank + 3) / 4, nct = (n + 7) / 8, mout_g = cm.mout;
      int loc[4][2];
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int cc = q * 8 + 2 * t + i;
          loc[q][i] = cc < n ? (int)sloc[d][cc] : -1;
        }
      const double2* Td = Ts + (size_t)d * MB_P * ldt;
      for (int mt = rw; mt < mout_g; mt += nrw) {
        double acc[4][3][2];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int e = 0; e < 3; ++e) acc[q][e][0] = acc[q][e][1] = 0.0;
#pragma unroll
        for (int kt = 0; kt < MB_KT; ++kt)
          if (kt < kt2) {
            const double ar = ur[kt], ai = ui[kt], as = ar + ai;
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (q < nct && (q % split) == half) {
                const double2 b = Td[(q * 8 + g) * ldt + kt * 4 + t];
                dmma_b(acc[q][0][0], acc[q][0][1], ar, b.x);
                dmma_b(acc[q][1][0], acc[q][1][1], ai, b.y);
                dmma_b(acc[q][2][0], acc[q][2][1], as, b.x + b.y);
              }
          }
        // U fragments for what comes next (this chunk's next row tile, or the next chunk's first), issued
        // before the Y_s update so their latency overlaps it
        if (mt + nrw < mout_g) {
          load_u(cm, mt + nrw);
        } else if (j + 1 < nch) {
          const int dn = (int)((j + 1) % MB_D);
          mbar_wait(&bar_full[dn], (unsigned)(((j + 1) / MB_D) & 1));
          load_u(meta[dn], rw);
        }
        const int row = mt * 8 + g;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (q < nct && (q % split) == half)
#pragma unroll
            for (int i = 0; i < 2; ++i)
              if (loc[q][i] >= 0) {
                double2* y = Ys + (size_t)loc[q][i] * ldy + row;
                const double2 v = *y;
                *y = make_double2(v.x + acc[q][0][i] - acc[q][1][i], v.y + acc[q][2][i] - acc[q][0][i] - acc[q][1][i]);
              }
      }
      // a warp with no row tile in this chunk still prefetches the next chunk's U
      if (rw >= mout_g && j + 1 < nch) {
        const int dn = (int)((j + 1) % MB_D);
        mbar_wait(&bar_full[dn], (unsigned)(((j + 1) / MB_D) & 1));
        load_u(meta[dn], rw);
      }
      if (j + 1 < nch) cm = meta[(j + 1) % MB_D];  // its full barrier was awaited above
      mbar_arrive(&bar_empty[d]);
      // the warps sharing a row tile stay on one chunk: their column tiles hold distinct targets within a
      // chunk, not across chunks
      if (split > 1) named_bar_sync(1 + rw, 32 * split);
    }
  }
  __syncthreads();
  // the block's Y rows: one plain store per element (this launch owns them)
  for (int64_t i = tid; i < ns * s_out; i += blockDim.x) {
    const int64_t sl = i / s_out;
    const int r = (int)(i - sl * s_out);
    Y[(int64_t)B.blk_slot[sb + sl] * s_out + r] = Ys[sl * ldy + r];
  }
}

int m2l_block_ldt(int rmax8) { return ((rmax8 + 3) / 8) * 8 + 4; }  // >= rmax8, = 4 mod 8 (conflict-free B loads)
static int tv_ldx(int s_in) {
  const int k4 = (s_in + 3) / 4 * 4;
  return k4 + 4 - (k4 & 4);
}
size_t m2l_block_smem(int s_out, int rmax8, int bmax) {
  const int ldy = (s_out + 7) / 8 * 8;
  return ((size_t)bmax * ldy + (size_t)MB_D * MB_P * m2l_block_ldt(rmax8)) * sizeof(double2);
}
static size_t tv_smem(int s_in, int rmax8) {
  return (size_t)(rmax8 / 8) * ((s_in + 3) / 4) * 64 * sizeof(double) + (size_t)MB_D1 * MB_P * tv_ldx(s_in) * sizeof(double2);
}
int m2l_block_bmax(int s_out, int rmax8, size_t smem_limit) {
  if (rmax8 > 4 * MB_KT || rmax8 <= 0) return 0;
  if (tv_smem(s_out, rmax8) + 1024 > smem_limit) return 0;
  const size_t ring = (size_t)MB_D * MB_P * m2l_block_ldt(rmax8) * sizeof(double2);
  const size_t stat = MB_D * (2 * sizeof(uint64_t) + sizeof(ChunkMeta) + MB_P) + 1024;  // static shared memory + reserve
  if (smem_limit <= ring + stat) return 0;
  const size_t per = (size_t)((s_out + 7) / 8 * 8) * sizeof(double2);
  return (int)std::min<size_t>(255, (smem_limit - ring - stat) / per);
}
// compute warps and split for a level with mout row tiles: warp pairs per row tile for short expansions,
// else one warp per row tile up to 19 warps (a warp walks row tiles rw, rw + 19, ...)
static void bu_shape(int mout, int* nw, int* split) {
  if (mout <= 9) {
    *split = 2, *nw = 2 * mout;
  } else {
    *split = 1, *nw = std::min(mout, 19);  // <= 20 warps with the producer (__launch_bounds__)
  }
}

cudaError_t launch_m2l_block(const BTrans& B, const double2* X, double2* T, double2* Y, cudaStream_t st, int passes) {
  if (B.n_blocks <= 0) return cudaSuccess;
  if (passes & 1) {
    const size_t sm1 = tv_smem(B.s_in, B.rmax8);
    cudaError_t e = cudaFuncSetAttribute(k_m2l_tv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
    if (e != cudaSuccess) return e;
    k_m2l_tv<<<(unsigned)B.n_items1, 288, sm1, st>>>(B, X, T);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (!(passes & 2)) return cudaSuccess;
  const size_t sm = m2l_block_smem(B.s_out, B.rmax8, B.bmax);
  const cudaError_t e = cudaFuncSetAttribute(k_m2l_bu, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  int nw, split;
  bu_shape((B.s_out + 7) / 8, &nw, &split);
  k_m2l_bu<<<(unsigned)B.n_blocks, (nw + 1) * 32, sm, st>>>(B, T, Y, split);
  return cudaGetLastError();
}

}  // namespace fda
