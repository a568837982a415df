// Standalone launcher of the streaming ("strip") fused apply (strip_core.cuh) used by
// rsk_apply_shifted for large images in the SHIFTED and SPLIT modes. DESIGN.md §4.1b.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "strip_core.cuh"

namespace rsk {

bool make_map3(CUtensorMap* m, const double* base, int64_t nx, int64_t ny, int64_t ld, int64_t nvec, int bw, int bh);

template <int R>
__global__ void __launch_bounds__(kAT, kStripCtasPerSm)
    strip_apply_kernel(const __grid_constant__ StripParams p, const int* __restrict__ list, int nvec) {
  extern __shared__ __align__(128) double smem[];
  using Core = StripCore<R>;
  using C = StripCfg<R>;
  Core::init(smem, p);
  StripRing ring{0u, 0u};
  const int ipv = p.nseg * p.nstrip;
  const int nitems = ipv * nvec;
  // item order: vector fastest (the CTAs of one wave share a segment's weights and the
  // strips' column halos through L2), then strip, then segment
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    const int li = it % nvec;
    const int ss = it / nvec;
    const int strip = ss % p.nstrip, seg = ss / p.nstrip;
    const int s = list ? list[li] : li;
    double lo;
    const int ra = p.row0 + seg * p.seg_rows;
    const double dot = Core::item(p, smem, ring, s, strip, ra, min(p.row1, ra + p.seg_rows), false, &lo) + lo;
    if (p.want_dot) {
      const double bs = block_sum(dot, smem + C::OFF_RED);
      if (threadIdx.x == 0) p.part[(int64_t)li * ipv + ss] = bs;
    }
  }
}

extern "C" int rsk_debug_strip_prof(double* out8, int reset) {
#ifdef RSK_STRIP_PROF
  unsigned long long v[8];
  if (cudaMemcpyFromSymbol(v, g_strip_prof, sizeof(v)) != cudaSuccess) return -1;
  for (int i = 0; i < 8; ++i) out8[i] = (double)v[i];
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_strip_prof, z, sizeof(z));
  }
  return 0;
#else
  (void)out8; (void)reset;
  return -1;
#endif
}

__global__ void strip_dot_reduce(const double* part, int ipv, const int* list, double* xdoty) {
  const int li = blockIdx.x;
  const int s = list ? list[li] : li;
  double t = 0.0;
  for (int j = threadIdx.x; j < ipv; j += 32) t += part[(int64_t)li * ipv + j];
  t = warp_sum(t);
  if (threadIdx.x == 0) xdoty[s] = t;
}

// rows per segment: whole columns when the batch alone fills two waves of CTAs, else
// shorter segments (multiples of 8 rows)
int strip_seg_rows(int64_t ny, int64_t nx, int nvec, int ctas) {
  const int nstrip = (int)((nx + kStripW - 1) / kStripW);
  int64_t nseg = (2LL * ctas + (int64_t)nvec * nstrip - 1) / ((int64_t)nvec * nstrip);
  if (nseg < 1) nseg = 1;
  int64_t rows = (ny + nseg - 1) / nseg;
  rows = (rows + 7) / 8 * 8;
  if (rows < 64) rows = 64;
  return (int)rows;
}

bool strip_fill_params(Handle* h, StripParams& p, const double* X, int64_t ldx, const double* X2, int64_t ldx2,
                       int64_t nvec_map, double* Y, int64_t ldy, double* EY, int64_t ldey, const double* gamma,
                       int mode, int seg_rows) {
  std::memset(&p, 0, sizeof(p));
  const int r = h->r;
  const int px = pad4mod8(kStripW + 4 * r);
  if (!make_map3(&p.mapX, X, h->nx, h->ny, ldx, nvec_map, px, 8)) return false;
  if (X2 && !make_map3(&p.mapX2, X2, h->nx, h->ny, ldx2, nvec_map, px, 8)) return false;
  p.Y = Y; p.ldy = ldy; p.EY = EY; p.ldey = ldey;
  p.gamma = gamma;
  p.wx = h->wx; p.wy = h->wy;
  p.dcorr = h->dcorr;
  p.part = h->scratch;
  p.ny = (int)h->ny; p.nx = (int)h->nx;
  p.nstrip = (int)((h->nx + kStripW - 1) / kStripW);
  p.seg_rows = seg_rows;
  p.row0 = 0;
  p.row1 = (int)h->ny;
  p.nseg = (int)((h->ny + seg_rows - 1) / seg_rows);
  p.mode = mode;
  p.prefetch_w = getenv("RSK_STRIP_NOPF") ? 0 : 1;
  const int T = 4 * r + 1;
  for (int t = 0; t < T; ++t) { p.cx[t] = h->cBx[t]; p.cy[t] = h->cBy[t]; }
  return true;
}

template <int R>
static cudaError_t strip_launch_r(const StripParams& p, const int* list, int nvec, int sm_count, cudaStream_t st) {
  using C = StripCfg<R>;
  static int bps = 0;
  if (bps == 0) {
    cudaError_t e = cudaFuncSetAttribute(strip_apply_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, strip_apply_kernel<R>, kAT, C::SMEM);
    if (e != cudaSuccess) return e;
    if (bps < 1) bps = 1;
  }
  const int nitems = p.nseg * p.nstrip * nvec;
  int grid = bps * sm_count;
  if (grid > nitems) grid = nitems;
  count_launch();
  strip_apply_kernel<R><<<grid, kAT, C::SMEM, st>>>(p, list, nvec);
  return cudaGetLastError();
}

size_t strip_smem_bytes(int r) {
  switch (r) {
    case 1: return StripCfg<1>::SMEM; case 2: return StripCfg<2>::SMEM; case 3: return StripCfg<3>::SMEM;
    case 4: return StripCfg<4>::SMEM; case 5: return StripCfg<5>::SMEM; case 6: return StripCfg<6>::SMEM;
    case 7: return StripCfg<7>::SMEM; case 8: return StripCfg<8>::SMEM; case 9: return StripCfg<9>::SMEM;
    case 10: return StripCfg<10>::SMEM; case 11: return StripCfg<11>::SMEM; case 12: return StripCfg<12>::SMEM;
    default: return 0;
  }
}

// Returns cudaErrorNotSupported (nothing enqueued) when the strip path does not apply
// (odd widths / misaligned batches: no TMA map); the caller then uses the tiled core.
// rows [row0, row1) of the output only (row1 <= 0: the whole image)
cudaError_t launch_apply_strip(Handle* h, const ApplyLaunch& a, cudaStream_t st, int row0, int row1) {
  if (!(a.mode == RSK_APPLY_SHIFTED || a.mode == RSK_APPLY_SPLIT) || a.cg || a.nlist <= 0 || h->ct)
    return cudaErrorNotSupported;
  if (row1 <= 0) { row0 = 0; row1 = (int)h->ny; }
  const int64_t nv = (a.list || a.nvec_total > 0) ? a.nvec_total : a.nlist;
  const int ctas = kStripCtasPerSm * h->sm_count;
  const int seg = strip_seg_rows(row1 - row0, h->nx, a.nlist, ctas);
  StripParams p;
  if (!strip_fill_params(h, p, a.X, a.ldx, nullptr, 0, nv, a.Y, a.ldy, a.EY, a.ldey, a.gamma, a.mode, seg))
    return cudaErrorNotSupported;
  p.row0 = row0;
  p.row1 = row1;
  p.nseg = (row1 - row0 + seg - 1) / seg;
  p.want_dot = a.xdoty != nullptr;
  const int ipv = p.nseg * p.nstrip;
  if (a.xdoty && sizeof(double) * (size_t)ipv * (size_t)a.nlist > h->scratch_bytes) return cudaErrorNotSupported;
  cudaError_t e;
  const int smc = h->sm_count;
  switch (h->r) {
    case 1: e = strip_launch_r<1>(p, a.list, a.nlist, smc, st); break;
    case 2: e = strip_launch_r<2>(p, a.list, a.nlist, smc, st); break;
    case 3: e = strip_launch_r<3>(p, a.list, a.nlist, smc, st); break;
    case 4: e = strip_launch_r<4>(p, a.list, a.nlist, smc, st); break;
    case 5: e = strip_launch_r<5>(p, a.list, a.nlist, smc, st); break;
    case 6: e = strip_launch_r<6>(p, a.list, a.nlist, smc, st); break;
    case 7: e = strip_launch_r<7>(p, a.list, a.nlist, smc, st); break;
    case 8: e = strip_launch_r<8>(p, a.list, a.nlist, smc, st); break;
    case 9: e = strip_launch_r<9>(p, a.list, a.nlist, smc, st); break;
    case 10: e = strip_launch_r<10>(p, a.list, a.nlist, smc, st); break;
    case 11: e = strip_launch_r<11>(p, a.list, a.nlist, smc, st); break;
    case 12: e = strip_launch_r<12>(p, a.list, a.nlist, smc, st); break;
    default: return cudaErrorNotSupported;
  }
  if (e != cudaSuccess) return e;
  if (a.xdoty) {
    count_launch();
    strip_dot_reduce<<<a.nlist, 32, 0, st>>>(h->scratch, ipv, a.list, a.xdoty);
    e = cudaGetLastError();
  }
  return e;
}

}  // namespace rsk
