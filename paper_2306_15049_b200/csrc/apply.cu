// Standalone launcher of the fused shifted apply (rsk_apply_shifted); the work-item core
// is in apply_core.cuh. Also: TMA tensor-map encoding and the
// fragment-ordered edge tables of B = G^T G.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "apply_core.cuh"

namespace rsk {

// standalone tiles: 64 output rows for r <= 6 (a 64 x (64 + 4r) halo box, fewer items:
// C2 x 32 shifts is 512 items instead of 768 on 148 CTAs), else the default height
__host__ __device__ constexpr int std_tile_rows(int r) { return r <= 6 ? 64 : (r <= 8 ? 56 : tc_tile_rows(r)); }

template <int R, bool kTma>
__global__ void __launch_bounds__(kAT, kApplyCtasPerSm) apply_kernel(const __grid_constant__ ApplyParams p) {
  extern __shared__ __align__(128) double smem[];
  using Core = ApplyCore<R, kTma, std_tile_rows(R)>;
  Core::init_bars(smem, p);
  const int nl = p.nlist_dev ? *p.nlist_dev : p.nlist;
  const int nitems = nl * p.ntiles;
  const int per = (nitems + gridDim.x - 1) / gridDim.x;
  const int ibeg = blockIdx.x * per;
  const int iend = min(nitems, ibeg + per);
  ApplyPipe pp{{0u, 0u}, 0};
  Core::run(p, smem, ibeg, iend, nl, pp);
}

// plain-mode dot reduction: xdoty[s] = sum_tiles part[li][tile]
__global__ void apply_dot_reduce(const double* part, int ntiles, const int* list, double* xdoty) {
  const int li = blockIdx.x;
  const int s = list ? list[li] : li;
  double t = 0.0;
  for (int j = threadIdx.x; j < ntiles; j += 32) t += part[(int64_t)li * ntiles + j];
  t = warp_sum(t);
  if (threadIdx.x == 0) xdoty[s] = t;
}

int apply_tile_rows(int r) { return tc_tile_rows(r); }

// optional per-phase timestamps of block 0 (RSK_APPLY_PROF=1; debugging only)
static unsigned long long* apply_prof_buf() {
  static unsigned long long* ap = nullptr;
  static int on = -1;
  if (on < 0) {
    on = getenv("RSK_APPLY_PROF") ? 1 : 0;
    if (on && cudaMalloc(&ap, 8 * sizeof(unsigned long long)) == cudaSuccess)
      cudaMemset(ap, 0, 8 * sizeof(unsigned long long));
  }
  return ap;
}

extern "C" int rsk_debug_apply_prof(double* out8, int reset) {
  unsigned long long* ap = apply_prof_buf();
  if (!ap) return -1;
  unsigned long long v[8];
  if (cudaMemcpy(v, ap, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  for (int i = 0; i < 8; ++i) out8[i] = (double)v[i];
  if (reset) cudaMemset(ap, 0, sizeof(v));
  return 0;
}

int apply_tiles(const Handle* h) {
  const int ty = tc_tile_rows(h->r);
  const int tx = (int)((h->nx + kTX - 1) / kTX), tyc = (int)((h->ny + ty - 1) / ty);
  return tx * tyc;
}

// ---------------------------------------------------------------- tensor maps
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

// 3-D map {nx, ny, vectors} over a batch with leading dimension ld (elements), box
// {bw, bh, 1}; false if TMA cannot describe it (odd widths, misalignment)
bool make_map3(CUtensorMap* m, const double* base, int64_t nx, int64_t ny, int64_t ld, int64_t nvec, int bw, int bh) {
  auto fn = encode_fn();
  if (!fn || !base) return false;
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (nx & 1) || (ld & 1) || nvec < 1) return false;
  cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nvec};
  cuuint64_t strides[2] = {(cuuint64_t)nx * 8, (cuuint64_t)ld * 8};
  cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 2-D map {inner, outer} with an explicit outer pitch (elements), box {bw, bh}
bool make_map2s(CUtensorMap* m, const double* base, int64_t inner, int64_t outer, int64_t pitch, int bw, int bh) {
  auto fn = encode_fn();
  if (!fn || !base) return false;
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (pitch & 1) || outer < 1) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)pitch * 8};
  cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)bh};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_map2(CUtensorMap* m, const double* base, int64_t nx, int64_t ny, int bw, int bh) {
  auto fn = encode_fn();
  if (!fn || !base) return false;
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (nx & 1)) return false;
  cuuint64_t dims[2] = {(cuuint64_t)nx, (cuuint64_t)ny};
  cuuint64_t strides[1] = {(cuuint64_t)nx * 8};
  cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)bh};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ---------------------------------------------------------------- launch
template <int R>
static cudaError_t launch_r(const ApplyParams& prm, bool tma, int sm_count, cudaStream_t st) {
  using C = TcCfg<R, std_tile_rows(R)>;
  static int bps[2] = {0, 0};
  int& blocks_per_sm = bps[tma ? 1 : 0];
  if (blocks_per_sm == 0) {
    auto kfn = tma ? apply_kernel<R, true> : apply_kernel<R, false>;
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kfn, kAT, C::SMEM);
    if (e != cudaSuccess) return e;
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  const int nitems = prm.nlist * prm.ntiles;
  int grid = blocks_per_sm * sm_count;
  if (grid > nitems && !prm.nlist_dev) grid = nitems;
  count_launch();
  if (tma) apply_kernel<R, true><<<grid, kAT, C::SMEM, st>>>(prm);
  else apply_kernel<R, false><<<grid, kAT, C::SMEM, st>>>(prm);
  return cudaGetLastError();
}

bool fill_apply_params(Handle* h, const ApplyLaunch& a, ApplyParams& prm, int ty_override) {
  std::memset(&prm, 0, sizeof(prm));
  prm.X = a.X; prm.ldx = a.ldx;
  prm.X2 = a.X2; prm.ldx2 = a.ldx2;
  prm.Y = a.Y; prm.ldy = a.ldy;
  prm.EY = a.EY; prm.ldey = a.ldey;
  prm.gamma = a.gamma;
  prm.list = a.list;
  prm.wx = h->wx; prm.wy = h->wy;
  prm.dcorr = h->dcorr;
  prm.cg = a.cg;
  prm.ny = (int)h->ny; prm.nx = (int)h->nx;
  prm.tiles_x = (int)((h->nx + kTX - 1) / kTX);
  const int tyg = ty_override > 0 ? ty_override : tc_tile_rows(h->r);
  prm.ntiles = prm.tiles_x * (int)((h->ny + tyg - 1) / tyg);
  prm.nlist = a.nlist;
  prm.nlist_dev = a.nlist_dev;
  prm.mode = a.mode;
  prm.cg_alpha = a.cg_alpha ? 1 : 0;
  prm.src2_rconv = a.src2_rconv ? 1 : 0;
  prm.want_dot = (a.xdoty != nullptr || a.cg_alpha) ? 1 : 0;
  prm.part = h->scratch;
  prm.aprof = apply_prof_buf();
  prm.aprof_block = getenv("RSK_APPLY_PROF") ? atoi(getenv("RSK_APPLY_PROF")) : -1;
  const int T = 4 * h->r + 1;
  if (a.mode == RSK_APPLY_C_ONLY) {
    prm.edge_fix = 0;
    for (int t = 0; t < T; ++t) { prm.cx[t] = h->cCx[t]; prm.cy[t] = h->cCy[t]; }
  } else if (a.mode == RSK_APPLY_CT_ONLY) {
    prm.edge_fix = 0;
    for (int t = 0; t < T; ++t) { prm.cx[t] = h->cTx[t]; prm.cy[t] = h->cTy[t]; }
  } else {
    prm.edge_fix = 1;
    for (int t = 0; t < T; ++t) { prm.cx[t] = h->cBx[t]; prm.cy[t] = h->cBy[t]; }
  }
  // TMA map (box = the staged halo tile); any failure -> cp.async path
  const int r = h->r;
  const int ty = tyg;
  const int hy = ((ty + 4 * r + 7) / 8) * 8;
  const int px = pad4mod8(kTX + 4 * r);
  bool tma = getenv("RSK_NO_TMA") == nullptr;
  const int64_t nv = (a.list || a.nvec_total > 0) ? a.nvec_total : a.nlist;
  tma = tma && make_map3(&prm.mapX, a.X, h->nx, h->ny, a.ldx, nv, px, hy);
  if (tma && a.X2) tma = make_map3(&prm.mapX2, a.X2, h->nx, h->ny, a.ldx2, nv, px, hy);
  return tma;
}

cudaError_t launch_apply_taps(Handle* h, const ApplyLaunch& a, const double* cx, const double* cy, int edge_fix,
                              cudaStream_t st) {
  if (a.nlist <= 0) return cudaSuccess;
  if (a.cg || a.xdoty) return cudaErrorNotSupported;
  ApplyParams prm;
  const bool tma = fill_apply_params(h, a, prm, std_tile_rows(h->r));
  const int T = 4 * h->r + 1;
  for (int t = 0; t < T; ++t) { prm.cx[t] = cx ? cx[t] : 0.0; prm.cy[t] = cy ? cy[t] : 0.0; }
  prm.edge_fix = edge_fix;
  prm.want_dot = 0;
  const int smc = h->sm_count;
  switch (h->r) {
    case 1: return launch_r<1>(prm, tma, smc, st);
    case 2: return launch_r<2>(prm, tma, smc, st);
    case 3: return launch_r<3>(prm, tma, smc, st);
    case 4: return launch_r<4>(prm, tma, smc, st);
    case 5: return launch_r<5>(prm, tma, smc, st);
    case 6: return launch_r<6>(prm, tma, smc, st);
    case 7: return launch_r<7>(prm, tma, smc, st);
    case 8: return launch_r<8>(prm, tma, smc, st);
    case 9: return launch_r<9>(prm, tma, smc, st);
    case 10: return launch_r<10>(prm, tma, smc, st);
    case 11: return launch_r<11>(prm, tma, smc, st);
    case 12: return launch_r<12>(prm, tma, smc, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_apply(Handle* h, const ApplyLaunch& a, cudaStream_t st) {
  if (h->ct) return launch_ct_apply(h, a, st);   // CT: sparse C, C^T (ct.cu)
  if (a.nlist <= 0) return cudaSuccess;
  if (h->rank == 2) return launch_apply_rank2(h, a, st);
  {
    // large images: the streaming strip core (strip_core.cuh); RSK_APPLY_STRIP=0/1 forces
    const char* ev = getenv("RSK_APPLY_STRIP");
    const int force = ev ? atoi(ev) : -1;
    if (force == 1 || (force != 0 && h->ny * h->nx >= kStripMinN)) {
      cudaError_t es = launch_apply_strip(h, a, st);
      if (es != cudaErrorNotSupported) return es;
    }
  }
  ApplyParams prm;
  const bool tma = fill_apply_params(h, a, prm, std_tile_rows(h->r));
  if (a.xdoty && !a.cg) {
    const size_t need = sizeof(double) * (size_t)prm.ntiles * (size_t)a.nlist;
    if (need > h->scratch_bytes) return cudaErrorMemoryAllocation;
  }
  cudaError_t e;
  const int smc = h->sm_count;
  switch (h->r) {
    case 1: e = launch_r<1>(prm, tma, smc, st); break;
    case 2: e = launch_r<2>(prm, tma, smc, st); break;
    case 3: e = launch_r<3>(prm, tma, smc, st); break;
    case 4: e = launch_r<4>(prm, tma, smc, st); break;
    case 5: e = launch_r<5>(prm, tma, smc, st); break;
    case 6: e = launch_r<6>(prm, tma, smc, st); break;
    case 7: e = launch_r<7>(prm, tma, smc, st); break;
    case 8: e = launch_r<8>(prm, tma, smc, st); break;
    case 9: e = launch_r<9>(prm, tma, smc, st); break;
    case 10: e = launch_r<10>(prm, tma, smc, st); break;
    case 11: e = launch_r<11>(prm, tma, smc, st); break;
    case 12: e = launch_r<12>(prm, tma, smc, st); break;
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  {
    static int chk = -1;
    if (chk < 0) chk = getenv("RSK_APPLY_CHECK") ? 1 : 0;
    if (chk) {
      e = cudaStreamSynchronize(st);
      fprintf(stderr, "[apply] r=%d n=%dx%d tma=%d mode=%d nlist=%d ndev=%p list=%p X=%p ldx=%lld X2=%p Y=%p ldy=%lld EY=%p wx=%p wy=%p cg=%p -> %s\n",
              h->r, prm.ny, prm.nx, (int)tma, a.mode, a.nlist, (void*)a.nlist_dev, (void*)a.list, (void*)a.X,
              (long long)a.ldx, (void*)a.X2, (void*)a.Y, (long long)a.ldy, (void*)a.EY, (void*)h->wx, (void*)h->wy,
              (void*)a.cg, cudaGetErrorString(e));
      if (e != cudaSuccess) return e;
    }
  }
  if (a.xdoty && !a.cg) {
    count_launch();
    apply_dot_reduce<<<a.nlist, 32, 0, st>>>(h->scratch, prm.ntiles, a.list, a.xdoty);
    e = cudaGetLastError();
  }
  return e;
}

}  // namespace rsk
