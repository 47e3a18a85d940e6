// grid.cu -- candidate-pair generation on the GPU: the top-level
// structure before the path ("combining the fiber intersection with a top level hierarchy
// ... is straightforward").  A uniform grid over the segments' bounding boxes
// (control-point hull dilated by the largest radius control point: the convex hull bound of
// P:488-491), and a 3-D DDA per ray that emits every segment whose box the ray overlaps, in
// front-to-back cell order.
//
// Conservativeness (no missed candidate) in FP32: boxes are dilated by 1e-3 of a cell before
// they are registered, so a cell the DDA rounds past at an edge or corner is covered by its
// neighbours; a segment is emitted in the cell whose DDA t-range holds the ray's entry into
// its (dilated) box, clamped to the grid entry.  The t-ranges of consecutive cells share
// their end points exactly, so every entry lands in at least one visited cell; an entry on a
// shared end point is emitted twice (harmless for the nearest hit: equal results).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>

#include "fiber.h"
#include "fiber_internal.h"
#include "scan.cuh"

struct fiber_grid_s {
  float lo[3], cell[3], inv_cell[3];
  int dims[3];
  int64_t n_cells, n_entries, n_segs;
  int device;
  float4* box_lo;        // device [n_segs] dilated boxes
  float4* box_hi;
  uint32_t* cell_start;  // device [n_cells + 1]
  uint32_t* entries;     // device [n_entries] segment ids, ascending within a cell
};

namespace {

struct GridView {
  float lo[3], cell[3], inv_cell[3];
  int dims[3];
  const float4* box_lo;
  const float4* box_hi;
  const uint32_t* cell_start;
  const uint32_t* entries;
};

GridView view(const fiber_grid_s* g) {
  GridView v;
  for (int k = 0; k < 3; ++k) {
    v.lo[k] = g->lo[k];
    v.cell[k] = g->cell[k];
    v.inv_cell[k] = g->inv_cell[k];
    v.dims[k] = g->dims[k];
  }
  v.box_lo = g->box_lo;
  v.box_hi = g->box_hi;
  v.cell_start = g->cell_start;
  v.entries = g->entries;
  return v;
}

__host__ __device__ __forceinline__ unsigned int f2ord(float f) {
  unsigned int u;
  memcpy(&u, &f, sizeof u);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__host__ __device__ __forceinline__ float ord2f(unsigned int u) {
  const unsigned int b = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
  float f;
  memcpy(&f, &b, sizeof f);
  return f;
}

// segment boxes (undilated) and the scene bounds (ordered-int atomics)
__global__ void boxes_kernel(const float4* p0, const float4* p1, const float4* p2,
                             const float4* p3, int64_t n, float4* blo, float4* bhi,
                             unsigned int* bounds) {
  float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n;
       s += (int64_t)gridDim.x * blockDim.x) {
    const float4 P[4] = {p0[s], p1[s], p2[s], p3[s]};
    const float r = fmaxf(fmaxf(P[0].w, P[1].w), fmaxf(P[2].w, P[3].w));
    float4 lo = make_float4(INFINITY, INFINITY, INFINITY, 0.f), hi = make_float4(-INFINITY, -INFINITY, -INFINITY, 0.f);
    for (int i = 0; i < 4; ++i) {
      lo.x = fminf(lo.x, P[i].x), lo.y = fminf(lo.y, P[i].y), lo.z = fminf(lo.z, P[i].z);
      hi.x = fmaxf(hi.x, P[i].x), hi.y = fmaxf(hi.y, P[i].y), hi.z = fmaxf(hi.z, P[i].z);
    }
    lo.x -= r, lo.y -= r, lo.z -= r;
    hi.x += r, hi.y += r, hi.z += r;
    blo[s] = lo;
    bhi[s] = hi;
    mn[0] = fminf(mn[0], lo.x), mn[1] = fminf(mn[1], lo.y), mn[2] = fminf(mn[2], lo.z);
    mx[0] = fmaxf(mx[0], hi.x), mx[1] = fmaxf(mx[1], hi.y), mx[2] = fmaxf(mx[2], hi.z);
  }
  for (int k = 0; k < 3; ++k) {
    float a = mn[k], b = mx[k];
    for (int d = 16; d > 0; d >>= 1) {
      a = fminf(a, __shfl_xor_sync(0xffffffffu, a, d));
      b = fmaxf(b, __shfl_xor_sync(0xffffffffu, b, d));
    }
    if ((threadIdx.x & 31) == 0 && a <= b) {
      atomicMin(&bounds[k], f2ord(a));
      atomicMax(&bounds[3 + k], f2ord(b));
    }
  }
}

__device__ __forceinline__ void cell_range(const GridView& g, float4 lo, float4 hi, int c0[3],
                                           int c1[3]) {
  const float l[3] = {lo.x, lo.y, lo.z}, h[3] = {hi.x, hi.y, hi.z};
  for (int k = 0; k < 3; ++k) {
    c0[k] = max(0, min(g.dims[k] - 1, (int)floorf((l[k] - g.lo[k]) * g.inv_cell[k])));
    c1[k] = max(0, min(g.dims[k] - 1, (int)floorf((h[k] - g.lo[k]) * g.inv_cell[k])));
  }
}

// dilate the boxes (1e-3 cell) and count the cells each one overlaps
__global__ void register_count_kernel(GridView g, int64_t n, float4* blo, float4* bhi,
                                      uint32_t* cell_count) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n;
       s += (int64_t)gridDim.x * blockDim.x) {
    float4 lo = blo[s], hi = bhi[s];
    lo.x -= 1e-3f * g.cell[0], lo.y -= 1e-3f * g.cell[1], lo.z -= 1e-3f * g.cell[2];
    hi.x += 1e-3f * g.cell[0], hi.y += 1e-3f * g.cell[1], hi.z += 1e-3f * g.cell[2];
    blo[s] = lo;
    bhi[s] = hi;
    int c0[3], c1[3];
    cell_range(g, lo, hi, c0, c1);
    for (int z = c0[2]; z <= c1[2]; ++z)
      for (int y = c0[1]; y <= c1[1]; ++y)
        for (int x = c0[0]; x <= c1[0]; ++x)
          atomicAdd(&cell_count[((int64_t)z * g.dims[1] + y) * g.dims[0] + x], 1u);
  }
}

__global__ void register_fill_kernel(GridView g, int64_t n, const uint32_t* cell_start,
                                     uint32_t* cursor, uint32_t* entries) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n;
       s += (int64_t)gridDim.x * blockDim.x) {
    int c0[3], c1[3];
    cell_range(g, g.box_lo[s], g.box_hi[s], c0, c1);
    for (int z = c0[2]; z <= c1[2]; ++z)
      for (int y = c0[1]; y <= c1[1]; ++y)
        for (int x = c0[0]; x <= c1[0]; ++x) {
          const int64_t c = ((int64_t)z * g.dims[1] + y) * g.dims[0] + x;
          entries[cell_start[c] + atomicAdd(&cursor[c], 1u)] = (uint32_t)s;
        }
  }
}

// deterministic order inside each cell: insertion sort by segment id
__global__ void sort_cells_kernel(int64_t n_cells, const uint32_t* cell_start, uint32_t* entries) {
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n_cells;
       c += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t b = cell_start[c], e = cell_start[c + 1];
    for (uint32_t i = b + 1; i < e; ++i) {
      const uint32_t v = entries[i];
      uint32_t j = i;
      while (j > b && entries[j - 1] > v) {
        entries[j] = entries[j - 1];
        --j;
      }
      entries[j] = v;
    }
  }
}

// Ray entry/exit of a box (slab test); false if they do not overlap on [t0, t1].
__device__ __forceinline__ bool box_entry(const float o[3], const float id[3], float4 lo, float4 hi,
                                          float t0, float t1, float& te) {
  const float l[3] = {lo.x, lo.y, lo.z}, h[3] = {hi.x, hi.y, hi.z};
  float a = t0, b = t1;
  for (int k = 0; k < 3; ++k) {
    float x = (l[k] - o[k]) * id[k], y = (h[k] - o[k]) * id[k];
    if (isnan(x) || isnan(y)) {  // direction 0 on this axis: inside or outside the slab
      if (o[k] < l[k] || o[k] > h[k]) return false;
      continue;
    }
    a = fmaxf(a, fminf(x, y));
    b = fminf(b, fmaxf(x, y));
  }
  te = a;
  return a <= b;
}

// The DDA, resumable: per-ray constants and an 8-word state (the current cell, the axis
// crossings, the cell's entry t and a cursor into its segment list).  walk() emits every
// candidate of the ray in front-to-back cell order; dda_walk() emits up to kmax and can be
// resumed where it stopped, emitting the same sequence.
struct RayDDA {
  float o[3], d[3], id[3];
  float t0, t1;
  int step[3];
  float tdelta[3];
};
struct DDAState {
  int c[3];  // c[0] < 0: the walk is over
  float tnext[3];
  float tin;
  uint32_t cursor;
};

__device__ bool dda_setup(const GridView& g, float4 r0, float4 r1, RayDDA& R, DDAState& S) {
  R.o[0] = r0.x, R.o[1] = r0.y, R.o[2] = r0.z;
  R.d[0] = r1.x, R.d[1] = r1.y, R.d[2] = r1.z;
  for (int k = 0; k < 3; ++k) R.id[k] = 1.0f / R.d[k];  // +-inf for a zero component
  // clip [0, tmax) to the grid box
  float t0 = 0.0f, t1 = r0.w;
  for (int k = 0; k < 3; ++k) {
    const float lo = g.lo[k], hi = g.lo[k] + g.dims[k] * g.cell[k];
    if (R.d[k] == 0.0f) {
      if (R.o[k] < lo || R.o[k] > hi) t1 = -1.0f;
      continue;
    }
    float x = (lo - R.o[k]) * R.id[k], y = (hi - R.o[k]) * R.id[k];
    t0 = fmaxf(t0, fminf(x, y));
    t1 = fminf(t1, fmaxf(x, y));
  }
  R.t0 = t0;
  R.t1 = t1;
  for (int k = 0; k < 3; ++k) {
    const float p = R.o[k] + t0 * R.d[k];
    S.c[k] = max(0, min(g.dims[k] - 1, (int)floorf((p - g.lo[k]) * g.inv_cell[k])));
    if (R.d[k] > 0.0f) {
      R.step[k] = 1;
      S.tnext[k] = (g.lo[k] + (S.c[k] + 1) * g.cell[k] - R.o[k]) * R.id[k];
      R.tdelta[k] = g.cell[k] * R.id[k];
    } else if (R.d[k] < 0.0f) {
      R.step[k] = -1;
      S.tnext[k] = (g.lo[k] + S.c[k] * g.cell[k] - R.o[k]) * R.id[k];
      R.tdelta[k] = -g.cell[k] * R.id[k];
    } else {
      R.step[k] = 0;
      S.tnext[k] = INFINITY;
      R.tdelta[k] = INFINITY;
    }
  }
  S.tin = t0;
  S.cursor = 0;
  if (!(t0 <= t1)) S.c[0] = -1;
  return S.c[0] >= 0;
}

// Re-derive the constants of a ray whose state is stored (the setup is deterministic).
__device__ void dda_consts(const GridView& g, float4 r0, float4 r1, RayDDA& R) {
  DDAState tmp;
  dda_setup(g, r0, r1, R, tmp);
}

template <class Emit>
__device__ uint32_t dda_walk(const GridView& g, const RayDDA& R, DDAState& S, uint32_t kmax,
                             Emit emit) {
  uint32_t n = 0;
  while (S.c[0] >= 0) {
    const int ax = S.tnext[0] <= S.tnext[1] ? (S.tnext[0] <= S.tnext[2] ? 0 : 2)
                                            : (S.tnext[1] <= S.tnext[2] ? 1 : 2);
    // the last cell (the ray ends in it, or the next step leaves the grid) extends to t1, so
    // a rounding disagreement between the DDA and the clipped interval loses nothing
    const bool last = S.tnext[ax] >= R.t1 || S.c[ax] + R.step[ax] < 0 ||
                      S.c[ax] + R.step[ax] >= g.dims[ax];
    const float tout = last ? R.t1 : S.tnext[ax];
    const int64_t cell = ((int64_t)S.c[2] * g.dims[1] + S.c[1]) * g.dims[0] + S.c[0];
    const uint32_t b = g.cell_start[cell], e = g.cell_start[cell + 1];
    for (uint32_t i = b + S.cursor; i < e; ++i) {
      const uint32_t s = g.entries[i];
      float te;
      if (box_entry(R.o, R.id, g.box_lo[s], g.box_hi[s], R.t0, R.t1, te) && te >= S.tin &&
          te <= tout) {
        emit(s);
        if (++n == kmax) {
          S.cursor = i + 1 - b;
          return n;
        }
      }
    }
    S.cursor = 0;
    if (last) {
      S.c[0] = -1;
      break;
    }
    S.c[ax] += R.step[ax];
    S.tin = tout;
    S.tnext[ax] += R.tdelta[ax];
  }
  return n;
}

template <class Emit>
__device__ void walk(const GridView& g, float4 r0, float4 r1, Emit emit) {
  RayDDA R;
  DDAState S;
  if (dda_setup(g, r0, r1, R, S)) dda_walk(g, R, S, 0xffffffffu, emit);
}

__global__ void __launch_bounds__(128) count_kernel(GridView g, const float4* rays, int64_t n_rays,
                                                   uint32_t* cnt, unsigned int* maxc) {
  uint32_t mymax = 0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rays;
       r += (int64_t)gridDim.x * blockDim.x) {
    uint32_t c = 0;
    walk(g, rays[2 * r], rays[2 * r + 1], [&](uint32_t) { ++c; });
    cnt[r] = c;
    mymax = max(mymax, c);
  }
  for (int d = 16; d > 0; d >>= 1) mymax = max(mymax, __shfl_xor_sync(0xffffffffu, mymax, d));
  if ((threadIdx.x & 31) == 0) atomicMax(maxc, mymax);
}

__global__ void __launch_bounds__(128) write_kernel(GridView g, const float4* rays, int64_t n_rays,
                                                   const uint32_t* off, uint2* pairs) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rays;
       r += (int64_t)gridDim.x * blockDim.x) {
    uint32_t k = off[r];
    walk(g, rays[2 * r], rays[2 * r + 1], [&](uint32_t s) { pairs[k++] = make_uint2((uint32_t)r, s); });
  }
}

// Rounds order: the k-th candidates of all rays (ray order), then the (k+1)-th, ...
// Per block of 1024 rays and rank k: how many of its rays have more than k candidates
// (a histogram of the block's counts, summed from the top), k-major for the scan.
constexpr int kRB = 1024;
__global__ void __launch_bounds__(256) rank_counts_kernel(const uint32_t* off, int64_t n_rays,
                                                         uint32_t max_count, int64_t nblocks,
                                                         uint32_t* bk) {
  extern __shared__ uint32_t hist[];  // [max_count + 1]
  const int64_t b = blockIdx.x;
  for (uint32_t k = threadIdx.x; k <= max_count; k += blockDim.x) hist[k] = 0u;
  __syncthreads();
  for (int j = threadIdx.x; j < kRB; j += blockDim.x) {
    const int64_t r = b * kRB + j;
    if (r < n_rays) atomicAdd(&hist[off[r + 1] - off[r]], 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // suffix sums: #{rays with count > k}
    uint32_t above = 0;
    for (int64_t k = (int64_t)max_count - 1; k >= 0; --k) {
      above += hist[k + 1];
      hist[k + 1] = above;
    }
  }
  __syncthreads();
  for (uint32_t k = threadIdx.x; k < max_count; k += blockDim.x)
    bk[(int64_t)k * nblocks + b] = hist[k + 1];
}

__global__ void __launch_bounds__(256) rounds_scatter_kernel(const uint32_t* off, int64_t n_rays,
                                                            int64_t nblocks,
                                                            const uint32_t* bstart,
                                                            const uint2* csr, uint2* out) {
  __shared__ uint32_t bmax;
  const int64_t b = blockIdx.x;
  // thread t owns rays b*1024 + 4t .. +3 (contiguous: block ranks follow ray order)
  uint32_t cnt[4], base[4], mine = 0;
  for (int j = 0; j < 4; ++j) {
    const int64_t r = b * kRB + 4 * threadIdx.x + j;
    cnt[j] = r < n_rays ? off[r + 1] - off[r] : 0u;
    base[j] = r < n_rays ? off[r] : 0u;
    mine = max(mine, cnt[j]);
  }
  if (threadIdx.x == 0) bmax = 0;
  __syncthreads();
  atomicMax(&bmax, mine);
  __syncthreads();
  const uint32_t kend = bmax;
  for (uint32_t k = 0; k < kend; ++k) {
    uint32_t f = 0;
    for (int j = 0; j < 4; ++j) f += cnt[j] > k;
    uint32_t total;
    uint32_t rank = fiberscan::block_excl(f, &total) + bstart[(int64_t)k * nblocks + b];
    for (int j = 0; j < 4; ++j)
      if (cnt[j] > k) out[rank++] = csr[base[j] + k];
  }
}

// ---- closest hit with early termination (fiber_grid_closest) ----------------------------
__global__ void closest_init_kernel(GridView g, const float4* rays, int64_t n_rays,
                                    DDAState* st, uint32_t* active) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rays;
       r += (int64_t)gridDim.x * blockDim.x) {
    RayDDA R;
    DDAState S;
    dda_setup(g, rays[2 * r], rays[2 * r + 1], R, S);
    st[r] = S;
    active[r] = (uint32_t)r;
  }
}

// One round: every active ray whose best hit is not strictly before its walk position emits
// its next k candidates into pairs[j*k ..] (unused slots: an out-of-range ray, a no-op pair);
// keep[j] = the ray still has candidates after this round.
__global__ void closest_walk_kernel(GridView g, const float4* rays, int64_t n_rays,
                                    DDAState* st, const uint32_t* active, int64_t n_active,
                                    uint32_t k, const unsigned long long* nearest, uint2* pairs,
                                    uint32_t* keep) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_active;
       j += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t r = active[j];
    DDAState S = st[r];
    const unsigned long long key = nearest[r];
    const float best = key == ~0ull ? INFINITY : __uint_as_float((uint32_t)(key >> 32));
    uint32_t n = 0;
    // every later candidate enters its box at t >= S.tin, and its hits lie in the box
    if (S.c[0] >= 0 && !(best < S.tin)) {
      RayDDA R;
      dda_consts(g, rays[2 * r], rays[2 * r + 1], R);
      uint32_t m = 0;
      n = dda_walk(g, R, S, k, [&](uint32_t s) { pairs[(uint64_t)j * k + m++] = make_uint2(r, s); });
      st[r] = S;
    }
    for (uint32_t q = n; q < k; ++q) pairs[(uint64_t)j * k + q] = make_uint2(0xffffffffu, 0u);
    keep[j] = S.c[0] >= 0 && n > 0 ? 1u : 0u;
  }
}

__global__ void compact_kernel(const uint32_t* active, const uint32_t* keep, const uint32_t* pos,
                               int64_t n, uint32_t* out) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x)
    if (keep[j]) out[pos[j]] = active[j];
}

int grid_blocks(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  return (int)(b > 148 * 64 ? 148 * 64 : (b < 1 ? 1 : b));
}

}  // namespace

extern "C" int fiber_grid_create(const fiber_segments* segs, float cells_per_segment,
                                 fiber_grid** out, void* cuda_stream) {
  if (!segs || !out || segs->n <= 0 || segs->n >= ((int64_t)1 << 32) || !segs->p0 ||
      !(cells_per_segment > 0.0f))
    return set_error(FIBER_EINVAL, "fiber_grid_create: bad arguments");
  *out = nullptr;
  int rc = check_device();
  if (rc != FIBER_OK) return rc;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  fiber_grid_s* g = new fiber_grid_s{};
  cudaGetDevice(&g->device);
  const int64_t n = segs->n;
  g->n_segs = n;
  unsigned int* bounds = nullptr;
  bool ok = cudaMalloc((void**)&g->box_lo, n * sizeof(float4)) == cudaSuccess &&
            cudaMalloc((void**)&g->box_hi, n * sizeof(float4)) == cudaSuccess &&
            cudaMalloc((void**)&bounds, 6 * sizeof(unsigned int)) == cudaSuccess;
  if (ok) {
    const unsigned int init[6] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0u, 0u, 0u};
    ok = cudaMemcpyAsync(bounds, init, sizeof(init), cudaMemcpyHostToDevice, st) == cudaSuccess;
  }
  unsigned int hb[6];
  if (ok) {
    boxes_kernel<<<grid_blocks(n, 256), 256, 0, st>>>(
        (const float4*)segs->p0, (const float4*)segs->p1, (const float4*)segs->p2,
        (const float4*)segs->p3, n, g->box_lo, g->box_hi, bounds);
    ok = cudaMemcpyAsync(hb, bounds, sizeof(hb), cudaMemcpyDeviceToHost, st) == cudaSuccess &&
         cudaStreamSynchronize(st) == cudaSuccess;
  }
  if (ok) {
    // cells: about cells_per_segment x n, cubic-ish, each axis in [1, 1024]
    float ext[3], lo[3];
    double vol = 1.0;
    for (int k = 0; k < 3; ++k) {
      lo[k] = ord2f(hb[k]);
      ext[k] = fmaxf(ord2f(hb[3 + k]) - lo[k], 1e-30f);
      vol *= ext[k];
    }
    const double target = fmax(1.0, (double)cells_per_segment * (double)n);
    double cs = cbrt(vol / target);
    for (int k = 0; k < 3; ++k) {
      int d = (int)fmin(1024.0, fmax(1.0, ceil(ext[k] / cs)));
      g->dims[k] = d;
      g->lo[k] = lo[k];
      g->cell[k] = ext[k] / d * (1.0f + 1e-6f);
      g->inv_cell[k] = 1.0f / g->cell[k];
    }
    g->n_cells = (int64_t)g->dims[0] * g->dims[1] * g->dims[2];
    ok = cudaMalloc((void**)&g->cell_start, (g->n_cells + 1) * sizeof(uint32_t)) == cudaSuccess &&
         cudaMemsetAsync(g->cell_start, 0, (g->n_cells + 1) * sizeof(uint32_t), st) == cudaSuccess;
  }
  uint32_t* sums = nullptr;
  uint32_t* cursor = nullptr;
  if (ok) {
    GridView v = view(g);
    register_count_kernel<<<grid_blocks(n, 256), 256, 0, st>>>(v, n, g->box_lo, g->box_hi, g->cell_start);
    ok = cudaMalloc((void**)&sums, fiberscan::scan_scratch(g->n_cells + 1) * sizeof(uint32_t)) == cudaSuccess;
    if (ok) {
      fiberscan::exclusive_scan(g->cell_start, g->cell_start, g->n_cells + 1, sums, st);
      uint32_t total = 0;
      ok = cudaMemcpyAsync(&total, g->cell_start + g->n_cells, sizeof(uint32_t),
                           cudaMemcpyDeviceToHost, st) == cudaSuccess &&
           cudaStreamSynchronize(st) == cudaSuccess;
      g->n_entries = total;
    }
  }
  if (ok) {
    ok = cudaMalloc((void**)&g->entries, (g->n_entries + 1) * sizeof(uint32_t)) == cudaSuccess &&
         cudaMalloc((void**)&cursor, g->n_cells * sizeof(uint32_t)) == cudaSuccess &&
         cudaMemsetAsync(cursor, 0, g->n_cells * sizeof(uint32_t), st) == cudaSuccess;
  }
  if (ok) {
    GridView v = view(g);
    register_fill_kernel<<<grid_blocks(n, 256), 256, 0, st>>>(v, n, g->cell_start, cursor, g->entries);
    sort_cells_kernel<<<grid_blocks(g->n_cells, 256), 256, 0, st>>>(g->n_cells, g->cell_start, g->entries);
    ok = cudaStreamSynchronize(st) == cudaSuccess && cudaGetLastError() == cudaSuccess;
  }
  cudaFree(bounds);
  cudaFree(sums);
  cudaFree(cursor);
  if (!ok) {
    fiber_grid_destroy(g);
    cudaGetLastError();
    return set_error(FIBER_ECUDA, "fiber_grid_create: CUDA failure");
  }
  *out = g;
  return FIBER_OK;
}

extern "C" int fiber_grid_destroy(fiber_grid* g) {
  if (!g) return FIBER_OK;
  cudaFree(g->box_lo);
  cudaFree(g->box_hi);
  cudaFree(g->cell_start);
  cudaFree(g->entries);
  delete g;
  return FIBER_OK;
}

extern "C" int fiber_grid_info(const fiber_grid* g, int32_t dims[3], int64_t* n_entries) {
  if (!g || !dims || !n_entries) return set_error(FIBER_EINVAL, "fiber_grid_info: NULL");
  for (int k = 0; k < 3; ++k) dims[k] = g->dims[k];
  *n_entries = g->n_entries;
  return FIBER_OK;
}

extern "C" int fiber_grid_count(const fiber_grid* g, const fiber_ray* rays, int64_t n_rays,
                                uint32_t* offsets, uint32_t* max_count, uint64_t* total,
                                void* cuda_stream) {
  if (!g || n_rays < 0 || n_rays >= ((int64_t)1 << 32) || (n_rays > 0 && !rays) || !offsets ||
      !max_count || !total)
    return set_error(FIBER_EINVAL, "fiber_grid_count: bad arguments");
  int rc = check_device();
  if (rc != FIBER_OK) return rc;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  unsigned int* dmax = nullptr;
  uint32_t* sums = nullptr;
  bool ok = cudaMalloc((void**)&dmax, sizeof(unsigned int)) == cudaSuccess &&
            cudaMemsetAsync(dmax, 0, sizeof(unsigned int), st) == cudaSuccess &&
            cudaMalloc((void**)&sums, fiberscan::scan_scratch(n_rays + 1) * sizeof(uint32_t)) == cudaSuccess &&
            cudaMemsetAsync(offsets + n_rays, 0, sizeof(uint32_t), st) == cudaSuccess;
  if (ok && n_rays > 0) {
    count_kernel<<<grid_blocks(n_rays, 128), 128, 0, st>>>(view(g), (const float4*)rays, n_rays,
                                                          offsets, dmax);
  }
  uint32_t tot = 0;
  if (ok) {
    fiberscan::exclusive_scan(offsets, offsets, n_rays + 1, sums, st);
    ok = cudaMemcpyAsync(max_count, dmax, sizeof(uint32_t), cudaMemcpyDeviceToHost, st) == cudaSuccess &&
         cudaMemcpyAsync(&tot, offsets + n_rays, sizeof(uint32_t), cudaMemcpyDeviceToHost, st) == cudaSuccess &&
         cudaStreamSynchronize(st) == cudaSuccess && cudaGetLastError() == cudaSuccess;
  }
  *total = tot;
  cudaFree(dmax);
  cudaFree(sums);
  if (!ok) return set_error(FIBER_ECUDA, "fiber_grid_count: CUDA failure");
  return FIBER_OK;
}

extern "C" int fiber_grid_candidates(const fiber_grid* g, const fiber_ray* rays, int64_t n_rays,
                                     const uint32_t* offsets, uint32_t max_count, int order,
                                     fiber_pair* pairs, void* cuda_stream) {
  if (!g || n_rays < 0 || n_rays >= ((int64_t)1 << 32) || (n_rays > 0 && (!rays || !offsets || !pairs)) ||
      (order != 0 && order != 1))
    return set_error(FIBER_EINVAL, "fiber_grid_candidates: bad arguments");
  int rc = check_device();
  if (rc != FIBER_OK) return rc;
  if (n_rays == 0) return FIBER_OK;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  GridView v = view(g);
  if (order == 0) {
    write_kernel<<<grid_blocks(n_rays, 128), 128, 0, st>>>(v, (const float4*)rays, n_rays, offsets,
                                                          (uint2*)pairs);
    return check_launch("fiber_grid_candidates");
  }
  // rounds: CSR first, then the deterministic scatter
  uint32_t total = 0;
  if (cudaMemcpyAsync(&total, offsets + n_rays, sizeof(uint32_t), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return set_error(FIBER_ECUDA, "fiber_grid_candidates: CUDA failure");
  const int64_t nb = (n_rays + kRB - 1) / kRB;
  uint2* csr = nullptr;
  uint32_t *bk = nullptr, *sums = nullptr;
  const int64_t nbk = (int64_t)max_count * nb;
  bool ok = cudaMalloc((void**)&csr, ((size_t)total + 1) * sizeof(uint2)) == cudaSuccess &&
            cudaMalloc((void**)&bk, (nbk + 1) * sizeof(uint32_t)) == cudaSuccess &&
            cudaMalloc((void**)&sums, fiberscan::scan_scratch(nbk + 1) * sizeof(uint32_t)) == cudaSuccess;
  if (ok) {
    write_kernel<<<grid_blocks(n_rays, 128), 128, 0, st>>>(v, (const float4*)rays, n_rays, offsets, csr);
    if (max_count > 0) {
      const size_t hbytes = ((size_t)max_count + 1) * sizeof(uint32_t);
      if (hbytes > 200 * 1024) {
        ok = false;  // counts beyond 51k candidates per ray: use order 0
      } else {
        if (hbytes > 48 * 1024)
          cudaFuncSetAttribute(rank_counts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)hbytes);
        rank_counts_kernel<<<(unsigned)nb, 256, hbytes, st>>>(offsets, n_rays, max_count, nb, bk);
        fiberscan::exclusive_scan(bk, bk, nbk, sums, st);
        rounds_scatter_kernel<<<(unsigned)nb, 256, 0, st>>>(offsets, n_rays, nb, bk, csr,
                                                           (uint2*)pairs);
      }
    }
    ok = cudaStreamSynchronize(st) == cudaSuccess && cudaGetLastError() == cudaSuccess;
  }
  cudaFree(csr);
  cudaFree(bk);
  cudaFree(sums);
  if (!ok) return set_error(FIBER_ECUDA, "fiber_grid_candidates: CUDA failure");
  return FIBER_OK;
}

extern "C" int fiber_grid_closest(const fiber_grid* g, const fiber_ray* rays, int64_t n_rays,
                                  const fiber_segments* segs, int max_depth, uint64_t* nearest,
                                  int* rounds_out, void* cuda_stream) {
  if (!g || !segs || n_rays < 0 || n_rays >= ((int64_t)1 << 31) || (n_rays > 0 && (!rays || !nearest)) ||
      max_depth < 0 || max_depth > FIBER_MAX_DEPTH || segs->n != g->n_segs)
    return set_error(FIBER_EINVAL, "fiber_grid_closest: bad arguments");
  int rc = check_device();
  if (rc != FIBER_OK) return rc;
  if (rounds_out) *rounds_out = 0;
  if (n_rays == 0) return FIBER_OK;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  GridView v = view(g);
  DDAState* state = nullptr;
  uint32_t *act[2] = {nullptr, nullptr}, *keep = nullptr, *pos = nullptr, *sums = nullptr;
  uint2* pairs = nullptr;
  const uint32_t kmax = 256;
  bool ok = cudaMalloc((void**)&state, n_rays * sizeof(DDAState)) == cudaSuccess &&
            cudaMalloc((void**)&act[0], n_rays * sizeof(uint32_t)) == cudaSuccess &&
            cudaMalloc((void**)&act[1], n_rays * sizeof(uint32_t)) == cudaSuccess &&
            cudaMalloc((void**)&keep, (n_rays + 1) * sizeof(uint32_t)) == cudaSuccess &&
            cudaMalloc((void**)&pos, (n_rays + 1) * sizeof(uint32_t)) == cudaSuccess &&
            cudaMalloc((void**)&sums, fiberscan::scan_scratch(n_rays + 1) * sizeof(uint32_t)) == cudaSuccess;
  // the pair buffer of a round: n_active * k <= max over rounds; grown on demand
  size_t pair_cap = 0;
  int64_t n_active = n_rays;
  uint32_t k = 8;
  int rounds = 0;
  if (ok) {
    closest_init_kernel<<<grid_blocks(n_rays, 256), 256, 0, st>>>(v, (const float4*)rays, n_rays,
                                                                  state, act[0]);
    ok = cudaGetLastError() == cudaSuccess;
  }
  int cur = 0;
  while (ok && n_active > 0) {
    const size_t need = (size_t)n_active * k;
    if (need > pair_cap) {
      cudaFree(pairs);
      pairs = nullptr;
      pair_cap = need;
      ok = cudaMalloc((void**)&pairs, pair_cap * sizeof(uint2)) == cudaSuccess;
      if (!ok) break;
    }
    closest_walk_kernel<<<grid_blocks(n_active, 128), 128, 0, st>>>(
        v, (const float4*)rays, n_rays, state, act[cur], n_active, k,
        (const unsigned long long*)nearest, pairs, keep);
    ok = cudaGetLastError() == cudaSuccess;
    if (!ok) break;
    rc = launch_intersect_mode(rays, n_rays, segs, (const fiber_pair*)pairs, (int64_t)need,
                               max_depth, nearest, cuda_stream, 3);
    if (rc != FIBER_OK) {
      ok = false;
      break;
    }
    cudaMemsetAsync(keep + n_active, 0, sizeof(uint32_t), st);
    fiberscan::exclusive_scan(keep, pos, n_active + 1, sums, st);
    compact_kernel<<<grid_blocks(n_active, 256), 256, 0, st>>>(act[cur], keep, pos, n_active,
                                                               act[cur ^ 1]);
    uint32_t next = 0;
    ok = cudaMemcpyAsync(&next, pos + n_active, sizeof(uint32_t), cudaMemcpyDeviceToHost, st) == cudaSuccess &&
         cudaStreamSynchronize(st) == cudaSuccess;
    n_active = next;
    cur ^= 1;
    k = k * 2 > kmax ? kmax : k * 2;
    ++rounds;
  }
  cudaFree(state);
  cudaFree(act[0]);
  cudaFree(act[1]);
  cudaFree(keep);
  cudaFree(pos);
  cudaFree(sums);
  cudaFree(pairs);
  if (rounds_out) *rounds_out = rounds;
  if (rc != FIBER_OK) return rc;
  if (!ok) return set_error(FIBER_ECUDA, "fiber_grid_closest: CUDA failure");
  return FIBER_OK;
}
