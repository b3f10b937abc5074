// Passable-set predicate and connected-component labelling for sm_100a.
//
// Predicate (bit-exact with the reference): depth
// z = (fx*b)/d valid iff d finite, d > 0 and z finite (geometry.py:39-45,
// 169-172); edge e = |((((4c - left) - right) - up) - down)| evaluated in
// numpy's left-to-right order with correctly rounded fp64 operations
// (adaptive.py:80-97), valid only at interior pixels with all five depths
// valid; passable = edge valid and e <= t (the ST ray test,
// adaptive.py:130-132, 218-221).  The labeller evaluates it as an fp32
// filter with a rigorous error bound and falls back to the exact fp64
// evaluation only when |e32 - t| is inside the bound, so every decision is
// the fp64 decision (see fast_passable below).
//
// Labelling (no reference function): 8-connected
// components of the passable set, canonical label = smallest raster index in
// the component.  The passable set is a BIT mask (one uint32 word per 32
// pixels of a row) and the union-find runs over band runs (maximal runs of
// set bits of two OR-ed rows inside one word), not pixels.  Every link goes
// from the larger node to the smaller (atomicMin), so a root is always its
// component's minimum and the result is independent of scheduling.  Three
// launches per batch:
//
//   1. ccl_tile_kernel   128x128 tile per CTA, 256 threads = (2-row band,
//      word); bits from passable_bits_kernel (or a uint8 grid), band-run
//      union-find in shared memory, tile-border labels -> compact seam rows
//      / columns, global node init G[root] = root for border-touching roots,
//      the slot labels (16-bit tile pixel index per band-run slot) and the
//      border-root flags for pass 3.
//   2. ccl_seam_kernel   unions across tile seams in global memory (G is the
//      label array itself; only border-touching roots are ever nodes).
//   3. ccl_resolve_kernel  walks G once per border-touching root, then maps
//      each pixel to its band run (bit ops), the run to its tile label (the
//      slot labels) and that to its final label, with coalesced stores.
//
// HBM traffic per pixel from the bit mask: 1/8 B bits in (twice), 1/2 B slot
// labels out and back, 4 B labels out (+ the sparse seam / root traffic),
// against the 4 B/px floor of writing the labels.

#include <cuda_runtime.h>
#include <float.h>
#include <stdint.h>

#include <algorithm>

#include "sn_internal.h"

namespace sn {

constexpr int kLTW = 128;             // label tile columns
constexpr int kLTH = 128;             // label tile rows
constexpr int kLWords = kLTW / 32;    // words per tile row
constexpr int kRowWords = kLTH * kLWords;  // 512 row-words per tile
constexpr int kBands = kLTH / 2;      // 2-row bands per tile
constexpr int kLThreads = kBands * kLWords;  // 256: one thread per (band, word)
// node slots: a word holds at most 16 band runs, so the slot of a band run is
// band * 64 + word * 16 + (its rank among the word's runs) -- dense per word,
// no block scan: the rank is a popcount of the word's run starts below it
constexpr int kWordSlots = 16;
constexpr int kBandSlots = kLWords * kWordSlots;  // 64
constexpr int kSlots = kBands * kBandSlots;       // 4096
static_assert(kLThreads * kWordSlots == kSlots, "slot export: one word's slots per thread");

__device__ __forceinline__ double edge_value(double c, double l, double r, double u, double dn) {
  return fabs(__dsub_rn(__dsub_rn(__dsub_rn(__dsub_rn(__dmul_rn(4.0, c), l), r), u), dn));
}

__device__ __forceinline__ bool valid_z(double z) { return z == z; }

// ---------------------------------------------------------------------------
// standalone predicate (API sn_passable; exact fp64 per pixel, optional edges)

template <typename T>
__global__ void passable_kernel(const T* __restrict__ disp, const CclParams p,
                                uint8_t* __restrict__ pas, double* __restrict__ edges) {
  const int64_t total = p.B * p.H * p.W;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = idx % p.W;
    const int64_t y = (idx / p.W) % p.H;
    const T* f = disp + (idx - y * p.W - x);
    bool ok = false;
    double e = __longlong_as_double(0x7ff8000000000000ll);
    if (x >= 1 && x + 1 < p.W && y >= 1 && y + 1 < p.H) {
      const double c = pred_depth(f[y * p.W + x], p.fxb);
      const double l = pred_depth(f[y * p.W + x - 1], p.fxb);
      const double r = pred_depth(f[y * p.W + x + 1], p.fxb);
      const double u = pred_depth(f[(y - 1) * p.W + x], p.fxb);
      const double dn = pred_depth(f[(y + 1) * p.W + x], p.fxb);
      if (valid_z(c) && valid_z(l) && valid_z(r) && valid_z(u) && valid_z(dn)) {
        e = edge_value(c, l, r, u, dn);
        ok = true;
      }
    }
    if (pas) pas[idx] = (ok && e <= p.t) ? 1 : 0;
    if (edges) edges[idx] = e;
  }
}

// ---------------------------------------------------------------------------
// union-find helpers (indices only ever point to smaller indices)

// find with path halving: every write replaces a parent by an ancestor, so it
// commutes with concurrent unions (which only atomicMin roots).  The global
// array G of the seam pass: node = label = frame index.
__device__ __forceinline__ int uf_find(volatile int32_t* L, int x) {
  while (true) {
    const int p = L[x];
    SN_ASSERT(p >= 0 && p <= x);  // links only ever go to smaller nodes
    if (p == x) return x;
    const int gp = L[p];
    if (gp == p) return p;
    L[x] = gp;
    x = gp;
  }
}

// read-only find
__device__ __forceinline__ int uf_root(const volatile int32_t* L, int x) {
  int p = L[x];
  while (p != x) {
    x = p;
    p = L[x];
  }
  return x;
}

__device__ __forceinline__ void uf_unite(int32_t* L, int a, int b) {
  volatile int32_t* V = L;
  while (true) {
    a = uf_find(V, a);
    b = uf_find(V, b);
    if (a == b) return;
    if (a > b) {
      const int t = a;
      a = b;
      b = t;
    }
    const int old = atomicMin(&L[b], a);
    if (old == b) return;
    b = old;
  }
}

// The tile's parent array (shared memory) holds BYTE OFFSETS of padded slot
// entries: slot s lives at soff(s) = 4 (s + s/16), one pad word per word's
// 16 slots, so the lanes of a warp -- 8 bands x 4 words -- touching slots of
// equal rank in different words hit 32 different banks (4k + 17w mod 32).
// Offsets grow with the slot, so min-offset roots are min-slot roots; a
// parent value is directly the address of its entry (no index arithmetic in
// the find loops).  Roots' entries later hold label - kEnc (< 0).
__device__ __forceinline__ int soff(int s) { return (s + (s >> 4)) << 2; }
constexpr int kParentBytes = (kSlots + kSlots / 16) * 4;
static_assert(kParentBytes < 65536, "queued pairs pack two offsets into 16 bits each");
#define SN_CHECK_OFF(off) SN_ASSERT((off) >= 0 && (off) < kParentBytes && ((off) & 3) == 0)
__device__ __forceinline__ int ld_o(const volatile int32_t* L, int off) {
  SN_CHECK_OFF(off);
  return *reinterpret_cast<const volatile int32_t*>(reinterpret_cast<const volatile char*>(L) + off);
}
__device__ __forceinline__ void st_o(volatile int32_t* L, int off, int v) {
  SN_CHECK_OFF(off);
  *reinterpret_cast<volatile int32_t*>(reinterpret_cast<volatile char*>(L) + off) = v;
}
__device__ __forceinline__ int* at_o(int32_t* L, int off) {
  SN_CHECK_OFF(off);
  return reinterpret_cast<int*>(reinterpret_cast<char*>(L) + off);
}

__device__ __forceinline__ int uf_find_o(volatile int32_t* L, int x) {
  while (true) {
    const int p = ld_o(L, x);
    SN_ASSERT(p >= 0 && p <= x);  // links only ever go to smaller slots
    if (p == x) return x;
    const int gp = ld_o(L, p);
    if (gp == p) return p;
    st_o(L, x, gp);
    x = gp;
  }
}

__device__ __forceinline__ void uf_unite_o(int32_t* L, int a, int b) {
  volatile int32_t* V = L;
  while (true) {
    a = uf_find_o(V, a);
    b = uf_find_o(V, b);
    if (a == b) return;
    if (a > b) {
      const int t = a;
      a = b;
      b = t;
    }
    const int old = atomicMin(at_o(L, b), a);
    if (old == b) return;
    b = old;
  }
}

__device__ __forceinline__ uint32_t run_starts(uint32_t A) { return A & ~(A << 1); }

// bits 0 .. p of a word
__device__ __forceinline__ uint32_t upto_bit(int p) {
  return (p == 31) ? 0xffffffffu : ((2u << p) - 1u);
}

// rank (among the word's band runs, starts st) of the run that contains bit p
__device__ __forceinline__ int rank_at(uint32_t st, int p) { return __popc(st & upto_bit(p)) - 1; }

// rank of the word's last run (the one holding bit 31 if it is set)
__device__ __forceinline__ int last_rank(uint32_t st) { return __popc(st) - 1; }

// ---------------------------------------------------------------------------
// tile union-find over band runs
//
// A band is two consecutive rows; a band run is a maximal run of set bits of
// G = row0 | row1 inside one 32-bit word.  Every band run is 8-connected by
// itself (consecutive columns of G are 8-adjacent whichever row their pixels
// are in), so band runs are the union-find nodes: ~3x fewer than pixel runs
// of single rows on C3, and half the rows to merge.  A node's slot is
// band * 128 + column of the run's first column; links go to smaller slots
// (atomicMin), so roots are the minimum slot of their tile component and the
// result is schedule-independent.  The component's label is its smallest
// PIXEL index, reduced with atomicMin after compression.  Measured with
// tools/ccl_bench.cu on C3 bit masks: 2.1x faster than union-find over
// single-row word-runs (5.4 vs 11.2 us/frame), which was itself 2.3x faster
// than merging rows in log-depth rounds.
//
// On return L[slot] (for run-start slots) is the root slot (>= 0) of a
// non-root, or enc(label) = label - 2^30 (< 0) for a root.

constexpr int kEnc = 0x40000000;

__device__ __forceinline__ uint32_t band_word(const uint32_t* bits, int k, int w) {
  return bits[(2 * k) * kLWords + w] | bits[(2 * k + 1) * kLWords + w];
}

// bits [s, end of the run starting at s) of a word whose bit s is set
__device__ __forceinline__ uint32_t run_mask(uint32_t G, int s) {
  const uint32_t hi = 0xffffffffu << s;
  const uint32_t zer = ~G & hi;
  return zer ? ((zer & (0u - zer)) - 1u) & hi : hi;
}

// component label of the slot at byte offset `off`
__device__ __forceinline__ int slot_label(const int32_t* L, int off) {
  const int v = ld_o(L, off);
  return (v >= 0 ? ld_o(L, v) : v) + kEnc;
}

// offset of the band run holding pixel (r, c) of the tile (the pixel must be set)
__device__ __forceinline__ int pixel_slot(const uint32_t* bits, int r, int c) {
  const int k = r >> 1, w = c >> 5;
  return soff(k * kBandSlots + w * kWordSlots) +
         4 * rank_at(run_starts(band_word(bits, k, w)), c & 31);
}

// pairs per warp queue: the 8 queues (7 KB) share their shared memory with the
// tile's border flags (2 KB), which are only used after the unions -- 8 CTAs
// per SM need <= 27.5 KB each (160 / 192 / 224 pairs measured alike: the
// queues rarely fill)
constexpr int kUnionQueue = 224;
constexpr int kScratchWords = (kLThreads / 32) * kUnionQueue;

// One union of the tile pass.  A lane's first pair is united in place; the
// later ones go to the warp's queue while it has room (warp-aggregated: the
// active lanes take consecutive slots, one shared-memory atomic per call
// site), else in place too.  The queue is united by all 32 lanes after the
// pair walk: the per-lane pair counts differ a lot within a warp (a lane
// with many runs or overlaps kept the others idle), the queue spreads them.
__device__ __forceinline__ void unite_or_queue(int32_t* L, uint32_t* uq, int* uq_n, int a, int b,
                                               int& done) {
  if (done++ == 0) {
    uf_unite_o(L, a, b);
    return;
  }
  const uint32_t act = __activemask();
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(act) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(uq_n, __popc(act));
  base = __shfl_sync(act, base, leader);
  const int slot = base + __popc(act & ((1u << lane) - 1u));
  if (slot < kUnionQueue) {
    uq[slot] = ((uint32_t)a << 16) | (uint32_t)b;  // offsets < 2^16
    return;
  }
  uf_unite_o(L, a, b);
}

__device__ __forceinline__ void band_union_find(int32_t* L, const uint32_t* bits, int tid,
                                                uint32_t* uq, int* uq_n, uint32_t* flag) {
  const int k = tid >> 2, w = tid & 3;
  // byte offset of this word's first slot; the word's slots follow at +4,
  // the left word's at -68, the band above's at -272 (one band = 68 words)
  const int base = soff(k * kBandSlots + w * kWordSlots);
  constexpr int kWordOff = (kWordSlots + 1) * 4, kBandOff = kLWords * kWordOff;
  const uint32_t A0 = bits[(2 * k) * kLWords + w], A1 = bits[(2 * k + 1) * kLWords + w];
  const uint32_t G = A0 | A1, stG = run_starts(G);
  const int nr = __popc(stG);
  for (int i = 0; i < nr; ++i) st_o(L, base + 4 * i, base + 4 * i);
  if ((tid & 31) == 0) *uq_n = 0;
  int npairs = 0;  // this lane's pairs so far
  __syncthreads();
  // a band run crossing into this word from the left neighbour word
  if ((G & 1u) && w > 0) {
    const uint32_t Gl = band_word(bits, k, w - 1);
    if (Gl >> 31) unite_or_queue(L, uq, uq_n, base, base - kWordOff + 4 * last_rank(run_starts(Gl)), npairs);
  }
  // band k-1: only this band's first-row pixels touch it (its last row)
  if (k > 0) {
    const int rb = (2 * k - 1) * kLWords + w;
    const uint32_t B = bits[rb];
    const uint32_t stGb = run_starts(bits[rb - kLWords] | B);
    const uint32_t Gb = bits[rb - kLWords] | B;
    const uint32_t BL = w > 0 ? bits[rb - 1] : 0u, BR = w + 1 < kLWords ? bits[rb + 1] : 0u;
    const int bbase = base - kBandOff;
    int n = base;
    for (uint32_t m = stG; m; m &= m - 1u, n += 4) {
      const int s = __ffs(m) - 1;
      const uint32_t a = A0 & run_mask(G, s);
      if (!a) continue;
      uint32_t o = (a | (a << 1) | (a >> 1)) & B;
      while (o) {
        const int p = __ffs(o) - 1;
        unite_or_queue(L, uq, uq_n, n, bbase + 4 * rank_at(stGb, p), npairs);
        const uint32_t zb = ~Gb & ~upto_bit(p);  // zeros of band k-1 above p: end of that band run
        if (!zb) break;
        o &= ~((zb & (0u - zb)) - 1u);
      }
      if ((a & 1u) && (BL >> 31))
        unite_or_queue(L, uq, uq_n, n,
                       bbase - kWordOff + 4 * last_rank(run_starts(bits[rb - kLWords - 1] | BL)),
                       npairs);
      if ((a >> 31) && (BR & 1u)) unite_or_queue(L, uq, uq_n, n, bbase + kWordOff, npairs);
    }
  }
  // the queued pairs, one per lane (any union order gives the same min-slot
  // roots)
  __syncwarp();
  {
    const int cnt = min(*reinterpret_cast<volatile int*>(uq_n), kUnionQueue);
    for (int i = tid & 31; i < cnt; i += 32) {
      const uint32_t e = uq[i];
      uf_unite_o(L, (int)(e >> 16), (int)(e & 0xffffu));
    }
  }
  __syncthreads();
  // component label = smallest pixel index, reduced into the root's entry;
  // each node is pointed at its root on the way (roots may already hold a
  // label -- a negative value -- from another run's reduction: the walk
  // stops at a self-pointer or a negative entry)
  {
    int n = base;
    for (uint32_t m = stG; m; m &= m - 1u, n += 4) {
      const int s = __ffs(m) - 1;
      const uint32_t run = run_mask(G, s);
      const uint32_t a0 = A0 & run;
      const int mp = a0 ? (2 * k) * kLTW + w * 32 + __ffs(a0) - 1
                        : (2 * k + 1) * kLTW + w * 32 + __ffs(A1 & run) - 1;
      int x = n;
      for (int q = ld_o(L, x); q >= 0 && q != x; q = ld_o(L, x)) x = q;
      if (x != n) st_o(L, n, x);
      // the component's smallest pixel lies in its first band -- the root's
      // band (slots are band-major): only runs of that band reduce
      if (x >= k * kBandOff) atomicMin(at_o(L, x), mp - kEnc);
    }
  }
  // the union queues are spent: their memory becomes the border flags
  for (int i = tid; i < kLTW * kLTH / 32; i += kLThreads) flag[i] = 0u;
  __syncthreads();
}

constexpr int kTilePx = kLTW * kLTH;  // 16384: tile pixel index fits 14 bits

struct CclWorkspace {
  uint32_t* bits;   // [B][H][WW]
  uint16_t* lbl;    // [tile][kSlots] component label (tile pixel index) per band-run slot
  uint32_t* flags;  // [tile][kTilePx / 32] border-touching components (bit = label)
  int32_t* top;     // [B][n_ty][W]  first row of each tile row
  int32_t* bot;     // [B][n_ty][W]  last row of each tile row
  int32_t* left;    // [B][n_tx][H]  first column of each tile column
  int32_t* right;   // [B][n_tx][H]  last column of each tile column
  int WW, n_tx, n_ty;
};

__device__ __forceinline__ int frame_index(int px, int x0, int y0, int W) {
  return (y0 + (px >> 7)) * W + x0 + (px & (kLTW - 1));
}

// ---------------------------------------------------------------------------
// 1. tile pass.  MODE 1: uint8 passable input; MODE 2: the bit mask is the
// input (passable_bits_kernel).  Dynamic shared memory: the parent array only
// (kSlots int32 + pads = 17 KB; 8 CTAs/SM) -- the slot labels go straight to the
// workspace (measured: staging them in shared memory capped residency at 4
// CTAs/SM).

constexpr size_t kTileSmem = (size_t)(kSlots + kSlots / 16) * 4;

template <int MODE>
__global__ void __launch_bounds__(kLThreads, 8)
    ccl_tile_kernel(const uint8_t* __restrict__ pas_in, const CclParams p, const CclWorkspace ws,
                    int32_t* __restrict__ labels) {
  extern __shared__ __align__(16) int32_t smem[];
  __shared__ uint32_t bits[kRowWords];
  static_assert(kScratchWords >= kTilePx / 32, "the border flags live in the union queues");
  __shared__ uint32_t scratch[kScratchWords];
  uint32_t* flag = scratch;  // after the unions
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int W = (int)p.W, H = (int)p.H;
  const int tx = blockIdx.x, ty = blockIdx.y;
  const int x0 = tx * kLTW, y0 = ty * kLTH;
  const int64_t fbase = (int64_t)blockIdx.z * p.H * p.W;
  const int64_t frow = (int64_t)blockIdx.z * H;
  const int64_t tile = ((int64_t)blockIdx.z * ws.n_ty + ty) * ws.n_tx + tx;

  if (MODE == 1) {
    for (int rw = warp; rw < kRowWords; rw += kLThreads / 32) {
      const int r = rw >> 2, c = (rw & 3) * 32 + lane;
      const int gx = x0 + c, gy = y0 + r;
      const bool pk = gx < W && gy < H && pas_in[fbase + (int64_t)gy * W + gx] != 0;
      const uint32_t b = __ballot_sync(0xffffffffu, pk);
      if (lane == 0) bits[rw] = b;
    }
  } else {
    // both loads in flight before the stores (a rolled load -> store loop
    // waits one round trip per iteration)
    uint32_t bw[kRowWords / kLThreads];
#pragma unroll
    for (int k = 0; k < kRowWords / kLThreads; ++k) {
      const int i = k * kLThreads + tid;
      const int r = i >> 2, wc = tx * kLWords + (i & 3);
      bw[k] = (y0 + r < H && wc < ws.WW) ? __ldg(ws.bits + (frow + y0 + r) * ws.WW + wc) : 0u;
    }
#pragma unroll
    for (int k = 0; k < kRowWords / kLThreads; ++k) bits[k * kLThreads + tid] = bw[k];
  }
  __syncthreads();
  if (MODE == 1) {
    for (int i = tid; i < kRowWords; i += kLThreads) {
      const int r = i >> 2, wc = tx * kLWords + (i & 3);
      if (y0 + r < H && wc < ws.WW) ws.bits[(frow + y0 + r) * ws.WW + wc] = bits[i];
    }
  }

  int32_t* L = smem;
  __shared__ int union_n[kLThreads / 32];
  band_union_find(L, bits, tid, scratch + warp * kUnionQueue, &union_n[warp], flag);

  // every band run's entry becomes its component label, encoded as a root's
  // (label - kEnc; race-free: roots keep their value, and a non-root entry is
  // read by its owner only); flag components touching the tile border
  {
    const int k = tid >> 2, w = tid & 3;
    const uint32_t A0 = bits[(2 * k) * kLWords + w], A1 = bits[(2 * k + 1) * kLWords + w];
    const uint32_t G = A0 | A1;
    int n = soff(k * kBandSlots + w * kWordSlots);
    for (uint32_t m = run_starts(G); m; m &= m - 1u, n += 4) {
      const int s = __ffs(m) - 1;
      const int v = slot_label(L, n);
      st_o(L, n, v - kEnc);
      const uint32_t run = run_mask(G, s);
      if ((k == 0 && (A0 & run)) || (k == kBands - 1 && (A1 & run)) || (w == 0 && (run & 1u)) ||
          (w == kLWords - 1 && (run >> 31)))
        atomicOr(&flag[v >> 5], 1u << (v & 31));
    }
  }
  __syncthreads();
  // export the slot labels as 16-bit values, one word's 16 slots (32 B) per
  // thread: coalesced full-sector stores (slots that hold no run carry stale
  // values; the resolve pass reads run slots only)
  {
    const int* src = L + (soff(tid * kWordSlots) >> 2);
    uint32_t q[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      q[i] = ((uint32_t)(src[2 * i] + kEnc) & 0xffffu) | ((uint32_t)(src[2 * i + 1] + kEnc) << 16);
    SN_ASSERT(tile >= 0 && tile < p.B * ws.n_tx * ws.n_ty);
    uint4* dst = reinterpret_cast<uint4*>(ws.lbl + tile * kSlots + tid * kWordSlots);
    dst[0] = make_uint4(q[0], q[1], q[2], q[3]);
    dst[1] = make_uint4(q[4], q[5], q[6], q[7]);
  }

  // seam rows / columns: frame index of each border pixel's component, -1 if not passable
  const int64_t seam_row = ((int64_t)blockIdx.z * ws.n_ty + ty) * W;
  const int64_t seam_col = ((int64_t)blockIdx.z * ws.n_tx + tx) * H;
  // the 4 x 128 border positions over the whole block, two per thread: warps
  // 0-3 take 32-position pieces of the first row, then of the first column,
  // warps 4-7 of the last row, then of the last column (line warp-uniform,
  // coalesced stores)
  static_assert(kLTW == 128 && kLTH == 128 && kLThreads == 256, "border split");
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int q = j * kLThreads + tid;
    const int line = q >> 7, t = q & 127;  // 0 top, 1 bottom, 2 left, 3 right
    const bool row = line < 2;
    const int r = row ? (line == 0 ? 0 : kLTH - 1) : t;
    const int c = row ? t : (line == 2 ? 0 : kLTW - 1);
    if (y0 + r < H && (!row || x0 + c < W)) {
      int32_t v = -1;
      if ((bits[r * kLWords + (c >> 5)] >> (c & 31)) & 1u)
        v = frame_index(slot_label(L, pixel_slot(bits, r, c)), x0, y0, W);
      int32_t* dst = row ? (line == 0 ? ws.top : ws.bot) + seam_row + x0 + c
                         : (line == 2 ? ws.left : ws.right) + seam_col + y0 + r;
      *dst = v;
    }
  }
  // global union-find nodes: one per border-touching component, G[label] = label
  {
    int32_t* G = labels + fbase;
    for (int i = tid; i < kTilePx / 32; i += kLThreads) {
      const uint32_t fw = flag[i];
      ws.flags[tile * (kTilePx / 32) + i] = fw;
      for (uint32_t m = fw; m; m &= m - 1u) {
        const int g = frame_index(i * 32 + __ffs(m) - 1, x0, y0, W);
        SN_ASSERT(g >= 0 && (int64_t)g < p.H * p.W);
        G[g] = g;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// 2. seams between tiles (global union-find on G = labels)
//
// Horizontal seams: pixel (x, y) in the last row of tile row ty against
// (x-1 .. x+1, y+1) in the first row of tile row ty+1 -- diagonals across tile
// columns included, so tile corners need no extra case.  Vertical seams:
// (x, y) in the last column of tile column tx against (x+1, y-1 .. y+1).
// A straight neighbour makes the diagonal links redundant (the diagonal
// pixels are 8-adjacent to it along the seam row/column).

// One CTA per (seam line, 128-position chunk) and F frames: the line decode
// is block-uniform 32-bit arithmetic (a 64-bit division per position cost
// more than the unions).  F = 4 frames per thread (their seam loads issued
// together) from 128-frame launches, 1 below: smaller batches need the wider
// grid to hide the unions' latency (measured, DESIGN 4.3)
constexpr int kSeamThreads = 128;

template <int kSeamFrames>
__global__ void __launch_bounds__(kSeamThreads)
    ccl_seam_kernel(const CclParams p, const CclWorkspace ws, int32_t* __restrict__ labels) {
  const int W = (int)p.W, H = (int)p.H;
  const int chW = (W + kSeamThreads - 1) / kSeamThreads;
  const int chH = (H + kSeamThreads - 1) / kSeamThreads;
  const int nh = (ws.n_ty - 1) * chW;  // horizontal (line, chunk) pairs
  const int b = blockIdx.x;
  const bool horiz = b < nh;
  const int bb = horiz ? b : b - nh;
  const int ch = horiz ? chW : chH;
  const int s = bb / ch;
  const int i = (bb - s * ch) * kSeamThreads + threadIdx.x;
  const int n = horiz ? W : H;
  const int lane = threadIdx.x & 31;
  // kSeamFrames frames per thread, their seam loads issued together.  The
  // neighbour positions' values (dedupe and diagonals) come from the
  // neighbour lanes by shuffle -- positions are consecutive across a warp --
  // and lanes 0 / 31 load theirs with the batch (so the warp stays whole for
  // the shuffles: positions past the line's end carry -1)
  for (int64_t f0 = (int64_t)blockIdx.y * kSeamFrames; f0 < p.B;
       f0 += (int64_t)gridDim.y * kSeamFrames) {
    int32_t av[kSeamFrames], cv[kSeamFrames], ae[kSeamFrames], ce[kSeamFrames];
    const int ie = lane == 0 ? i - 1 : i + 1;  // edge lanes' outside neighbour
#pragma unroll
    for (int k = 0; k < kSeamFrames; ++k) {
      const int64_t f = f0 + k;
      const int32_t* a_row = horiz ? ws.bot + (f * ws.n_ty + s) * W : ws.right + (f * ws.n_tx + s) * H;
      const int32_t* b_row =
          horiz ? ws.top + (f * ws.n_ty + s + 1) * W : ws.left + (f * ws.n_tx + s + 1) * H;
      const bool fin = f < p.B;
      av[k] = fin && i < n ? a_row[i] : -1;
      cv[k] = fin && i < n ? b_row[i] : -1;
      const bool edge = fin && (lane == 0 || lane == 31) && ie >= 0 && ie < n;
      ae[k] = edge ? a_row[ie] : -1;
      ce[k] = edge ? b_row[ie] : -1;
    }
#pragma unroll 1
    for (int k = 0; k < kSeamFrames; ++k) {
      const int32_t a = av[k], c = cv[k];
      int32_t al = __shfl_up_sync(0xffffffffu, a, 1), cl = __shfl_up_sync(0xffffffffu, c, 1);
      int32_t ar = __shfl_down_sync(0xffffffffu, a, 1), cr = __shfl_down_sync(0xffffffffu, c, 1);
      if (lane == 0) al = ae[k], cl = ce[k];
      if (lane == 31) ar = ae[k], cr = ce[k];
      if (a < 0) continue;
      int32_t* G = labels + (f0 + k) * p.H * p.W;
      SN_ASSERT((int64_t)a < p.H * p.W && (int64_t)c < p.H * p.W);
      SN_ASSERT((int64_t)cl < p.H * p.W && (int64_t)cr < p.H * p.W);
      if (c >= 0) {
        // a run crossing the seam gives the same (a, c) pair at consecutive
        // positions: only its first position unites (the union is idempotent)
        if (a != c && !(al == a && cl == c)) uf_unite(G, a, c);
      } else {
        // diagonals; skipped where the neighbour position pairs the same a
        // with that pixel straight (it unites them itself)
        if (cl >= 0 && cl != a && al != a) uf_unite(G, a, cl);
        if (cr >= 0 && cr != a && ar != a) uf_unite(G, a, cr);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// 3. resolve: border-touching components through G (one walk each), then per
// pixel: band-run slot (bit ops) -> tile label -> final label, coalesced stores

__device__ __forceinline__ int lp(int slot) { return slot + (slot >> 4); }

__global__ void __launch_bounds__(kLThreads)
    ccl_resolve_kernel(const CclParams p, const CclWorkspace ws, int32_t* __restrict__ labels) {
  // slot label, then slot FINAL label; one pad word per word's 16 slots (lp)
  // so the lanes of a warp looking up runs of equal rank in different words
  // hit different banks
  __shared__ __align__(16) int32_t lab[kSlots + kSlots / 16];
  __shared__ uint32_t bits[kRowWords];
  __shared__ uint32_t flag[kTilePx / 32];
  __shared__ int32_t rank0[kTilePx / 32];  // flagged labels before word i
  __shared__ int32_t fin[512];  // final label per flagged component (<= border pixels)
  __shared__ int32_t warp_sum[kLThreads / 32];
  constexpr int FPT = kTilePx / 32 / kLThreads;  // flag words per thread (2)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int W = (int)p.W, H = (int)p.H;
  const int tx = blockIdx.x, ty = blockIdx.y;
  const int x0 = tx * kLTW, y0 = ty * kLTH;
  const int64_t fbase = (int64_t)blockIdx.z * p.H * p.W;
  const int64_t tile = ((int64_t)blockIdx.z * ws.n_ty + ty) * ws.n_tx + tx;
  {
    const uint4* src = reinterpret_cast<const uint4*>(ws.lbl + tile * kSlots);
#pragma unroll
    for (int i = 0; i < kSlots / 8 / kLThreads; ++i) {
      const int j = i * kLThreads + tid;  // slots 8j .. 8j+7, one 16-slot group
      const uint4 v = src[j];
      int32_t* d = lab + lp(8 * j);
      d[0] = v.x & 0xffff;
      d[1] = v.x >> 16;
      d[2] = v.y & 0xffff;
      d[3] = v.y >> 16;
      d[4] = v.z & 0xffff;
      d[5] = v.z >> 16;
      d[6] = v.w & 0xffff;
      d[7] = v.w >> 16;
    }
    for (int i = tid; i < kRowWords; i += kLThreads) {
      const int r = i >> 2, wc = tx * kLWords + (i & 3);
      bits[i] = (y0 + r < H && wc < ws.WW)
                    ? ws.bits[((int64_t)blockIdx.z * H + y0 + r) * ws.WW + wc]
                    : 0u;
    }
  }
  // flag words tid*FPT .. tid*FPT+FPT-1; exclusive prefix of their popcounts
  uint32_t fw[FPT];
  int c = 0;
#pragma unroll
  for (int j = 0; j < FPT; ++j) {
    fw[j] = ws.flags[tile * (kTilePx / 32) + tid * FPT + j];
    flag[tid * FPT + j] = fw[j];
    c += __popc(fw[j]);
  }
  int inc = c;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += v;
  }
  if (lane == 31) warp_sum[warp] = inc;
  __syncthreads();
  int off = 0;
  for (int i = 0; i < warp; ++i) off += warp_sum[i];
  int k = off + inc - c;
  // walk G once per flagged component.  Nodes are only ever tile-component
  // labels, and a concurrent resolve of another tile overwrites such a node
  // with its final label -- an ancestor -- so the read-only walk is valid.
  // The components' frame indices first (each thread its flag words), then
  // the walks spread over the block, one component per thread: a thread's
  // flag words can hold many components, and every walk is a chain of
  // dependent L2 loads
  int n_flagged = 0;
  for (int i = 0; i < kLThreads / 32; ++i) n_flagged += warp_sum[i];
  n_flagged = min(n_flagged, 512);
#pragma unroll
  for (int j = 0; j < FPT; ++j) {
    rank0[tid * FPT + j] = k;
    for (uint32_t m = fw[j]; m; m &= m - 1u) {
      const int v = (tid * FPT + j) * 32 + __ffs(m) - 1;
      SN_ASSERT(k < 512 && (int64_t)frame_index(v, x0, y0, W) < p.H * p.W);
      if (k < 512) fin[k] = frame_index(v, x0, y0, W);
      ++k;
    }
  }
  __syncthreads();
  {
    const volatile int32_t* G = labels + fbase;
    for (int i = tid; i < n_flagged; i += kLThreads) fin[i] = uf_root(G, fin[i]);
  }
  __syncthreads();
  // final label of every band-run slot, by the slot's owner thread (band, word)
  {
    const int kb = tid >> 2, w = tid & 3;
    const int base = lp(kb * kBandSlots + w * kWordSlots);
    const int nr = __popc(run_starts(band_word(bits, kb, w)));
    for (int i = 0; i < nr; ++i) {
      const int slot = base + i;
      SN_ASSERT(slot >= 0 && slot < kSlots + kSlots / 16);
      const int v = lab[slot];
      SN_ASSERT(v >= 0 && v < kTilePx);
      SN_ASSERT(!((flag[v >> 5] >> (v & 31)) & 1u) ||
                rank0[v >> 5] + __popc(flag[v >> 5] & ((1u << (v & 31)) - 1u)) < 512);
      const uint32_t fwv = flag[v >> 5];
      const uint32_t bit = 1u << (v & 31);
      lab[slot] = (fwv & bit) ? fin[rank0[v >> 5] + __popc(fwv & (bit - 1u))]
                              : frame_index(v, x0, y0, W);
    }
  }
  __syncthreads();
  // per pixel: band-run slot by bit ops -> final label; coalesced stores
  int32_t* out = labels + fbase;
  const bool full = x0 + kLTW <= W && y0 + kLTH <= H;
  if (full && (W & 3) == 0) {
    // a warp writes one 128-pixel tile row per step, 4 pixels (16 B) per lane
    const int w = lane >> 3, sub = (lane & 7) * 4;
    for (int r = warp; r < kLTH; r += kLThreads / 32) {
      const uint32_t A = bits[r * kLWords + w];
      const uint32_t st = run_starts(band_word(bits, r >> 1, w));
      const int base = lp((r >> 1) * kBandSlots + w * kWordSlots);  // a 16-slot group
      // rank of the run holding the lane's first pixel (starts <= sub, minus
      // one), then carried along the 4 pixels: a pixel in the band run starts
      // a new slot only where the band word has a run start
      const uint32_t ab = A >> sub, sb = st >> sub;
      int s = __popc(st & ((2u << sub) - 1u)) - 1;  // sub <= 28
      int v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j > 0 && ((sb >> j) & 1u)) ++s;
        SN_ASSERT(!((ab >> j) & 1u) || (s >= 0 && s < kWordSlots));
        v[j] = ((ab >> j) & 1u) ? lab[base + s] : -1;
      }
      __stcs(reinterpret_cast<int4*>(out + (y0 + r) * W + x0 + w * 32 + sub),
             make_int4(v[0], v[1], v[2], v[3]));
    }
  } else {
    const uint32_t upto = (lane == 31) ? 0xffffffffu : ((2u << lane) - 1u);
    for (int rw = warp; rw < kRowWords; rw += kLThreads / 32) {
      const int r = rw >> 2, w = rw & 3;
      const int gx = x0 + w * 32 + lane, gy = y0 + r;
      if (gx >= W || gy >= H) continue;
      const uint32_t A = bits[rw];
      int32_t v = -1;
      if ((A >> lane) & 1u) {
        const uint32_t st = run_starts(band_word(bits, r >> 1, w));
        v = lab[lp((r >> 1) * kBandSlots + w * kWordSlots) + __popc(st & upto) - 1];
      }
      out[gy * W + gx] = v;  // frame offsets fit int32 (host-checked)
    }
  }
}

__global__ void add_offset_kernel(int32_t* __restrict__ labels, int64_t n, int64_t base) {
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = labels[idx];
    if (v >= 0) labels[idx] = (int32_t)(v + base);
  }
}

// relabel: scatter the (key -> root) map into a dense scratch indexed by
// key - base, then gather per pixel
__global__ void relabel_scatter_kernel(int32_t* __restrict__ scratch, int64_t n, int64_t base,
                                       const int32_t* __restrict__ keys,
                                       const int32_t* __restrict__ vals,
                                       const int32_t* __restrict__ n_map) {
  const int m = *n_map;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int64_t k = (int64_t)keys[i] - base;
    if (k >= 0 && k < n) scratch[k] = vals[i];
  }
}

__global__ void relabel_gather_kernel(int32_t* __restrict__ labels, int64_t n, int64_t base,
                                      const int32_t* __restrict__ scratch) {
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = labels[idx];
    if (v >= 0) {
      const int64_t k = (int64_t)v - base;
      if (k >= 0 && k < n) {
        const int32_t r = scratch[k];
        if (r >= 0) labels[idx] = r;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// launchers

static unsigned grid_for(const LaunchCtx& ctx, int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  const int64_t cap = (int64_t)ctx.num_sms * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (unsigned)g;
}

CclParams make_ccl_params(int64_t B, int64_t H, int64_t W, double fxb, double t) {
  CclParams p{};
  p.B = B;
  p.H = H;
  p.W = W;
  p.fxb = fxb;
  p.t = t;
  p.fxb_f = (float)fxb;
  p.t_f = (float)t;
  // the filter's error bound assumes normal fp32 operands (fxb_f, t_f, zf)
  p.exact_only = !(fxb >= 1e-20 && fxb <= 1e20 && t >= 1e-30 && t <= 1e30);
  return p;
}

static size_t align256(size_t v) { return (v + 255) / 256 * 256; }

size_t ccl_workspace_bytes(int64_t B, int64_t H, int64_t W) {
  const size_t one = ccl_workspace_bytes_one(B, H, W);
  if (B < kCclSplitFrames) return one;
  const size_t halves = ccl_workspace_bytes_one(B / 2, H, W) + ccl_workspace_bytes_one(B - B / 2, H, W);
  return one > halves ? one : halves;
}

size_t ccl_workspace_bytes_one(int64_t B, int64_t H, int64_t W) {
  const int64_t WW = (W + 31) / 32;
  const int64_t n_tx = (W + kLTW - 1) / kLTW, n_ty = (H + kLTH - 1) / kLTH;
  const int64_t tiles = B * n_tx * n_ty;
  return align256((size_t)(B * H * WW) * 4) + 2 * align256((size_t)(B * n_ty * W) * 4) +
         2 * align256((size_t)(B * n_tx * H) * 4) + align256((size_t)(tiles * kSlots) * 2) +
         align256((size_t)(tiles * kTilePx / 32) * 4);
}

template <typename T>
int run_passable(const LaunchCtx& ctx, const T* disp, const CclParams& p, uint8_t* pas,
                 double* edges) {
  const int64_t n = p.B * p.H * p.W;
  if (n == 0) return SN_OK;
  passable_kernel<T><<<grid_for(ctx, n, 256), 256, 0, ctx.stream>>>(disp, p, pas, edges);
  return check_launch("passable_kernel");
}
template int run_passable<float>(const LaunchCtx&, const float*, const CclParams&, uint8_t*,
                                 double*);
template int run_passable<double>(const LaunchCtx&, const double*, const CclParams&, uint8_t*,
                                  double*);

// ST-passable bit mask (adaptive.py:80-97,130-132) as a streaming kernel.
//
// A warp owns 128 aligned columns x kPbRows rows of a frame; lane L owns the
// 4 consecutive columns 4L .. 4L+3 (one 16-byte load per row for fp32).  The
// rows stream through a 3-row register window of depths zf = fxb * rcp(d);
// the left / right neighbours of a lane's first / last column come from the
// neighbour lanes by shuffle (lanes 0 and 31 load the warp's outer columns),
// and the arithmetic runs on pixel pairs with packed f32x2 ops.  Per pixel the
// fp32 filter of sn_common.cuh decides passable (|e| < t - margin), not
// passable (|e| > t + margin) or undecided, where margin = 2^-20 S + 2^-21 t.
// Decisions need every depth of the 5-point stencil > 0: a row-lane whose
// window holds a non-positive depth (negative, zero or +inf disparities) is
// undecided as a whole; NaN samples propagate into e and leave the pixel
// undecided; infinite depths make the margin infinite (undecided as well).
// Undecided pixels -- ties, invalid or out-of-range samples -- take the exact
// fp64 path with the reference's op order (pred_exact_d), so every decision
// is the fp64 reference's.  The per-lane result is a nibble per row; an 8x8
// nibble transpose across each 8-lane group (3 xor-shuffle stages) turns
// them into the bit-mask words, one word per lane per 8 rows.  Reads 4 B/px
// (+ halo rows through L2), writes 1/8 B/px.
constexpr int kPbRows = 16;  // 32: spills at the 64-register cap (2.71 vs 2.44 us/frame)
constexpr int kPbCols = 128;

__device__ __forceinline__ float4 pb_depth4(float4 d, float fxb) {
  return make_float4(__fmul_rn(fxb, rcp_ftz(d.x)), __fmul_rn(fxb, rcp_ftz(d.y)),
                     __fmul_rn(fxb, rcp_ftz(d.z)), __fmul_rn(fxb, rcp_ftz(d.w)));
}

__device__ __forceinline__ float pb_min4(float4 z) {
  return fminf(fminf(z.x, z.y), fminf(z.z, z.w));
}
__device__ __forceinline__ float pb_max4(float4 z) {
  return fmaxf(fmaxf(z.x, z.y), fmaxf(z.z, z.w));
}

// One row of a lane's 4 pixels: sets bit b + j of `yes` (passable) or `no`
// (not passable) for every decided pixel j; `clean` = every non-NaN depth of
// the stencils in (0, 2^100).  e = 4c - ((u + d) + (l + r)) has the four
// roundings of the filter bound; lo / hi = t -/+ (2^-21 t + 2^-20 S).  In a
// clean window a NaN e can only come from a NaN (invalid) sample, so the
// unordered compare decides such pixels "not passable" at once.
__device__ __forceinline__ void pb_row(float4 zu, float4 zc, float4 zd, float lft, float rgt,
                                       bool clean, float2 qlo, float2 qhi, int b, uint32_t& yes,
                                       uint32_t& no) {
  // horizontal neighbour sums (scalar: the pairs would straddle registers)
  const float2 hs01 = make_float2(__fadd_rn(lft, zc.y), __fadd_rn(zc.x, zc.z));
  const float2 hs23 = make_float2(__fadd_rn(zc.y, zc.w), __fadd_rn(zc.z, rgt));
  const float2 P01 = __fadd2_rn(__fadd2_rn(make_float2(zu.x, zu.y), make_float2(zd.x, zd.y)), hs01);
  const float2 P23 = __fadd2_rn(__fadd2_rn(make_float2(zu.z, zu.w), make_float2(zd.z, zd.w)), hs23);
  const float2 four = make_float2(4.0f, 4.0f);
  const float2 e01 = __ffma2_rn(four, make_float2(zc.x, zc.y), make_float2(-P01.x, -P01.y));
  const float2 e23 = __ffma2_rn(four, make_float2(zc.z, zc.w), make_float2(-P23.x, -P23.y));
  const float2 S01 = __ffma2_rn(four, make_float2(zc.x, zc.y), P01);
  const float2 S23 = __ffma2_rn(four, make_float2(zc.z, zc.w), P23);
  const float2 km = make_float2(-9.5367431640625e-07f, -9.5367431640625e-07f);  // -2^-20
  const float2 kp = make_float2(9.5367431640625e-07f, 9.5367431640625e-07f);
  const float2 lo01 = __ffma2_rn(S01, km, qlo), lo23 = __ffma2_rn(S23, km, qlo);
  const float2 hi01 = __ffma2_rn(S01, kp, qhi), hi23 = __ffma2_rn(S23, kp, qhi);
  if (clean && fabsf(e01.x) < lo01.x) yes |= 1u << b;
  if (clean && fabsf(e01.y) < lo01.y) yes |= 2u << b;
  if (clean && fabsf(e23.x) < lo23.x) yes |= 4u << b;
  if (clean && fabsf(e23.y) < lo23.y) yes |= 8u << b;
  if (clean && !(fabsf(e01.x) <= hi01.x)) no |= 1u << b;
  if (clean && !(fabsf(e01.y) <= hi01.y)) no |= 2u << b;
  if (clean && !(fabsf(e23.x) <= hi23.x)) no |= 4u << b;
  if (clean && !(fabsf(e23.y) <= hi23.y)) no |= 8u << b;
}

// A row's 4 raw samples as loaded (converted to fp32 only when used, so a
// prefetched row does not wait for its load).  The caller clamps rows and
// columns into the frame: samples of clamped (outside) rows and columns only
// ever feed pixels that are not interior, whose bits are masked.
template <typename T, bool VEC>
struct PbRaw {
  T v[4];
  __device__ __forceinline__ void load(const T* row, int W) {
    if constexpr (VEC && sizeof(T) == 4) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(row));
      v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w;
    } else if constexpr (VEC) {
      const double2 a = __ldg(reinterpret_cast<const double2*>(row));
      const double2 b = __ldg(reinterpret_cast<const double2*>(row + 2));
      v[0] = a.x, v[1] = a.y, v[2] = b.x, v[3] = b.y;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) v[j] = __ldg(row + min(j, W - 1));
    }
  }
  __device__ __forceinline__ float4 depth(float fxb) const {
    return pb_depth4(make_float4(disp_f32(v[0]), disp_f32(v[1]), disp_f32(v[2]), disp_f32(v[3])),
                     fxb);
  }
};

// The rows of one warp task; rows outside the frame are clamped into it.
// Row r + 1 + PD is loaded while row r is evaluated (PD rows in flight).
template <typename T, bool VEC>
__device__ __forceinline__ void pb_task(const T* colp, const T* edgep, int y0, int H, int W, int xw,
                                        int lane, float fxb, bool pe, float2 qlo, float2 qhi,
                                        uint32_t* yes, uint32_t* no) {
  constexpr int PD = 2;  // measured flat for 1..3 (ptxas schedules the loads itself)
  auto rowoff = [&](int y) -> int {  // frame offsets fit int32 (host-checked)
    return min(max(y, 0), H - 1) * W;
  };
  PbRaw<T, VEC> raw[PD];
  T eraw[PD];
#pragma unroll
  for (int i = 0; i < PD; ++i) {
    raw[i].load(colp + rowoff(y0 + 1 + i), xw);
    eraw[i] = __ldg(edgep + rowoff(y0 + 1 + i));
  }
  PbRaw<T, VEC> r0;
  r0.load(colp + rowoff(y0 - 1), xw);
  float4 zu = r0.depth(fxb);
  r0.load(colp + rowoff(y0), xw);
  float4 zc = r0.depth(fxb);
  float ec = __fmul_rn(fxb, rcp_ftz(disp_f32(__ldg(edgep + rowoff(y0)))));
  float mu = pb_min4(zu), mc = pb_min4(zc), xu = pb_max4(zu), xcm = pb_max4(zc);
#pragma unroll
  for (int r = 0; r < kPbRows; ++r) {
    const float4 zd = raw[r % PD].depth(fxb);
    const float ed = __fmul_rn(fxb, rcp_ftz(disp_f32(eraw[r % PD])));
    if (r + PD < kPbRows) {
      const int off = rowoff(y0 + r + 1 + PD);
      raw[r % PD].load(colp + off, xw);
      eraw[r % PD] = __ldg(edgep + off);
    }
    const float md = pb_min4(zd), xd = pb_max4(zd);
    float lft = __shfl_up_sync(0xffffffffu, zc.w, 1);
    float rgt = __shfl_down_sync(0xffffffffu, zc.x, 1);
    if (lane == 0) lft = ec;
    if (lane == 31) rgt = ec;
    // every non-NaN depth of the lane's stencils in (0, 2^100): NaN samples
    // are skipped by min/max (a window of NaNs only is clean) and poison e
    const float lo = fminf(fminf(fminf(mu, mc), fminf(md, lft)), rgt);
    const float hi = fmaxf(fmaxf(fmaxf(xu, xcm), fmaxf(xd, lft)), rgt);
    const bool clean = !pe && !(lo <= 0.0f) && !(hi >= 1.2676506002282294e30f);
    pb_row(zu, zc, zd, lft, rgt, clean, qlo, qhi, 4 * (r & 7), yes[r >> 3], no[r >> 3]);
    zu = zc;
    zc = zd;
    mu = mc;
    mc = md;
    xu = xcm;
    xcm = xd;
    ec = ed;
  }
}

// One warp per block: the task loop and every shuffle are then in uniform
// control flow (no divergence-safe shuffle sequences in the hot loop); 32
// single-warp blocks per SM give the full 32 warps at 64 registers.
template <typename T, bool VEC>
__global__ void __launch_bounds__(32, 32)
    passable_bits_kernel(const T* __restrict__ disp, const FixedParams p,
                         uint32_t* __restrict__ bits, unsigned* __restrict__ next_task) {
  const int W = (int)p.W, H = (int)p.H, WW = p.bits_ww;
  const int lane = threadIdx.x;
  const unsigned tasks_x = (unsigned)((W + kPbCols - 1) / kPbCols);
  const unsigned strips_y = (unsigned)((H + kPbRows - 1) / kPbRows);
  const unsigned n_tasks = (unsigned)p.B * strips_y * tasks_x;  // < 2^31 (host-checked)
  const float tm = __fmul_rn(p.t_f, 4.76837158203125e-07f /* 2^-21 */);
  const float2 qlo = make_float2(__fsub_rn(p.t_f, tm), __fsub_rn(p.t_f, tm));
  const float2 qhi = make_float2(__fadd_rn(p.t_f, tm), __fadd_rn(p.t_f, tm));
  const bool pe = p.pred_exact != 0;
  const int g8 = lane & 7;
  // tasks handed out dynamically (their cost varies: exact-path pixels): the
  // first by block index, then from a counter whose next value is fetched
  // while the current task runs
  unsigned nraw = lane == 0 ? atomicAdd(next_task, 1u) : 0u;
  for (unsigned task = blockIdx.x; task < n_tasks;) {
    const unsigned rest = task / tasks_x;
    const int tx = (int)(task - rest * tasks_x);
    const unsigned f = rest / strips_y;
    const int y0 = (int)(rest - f * strips_y) * kPbRows;
    const int x0 = tx * kPbCols, xl = x0 + 4 * lane;
    const T* fr = disp + (int64_t)f * p.H * p.W;
    // clamped load columns (see PbRaw): a lane past the right edge
    // re-reads the last vector; the warp's outer columns (lane 0: left, lane
    // 31: right; the other lanes' copy is unused) stay in the frame
    const int xc = VEC ? min(xl, W - 4) : xl;
    const int xe = min(max(lane == 0 ? x0 - 1 : x0 + kPbCols, 0), W - 1);
    uint32_t yes[kPbRows / 8] = {}, no[kPbRows / 8] = {};
    pb_task<T, VEC>(fr + xc, fr + xe, y0, H, W, VEC ? 4 : W - xc, lane, p.fxb_f, pe, qlo, qhi, yes,
                    no);
    // interior pixels only (the reference has no padding): columns 1 .. W-2
    // (per lane, replicated over the rows' nibbles), rows 1 .. H-2
    uint32_t cm = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) cm |= (xl + j >= 1 && xl + j + 1 < W) ? (0x11111111u << j) : 0u;
    uint32_t und[kPbRows / 8], anyu = 0;
#pragma unroll
    for (int k = 0; k < kPbRows / 8; ++k) {
      const int ya = y0 + 8 * k;  // rows ya .. ya+7 -> nibbles 0 .. 7
      uint32_t rows = 0xffffffffu;
      if (ya < 1) rows &= 0xfffffff0u;
      if (ya + 8 > H - 1) rows &= (H - 1 - ya) <= 0 ? 0u : (0xffffffffu >> (4 * (8 - (H - 1 - ya))));
      const uint32_t m = cm & rows;
      yes[k] &= m;
      und[k] = m & ~(yes[k] | no[k]);
      anyu |= und[k];
    }
    // rare exact decisions (fp64, reference op order)
    if (__any_sync(0xffffffffu, anyu != 0u)) {
#pragma unroll
      for (int k = 0; k < kPbRows / 8; ++k) {
        for (uint32_t m = und[k]; m; m &= m - 1u) {
          const int b = __ffs(m) - 1;
          const int y = y0 + 8 * k + (b >> 2), x = xl + (b & 3);
          const T* c = fr + (int64_t)y * W + x;
          if (pred_exact_d(c[0], c[-1], c[1], c[-W], c[W], p.fxb, p.t)) yes[k] |= 1u << b;
        }
      }
    }
    // 8x8 nibble transpose inside each 8-lane group: lane 8g+i ends with the
    // word of row 8k+i, columns x0 + 32g .. +31.  Stage s: the partner is
    // lane ^ s; a lane keeps the nibbles whose row bit s equals its own lane
    // bit s and takes the others from the partner, rotated into place (the
    // rotation's wrapped-around bits land in the kept half and are masked).
    const int gw = tx * (kPbCols / 32) + (lane >> 3);
#pragma unroll
    for (int k = 0; k < kPbRows / 8; ++k) {
      uint32_t v = yes[k];
#pragma unroll
      for (int s = 4; s >= 1; s >>= 1) {
        const uint32_t mc_ = s == 1 ? 0x0F0F0F0Fu : (s == 2 ? 0x00FF00FFu : 0x0000FFFFu);
        const bool hi = (g8 & s) != 0;
        const uint32_t keep = hi ? ~mc_ : mc_;
        const uint32_t t = __shfl_xor_sync(0xffffffffu, v, s);
        const uint32_t rot = __funnelshift_r(t, t, hi ? 4 * s : 32 - 4 * s);
        v = (v & keep) | (rot & ~keep);
      }
      const int y = y0 + 8 * k + g8;
      SN_ASSERT(f < p.B);
    if (y < H && gw < WW) bits[((int64_t)f * p.H + y) * WW + gw] = v;
    }
    task = gridDim.x + __shfl_sync(0xffffffffu, nraw, 0);
    if (task < n_tasks && lane == 0) nraw = atomicAdd(next_task, 1u);
  }
}

template <typename T>
int run_passable_bits(const LaunchCtx& ctx, const T* disp, const FixedParams& p,
                      uint32_t* bits) {
  const int64_t tasks = p.B * ((p.H + kPbRows - 1) / kPbRows) * ((p.W + kPbCols - 1) / kPbCols);
  if (tasks == 0) return SN_OK;
  if (p.H * p.W > 0x7fffffffLL || tasks > 0x7fffffffLL)
    return set_error(SN_EINVAL, "frame or batch too large for the passable-bit kernel");
  const bool vec = p.W % 4 == 0 && reinterpret_cast<uintptr_t>(disp) % 16 == 0 && p.W >= 4;
  int64_t g = tasks;
  if (g > (int64_t)ctx.num_sms * 32) g = (int64_t)ctx.num_sms * 32;
  // the task counter: stream-ordered scratch (concurrent calls on other
  // streams get their own)
  unsigned* next_task = nullptr;
  int rc = scratch_alloc(ctx, sizeof(unsigned), reinterpret_cast<void**>(&next_task));
  if (rc) return rc;
  if (cudaMemsetAsync(next_task, 0, sizeof(unsigned), ctx.stream) != cudaSuccess) {
    scratch_free(ctx, next_task);
    return set_cuda_error("cudaMemsetAsync(task counter)");
  }
  if (vec)
    passable_bits_kernel<T, true><<<(unsigned)g, 32, 0, ctx.stream>>>(disp, p, bits, next_task);
  else
    passable_bits_kernel<T, false><<<(unsigned)g, 32, 0, ctx.stream>>>(disp, p, bits, next_task);
  rc = check_launch("passable_bits_kernel");
  scratch_free(ctx, next_task);
  return rc;
}
template int run_passable_bits<float>(const LaunchCtx&, const float*, const FixedParams&,
                                      uint32_t*);
template int run_passable_bits<double>(const LaunchCtx&, const double*, const FixedParams&,
                                       uint32_t*);

template <typename T>
int run_ccl(const LaunchCtx& ctx, const T* disp, const uint8_t* pas, const CclParams& p,
            int64_t index_base, int32_t* labels, void* workspace, size_t ws_bytes,
            const uint32_t* bits_in) {
  const int64_t n = p.B * p.H * p.W;
  if (n == 0) return SN_OK;
  if (p.H * p.W > 0x7fffffffLL) return set_error(SN_EINVAL, "frame too large for int32 labels");
  if (!workspace || ws_bytes < ccl_workspace_bytes_one(p.B, p.H, p.W))
    return set_error(SN_EINVAL, "labeller workspace too small (%zu < %zu bytes)", ws_bytes,
                     ccl_workspace_bytes_one(p.B, p.H, p.W));
  constexpr int64_t kMaxFrames = 65535;  // grid.z
  if (p.B > kMaxFrames) {
    // frames are independent: consecutive launches of <= 65535 frames, each
    // reusing the front of the workspace (stream order serialises them)
    const int64_t HW = p.H * p.W, WW = (p.W + 31) / 32;
    for (int64_t f0 = 0; f0 < p.B; f0 += kMaxFrames) {
      CclParams q = p;
      q.B = std::min<int64_t>(kMaxFrames, p.B - f0);
      const int rc = run_ccl(ctx, disp ? disp + f0 * HW : nullptr, pas ? pas + f0 * HW : nullptr, q,
                             index_base, labels + f0 * HW, workspace, ws_bytes,
                             bits_in ? bits_in + f0 * p.H * WW : nullptr);
      if (rc) return rc;
    }
    return SN_OK;
  }
  CclWorkspace ws;
  ws.WW = (int)((p.W + 31) / 32);
  ws.n_tx = (int)((p.W + kLTW - 1) / kLTW);
  ws.n_ty = (int)((p.H + kLTH - 1) / kLTH);
  uint8_t* q = static_cast<uint8_t*>(workspace);
  ws.bits = reinterpret_cast<uint32_t*>(q);
  q += align256((size_t)(p.B * p.H * ws.WW) * 4);
  ws.top = reinterpret_cast<int32_t*>(q);
  q += align256((size_t)(p.B * ws.n_ty * p.W) * 4);
  ws.bot = reinterpret_cast<int32_t*>(q);
  q += align256((size_t)(p.B * ws.n_ty * p.W) * 4);
  ws.left = reinterpret_cast<int32_t*>(q);
  q += align256((size_t)(p.B * ws.n_tx * p.H) * 4);
  ws.right = reinterpret_cast<int32_t*>(q);
  q += align256((size_t)(p.B * ws.n_tx * p.H) * 4);
  const int64_t tiles = p.B * ws.n_tx * ws.n_ty;
  ws.lbl = reinterpret_cast<uint16_t*>(q);
  q += align256((size_t)(tiles * kSlots) * 2);
  ws.flags = reinterpret_cast<uint32_t*>(q);

  int rc = ensure_dyn_smem(reinterpret_cast<const void*>(ccl_tile_kernel<1>), (int)kTileSmem,
                           ctx.device, "ccl_tile_kernel<1>");
  if (!rc)
    rc = ensure_dyn_smem(reinterpret_cast<const void*>(ccl_tile_kernel<2>), (int)kTileSmem,
                         ctx.device, "ccl_tile_kernel<2>");
  if (rc) return rc;
  if (disp) {
    // predicate from fp32 disparity: the streaming bit-mask kernel first
    FixedParams fp{};
    fp.B = p.B;
    fp.H = p.H;
    fp.W = p.W;
    fp.fxb = p.fxb;
    fp.fxb_f = (float)p.fxb;
    fill_predicate(fp, p.fxb, p.t, ws.bits);
    const int rc0 = run_passable_bits<T>(ctx, disp, fp, ws.bits);
    if (rc0) return rc0;
    bits_in = ws.bits;
  }
  if (bits_in) ws.bits = const_cast<uint32_t*>(bits_in);  // read-only in MODE 2
  dim3 grid((unsigned)ws.n_tx, (unsigned)ws.n_ty, (unsigned)p.B);
  if (bits_in)
    ccl_tile_kernel<2><<<grid, kLThreads, kTileSmem, ctx.stream>>>(nullptr, p, ws, labels);
  else
    ccl_tile_kernel<1><<<grid, kLThreads, kTileSmem, ctx.stream>>>(pas, p, ws, labels);
  rc = check_launch("ccl_tile_kernel");
  if (rc) return rc;
  const int64_t seam_blocks =
      (int64_t)(ws.n_ty - 1) * ((p.W + kSeamThreads - 1) / kSeamThreads) +
      (int64_t)(ws.n_tx - 1) * ((p.H + kSeamThreads - 1) / kSeamThreads);
  if (seam_blocks > 0) {
    const int F = p.B >= 128 ? 4 : 1;
    const int64_t gy = (p.B + F - 1) / F;
    dim3 sg((unsigned)seam_blocks, (unsigned)(gy < 65535 ? gy : 65535));
    if (F == 4)
      ccl_seam_kernel<4><<<sg, kSeamThreads, 0, ctx.stream>>>(p, ws, labels);
    else
      ccl_seam_kernel<1><<<sg, kSeamThreads, 0, ctx.stream>>>(p, ws, labels);
    if ((rc = check_launch("ccl_seam_kernel"))) return rc;
  }
  ccl_resolve_kernel<<<grid, kLThreads, 0, ctx.stream>>>(p, ws, labels);
  if ((rc = check_launch("ccl_resolve_kernel"))) return rc;
  if (index_base != 0) {
    add_offset_kernel<<<grid_for(ctx, n, 256), 256, 0, ctx.stream>>>(labels, n, index_base);
    rc = check_launch("add_offset_kernel");
  }
  return rc;
}
template int run_ccl<float>(const LaunchCtx&, const float*, const uint8_t*, const CclParams&,
                            int64_t, int32_t*, void*, size_t, const uint32_t*);
template int run_ccl<double>(const LaunchCtx&, const double*, const uint8_t*, const CclParams&,
                             int64_t, int32_t*, void*, size_t, const uint32_t*);

// ---------------------------------------------------------------------------
// strip seams on the device: the gathered first / last owned
// label rows of every strip ([n_strips][2][W], global raster indices) are
// merged with the labeller's own min-root union-find, on a table indexed by
// label value (entries of labels that are not on a seam stay -1), then every
// strip relabels its pixels through the table.  Deterministic: the roots are
// the minimum labels, whatever the order of the unions -- every rank builds
// the same table from the same gathered rows, with no host round trip.

__global__ void seam_init_kernel(const int32_t* __restrict__ seams, int64_t n, int32_t* table) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = seams[i];
    if (v >= 0) table[v] = v;
  }
}

// position u of seam s: strip s+1's first-row pixel u against strip s's
// last-row pixels u-1, u, u+1 (8-connected; all three, as the host merge, so
// the result does not rely on row neighbours sharing a label)
__global__ void seam_unite_kernel(const int32_t* __restrict__ seams, int n_strips, int W,
                                  int32_t* table) {
  const int64_t total = (int64_t)(n_strips - 1) * W;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int s = (int)(i / W), u = (int)(i - (int64_t)s * W);
    const int32_t* a = seams + ((int64_t)s * 2 + 1) * W;   // last owned row of strip s
    const int32_t* b = seams + ((int64_t)s + 1) * 2 * W;   // first owned row of strip s+1
    const int32_t x = b[u];
    if (x < 0) continue;
    for (int du = -1; du <= 1; ++du) {
      const int uu = u + du;
      if (uu < 0 || uu >= W) continue;
      const int32_t y = a[uu];
      if (y >= 0 && y != x) uf_unite(table, x, y);
    }
  }
}

__global__ void seam_compress_kernel(const int32_t* __restrict__ seams, int64_t n, int32_t* table) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = seams[i];
    if (v >= 0) table[v] = uf_root(table, v);
  }
}

__global__ void relabel_table_kernel(int32_t* __restrict__ labels, int64_t n,
                                     const int32_t* __restrict__ table, int64_t table_n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = labels[i];
    if (v >= 0 && v < table_n) {
      const int32_t r = __ldg(table + v);
      if (r >= 0) labels[i] = r;
    }
  }
}

int run_seam_merge(const LaunchCtx& ctx, const int32_t* seams, int n_strips, int64_t W,
                   int32_t* table, int64_t table_n) {
  if (table_n > 0 && cudaMemsetAsync(table, 0xff, (size_t)table_n * 4, ctx.stream) != cudaSuccess)
    return set_cuda_error("cudaMemsetAsync(seam table)");
  const int64_t n = (int64_t)n_strips * 2 * W;
  if (n == 0) return SN_OK;
  seam_init_kernel<<<grid_for(ctx, n, 256), 256, 0, ctx.stream>>>(seams, n, table);
  int rc = check_launch("seam_init_kernel");
  if (rc) return rc;
  if (n_strips > 1) {
    seam_unite_kernel<<<grid_for(ctx, (int64_t)(n_strips - 1) * W, 256), 256, 0, ctx.stream>>>(
        seams, n_strips, (int)W, table);
    if ((rc = check_launch("seam_unite_kernel"))) return rc;
  }
  seam_compress_kernel<<<grid_for(ctx, n, 256), 256, 0, ctx.stream>>>(seams, n, table);
  return check_launch("seam_compress_kernel");
}

int run_relabel_table(const LaunchCtx& ctx, int32_t* labels, int64_t n, const int32_t* table,
                      int64_t table_n) {
  if (n == 0) return SN_OK;
  relabel_table_kernel<<<grid_for(ctx, n, 256), 256, 0, ctx.stream>>>(labels, n, table, table_n);
  return check_launch("relabel_table_kernel");
}

int run_relabel(const LaunchCtx& ctx, int32_t* labels, int64_t n, int64_t base,
                const int32_t* keys, const int32_t* vals, const int32_t* n_map, int32_t cap,
                int32_t* scratch) {
  if (n == 0) return SN_OK;
  if (cudaMemsetAsync(scratch, 0xff, (size_t)n * sizeof(int32_t), ctx.stream) != cudaSuccess)
    return set_cuda_error("cudaMemsetAsync(relabel scratch)");
  relabel_scatter_kernel<<<grid_for(ctx, cap, 256), 256, 0, ctx.stream>>>(scratch, n, base, keys,
                                                                          vals, n_map);
  int rc = check_launch("relabel_scatter_kernel");
  if (rc) return rc;
  relabel_gather_kernel<<<grid_for(ctx, n, 256), 256, 0, ctx.stream>>>(labels, n, base, scratch);
  return check_launch("relabel_gather_kernel");
}

}  // namespace sn
