// gs_common.cuh — device-side arithmetic shared by every GridShift kernel.
//
// Every floating-point expression here is pinned to the CPU oracle (oracle/gs_oracle.cpp,
// pins P1-P6) with explicit _rn intrinsics so nvcc can never contract them into DFMA.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#define GS_APRON 2       // empty cells around the data key box on each side, every dim
#define GS_DMAX 12

// error bits (errflag[0]): 1 non-finite input, 2 point outside the key box (invariant), 4
// centroid left the box, 8 watchdog, 16 frame beyond K8's capacity, 32 key box larger than the
// grid, 64 keys beyond the int64 range, 128 point outside the PREDICTED box (rerun with bounds)
constexpr int GS_ERR_SKIP = 1 | 32 | 64 | 128;  // binning did not complete: later kernels skip

// The IEEE division as an out-of-line call for the rare-operand fallbacks of the reciprocal
// divisions: inlined, the compiler if-converts it and runs its whole ~12-op FP64 sequence
// speculatively on the common path (measured ~150 cycles per sweep level on a lone warp).
__device__ __noinline__ double gs_ddiv_slow(double a, double b) { return __ddiv_rn(a, b); }

// Geometry of the dense cell grid: frame-major, then lexicographic row-major over the d dims
// (dim 0 slowest), so the linear cell index order IS the SPEC's lexicographic key order
// within a frame, and frames never neighbour each other.
struct GsBox {
  int32_t d;
  int32_t F;            // fixed-point exponent of the binning sums
  double h;
  double inv_h;         // RN(1/h): only a fast-path hint, see gs_grid_coord
  double scale;         // 2^F
  double inv_scale;     // 2^-F
  int64_t n;            // points per frame
  int64_t nframes;
  int64_t vol_frame;    // cells per frame
  int64_t vol_total;    // cells in all frames
  int64_t kmin[GS_DMAX];    // key of the box origin per dim (data min key - apron)
  int64_t ext[GS_DMAX];     // box extent per dim (apron included)
  int64_t stride[GS_DMAX];  // linear stride per dim (stride[d-1] = 1)
};

// grid_index component (pin P1): floor(RN(x/h)), floor toward -inf, integral
// quotients go to the upper cell.  Fast path: q = RN(x*RN(1/h)) is within 4u|x/h| of the IEEE
// quotient, so when q's fractional part is farther than 2^-50*max(|q|,1) from an integer,
// floor(q) == floor(RN(x/h)); otherwise take the exact IEEE division.  Bit-identical to
// std::floor(x / h) for every finite x.
__device__ __forceinline__ int64_t gs_grid_coord(double x, double h, double inv_h) {
  double q = __dmul_rn(x, inv_h);
  double fl = floor(q);
  double fr = __dsub_rn(q, fl);
  double tol = 0x1p-50 * fmax(fabs(q), 1.0);
  if (!(fr >= tol && fr <= 1.0 - tol)) fl = floor(gs_ddiv_slow(x, h));
  return (int64_t)fl;
}

// ---- segmentation front end fused into the point readers: 8-bit RGB
// pixels are read as 3 bytes and turned into features on the fly -- rgb: channel / 255;
// rgbxy: + x = col / (W-1), y = row / (H-1) -- instead of a 12-24 B/pixel fp32 feature array.
// Every quotient is RN(a / b) for a small non-negative integer a: Markstein's form from
// y = RN(1/b) is the correctly rounded quotient there (see rs_div), so the features equal the
// oracle's `img / 255.0` bit for bit.
struct GsImg {
  int W = 0, H = 0;       // rgbxy image width / height (0: rgb only)
  double wm1 = 0, hm1 = 0, rw = 0, rh = 0;
};

__device__ __forceinline__ double gs_div_small(double a, double b, double y) {
  const double q0 = __dmul_rn(a, y);
  return __fma_rn(__fma_rn(-q0, b, a), y, q0);
}

template <typename T, int D>
__host__ __device__ constexpr int gs_raw_cols() {
  return sizeof(T) == 1 ? 3 : D;  // uint8_t: r, g, b bytes per pixel
}

// feature c of a point from its raw row; pl = the point's index within its frame
template <typename T, int D>
__device__ __forceinline__ double gs_feature(const T* raw, int c, int64_t pl, const GsImg& im) {
  if constexpr (sizeof(T) == 1) {
    if (c < 3) return gs_div_small((double)raw[c], 255.0, 1.0 / 255.0);
    const uint32_t ul = (uint32_t)pl, col = ul % (uint32_t)im.W, row = ul / (uint32_t)im.W;
    return c == 3 ? gs_div_small((double)col, im.wm1, im.rw)
                  : gs_div_small((double)row, im.hm1, im.rh);
  } else {
    return (double)raw[c];
  }
}

__device__ __forceinline__ GsImg gs_img(int W, int64_t n) {
  GsImg im;
  if (W > 1) {
    im.W = W;
    im.H = (int)(n / W);
    im.wm1 = (double)(W - 1);
    im.hm1 = (double)(im.H - 1);
    im.rw = __drcp_rn(im.wm1);
    im.rh = __drcp_rn(im.hm1);
  }
  return im;
}

// Fixed-point offset of coordinate x inside its cell k (oracle build mode 1):
// nearbyint((x - k*h) * 2^F) as int64.
__device__ __forceinline__ long long gs_fixq(double x, int64_t k, double h, double scale) {
  double base = __dmul_rn((double)k, h);
  double off = __dsub_rn(x, base);
  return __double2ll_rn(__dmul_rn(off, scale));
}

// Centroid coordinate from a fixed-point cell sum: k*h + ((double)sum / (double)count) * 2^-F.
__device__ __forceinline__ double gs_fix_centroid(int64_t k, long long qsum, uint32_t count,
                                                  double h, double inv_scale) {
  double base = __dmul_rn((double)k, h);
  double mq = __ddiv_rn(__ll2double_rn(qsum), (double)count);
  return __dadd_rn(base, __dmul_rn(mq, inv_scale));
}

// slot[] readers: a point's dense grid cell.  slot holds u16 frame-local cells when the frame
// volume fits 16 bits (image frames: half the bytes), else u32 global cells.
__device__ __forceinline__ uint32_t gs_slot_cell(const void* slot, bool s16, int64_t p,
                                                 uint32_t fbase) {
  return s16 ? fbase + ((const uint16_t*)slot)[p] : ((const uint32_t*)slot)[p];
}

// Key of dim c of a linear cell index (within its frame).
__device__ __forceinline__ int64_t gs_key_of(const GsBox& b, int64_t L, int c) {
  int64_t local = L % b.vol_frame;
  return (local / b.stride[c]) % b.ext[c] + b.kmin[c];
}

// Linear offset of the lexicographic neighbour offset #t (v in {-1,0,1}^d, dim 0 most
// significant digit; SPEC.md:49-57 / pin P2) — odometer form used by the kernels.
struct GsNbrOdometer {
  int8_t v[GS_DMAX];
  int64_t off;
  __device__ __forceinline__ void init(const GsBox& b) {
    off = 0;
    for (int c = 0; c < b.d; ++c) {
      v[c] = -1;
      off -= b.stride[c];
    }
  }
  // advance to the next offset in lexicographic order
  __device__ __forceinline__ void next(const GsBox& b) {
    for (int c = b.d - 1; c >= 0; --c) {
      if (v[c] < 1) {
        ++v[c];
        off += b.stride[c];
        return;
      }
      v[c] = -1;
      off -= 2 * b.stride[c];
    }
  }
};

__device__ __forceinline__ uint32_t gs_ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void gs_st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
