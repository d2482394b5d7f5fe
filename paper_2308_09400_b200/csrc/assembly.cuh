// Shared state of the assembly translation units (assembly.cu: sort-based symbolic phase, numeric kernels,
// gradient scatter; symbolic_rows.cu: row-wise symbolic phase).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace b200ipc {

constexpr int kMaxFam = 7;  // family ids 0..6; 7 tags the diagonal mass slot in source descriptors
constexpr int kAT = 256;

struct FamDesc {
  int32_t s[kMaxFam];
  int64_t nb[kMaxFam];
  int64_t ent_off[kMaxFam + 1];   // prefix of nb*s*s  (matrix slots, after the N diagonal slots)
  int64_t vert_off[kMaxFam + 1];  // prefix of nb*s    (gradient slots)
  const int64_t* vids[kMaxFam];
  int32_t nfam;
  // dense-block layout of a family: 1 = the reference's row-major (nb, 3s, 3s); 3 = sub-block-major
  // (nb, s, s, 3, 3), every 3x3 sub-block 72 contiguous bytes.  It is the factor of c in the element
  // offset / 3 of sub-block (a, c): 3 (b s + a) s + cmul c.
  int32_t cmul[kMaxFam];
};

struct HessPtrs {
  const double* p[kMaxFam + 1];  // slot 7 = "no source" (null)
};

template <typename T>
struct DevBuf {
  T* ptr = nullptr;
  size_t cap = 0;
  cudaError_t reserve(size_t n) {
    if (n <= cap) return cudaSuccess;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(&ptr, n * sizeof(T));
    if (e == cudaSuccess) cap = n;
    return e;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
  }
};

}  // namespace b200ipc

struct b200ipc_assembly {
  int64_t nverts = 0;
  int64_t nslots = 0;      // N + sum nb*s*s
  int64_t nvalid = 0;      // slots that survive the fixed-vertex filter
  int64_t nnzb = 0;
  int64_t ngslots = 0;     // sum nb*s
  bool ready = false;
  bool have_desc = false, have_fdesc = false, have_rows = false;   // descriptor tables are built on first use
  int variant = 0;         // numeric kernel: 0 auto (per-block runs when applicable), 1 runs, 4 row-wise
  int symbolic_mode = 0;   // 0 auto (row-wise, sort path when a row is too long), 1 sort path always
  uint32_t tiled_next = 0; // bit f: family f of the NEXT pattern delivers its dense blocks sub-block-major
  uint32_t tiled = 0;      // the same for the current pattern
  int symbolic_used = 0;   // which path built the current pattern: 1 sort, 2 row-wise
  int64_t max_row = -1;    // longest block row of the current pattern (-1: not measured yet)
  b200ipc::FamDesc fam;
  b200ipc::DevBuf<uint8_t> fixed;
  b200ipc::DevBuf<uint64_t> keys_a, keys_b;
  b200ipc::DevBuf<uint32_t> slot_a, slot_b;   // slot_b ends up as the sorted permutation
  b200ipc::DevBuf<int32_t> head, useg;        // head flags / scan, run starts (nnzb+1)
  b200ipc::DevBuf<uint32_t> desc;             // per sorted source: family << 30 | element offset / 3 (3 = mass slot)
  b200ipc::DevBuf<uint32_t> fdesc;            // per sorted source, factor form: family | c-a+3 | b*D+3a
  b200ipc::DevBuf<int32_t> rowptr, colidx;
  b200ipc::DevBuf<uint32_t> gkeys_a, gkeys_b, gslot_a, gslot_b;
  b200ipc::DevBuf<int32_t> gseg;              // (N+1) run starts per vertex
  b200ipc::DevBuf<uint64_t> rs_desc, rs_dst;  // per row-source: chunk offset|family, 4 x u16 destination block
  b200ipc::DevBuf<uint8_t> temp;
  b200ipc::DevBuf<int64_t> scalars;           // device scratch for counts
  b200ipc::DevBuf<int32_t> uend;                // run ends (a run is [useg[u], uend[u]); slab-spaced after the row-wise phase)
  b200ipc::DevBuf<int32_t> row_len, slab_col, slab_beg, slab_end;   // row-wise symbolic phase: per-row slabs
};

