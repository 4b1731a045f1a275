// Device-side tensor-language analysis: Value payloads, interned split-origin
// cut trees, shape inference, make / merge / same_data.
//
// Semantics follow the reference TensorAnalysis (reference:
// pkg/src/tensorsat/tensor_lang.py:72-136 Value/merge_values, :293-515
// infer_shape + _infer_*, :730-746 TensorAnalysis.make/merge).  Shapes are
// rank <= 4 (MAX_RANK, tensor_lang.py:42).  Cut trees are hash-consed into a
// device table so structural equality is id equality; an origin set is a
// small sorted array of (axis << 28 | tree id).
#pragma once
#include "common.cuh"

#define MAXO 6            // origin entries per side of a Value
#define TREE_MAXPOS 5     // concat_6 -> 5 interior cuts
#define TREE_NONE 0x0FFFFFFFu

enum OpCode : int {
  OP_EWADD = 0, OP_EWMUL, OP_MATMUL, OP_CONV, OP_RELU, OP_TANH, OP_SIGMOID,
  OP_POOLMAX, OP_POOLAVG, OP_TRANSPOSE, OP_ENLARGE, OP_SPLIT, OP_SPLIT0, OP_SPLIT1,
  OP_MERGE, OP_RESHAPE, OP_INPUT, OP_WEIGHT, OP_NOOP,
  OP_CONCAT2, OP_CONCAT3, OP_CONCAT4, OP_CONCAT5, OP_CONCAT6,
  OP_COUNT
};

enum ValKind : int8_t { VK_NONE = 0, VK_N = 1, VK_S = 2, VK_T = 3, VK_TT = 4 };

// analysis status codes (0 = ok)
enum AnaStatus : int { AS_OK = 0, AS_SHAPE = 1, AS_SPLIT_ORIGIN = 2, AS_ORIGIN_OVERFLOW = 3, AS_TREE_FULL = 4 };

struct AtomInfo {
  int32_t kind;    // 0 = int atom, 1 = str atom
  int32_t opcode;  // OpCode for operator names, -1 otherwise
  i64 ival;        // int atoms
  int32_t ndims;   // parse_dims(str): number of parts, -1 when unparsable
  int32_t nident;  // parse_identifier(str): rank, -1 when invalid
  i64 dims[4];
  i64 idims[4];
};

struct __align__(16) Val {
  int8_t kind;
  int8_t r0, r1;   // ranks of shape / pair halves
  int8_t n0, n1;   // origin counts
  int8_t pad[3];
  i64 iv;          // N: ival, S: atom id
  i64 d0[4];
  i64 d1[4];
  u32 o0[MAXO];
  u32 o1[MAXO];
};

// One tree per 128-byte line: a published tree is immutable and no other
// tree shares its line, so readers may cache it in L1 (a popular tree --
// every combo of a merge rule builds the same concat -- otherwise turns into
// one hot L2 line read by every thread of the wave)
struct __align__(128) Tree {
  int32_t npos;
  int32_t pad;
  i64 pos[TREE_MAXPOS];
  u32 kid[TREE_MAXPOS + 1];  // TREE_NONE = no subtree
  u32 pad2[14];
};
static_assert(sizeof(Tree) == 128, "one tree per 128-byte line");

struct TreeTab {
  Tree* trees;
  u32* hc;        // open addressing, TSAT_NONE = empty
  u32 hc_mask;
  u32* count;
  u32 cap;
};

__constant__ int8_t c_sig_n[OP_COUNT] = {2, 2, 3, 6, 1, 1, 1, 7, 7, 2, 2, 2, 1, 1, 2, 2, 1, 1, 2, 3, 4, 5, 6, 7};
// argument kinds per op, VK_* codes; row = op
__constant__ int8_t c_sig_k[OP_COUNT][7] = {
    {3, 3}, {3, 3}, {1, 3, 3}, {1, 1, 1, 1, 3, 3}, {3}, {3}, {3},
    {3, 1, 1, 1, 1, 1, 1}, {3, 1, 1, 1, 1, 1, 1}, {3, 2}, {3, 3}, {1, 3}, {4}, {4},
    {3, 1}, {3, 2}, {2}, {2}, {3, 3},
    {1, 3, 3}, {1, 3, 3, 3}, {1, 3, 3, 3, 3}, {1, 3, 3, 3, 3, 3}, {1, 3, 3, 3, 3, 3, 3}};

__device__ __forceinline__ u32 orig_axis(u32 e) { return e >> 28; }
__device__ __forceinline__ u32 orig_tree(u32 e) { return e & 0x0FFFFFFFu; }
__device__ __forceinline__ u32 orig_pack(u32 axis, u32 tree) { return (axis << 28) | tree; }

__device__ __forceinline__ void val_clear(Val& v) {
  v.kind = VK_NONE;
  v.r0 = v.r1 = v.n0 = v.n1 = 0;
  v.pad[0] = v.pad[1] = v.pad[2] = 0;
  v.iv = 0;
#pragma unroll
  for (int i = 0; i < 4; i++) v.d0[i] = v.d1[i] = 0;
#pragma unroll
  for (int i = 0; i < MAXO; i++) v.o0[i] = v.o1[i] = 0;
}

// ---------------------------------------------------------------- origin sets

// insert into sorted unique array; returns false on overflow
__device__ __forceinline__ bool oset_add(u32* o, int8_t& n, u32 e) {
  int i = 0;
  while (i < n && o[i] < e) i++;
  if (i < n && o[i] == e) return true;
  if (n >= MAXO) return false;
  for (int j = n; j > i; j--) o[j] = o[j - 1];
  o[i] = e;
  n++;
  return true;
}

__device__ __forceinline__ bool oset_union(u32* o, int8_t& n, const u32* b, int8_t nb) {
  for (int i = 0; i < nb; i++)
    if (!oset_add(o, n, b[i])) return false;
  return true;
}

__device__ __forceinline__ bool oset_subset(const u32* a, int8_t na, const u32* b, int8_t nb) {
  for (int i = 0; i < na; i++) {
    bool f = false;
    for (int j = 0; j < nb; j++) f |= (a[i] == b[j]);
    if (!f) return false;
  }
  return true;
}

// number of trees recorded on ``axis`` and the first one
__device__ __forceinline__ int oset_on_axis(const u32* o, int8_t n, u32 axis, u32& tree) {
  int c = 0;
  for (int i = 0; i < n; i++)
    if (orig_axis(o[i]) == axis) {
      if (c == 0) tree = orig_tree(o[i]);
      c++;
    }
  return c;
}

// ---------------------------------------------------------------- tree interning

__device__ __forceinline__ u64 tree_hash(int npos, const i64* pos, const u32* kid) {
  u64 h = 0x51ed270b27d2d0c1ULL ^ (u64)npos;
  for (int i = 0; i < npos; i++) h = hash_mix(h, (u64)pos[i]);
  for (int i = 0; i <= npos; i++) h = hash_mix(h, (u64)kid[i]);
  return h;
}

// cached loads: t was published (its id read from the table) after the
// inserter fenced its contents, and its line holds no other tree
__device__ __forceinline__ bool tree_eq(const Tree* t, int npos, const i64* pos, const u32* kid) {
  if (t->npos != npos) return false;
  for (int i = 0; i < npos; i++)
    if (t->pos[i] != pos[i]) return false;
  for (int i = 0; i <= npos; i++)
    if (t->kid[i] != kid[i]) return false;
  return true;
}

// returns tree id, or TSAT_NONE when the table is full
static __device__ u32 tree_intern(const TreeTab& tt, int npos, const i64* pos, const u32* kid) {
  u64 h = tree_hash(npos, pos, kid);
  u32 slot = (u32)h & tt.hc_mask;
  u32 mine = TSAT_NONE;
  for (u32 probe = 0; probe <= tt.hc_mask; probe++) {
    // a slot goes NONE -> id once per engine lifetime: a stale NONE only
    // sends this thread to the CAS below, which returns the published id
    u32 cur = tt.hc[slot];
    if (cur == TSAT_NONE) {
      if (mine == TSAT_NONE) {
        mine = atomicAdd(tt.count, 1u);
        if (mine >= tt.cap || mine >= TREE_NONE) return TSAT_NONE;
        Tree* t = &tt.trees[mine];
        t->npos = npos;
        t->pad = 0;
        for (int i = 0; i < TREE_MAXPOS; i++) t->pos[i] = i < npos ? pos[i] : 0;
        for (int i = 0; i <= TREE_MAXPOS; i++) t->kid[i] = i <= npos ? kid[i] : TREE_NONE;
        __threadfence();
      }
      u32 prev = atomicCAS(&tt.hc[slot], TSAT_NONE, mine);
      if (prev == TSAT_NONE) return mine;
      cur = prev;
    }
    // no fence here: the inserter fenced its tree before publishing the id,
    // and tree_eq's volatile (L2) loads are address-dependent on that id
    if (tree_eq(&tt.trees[cur], npos, pos, kid)) return cur;
    slot = (slot + 1) & tt.hc_mask;
  }
  return TSAT_NONE;
}

__device__ __forceinline__ void tree_read(const TreeTab& tt, u32 id, int& npos, i64* pos, u32* kid) {
  const Tree* t = &tt.trees[id];  // published, immutable, alone in its line
  npos = t->npos;
  for (int i = 0; i < TREE_MAXPOS; i++) pos[i] = t->pos[i];
  for (int i = 0; i <= TREE_MAXPOS; i++) kid[i] = t->kid[i];
}

// ---------------------------------------------------------------- helpers

__device__ __forceinline__ bool shape_eq(const i64* a, int ra, const i64* b, int rb) {
  if (ra != rb) return false;
  for (int i = 0; i < ra; i++)
    if (a[i] != b[i]) return false;
  return true;
}

// 16-byte-word copy (eight vector loads, then eight vector stores)
__device__ __forceinline__ void val_copy(Val& d, const Val& s) {
  const uint4* a = reinterpret_cast<const uint4*>(&s);
  uint4* b = reinterpret_cast<uint4*>(&d);
  uint4 w[sizeof(Val) / 16];
#pragma unroll
  for (int i = 0; i < (int)(sizeof(Val) / 16); i++) w[i] = a[i];
#pragma unroll
  for (int i = 0; i < (int)(sizeof(Val) / 16); i++) b[i] = w[i];
}

__device__ __forceinline__ bool val_same_data(const Val& a, const Val& b) {
  if (a.kind != b.kind) return false;
  switch (a.kind) {
    case VK_N:
    case VK_S:
      return a.iv == b.iv;
    case VK_T:
      return shape_eq(a.d0, a.r0, b.d0, b.r0);
    case VK_TT:
      return shape_eq(a.d0, a.r0, b.d0, b.r0) && shape_eq(a.d1, a.r1, b.d1, b.r1);
    default:
      return true;
  }
}

// merged origins differ from a's?  (used to detect analysis change on union)
__device__ __forceinline__ bool val_merge_grows(const Val& a, const Val& b) {
  if (a.kind == VK_T) return !oset_subset(b.o0, b.n0, a.o0, a.n0);
  if (a.kind == VK_TT)
    return !oset_subset(b.o0, b.n0, a.o0, a.n0) || !oset_subset(b.o1, b.n1, a.o1, a.n1);
  return false;
}

// a := merge(a, b); assumes same_data already checked.  returns AnaStatus
__device__ __forceinline__ int val_merge_into(Val& a, const Val& b) {
  if (a.kind == VK_T) return oset_union(a.o0, a.n0, b.o0, b.n0) ? AS_OK : AS_ORIGIN_OVERFLOW;
  if (a.kind == VK_TT) {
    if (!oset_union(a.o0, a.n0, b.o0, b.n0)) return AS_ORIGIN_OVERFLOW;
    if (!oset_union(a.o1, a.n1, b.o1, b.n1)) return AS_ORIGIN_OVERFLOW;
  }
  return AS_OK;
}

__device__ __forceinline__ void set_tensor(Val& o, const i64* d, int r) {
  val_clear(o);
  o.kind = VK_T;
  o.r0 = (int8_t)r;
  for (int i = 0; i < r; i++) o.d0[i] = d[i];
}

__device__ __forceinline__ bool check_shape(const i64* d, int r) {
  if (r < 1 || r > 4) return false;
  for (int i = 0; i < r; i++)
    if (d[i] < 1) return false;
  return true;
}

__device__ __forceinline__ bool in_range(i64 v, i64 lo, i64 hi) { return v >= lo && v <= hi; }
#define I64_MAX_ 0x7fffffffffffffffLL

// conv_out_hw (tensor_lang.py:269-279); SAME uses float ceil like math.ceil(h / s)
__device__ __forceinline__ int conv_out(i64 h, i64 w, i64 kh, i64 kw, i64 sh, i64 sw, i64 pad,
                                        i64& oh, i64& ow) {
  if (sh < 1 || sw < 1) return AS_SHAPE;
  if (pad == 0) {
    oh = (i64)ceil((double)h / (double)sh);
    ow = (i64)ceil((double)w / (double)sw);
    return AS_OK;
  }
  if (pad == 1) {
    if (h < kh || w < kw) return AS_SHAPE;
    oh = (h - kh) / sh + 1;
    ow = (w - kw) / sw + 1;
    return AS_OK;
  }
  return AS_SHAPE;
}

// ---------------------------------------------------------------- infer_shape

// Argument values by reference: an array of pointers into the node table /
// wave table (no 128-byte copies into local memory).
struct ValRefs {
  const Val* const* p;
  __device__ __forceinline__ const Val& operator[](int i) const { return *p[i]; }
};

// Output value of operator ``op`` for argument values ``a`` (n of them).
static __device__ int infer_shape_dev(int op, ValRefs a, int n, Val& out, const AtomInfo* atoms,
                               const TreeTab& tt) {
  if (op < 0 || op >= OP_COUNT) return AS_SHAPE;
  if (n != c_sig_n[op]) return AS_SHAPE;
  for (int i = 0; i < n; i++)
    if (a[i].kind != c_sig_k[op][i]) return AS_SHAPE;
  switch (op) {
    case OP_EWADD:
    case OP_EWMUL: {
      if (!shape_eq(a[0].d0, a[0].r0, a[1].d0, a[1].r0)) return AS_SHAPE;
      set_tensor(out, a[0].d0, a[0].r0);
      out.n0 = a[0].n0;
      for (int i = 0; i < a[0].n0; i++) out.o0[i] = a[0].o0[i];
      return oset_union(out.o0, out.n0, a[1].o0, a[1].n0) ? AS_OK : AS_ORIGIN_OVERFLOW;
    }
    case OP_MATMUL: {
      if (!in_range(a[0].iv, 0, 3)) return AS_SHAPE;
      const Val &x = a[1], &y = a[2];
      int r = x.r0;
      if (x.r0 < 2 || y.r0 < 2 || x.r0 != y.r0) return AS_SHAPE;
      for (int i = 0; i < r - 2; i++)
        if (x.d0[i] != y.d0[i]) return AS_SHAPE;
      if (x.d0[r - 1] != y.d0[r - 2]) return AS_SHAPE;
      i64 d[4];
      for (int i = 0; i < r - 1; i++) d[i] = x.d0[i];
      d[r - 1] = y.d0[r - 1];
      set_tensor(out, d, r);
      for (int i = 0; i < x.n0; i++)
        if (orig_axis(x.o0[i]) == (u32)(r - 2))
          if (!oset_add(out.o0, out.n0, x.o0[i])) return AS_ORIGIN_OVERFLOW;
      for (int i = 0; i < y.n0; i++)
        if (orig_axis(y.o0[i]) == (u32)(y.r0 - 1))
          if (!oset_add(out.o0, out.n0, orig_pack(r - 1, orig_tree(y.o0[i])))) return AS_ORIGIN_OVERFLOW;
      return AS_OK;
    }
    case OP_CONV: {
      i64 sh = a[0].iv, sw = a[1].iv, pad = a[2].iv, act = a[3].iv;
      if (sh < 1 || sw < 1 || !in_range(pad, 0, 1) || !in_range(act, 0, 3)) return AS_SHAPE;
      const Val &x = a[4], &w = a[5];
      if (x.r0 != 4 || w.r0 != 4) return AS_SHAPE;
      i64 c = x.d0[1], cin = w.d0[1], cout = w.d0[0];
      if (c % cin != 0) return AS_SHAPE;
      i64 groups = c / cin;
      if (cout % groups != 0) return AS_SHAPE;
      i64 oh, ow;
      if (conv_out(x.d0[2], x.d0[3], w.d0[2], w.d0[3], sh, sw, pad, oh, ow)) return AS_SHAPE;
      i64 d[4] = {x.d0[0], cout, oh, ow};
      set_tensor(out, d, 4);
      for (int i = 0; i < w.n0; i++)
        if (orig_axis(w.o0[i]) == 0)
          if (!oset_add(out.o0, out.n0, orig_pack(1, orig_tree(w.o0[i])))) return AS_ORIGIN_OVERFLOW;
      return AS_OK;
    }
    case OP_RELU:
    case OP_TANH:
    case OP_SIGMOID: {
      out = a[0];
      return AS_OK;
    }
    case OP_POOLMAX:
    case OP_POOLAVG: {
      const Val& x = a[0];
      i64 kh = a[1].iv, kw = a[2].iv, sh = a[3].iv, sw = a[4].iv, pad = a[5].iv, act = a[6].iv;
      if (kh < 1 || kw < 1 || sh < 1 || sw < 1 || !in_range(pad, 0, 1) || !in_range(act, 0, 3))
        return AS_SHAPE;
      if (x.r0 != 4) return AS_SHAPE;
      i64 oh, ow;
      if (conv_out(x.d0[2], x.d0[3], kh, kw, sh, sw, pad, oh, ow)) return AS_SHAPE;
      i64 d[4] = {x.d0[0], x.d0[1], oh, ow};
      set_tensor(out, d, 4);
      for (int i = 0; i < x.n0; i++)
        if (orig_axis(x.o0[i]) <= 1) out.o0[out.n0++] = x.o0[i];
      return AS_OK;
    }
    case OP_TRANSPOSE: {
      const Val& x = a[0];
      const AtomInfo& p = atoms[a[1].iv];
      if (p.ndims < 0) return AS_SHAPE;
      int r = x.r0;
      if (p.ndims != r) return AS_SHAPE;
      // sorted(perm) == range(rank)
      int seen = 0;
      for (int i = 0; i < r; i++) {
        i64 q = p.dims[i];
        if (q < 0 || q >= r || (seen >> q) & 1) return AS_SHAPE;
        seen |= 1 << q;
      }
      i64 d[4];
      int inv[4];
      for (int i = 0; i < r; i++) {
        d[i] = x.d0[p.dims[i]];
        inv[p.dims[i]] = i;
      }
      set_tensor(out, d, r);
      for (int i = 0; i < x.n0; i++) {
        u32 ax = orig_axis(x.o0[i]);
        if ((int)ax >= r) return AS_SHAPE;  // KeyError in the reference; unreachable
        if (!oset_add(out.o0, out.n0, orig_pack(inv[ax], orig_tree(x.o0[i])))) return AS_ORIGIN_OVERFLOW;
      }
      return AS_OK;
    }
    case OP_ENLARGE: {
      const Val &x = a[0], &ref = a[1];
      if (x.r0 != 4 || ref.r0 != 4) return AS_SHAPE;
      if (x.d0[2] > ref.d0[2] || x.d0[3] > ref.d0[3]) return AS_SHAPE;
      i64 d[4] = {x.d0[0], x.d0[1], ref.d0[2], ref.d0[3]};
      set_tensor(out, d, 4);
      for (int i = 0; i < x.n0; i++)
        if (orig_axis(x.o0[i]) <= 1) out.o0[out.n0++] = x.o0[i];
      return AS_OK;
    }
    case OP_CONCAT2:
    case OP_CONCAT3:
    case OP_CONCAT4:
    case OP_CONCAT5:
    case OP_CONCAT6: {
      int k = n - 1;
      ValRefs in{a.p + 1};
      int r = in[0].r0;
      i64 axis = a[0].iv;
      if (!in_range(axis, 0, r - 1)) return AS_SHAPE;
      for (int j = 1; j < k; j++) {
        if (in[j].r0 != r) return AS_SHAPE;
        for (int ax = 0; ax < r; ax++)
          if (ax != axis && in[j].d0[ax] != in[0].d0[ax]) return AS_SHAPE;
      }
      i64 total = 0, pos[TREE_MAXPOS];
      u32 kid[TREE_MAXPOS + 1];
      for (int j = 0; j < k; j++) {
        total += in[j].d0[axis];
        if (j < k - 1) pos[j] = total;
        u32 t = TREE_NONE;
        int c = oset_on_axis(in[j].o0, in[j].n0, (u32)axis, t);
        kid[j] = c == 1 ? t : TREE_NONE;
      }
      u32 id = tree_intern(tt, k - 1, pos, kid);
      if (id == TSAT_NONE) return AS_TREE_FULL;
      i64 d[4];
      for (int i = 0; i < r; i++) d[i] = in[0].d0[i];
      d[axis] = total;
      if (!check_shape(d, r)) return AS_SHAPE;
      set_tensor(out, d, r);
      out.o0[0] = orig_pack((u32)axis, id);
      out.n0 = 1;
      return AS_OK;
    }
    case OP_SPLIT: {
      const Val& x = a[1];
      int r = x.r0;
      i64 axis = a[0].iv;
      if (!in_range(axis, 0, r - 1)) return AS_SHAPE;
      u32 t = 0;
      int c = oset_on_axis(x.o0, x.n0, (u32)axis, t);
      if (c == 0) return AS_SPLIT_ORIGIN;
      if (c > 1) return AS_SHAPE;
      int np;
      i64 pos[TREE_MAXPOS];
      u32 kid[TREE_MAXPOS + 1];
      tree_read(tt, t, np, pos, kid);
      i64 cut = pos[0], total = x.d0[axis];
      if (!(0 < cut && cut < total)) return AS_SHAPE;
      val_clear(out);
      out.kind = VK_TT;
      out.r0 = out.r1 = (int8_t)r;
      for (int i = 0; i < r; i++) out.d0[i] = out.d1[i] = x.d0[i];
      out.d0[axis] = cut;
      out.d1[axis] = total - cut;
      u32 rtree, ltree = kid[0];
      if (np > 1) {
        i64 rest[TREE_MAXPOS];
        for (int i = 1; i < np; i++) rest[i - 1] = pos[i] - cut;
        rtree = tree_intern(tt, np - 1, rest, kid + 1);
        if (rtree == TSAT_NONE) return AS_TREE_FULL;
      } else {
        rtree = kid[1];
      }
      for (int i = 0; i < x.n0; i++)
        if (orig_axis(x.o0[i]) != (u32)axis) {
          out.o0[out.n0++] = x.o0[i];
          out.o1[out.n1++] = x.o0[i];
        }
      if (ltree != TREE_NONE && !oset_add(out.o0, out.n0, orig_pack((u32)axis, ltree))) return AS_ORIGIN_OVERFLOW;
      if (rtree != TREE_NONE && !oset_add(out.o1, out.n1, orig_pack((u32)axis, rtree))) return AS_ORIGIN_OVERFLOW;
      return AS_OK;
    }
    case OP_SPLIT0:
    case OP_SPLIT1: {
      // every load before the first store: out may alias a generic argument
      // pointer as far as the compiler knows, so interleaved field copies
      // would serialise load -> store -> load
      const Val& p = a[0];
      const bool lo = op == OP_SPLIT0;
      const int8_t r = lo ? p.r0 : p.r1, no = lo ? p.n0 : p.n1;
      i64 d[4];
      u32 o[MAXO];
#pragma unroll
      for (int i = 0; i < 4; i++) d[i] = lo ? p.d0[i] : p.d1[i];
#pragma unroll
      for (int i = 0; i < MAXO; i++) o[i] = lo ? p.o0[i] : p.o1[i];
      val_clear(out);
      out.kind = VK_T;
      out.r0 = r;
      out.n0 = no;
#pragma unroll
      for (int i = 0; i < 4; i++) out.d0[i] = d[i];
#pragma unroll
      for (int i = 0; i < MAXO; i++) out.o0[i] = o[i];
      return AS_OK;
    }
    case OP_MERGE: {
      const Val& w = a[0];
      i64 count = a[1].iv;
      if (count < 1) return AS_SHAPE;
      if (w.r0 != 4) return AS_SHAPE;
      i64 d[4] = {w.d0[0], w.d0[1] * count, w.d0[2], w.d0[3]};
      set_tensor(out, d, 4);
      return AS_OK;
    }
    case OP_RESHAPE: {
      const AtomInfo& s = atoms[a[1].iv];
      if (s.ndims < 0) return AS_SHAPE;
      if (!check_shape(s.dims, s.ndims)) return AS_SHAPE;
      i64 p1 = 1, p2 = 1;
      for (int i = 0; i < s.ndims; i++) p1 *= s.dims[i];
      for (int i = 0; i < a[0].r0; i++) p2 *= a[0].d0[i];
      if (p1 != p2) return AS_SHAPE;
      set_tensor(out, s.dims, s.ndims);
      return AS_OK;
    }
    case OP_INPUT:
    case OP_WEIGHT: {
      const AtomInfo& s = atoms[a[0].iv];
      if (s.nident < 0) return AS_SHAPE;
      if (!check_shape(s.idims, s.nident)) return AS_SHAPE;
      set_tensor(out, s.idims, s.nident);
      return AS_OK;
    }
    case OP_NOOP: {
      i64 d[1] = {1};
      set_tensor(out, d, 1);
      return AS_OK;
    }
  }
  return AS_SHAPE;
}

// TensorAnalysis.make (tensor_lang.py:734-743)
__device__ __forceinline__ int val_make(u32 atom, ValRefs kids, int n, Val& out,
                                        const AtomInfo* atoms, const TreeTab& tt) {
  const AtomInfo& ai = atoms[atom];
  if (n == 0) {
    val_clear(out);
    if (ai.kind == 0) {
      out.kind = VK_N;
      out.iv = ai.ival;
      return AS_OK;
    }
    if (ai.opcode < 0) {
      out.kind = VK_S;
      out.iv = atom;
      return AS_OK;
    }
    return AS_SHAPE;  // operator used without arguments
  }
  if (ai.kind != 1 || ai.opcode < 0) return AS_SHAPE;  // unknown operator
  return infer_shape_dev(ai.opcode, kids, n, out, atoms, tt);
}
