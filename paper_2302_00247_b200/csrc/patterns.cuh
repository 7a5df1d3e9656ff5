// Pattern registry, shard-state conversions and the collective cost model,
// usable from host and device.  Every fp64 expression keeps CPython's
// operation order with explicit round-to-nearest intrinsics on the device, so
// costs are bit-identical to the reference's floats.
//
//   registry              patterns.py:118-159 (LAST = -1, patterns.py:23)
//   ShardSpec.normalized  patterns.py:44-50
//   conversion_collective patterns.py:202-221 (+ _convert divisibility, search.py:227-233)
//   apply_collective      patterns.py:173-185
//   collective_cost_bytes costmodel.py:122-134, collective_call_cost 141-145
#pragma once

#include <cstdint>

#include "../../include/shardsearch.h"

#if defined(__CUDACC__)
#define SP_HD __host__ __device__ __forceinline__
#else
#define SP_HD inline
#endif

namespace sp {

enum SpecKind : int8_t { K_R = 0, K_S = 1, K_P = 2, K_NONE = 3 };
enum CollKind : int8_t { C_ID = 0, C_AR = 1, C_AG = 2, C_RS = 3, C_A2A = 4 };

struct PSpec {
  int8_t kind;
  int8_t axis;  // split axis as registered (may be -1 == LAST)
};
struct Pattern {
  PSpec in, w, out;
  int8_t coll;  // C_ID or C_AR
};

SP_HD PSpec R_() { return PSpec{K_R, 0}; }
SP_HD PSpec S_(int a) { return PSpec{K_S, (int8_t)a}; }
SP_HD PSpec P_() { return PSpec{K_P, 0}; }
SP_HD PSpec N_() { return PSpec{K_NONE, 0}; }

// patterns_for(op): number of patterns (<= 4), -1 for non-shardable kinds.
SP_HD int patterns_for(int op, Pattern* p) {
  switch (op) {
    case SP_OP_MATMUL:
      p[0] = Pattern{R_(), R_(), R_(), C_ID};
      p[1] = Pattern{R_(), S_(1), S_(-1), C_ID};
      p[2] = Pattern{S_(-1), S_(0), P_(), C_AR};
      p[3] = Pattern{S_(0), R_(), S_(0), C_ID};
      return 4;
    case SP_OP_ELEMENTWISE:
      p[0] = Pattern{R_(), R_(), R_(), C_ID};
      p[1] = Pattern{S_(0), R_(), S_(0), C_ID};
      p[2] = Pattern{S_(-1), S_(0), S_(-1), C_ID};
      return 3;
    case SP_OP_LAYERNORM:
    case SP_OP_SOFTMAX:
      p[0] = Pattern{R_(), N_(), R_(), C_ID};
      p[1] = Pattern{S_(0), N_(), S_(0), C_ID};
      return 2;
    case SP_OP_EMBEDDING:
      p[0] = Pattern{R_(), R_(), R_(), C_ID};
      p[1] = Pattern{R_(), S_(1), S_(-1), C_ID};
      p[2] = Pattern{S_(0), R_(), S_(0), C_ID};
      return 3;
    case SP_OP_RESHAPE:
    case SP_OP_INPUT:
    case SP_OP_OUTPUT:
      p[0] = Pattern{R_(), N_(), R_(), C_ID};
      return 1;
    default:
      return -1;
  }
}

// Normalised spec: kind + concrete axis.  Returns false on SpecMismatch.
struct NSpec {
  int8_t kind;
  int8_t axis;
};
SP_HD bool normalize(PSpec s, int rank, NSpec* out) {
  if (s.kind == K_S) {
    int a = s.axis >= 0 ? s.axis : rank + s.axis;
    if (a < 0 || a >= rank) return false;
    *out = NSpec{K_S, (int8_t)a};
    return true;
  }
  *out = NSpec{s.kind, 0};
  return true;
}
SP_HD bool nspec_eq(NSpec a, NSpec b) { return a.kind == b.kind && (a.kind != K_S || a.axis == b.axis); }

// Reachable node states are R, S(0), S(rank-1) (PARTIAL only ever leaves a
// pattern with its AllReduce, which restores R).  Index them 0 / 1 / 2.
SP_HD NSpec state_spec(int idx, int rank) {
  if (idx == 0) return NSpec{K_R, 0};
  if (idx == 1) return NSpec{K_S, 0};
  return NSpec{K_S, (int8_t)(rank - 1)};
}
SP_HD int state_index(NSpec s, int rank) {
  if (s.kind != K_S) return 0;
  if (s.axis == 0) return 1;
  return 2;  // axis == rank-1 (the only other reachable split)
}

// conversion_collective + _convert: false on NoRouteError.
SP_HD bool convert(NSpec a, NSpec b, const int64_t* shape, int64_t d, int8_t* kind, int8_t* axis) {
  if (nspec_eq(a, b)) {
    *kind = C_ID;
    *axis = -1;
  } else if (b.kind == K_R && a.kind == K_S) {
    *kind = C_AG;
    *axis = a.axis;
  } else if (b.kind == K_R && a.kind == K_P) {
    *kind = C_AR;
    *axis = -1;
  } else if (a.kind == K_S && b.kind == K_S) {
    *kind = C_A2A;
    *axis = b.axis;
  } else if (a.kind == K_P && b.kind == K_S) {
    *kind = C_RS;
    *axis = b.axis;
  } else {
    return false;
  }
  if (b.kind == K_S && (shape[b.axis] % d) != 0) return false;
  return true;
}

// Round-to-nearest fp64 primitives (no FMA contraction on either side).
SP_HD double dadd(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dadd_rn(a, b);
#else
  volatile double r = a + b;
  return r;
#endif
}
SP_HD double dmul(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dmul_rn(a, b);
#else
  volatile double r = a * b;
  return r;
#endif
}
SP_HD double ddiv(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __ddiv_rn(a, b);
#else
  volatile double r = a / b;
  return r;
#endif
}

struct MeshC {
  int64_t d;
  double bw, setup;
  double eff[5];  // by CollKind
};

SP_HD MeshC mesh_consts(const sp_mesh& m) {
  MeshC c;
  c.d = m.m * m.n;
  c.bw = m.m > 1 ? m.inter_bw : m.intra_bw;
  c.setup = m.setup_latency_s;
  c.eff[C_ID] = 1.0;
  c.eff[C_AR] = m.eff_allreduce;
  c.eff[C_AG] = m.eff_allgather;
  c.eff[C_RS] = m.eff_reducescatter;
  c.eff[C_A2A] = m.eff_alltoall;
  return c;
}

// collective_cost_bytes: AR volume ((2.0*(d-1))/d)*B, others ((d-1)/d)*B; t = (v/bw)*eff
SP_HD double cost_bytes(int kind, int64_t nbytes, const MeshC& m) {
  if (kind == C_ID || m.d == 1) return 0.0;
  double vol;
  if (kind == C_AR)
    vol = dmul(ddiv(dmul(2.0, (double)(m.d - 1)), (double)m.d), (double)nbytes);
  else
    vol = dmul(ddiv((double)(m.d - 1), (double)m.d), (double)nbytes);
  return dmul(ddiv(vol, m.bw), m.eff[kind]);
}

// collective_call_cost: setup + transfer; identity or one device is free
SP_HD double call_cost(int kind, int64_t nbytes, const MeshC& m) {
  if (kind == C_ID || m.d == 1) return 0.0;
  return dadd(m.setup, cost_bytes(kind, nbytes, m));
}

}  // namespace sp
