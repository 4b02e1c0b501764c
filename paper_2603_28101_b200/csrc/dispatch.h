// Kernel dispatch tables shared by the host code (heddle_place.cu) and the translation units
// that instantiate the large kernel families (inst_*.cu, compiled in parallel; a -DHEDDLE_UNITY
// build includes them into heddle_place.cu instead).  Each getter returns the kernel variant for a
// dtype / semiring / feature combination; the launch stays in heddle_place.cu.
#pragma once
#include <cstdint>

#include "backtrack.cuh"
#include "dp_batched.cuh"
#include "dp_layered.cuh"
#include "heddle_place.h"
#include "valley.cuh"

using K2Fn = void (*)(hp::SolveArgs);
using K4Fn = void (*)(hp::SolveArgs, int32_t*);
using K4QFn = void (*)(hp::SolveArgs, int, const int32_t*, const int32_t*, const int32_t*, void*, int32_t*);
using K3Fn = void (*)(hp::LayerArgs);
using K5Fn = void (*)(hp::PersistArgs);
using KPro = void (*)(hp::SolveArgs);
using K8Fn = void (*)(hp::SolveArgs);
using K8LFn = void (*)(hp::SolveArgs, int, hp::ValleyWs);

// dt: heddle_dtype, sr: heddle_semiring
// (HEDDLE_F32X exists only with MINPLUS; heddle_place_init rejects the other combination)
#define HP_DISPATCH(NAME, ...)                                                                          \
  (dt == HEDDLE_F32X ? NAME<HEDDLE_F32X, HEDDLE_MINPLUS>(__VA_ARGS__)                                  \
   : dt == HEDDLE_F32 ? (sr == HEDDLE_MINMAX ? NAME<HEDDLE_F32, HEDDLE_MINMAX>(__VA_ARGS__)             \
                                           : NAME<HEDDLE_F32, HEDDLE_MINPLUS>(__VA_ARGS__))             \
   : dt == HEDDLE_F64 ? (sr == HEDDLE_MINMAX ? NAME<HEDDLE_F64, HEDDLE_MINMAX>(__VA_ARGS__)             \
                                             : NAME<HEDDLE_F64, HEDDLE_MINPLUS>(__VA_ARGS__))           \
                      : (sr == HEDDLE_MINMAX ? NAME<HEDDLE_U32, HEDDLE_MINMAX>(__VA_ARGS__)             \
                                             : NAME<HEDDLE_U32, HEDDLE_MINPLUS>(__VA_ARGS__)))

K2Fn k2_for(int dt, int sr, bool kp, bool kv, bool w = false);   // inst_k2.cu
K4Fn k4_for(int dt, int sr, bool kv, bool w);                     // inst_k4.cu
K4Fn k4c_for(int dt, int sr, bool kv, bool w);
K4QFn k4q_for(int dt, int sr, bool kv, bool w);
K3Fn k3_for(int dt, int sr, bool kp, bool kv, bool w = false);                    // inst_k35.cu
KPro pro_for(int dt, int sr, bool kp, bool kv);
K5Fn k5_for(int dt, int sr);
K8Fn k8c_for(int dt, bool kv, bool w, int v);                       // inst_k8.cu: cluster variants (kK8Cluster CTAs)
K8Fn k8_for(int dt, bool kp, bool kv, bool w, int wide);          // inst_k8.cu (0: 128, 1: 1024, 2: 512 threads)
K8LFn k8l_for(int dt, bool kp, bool kv, bool w = false);
