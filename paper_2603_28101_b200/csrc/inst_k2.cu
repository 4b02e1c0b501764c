// K2 (dp_batched.cuh): every dtype / semiring / feature variant.
#ifndef HEDDLE_UNITY
#define HEDDLE_INST_TU   // the non-template kernels live in heddle_place.cu's translation unit
#endif
#include "dispatch.h"

using namespace hp;

template <int DT, int SR>
K2Fn pick_k2(bool kp, bool kv, bool w) {
  if (w) {
    if (kp) return kv ? k2_dp_batched<DT, SR, true, true, true> : k2_dp_batched<DT, SR, true, false, true>;
    return kv ? k2_dp_batched<DT, SR, false, true, true> : k2_dp_batched<DT, SR, false, false, true>;
  }
  if (kp) return kv ? k2_dp_batched<DT, SR, true, true> : k2_dp_batched<DT, SR, true, false>;
  return kv ? k2_dp_batched<DT, SR, false, true> : k2_dp_batched<DT, SR, false, false>;
}

K2Fn k2_for(int dt, int sr, bool kp, bool kv, bool w) {
  if (dt == HEDDLE_F32X) return pick_k2<HEDDLE_F32X, HEDDLE_MINPLUS>(kp, kv, w);
  if (dt == HEDDLE_F32) return sr == HEDDLE_MINMAX ? pick_k2<HEDDLE_F32, HEDDLE_MINMAX>(kp, kv, w) : pick_k2<HEDDLE_F32, HEDDLE_MINPLUS>(kp, kv, w);
  if (dt == HEDDLE_F64) return sr == HEDDLE_MINMAX ? pick_k2<HEDDLE_F64, HEDDLE_MINMAX>(kp, kv, w) : pick_k2<HEDDLE_F64, HEDDLE_MINPLUS>(kp, kv, w);
  return sr == HEDDLE_MINMAX ? pick_k2<HEDDLE_U32, HEDDLE_MINMAX>(kp, kv, w) : pick_k2<HEDDLE_U32, HEDDLE_MINPLUS>(kp, kv, w);
}
