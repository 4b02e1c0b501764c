// K4 (backtrack.cuh): warp-per-problem and CTA-per-problem variants.
#ifndef HEDDLE_UNITY
#define HEDDLE_INST_TU   // the non-template kernels live in heddle_place.cu's translation unit
#endif
#include "dispatch.h"

using namespace hp;

template <int DT, int SR>
K4Fn pick_k4(bool kv, bool w) {
  if (w) return kv ? k4_backtrack<DT, SR, true, true> : k4_backtrack<DT, SR, false, true>;
  return kv ? k4_backtrack<DT, SR, true> : k4_backtrack<DT, SR, false>;
}
template <int DT, int SR>
K4Fn pick_k4c(bool kv, bool w) {
  if (w) return kv ? k4_backtrack_cta<DT, SR, true, true> : k4_backtrack_cta<DT, SR, false, true>;
  return kv ? k4_backtrack_cta<DT, SR, true> : k4_backtrack_cta<DT, SR, false>;
}


K4Fn k4_for(int dt, int sr, bool kv, bool w) {
  if (dt == HEDDLE_F32X) return pick_k4<HEDDLE_F32X, HEDDLE_MINPLUS>(kv, w);
  if (dt == HEDDLE_F32) return sr == HEDDLE_MINMAX ? pick_k4<HEDDLE_F32, HEDDLE_MINMAX>(kv, w) : pick_k4<HEDDLE_F32, HEDDLE_MINPLUS>(kv, w);
  if (dt == HEDDLE_F64) return sr == HEDDLE_MINMAX ? pick_k4<HEDDLE_F64, HEDDLE_MINMAX>(kv, w) : pick_k4<HEDDLE_F64, HEDDLE_MINPLUS>(kv, w);
  return sr == HEDDLE_MINMAX ? pick_k4<HEDDLE_U32, HEDDLE_MINMAX>(kv, w) : pick_k4<HEDDLE_U32, HEDDLE_MINPLUS>(kv, w);
}

K4Fn k4c_for(int dt, int sr, bool kv, bool w) { return HP_DISPATCH(pick_k4c, kv, w); }

template <int DT, int SR>
K4QFn pick_k4q(bool kv, bool w) {
  if (w) return kv ? k4_query<DT, SR, true, true> : k4_query<DT, SR, false, true>;
  return kv ? k4_query<DT, SR, true> : k4_query<DT, SR, false>;
}

K4QFn k4q_for(int dt, int sr, bool kv, bool w) { return HP_DISPATCH(pick_k4q, kv, w); }
