// K3 per-layer kernel, layered prologue and K5 persistent kernel (dp_layered.cuh).
#ifndef HEDDLE_UNITY
#define HEDDLE_INST_TU   // the non-template kernels live in heddle_place.cu's translation unit
#endif
#include "dispatch.h"

using namespace hp;

template <int DT, int SR>
K3Fn pick_k3(bool kp, bool kv, bool w) {
  if (w) {
    if (kp) return kv ? k3_layer<DT, SR, true, true, true> : k3_layer<DT, SR, true, false, true>;
    return kv ? k3_layer<DT, SR, false, true, true> : k3_layer<DT, SR, false, false, true>;
  }
  if (kp) return kv ? k3_layer<DT, SR, true, true> : k3_layer<DT, SR, true, false>;
  return kv ? k3_layer<DT, SR, false, true> : k3_layer<DT, SR, false, false>;
}
template <int DT, int SR>
KPro pick_pro(bool kp, bool kv) {
  if (kp) return kv ? k3_prologue<DT, SR, true, true> : k3_prologue<DT, SR, true, false>;
  return kv ? k3_prologue<DT, SR, false, true> : k3_prologue<DT, SR, false, false>;
}
K3Fn k3_for(int dt, int sr, bool kp, bool kv, bool w) { return HP_DISPATCH(pick_k3, kp, kv, w); }
KPro pro_for(int dt, int sr, bool kp, bool kv) { return HP_DISPATCH(pick_pro, kp, kv); }
template <int DT, int SR>
K5Fn pick_k5() { return k5_persistent<DT, SR>; }
K5Fn k5_for(int dt, int sr) { return HP_DISPATCH(pick_k5); }
