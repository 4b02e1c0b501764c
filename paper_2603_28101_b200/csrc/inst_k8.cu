// K8 / K8L valley kernels (valley.cuh, min-max only).
#ifndef HEDDLE_UNITY
#define HEDDLE_INST_TU   // the non-template kernels live in heddle_place.cu's translation unit
#endif
#include "dispatch.h"

using namespace hp;

template <int DT, int NT>
K8Fn pick_k8n(bool kp, bool kv, bool w) {
  if (kp) {
    if (w) return kv ? k8_valley<DT, true, true, true, NT> : k8_valley<DT, true, false, true, NT>;
    return kv ? k8_valley<DT, true, true, false, NT> : k8_valley<DT, true, false, false, NT>;
  }
  if (w) return kv ? k8_valley<DT, false, true, true, NT> : k8_valley<DT, false, false, true, NT>;
  return kv ? k8_valley<DT, false, true, false, NT> : k8_valley<DT, false, false, false, NT>;
}
template <int DT>
K8Fn pick_k8(bool kp, bool kv, bool w, int wide) {
  return wide == 2 ? pick_k8n<DT, kK8ThreadsMid>(kp, kv, w)
                   : wide ? pick_k8n<DT, kK8ThreadsWide>(kp, kv, w) : pick_k8n<DT, kK8Threads>(kp, kv, w);
}
K8Fn k8_for(int dt, bool kp, bool kv, bool w, int wide) {
  if (dt == HEDDLE_F32) return pick_k8<HEDDLE_F32>(kp, kv, w, wide);
  if (dt == HEDDLE_F64) return pick_k8<HEDDLE_F64>(kp, kv, w, wide);
  return pick_k8<HEDDLE_U32>(kp, kv, w, wide);
}
// cluster variants (no parents): 0 = 512 threads x 8 CTAs, 1 = 512 x 4, 2 = 1024 x 4
template <int DT, int NT, int CL>
K8Fn pick_k8c_n(bool kv, bool w) {
  if (w) return kv ? k8_valley<DT, false, true, true, NT, CL> : k8_valley<DT, false, false, true, NT, CL>;
  return kv ? k8_valley<DT, false, true, false, NT, CL> : k8_valley<DT, false, false, false, NT, CL>;
}
template <int DT>
K8Fn pick_k8c(bool kv, bool w, int v) {
  return v == 0 ? pick_k8c_n<DT, 512, 2 * kK8Cluster>(kv, w)
                : v == 1 ? pick_k8c_n<DT, 512, kK8Cluster>(kv, w) : pick_k8c_n<DT, 1024, kK8Cluster>(kv, w);
}
K8Fn k8c_for(int dt, bool kv, bool w, int v) {
  if (dt == HEDDLE_F32) return pick_k8c<HEDDLE_F32>(kv, w, v);
  if (dt == HEDDLE_F64) return pick_k8c<HEDDLE_F64>(kv, w, v);
  return pick_k8c<HEDDLE_U32>(kv, w, v);
}
template <int DT>
K8LFn pick_k8l(bool kp, bool kv, bool w) {
  if (w) {
    if (kp) return kv ? k8l_layer<DT, true, true, true> : k8l_layer<DT, true, false, true>;
    return kv ? k8l_layer<DT, false, true, true> : k8l_layer<DT, false, false, true>;
  }
  if (kp) return kv ? k8l_layer<DT, true, true> : k8l_layer<DT, true, false>;
  return kv ? k8l_layer<DT, false, true> : k8l_layer<DT, false, false>;
}
K8LFn k8l_for(int dt, bool kp, bool kv, bool w) {
  if (dt == HEDDLE_F32) return pick_k8l<HEDDLE_F32>(kp, kv, w);
  if (dt == HEDDLE_F64) return pick_k8l<HEDDLE_F64>(kp, kv, w);
  return pick_k8l<HEDDLE_U32>(kp, kv, w);
}
