// mfcg_inst.cu -- one translation unit per polynomial degree (compiled with
// -DMFCG_P=1..8) so the heavy brick-kernel templates build in parallel.
#include "mfcg_engine.cuh"

#ifndef MFCG_P
#error "compile with -DMFCG_P=<degree>"
#endif

namespace mfcg {

#define MFCG_CAT2(a, b) a##b
#define MFCG_CAT(a, b) MFCG_CAT2(a, b)

#ifdef MFCG_STUB
// variant builds for timing experiments carry one degree only (tools/varlibs, build.build_variant)
EngineBase* MFCG_CAT(make_engine_p, MFCG_P)(OpCommon*, int* status) {
  set_error("this variant build does not contain the degree");
  *status = MFCG_EUNSUPPORTED;
  return nullptr;
}
#else
EngineBase* MFCG_CAT(make_engine_p, MFCG_P)(OpCommon* c, int* status) {
  if (c->precision == 0) {
    auto* e = new Engine<MFCG_P, double>(c);
    if ((*status = e->init()) != MFCG_OK) { delete e; return nullptr; }
    return e;
  }
  auto* e = new Engine<MFCG_P, float>(c);
  if ((*status = e->init()) != MFCG_OK) { delete e; return nullptr; }
  return e;
}
#endif

}  // namespace mfcg
