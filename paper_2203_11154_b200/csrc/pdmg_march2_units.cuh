// pdmg_march2_units.cuh -- the k_march2 instantiations, split over translation units so that `make -j` compiles
// them in parallel (each fused-pass kernel is 4-10 thousand instructions; ~80 instantiations).  A unit defines
// PDMG_M2_UNIT_T (double / float) and either PDMG_M2_UNIT_TWO (0 / 1: the generic kernels of that sweep count) or
// PDMG_M2_UNIT_NF (256 / 512 / 1024: the hot variants with the level's n compiled in, for PDMG_M2_UNIT_T), then includes
// this file.  Engine<T> fills its March2Table through the march2_fill_* functions declared in pdmg_march2_table.h.
#pragma once
#include "pdmg_kernels.cuh"
#include "pdmg_march2_table.h"

namespace pdmg_b200 {

#ifdef PDMG_M2_UNIT_NF
#ifndef PDMG_M2_UNIT_T
#define PDMG_M2_UNIT_T double
#endif
template <bool LU, bool PR, int PO, bool NI, bool TWO>
static void reg_hot_one(March2Fn<PDMG_M2_UNIT_T>* eN, March2Fn<PDMG_M2_UNIT_T>* e1N) {
  (TWO ? eN : e1N)[march2_key(LU, PR, PO, NI)] = &k_march2<PDMG_M2_UNIT_T, LU, PR, PO, NI, TWO, PDMG_M2_UNIT_NF>;
}
#define PDMG_M2_CAT2(a, b) a##b
#define PDMG_M2_CAT(a, b) PDMG_M2_CAT2(a, b)
void PDMG_M2_CAT(march2_fill_hot_, PDMG_M2_UNIT_NF)(March2Fn<PDMG_M2_UNIT_T>* eN, March2Fn<PDMG_M2_UNIT_T>* e1N) {
  reg_hot_one<true, true, POST_NONE, false, true>(eN, e1N);        // prolong+vanka2
  reg_hot_one<true, false, POST_RESTRICT, true, true>(eN, e1N);    // vanka2+restrict+norm_in
  reg_hot_one<false, false, POST_RESTRICT, true, true>(eN, e1N);   // zero+vanka2+restrict+norm_in
  reg_hot_one<false, false, POST_RESTRICT, false, true>(eN, e1N);  // zero+vanka2+restrict (coarse levels)
  reg_hot_one<true, true, POST_NONE, false, false>(eN, e1N);       // prolong+vanka (V(1,1))
  reg_hot_one<true, false, POST_RESTRICT, true, false>(eN, e1N);   // vanka+restrict+norm_in (V(1,1))
  reg_hot_one<false, false, POST_RESTRICT, true, false>(eN, e1N);  // zero+vanka+restrict+norm_in
  reg_hot_one<false, false, POST_RESTRICT, false, false>(eN, e1N); // zero+vanka+restrict
}
#else
template <bool LU, bool PR, int PO, bool NI = false>
static void reg_gen_one(March2Fn<PDMG_M2_UNIT_T>* e) {
  e[march2_key(LU, PR, PO, NI)] = &k_march2<PDMG_M2_UNIT_T, LU, PR, PO, NI, PDMG_M2_UNIT_TWO != 0>;
}
template <bool LU>
static void reg_gen_lu(March2Fn<PDMG_M2_UNIT_T>* e) {
  reg_gen_one<LU, false, POST_NONE>(e);
  reg_gen_one<LU, false, POST_RESTRICT>(e);
  reg_gen_one<LU, false, POST_NORM>(e);
  reg_gen_one<LU, true, POST_NONE>(e);
  reg_gen_one<LU, true, POST_NORM>(e);
  reg_gen_one<LU, false, POST_RESTRICT, true>(e);
  reg_gen_one<LU, false, POST_NONE, true>(e);
}
#if PDMG_M2_UNIT_TWO
void march2_fill_two(March2Fn<PDMG_M2_UNIT_T>* e) {
#else
void march2_fill_one(March2Fn<PDMG_M2_UNIT_T>* e) {
#endif
  reg_gen_lu<false>(e);
  reg_gen_lu<true>(e);
}
#endif

}  // namespace pdmg_b200
