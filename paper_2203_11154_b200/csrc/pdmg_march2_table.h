// pdmg_march2_table.h -- the function-pointer table of the fused Vanka passes (k_march2) and the per-unit fill
// functions that populate it (pdmg_march2_units.cuh).  key = loadu | prolong << 1 | post << 2 | norm_in << 4
#pragma once
#include "pdmg_kernels.cuh"

namespace pdmg_b200 {

template <class T>
using March2Fn = void (*)(MarchArgs<T>, CoefPack);
inline int march2_key(bool lu, bool pr, int post, bool nin = false) {
  return (lu ? 1 : 0) | (pr ? 2 : 0) | (post << 2) | (nin ? 16 : 0);
}
void march2_fill_two(March2Fn<double>* e);
void march2_fill_one(March2Fn<double>* e);
void march2_fill_two(March2Fn<float>* e);
void march2_fill_one(March2Fn<float>* e);
void march2_fill_hot_128(March2Fn<double>* eN, March2Fn<double>* e1N);
void march2_fill_hot_256(March2Fn<double>* eN, March2Fn<double>* e1N);
void march2_fill_hot_512(March2Fn<double>* eN, March2Fn<double>* e1N);
void march2_fill_hot_1024(March2Fn<double>* eN, March2Fn<double>* e1N);
void march2_fill_hot_128(March2Fn<float>* eN, March2Fn<float>* e1N);
void march2_fill_hot_256(March2Fn<float>* eN, March2Fn<float>* e1N);
void march2_fill_hot_512(March2Fn<float>* eN, March2Fn<float>* e1N);
void march2_fill_hot_1024(March2Fn<float>* eN, March2Fn<float>* e1N);

}  // namespace pdmg_b200
