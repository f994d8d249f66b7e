// pdmg_m2_hot128_c64.cu -- one unit of k_march2 instantiations (pdmg_march2_units.cuh)
#define PDMG_M2_UNIT_T float
#define PDMG_M2_UNIT_NF 128
#include "pdmg_march2_units.cuh"
