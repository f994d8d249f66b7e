// pdmg_m2_c128_two.cu -- one unit of k_march2 instantiations (pdmg_march2_units.cuh)
#define PDMG_M2_UNIT_T double
#define PDMG_M2_UNIT_TWO 1
#include "pdmg_march2_units.cuh"
