// pdmg_m2_c64_one.cu -- one unit of k_march2 instantiations (pdmg_march2_units.cuh)
#define PDMG_M2_UNIT_T float
#define PDMG_M2_UNIT_TWO 0
#include "pdmg_march2_units.cuh"
