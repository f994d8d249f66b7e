// pdmg_engine_c128.cu -- Engine<double> (complex128) and its kernels.
#include "pdmg_engine.cuh"

namespace pdmg_b200 {

template struct Engine<double>;
std::unique_ptr<EngineBase> make_engine_c128() { return std::make_unique<Engine<double>>(); }

}  // namespace pdmg_b200
