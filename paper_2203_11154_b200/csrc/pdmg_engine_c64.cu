// pdmg_engine_c64.cu -- Engine<float> (complex64: fp32 storage) and its kernels.
#include "pdmg_engine.cuh"

namespace pdmg_b200 {

template struct Engine<float>;
std::unique_ptr<EngineBase> make_engine_c64() { return std::make_unique<Engine<float>>(); }

}  // namespace pdmg_b200
