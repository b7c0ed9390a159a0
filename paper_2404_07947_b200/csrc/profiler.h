// XProfiler entry point (see profiler.cu).
#pragma once
#include "../../include/exegpt.h"
#include "engine.cuh"
#include "planner.h"

namespace exg {
void profile_layers(Engine& E, const exg_model_spec& spec, const exg_profile_grid& g, plan::Profile* out);
}
