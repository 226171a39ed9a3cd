// Device step (K7) entry points; see step.cu.
#pragma once

#include "engine.h"

namespace edx {

struct StepResult {
  int launches = 0;
  int evicting_workers = 0;
};

// Allocates and initialises the cache tables and step scratch of an engine.
void step_init_state(edx_engine* e);
// Enqueues SimState::step for the engine's current batch and d_decision; on
// return the per-worker counters are being copied to e->h_counters (the
// caller synchronises the stream).
void step_run(edx_engine* e, const int32_t* d_decision, StepResult* out);
// True when step_run decides every victim on the device (no host round trip),
// i.e. the step can be captured into a CUDA graph.
bool step_device_only(const edx_engine* e);

}  // namespace edx
