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
// Enqueues the decision-independent head of the step (clock, counters, the
// batch's unique ids) on e->step_side, forked from and later joined into
// e->stream by step_run.  Used by the fused iteration so the head overlaps
// the cost build and the dispatch.
void step_head(edx_engine* e);
// Undoes a launched head whose step will not run (the iteration failed).
void step_head_abandon(edx_engine* e);
// True when step_run decides every victim on the device (no host round trip),
// i.e. the step can be captured into a CUDA graph.
bool step_device_only(const edx_engine* e);

}  // namespace edx
