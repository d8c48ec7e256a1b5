// dpd/integrate.hpp -- declarations of the reference's `integrate` module
// for the B200 drop-in (dropin/integrate.cpp); the
// reference lists src/integrate.cpp (CMakeLists.txt:23) but ships neither it
// nor a header.  The box (wrap / walls) and the wall mode are
// explicit arguments.
#pragma once

#include "dpd/core.hpp"

namespace dpd {

enum class StepPhase { Phase1, Phase2 };

// Phase1: v += dt/2 f, x += dt v, then the box's boundary (periodic
// wrap S:524, walls S:506-514); Phase2: v += dt/2 f.  Non-finite state is a
// physics error naming the particle.
void verlet_step(ParticleStore& store, const PairParams& params, StepPhase phase, const SimBox& box,
                 WallMode wall_mode = WallMode::specular);

}  // namespace dpd
