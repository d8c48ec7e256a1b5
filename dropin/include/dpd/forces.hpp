// dpd/forces.hpp -- declarations of the reference's `forces` module
// (SPEC.md:405-475).  The reference lists src/forces.cpp in its build
// (CMakeLists.txt:22) but ships neither it nor this header; this is the header
// the B200 drop-in (dropin/forces.cpp) implements, named and shaped after the
// SPEC's operations.  One addition to SPEC's compute_forces listing: the box,
// which the minimum image (src/core.cpp:129-139) needs.
#pragma once

#include <cstdint>

#include "dpd/core.hpp"
#include "dpd/neighbor_table.hpp"
#include "dpd/rng.hpp"

namespace dpd {

// for every particle i, the sum over row(i) of F_C + F_D + F_R for
// the entries with |r_ij| <= r_c this step, plus the harmonic bond forces of
// `bonds`; written to store.force.  The pair random numbers come
// from store.tag / the velocities' signatures and state.step_mix (inc/rng.hpp:65-83).
void compute_forces(ParticleStore& store, const NeighborTable& table, const PairParams& params,
                    const BondTopology& bonds, const PairRandomState& state, const SimBox& box);

}  // namespace dpd
