// catsim/catsim.hpp -- umbrella header of this repo's drop-in catsim API (the
// reference has no umbrella; its headers are included one by one and work
// the same here).
#pragma once

#include "catsim/bench.hpp"
#include "catsim/cat_engine.hpp"
#include "catsim/engines.hpp"
#include "catsim/fragment.hpp"
#include "catsim/grid.hpp"
#include "catsim/layout.hpp"
#include "catsim/reference.hpp"
#include "catsim/rule.hpp"
#include "catsim/snapshot.hpp"
