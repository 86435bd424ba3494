// catsim/catsim.hpp -- the whole catsim C++ API of this repo (drop-in for the
// reference's CAT-engine path), header-only over include/ltl_b200.h.
#pragma once

#include "catsim/cat_engine.hpp"
#include "catsim/engines.hpp"
#include "catsim/fragment.hpp"
#include "catsim/grid.hpp"
#include "catsim/layout.hpp"
#include "catsim/rule.hpp"
#include "catsim/snapshot.hpp"
