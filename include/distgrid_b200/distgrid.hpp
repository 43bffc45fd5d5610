// distgrid_b200/distgrid.hpp — umbrella include of the C++ facade.  The facade mirrors the
// reference's headers one for one under include/distgrid/ (so `#include "distgrid/worker.hpp"`
// resolves to it with -I include); this header pulls in all of them.
#pragma once

#include "distgrid/config.hpp"
#include "distgrid/dataset.hpp"
#include "distgrid/field.hpp"
#include "distgrid/geometry.hpp"
#include "distgrid/grid.hpp"
#include "distgrid/mlp.hpp"
#include "distgrid/partition.hpp"
#include "distgrid/render.hpp"
#include "distgrid/rng.hpp"
#include "distgrid/train.hpp"
#include "distgrid/vecmath.hpp"
#include "distgrid/worker.hpp"
