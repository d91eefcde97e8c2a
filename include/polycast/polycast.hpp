// polycast-b200 umbrella header (reference: proj/include/polycast/polycast.hpp:5-8).
// The reference also pulls in io.hpp and bench.hpp (CSV/GeoJSON I/O and the
// LSQ benchmark harness); those are outside this build's scope (SURVEY §2 rows
// 4-5) and are not provided.
#pragma once

#include "batch.hpp"
#include "device.hpp"
#include "geometry.hpp"
