// polycast-b200 umbrella header: the reference's public API
// (proj/include/polycast/polycast.hpp:5-8 includes batch, bench, geometry and io)
// on the GPU engine, plus the device-context controls.
#pragma once

#include "batch.hpp"
#include "bench.hpp"
#include "device.hpp"
#include "geometry.hpp"
#include "io.hpp"
