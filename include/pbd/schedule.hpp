// Forwarding header: the reference API of proj/core/include/pbd/schedule.hpp lives in pbd/core.hpp.
#pragma once
#include "pbd/core.hpp"
