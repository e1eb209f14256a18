// loadflow/profiler.hpp -- forwards to the single API header (reference layout: proj/include/loadflow/profiler.hpp).
#pragma once
#include "loadflow/api.hpp"
