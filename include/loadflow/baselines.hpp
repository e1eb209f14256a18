// loadflow/baselines.hpp -- forwards to the single API header (reference layout: proj/include/loadflow/baselines.hpp).
#pragma once
#include "loadflow/api.hpp"
