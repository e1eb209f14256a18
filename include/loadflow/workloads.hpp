// loadflow/workloads.hpp -- forwards to the single API header (reference layout: proj/include/loadflow/workloads.hpp).
#pragma once
#include "loadflow/api.hpp"
