// loadflow/balancer.hpp -- forwards to the single API header (reference layout: proj/include/loadflow/balancer.hpp).
#pragma once
#include "loadflow/api.hpp"
