// loadflow/scheduler.hpp -- forwards to the single API header (reference layout: proj/include/loadflow/scheduler.hpp).
#pragma once
#include "loadflow/api.hpp"
