// loadflow/worker_pool.hpp -- forwards to the single API header (reference layout: proj/include/loadflow/worker_pool.hpp).
#pragma once
#include "loadflow/api.hpp"
