// loadflow/queue.hpp -- forwards to the single API header (reference layout: proj/include/loadflow/queue.hpp).
#pragma once
#include "loadflow/api.hpp"
