// loadflow/trainer.hpp -- forwards to the single API header (reference layout: proj/include/loadflow/trainer.hpp).
#pragma once
#include "loadflow/api.hpp"
