// shim: the reference header config.hpp maps onto the B200 drop-in
#pragma once
#include "loadsched_gpu.hpp"
