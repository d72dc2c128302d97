// shim: the reference header prng.hpp maps onto the B200 drop-in
#pragma once
#include "loadsched_gpu.hpp"
