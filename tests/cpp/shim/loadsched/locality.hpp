// shim: the reference header locality.hpp maps onto the B200 drop-in
#pragma once
#include "loadsched_gpu.hpp"
