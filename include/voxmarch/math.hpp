// Forwarding header: the reference's voxmarch/math.hpp maps to the B200 facade.
#pragma once
#include "voxmarch/voxmarch.hpp"
