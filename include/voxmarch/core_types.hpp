// Forwarding header: the reference's voxmarch/core_types.hpp maps to the B200 facade.
#pragma once
#include "voxmarch/voxmarch.hpp"
