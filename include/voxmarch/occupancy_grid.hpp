// Forwarding header: the reference's voxmarch/occupancy_grid.hpp maps to the B200 facade.
#pragma once
#include "voxmarch/voxmarch.hpp"
