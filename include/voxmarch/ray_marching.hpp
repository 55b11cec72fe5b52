// Forwarding header: the reference's voxmarch/ray_marching.hpp maps to the B200 facade.
#pragma once
#include "voxmarch/voxmarch.hpp"
