// Forwarding header: the reference's voxmarch/rendering.hpp maps to the B200 facade.
#pragma once
#include "voxmarch/voxmarch.hpp"
