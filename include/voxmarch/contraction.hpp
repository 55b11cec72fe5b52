// Forwarding header: the reference's voxmarch/contraction.hpp maps to the B200 facade.
#pragma once
#include "voxmarch/voxmarch.hpp"
