// Forwarding header: the reference's voxmarch/fields.hpp maps to the B200 facade.
#pragma once
#include "voxmarch/voxmarch.hpp"
