// Forwarding header: the reference's voxmarch/scene_camera.hpp maps to the B200 facade.
#pragma once
#include "voxmarch/voxmarch.hpp"
