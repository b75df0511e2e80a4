// Reference include path compatibility: proj/include/cgvariants/types.hpp
#pragma once
#include "cgvariants/cgv.hpp"
