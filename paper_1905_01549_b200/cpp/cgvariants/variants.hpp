// Reference include path compatibility: proj/include/cgvariants/variants.hpp
#pragma once
#include "cgvariants/cgv.hpp"
