// Reference include path compatibility: proj/include/cgvariants/preconditioner.hpp
#pragma once
#include "cgvariants/cgv.hpp"
