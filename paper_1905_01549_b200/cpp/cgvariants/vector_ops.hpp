// Reference include path compatibility: proj/include/cgvariants/vector_ops.hpp
#pragma once
#include "cgvariants/cgv.hpp"
