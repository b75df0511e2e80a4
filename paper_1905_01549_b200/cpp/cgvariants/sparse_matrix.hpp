// Reference include path compatibility: proj/include/cgvariants/sparse_matrix.hpp
#pragma once
#include "cgvariants/cgv.hpp"
