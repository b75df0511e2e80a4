// Reference include path compatibility: proj/include/cgvariants/runner.hpp
#pragma once
#include "cgvariants/cgv.hpp"
