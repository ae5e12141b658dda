// ecc.hpp -- umbrella header of the C++ drop-in API (include/ecc/*).
#pragma once
#include "ecc/common.hpp"
#include "ecc/context.hpp"
#include "ecc/image.hpp"
#include "ecc/chunk.hpp"
#include "ecc/value_index.hpp"
#include "ecc/kernel.hpp"
#include "ecc/vcec.hpp"
#include "ecc/curve.hpp"
#include "ecc/device.hpp"
#include "ecc/streaming.hpp"
#include "ecc/datagen.hpp"
#include "ecc/pipeline.hpp"
