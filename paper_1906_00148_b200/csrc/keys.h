// keys.h — host-side key objects (opaque handles of include/she.h).
#pragma once
#include <stdint.h>

#include <vector>

#include "../../include/she.h"

struct she_secret_key {
  she_params p;
  std::vector<uint8_t> s;  // LWE key, n bits
  std::vector<uint8_t> S;  // TRLWE key, N bits
};

struct she_cloud_key {
  she_params p;
  std::vector<uint32_t> bk;   // [n][2l][2][N]        torus32, coefficient domain
  std::vector<uint32_t> ksk;  // [N][t][base][n+1]    v = 0 rows zero
};
