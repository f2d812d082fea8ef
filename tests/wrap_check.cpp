// Host build of the engine's wrap_angle (csrc/common.cuh) for tests/test_wrap_host.py:
// reads n float64 from argv[1], writes wrap_angle of each to argv[2].
#include <cstdio>
#include <vector>

#include "common.cuh"

int main(int argc, char **argv) {
  if (argc != 3) return 2;
  FILE *f = std::fopen(argv[1], "rb");
  if (!f) return 3;
  std::vector<double> v;
  double x;
  while (std::fread(&x, sizeof x, 1, f) == 1) v.push_back(pi2::wrap_angle(x));
  std::fclose(f);
  FILE *g = std::fopen(argv[2], "wb");
  if (!g) return 4;
  std::fwrite(v.data(), sizeof(double), v.size(), g);
  std::fclose(g);
  return 0;
}
