// Host build of csrc/eig9.cuh for tests/test_eig9.py: reads n packed 9x9 matrices (45 doubles
// each) from stdin, writes for each the status (as a double) and the 45 entries of P+(M).
#include <cstdio>
#include <vector>
#include "eig9.cuh"

int main() {
  std::vector<double> buf(45);
  double out[45], scratch[35 + 9 * 9];
  while (fread(buf.data(), sizeof(double), 45, stdin) == 45) {
    double M[45];
    for (int q = 0; q < 45; ++q) M[q] = buf[q];
    for (int q = 0; q < 45; ++q) out[q] = 0.0;
    const double st = (double)e9::psd_project<9>(M, out, scratch, 1);
    fwrite(&st, sizeof(double), 1, stdout);
    fwrite(out, sizeof(double), 45, stdout);
  }
  return 0;
}
