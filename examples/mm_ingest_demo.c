/* Matrix Market ingest through the C ABI from plain C (host side only):
 *   mm_ingest_demo file.mtx [threads]
 * prints the header and the first entries of the parsed COO (0-based), or
 * the reference-style "path:line: reason" error.  No GPU needed. */
#include <stdio.h>
#include <stdlib.h>

#include "sketch_b200.h"

int main(int argc, char **argv) {
  if (argc < 2) {
    fprintf(stderr, "usage: %s file.mtx [threads]\n", argv[0]);
    return 2;
  }
  skt_mm_info info;
  if (skt_mm_probe(argv[1], &info) != SKT_OK) {
    printf("error = %s\n", skt_last_error());
    return 1;
  }
  const int64_t cap = info.n_entries * (info.symmetric ? 2 : 1);
  int64_t *rows = malloc(sizeof(int64_t) * (size_t)(cap > 0 ? cap : 1));
  int64_t *cols = malloc(sizeof(int64_t) * (size_t)(cap > 0 ? cap : 1));
  double *vals = malloc(sizeof(double) * (size_t)(cap > 0 ? cap : 1));
  int64_t count = 0;
  const int threads = argc > 2 ? atoi(argv[2]) : 0;
  if (skt_mm_read_coo(argv[1], cap, rows, cols, vals, &count, threads) != SKT_OK) {
    printf("error = %s\n", skt_last_error());
    return 1;
  }
  printf("shape = %lld %lld\n", (long long)info.n_rows, (long long)info.n_cols);
  printf("declared = %lld\n", (long long)info.n_entries);
  printf("count = %lld\n", (long long)count);
  printf("field symmetric = %d %d\n", info.field, info.symmetric);
  for (int64_t e = 0; e < count && e < 3; ++e)
    printf("entry%lld = %lld %lld %.17g\n", (long long)e, (long long)rows[e], (long long)cols[e], vals[e]);
  free(rows);
  free(cols);
  free(vals);
  return 0;
}
