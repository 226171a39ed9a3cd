/* ORACLE — TEST INFRASTRUCTURE ONLY.
 * Runs the compiled reference's TraceStream (orc_trace_dump, ref_shim.cpp) in
 * its own process -- numpy's bundled C++ runtime and the reference's iostreams
 * do not share a Python process safely.  Prints "OK\n<dump>" or "ERR\n<what()>".
 * Usage: trace_dump PATH SCHEMA|- N M CAPACITY */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "edx_oracle.h"

int main(int argc, char** argv) {
  if (argc != 6) return 2;
  const char* schema = strcmp(argv[2], "-") ? argv[2] : NULL;
  const int n = atoi(argv[3]), m = atoi(argv[4]);
  const uint64_t cap = strtoull(argv[5], NULL, 10);
  uint64_t len = 0;
  if (orc_trace_dump(argv[1], schema, n, m, cap, NULL, 0, &len) != ORC_OK) {
    printf("ERR\n%s", orc_last_error());
    return 0;
  }
  char* buf = malloc(len + 1);
  orc_trace_dump(argv[1], schema, n, m, cap, buf, len + 1, &len);
  fputs("OK\n", stdout);
  fwrite(buf, 1, len, stdout);
  free(buf);
  return 0;
}
