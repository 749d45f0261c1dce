// Native probe of luda_files_read (bounce / cuFile) with a SIGSEGV backtrace.
#include <execinfo.h>
#include <signal.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>
#include "../../include/luda_b200.h"
static void on_segv(int) {
  void* bt[64];
  int n = backtrace(bt, 64);
  backtrace_symbols_fd(bt, n, 2);
  _exit(139);
}
int main(int argc, char** argv) {
  signal(SIGSEGV, on_segv);
  int mode = argc > 1 ? atoi(argv[1]) : 2;
  const char* p = "/tmp/io_probe.bin";
  FILE* f = fopen(p, "wb");
  static char buf[3 << 20];
  for (size_t i = 0; i < sizeof buf; ++i) buf[i] = (char)(i * 131);
  fwrite(buf, 1, sizeof buf, f);
  fclose(f);
  fprintf(stderr, "init %d\n", luda_init(0));
  void* dev = nullptr;
  fprintf(stderr, "alloc %d\n", luda_region_alloc(sizeof buf + 64, &dev));
  const char* paths[1] = {p};
  uint64_t off[1] = {0}, len[1] = {sizeof buf};
  int used = -1;
  fprintf(stderr, "calling mode %d\n", mode);
  int rc = luda_files_read(paths, 1, dev, off, len, mode, &used);
  fprintf(stderr, "rc %d used %d err %s\n", rc, used, luda_last_error());
  return 0;
}
