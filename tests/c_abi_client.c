/* A plain-C client of libpipesgd (what a cgo / JNI / ctypes binding sees):
 * compiled with gcc -std=c11 against include/pipesgd.h and linked with
 * -lpipesgd by tests/test_cabi.py. Uses only entries that need no GPU. */
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "pipesgd.h"

int main(void) {
  int64_t plan[5];
  if (gp_version() != 1) return 1;
  /* C2 gradient over 2 ranks, trunc16, the standalone CTA budget */
  if (gp_ring_plan(4710538u, 2, 592, GP_CODEC_TRUNC16, 0, 4710538u, plan) != GP_OK) return 2;
  printf("chunk=%lld ctas=%lld ll=%lld nch=%lld\n", (long long)plan[0], (long long)plan[1], (long long)plan[2],
         (long long)plan[3]);
  /* argument errors come back as codes plus the thread's message */
  if (gp_encode(7, NULL, 0, NULL, NULL, NULL) != GP_ERR_ARG) return 3;
  if (strstr(gp_last_error_string(), "unknown codec") == NULL) return 4;
  if (gp_ring_plan(1, 1, 592, GP_CODEC_NONE, 0, 1, plan) != GP_ERR_ARG) return 5;
  printf("errors ok: %s\n", gp_last_error_string());
  return 0;
}
