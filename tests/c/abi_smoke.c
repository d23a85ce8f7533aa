/* abi_smoke.c -- a plain C consumer of include/pms.h (no C++, no CUDA
 * headers): reads an n x t sequence file, calls the north-star entry points
 * pms_find / pms_find64 and prints what they return, so tests/test_c_abi.py
 * can compare it with the CPU oracle.  Also exercises the documented
 * argument errors (PAPER.md:23 problem statement; include/pms.h).
 *
 *   abi_smoke FILE l d        FILE: "n t\n" then n*t bytes (rows of A/C/G/T)
 * Output lines: "find <status> <count> <code> <code> ...", "find64 ...",
 * "errors <status list>". */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "pms.h"

int main(int argc, char **argv) {
    if (argc != 4) {
        fprintf(stderr, "usage: %s FILE l d\n", argv[0]);
        return 2;
    }
    FILE *f = fopen(argv[1], "rb");
    if (!f) return 2;
    int n = 0, t = 0;
    if (fscanf(f, "%d %d", &n, &t) != 2 || n < 1 || t < 1) return 2;
    fgetc(f); /* the newline */
    uint8_t *seqs = (uint8_t *)malloc((size_t)n * t);
    if (!seqs || fread(seqs, 1, (size_t)n * t, f) != (size_t)n * t) return 2;
    fclose(f);
    const int l = atoi(argv[2]), d = atoi(argv[3]);

    enum { CAP = 1 << 16 };
    uint32_t *codes = (uint32_t *)malloc(CAP * sizeof(uint32_t));
    uint64_t *codes64 = (uint64_t *)malloc(CAP * sizeof(uint64_t));
    uint64_t count = 0;
    int st = pms_find(seqs, n, t, l, d, codes, CAP, &count);
    printf("find %d %llu", st, (unsigned long long)count);
    for (uint64_t i = 0; st == PMS_OK && i < count; ++i) printf(" %u", codes[i]);
    printf("\n");
    uint64_t count64 = 0;
    st = pms_find64(seqs, n, t, l, d, codes64, CAP, &count64);
    printf("find64 %d %llu", st, (unsigned long long)count64);
    for (uint64_t i = 0; st == PMS_OK && i < count64; ++i) printf(" %llu", (unsigned long long)codes64[i]);
    printf("\n");
    /* documented errors, in check order (include/pms.h) */
    uint64_t c = 0;
    printf("errors %d %d %d %d %d %d %d\n",
           pms_find(NULL, n, t, l, d, codes, CAP, &c),          /* NULL seqs      -> ARG */
           pms_find(seqs, n, t, l, d, codes, CAP, NULL),        /* NULL count     -> ARG */
           pms_find(seqs, n, t, l, d, NULL, 1, &c),             /* NULL out, cap  -> ARG */
           pms_find(seqs, n, t, 17, d, codes, CAP, &c),         /* l > 16 (u32)   -> ARG */
           pms_find(seqs, n, t, t + 1, 0, codes, CAP, &c),      /* l > t          -> ARG */
           pms_find(seqs, n, t, l, -1, codes, CAP, &c),         /* d < 0          -> ARG */
           pms_find(seqs, n, t, l, d, codes, 0, &c));           /* size query: TRUNCATED or OK */
    printf("strerror %s\n", pms_strerror(PMS_E_CHAR));
    free(seqs);
    free(codes);
    free(codes64);
    return 0;
}
