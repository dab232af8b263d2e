/* A C host of the drop-in boundary (include/contactsim_b200.h): no Python, no torch.
 *
 *   gcc -O2 -I include examples/collide_demo.c -L paper_2205_03532_b200/_lib \
 *       -lcontactsim_b200 -Wl,-rpath,$PWD/paper_2205_03532_b200/_lib -o examples/collide_demo
 *   examples/collide_demo input.bin
 *
 * input.bin (little endian): int64 nv, nt, nx, ny, nz, E; float64 origin[3], voxel,
 * aabb_lo[3], aabb_hi[3]; float64 vertices[nv*3]; int32 triangles[nt*3]; float32
 * values[nx*ny*nz]; float64 sdf_pose[E*7], mesh_pose[E*7], contact_distance[E].
 * Registers the grid and the mesh, runs one collide step through the host-buffer
 * call (cs_collide_host: H2D poses, generation + reduction, D2H stats) and prints
 * one line per env: n_cand n_patch n_kept max_kept_depth. Exit status: 0 ok,
 * else the cs_status of the failing call (message on stderr). */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "contactsim_b200.h"

static int check(int st, const char *what) {
    if (st != CS_OK) fprintf(stderr, "%s failed (%d): %s\n", what, st, cs_last_error());
    return st;
}

static void *take(FILE *f, size_t n) {
    void *p = malloc(n ? n : 1);
    if (!p || fread(p, 1, n, f) != n) { fprintf(stderr, "short input\n"); exit(CS_ERR_VALUE); }
    return p;
}

int main(int argc, char **argv) {
    if (argc != 2) { fprintf(stderr, "usage: %s input.bin\n", argv[0]); return CS_ERR_VALUE; }
    FILE *f = fopen(argv[1], "rb");
    if (!f) { perror(argv[1]); return CS_ERR_VALUE; }
    int64_t *hd = take(f, 6 * sizeof(int64_t));
    const int64_t nv = hd[0], nt = hd[1], nx = hd[2], ny = hd[3], nz = hd[4], E = hd[5];
    double *geo = take(f, 10 * sizeof(double));  /* origin[3], voxel, lo[3], hi[3] */
    double *verts = take(f, (size_t)nv * 3 * sizeof(double));
    int32_t *tris = take(f, (size_t)nt * 3 * sizeof(int32_t));
    float *values = take(f, (size_t)(nx * ny * nz) * sizeof(float));
    double *sp = take(f, (size_t)E * 7 * sizeof(double)), *mp = take(f, (size_t)E * 7 * sizeof(double));
    double *cd = take(f, (size_t)E * sizeof(double));
    fclose(f);

    int32_t hs, hm;
    int st;
    if ((st = check(cs_sdf_register(values, 0, (int32_t)nx, (int32_t)ny, (int32_t)nz, geo, geo[3], geo + 4, geo + 7,
                                    &hs), "cs_sdf_register"))) return st;
    if ((st = check(cs_mesh_register(verts, nv, tris, nt, &hm), "cs_mesh_register"))) return st;
    int32_t *hsv = malloc(sizeof(int32_t) * E), *hmv = malloc(sizeof(int32_t) * E);
    for (int64_t e = 0; e < E; ++e) { hsv[e] = hs; hmv[e] = hm; }
    /* ReductionParams() defaults (contacts/types.py:62-78); min_depth None -> -cd per env */
    cs_reduction_params rp = {128, 6, 1024, 0, 0.9396926207859084, 0.0};
    cs_plan *plan = NULL;
    if ((st = check(cs_plan_create(E, hsv, hmv, &rp, CS_STAGE_ALL, &plan), "cs_plan_create"))) return st;
    float *stats = malloc(sizeof(float) * 4 * E);
    if ((st = check(cs_collide_host(plan, sp, mp, CS_POSE7, cd, stats, NULL), "cs_collide_host"))) return st;
    for (int64_t e = 0; e < E; ++e)
        printf("%d %d %d %.9g\n", (int)stats[4 * e], (int)stats[4 * e + 1], (int)stats[4 * e + 2], stats[4 * e + 3]);
    cs_plan_destroy(plan);
    cs_mesh_free(hm);
    cs_sdf_free(hs);
    return 0;
}
