/*
 * TEST INFRASTRUCTURE — plain-C restatement of the reference hot path (FP64).
 *
 * A second, self-contained oracle for the per-pixel path of voxanim's
 * render_frame, written from the reference's algorithm (no reference code is
 * linked). It is checked bit for bit against the reference itself
 * (oracle/_ref, tests/test_oracle_restatement.py) and against the committed
 * golden fixtures (tests/golden/), and needs nothing but a C compiler, so it
 * also runs where /root/reference is absent. Only tests/ may use it; the
 * product never does.
 *
 * Followed operation by operation (compile with -ffp-contract=off):
 *   ray generation       proj/src/renderer.cpp:11-23
 *   sphere test          proj/src/renderer.cpp:25-43, bounding_sphere scene.cpp:16-20
 *   candidate order      proj/src/renderer.cpp:134-141,171-203 (no hit buffer)
 *   trace_ray            proj/src/renderer.cpp:63-100
 *   ray transform        proj/include/voxanim/math.hpp:206-224
 *   ray_box_params       proj/src/traversal.cpp:30-61
 *   first/next_node      proj/src/traversal.cpp:63-103
 *   traverse_impl        proj/src/traversal.cpp:115-245
 *   node_child           proj/src/svo.cpp:21-39
 *   shade                proj/src/renderer.cpp:102-113
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    uint32_t child_base, attr_base;
    uint8_t valid, leaf, pad[2];
} vo_node; /* the 12-byte SvoNode record */

typedef struct {
    const vo_node* nodes;
    const uint8_t* attrs; /* RGBA8 */
    uint32_t depth;
} vo_model;

typedef struct {
    int32_t id;
    int32_t model; /* index into the model table, -1: none */
    double R[9], t[3], s[3];
} vo_object;

typedef struct {
    double pos[3], C[9], fov_deg;
    int32_t width, height;
    uint8_t background[3];
} vo_camera;

/* per-pixel output: the vxa_pixel_aov layout (48 bytes) */
typedef struct {
    double t;
    int32_t object_id;
    uint32_t node_index, attr_index, voxel[3];
    uint8_t level, kind, entry_axis, pad0;
    uint32_t traversals, node_fetches, pad1;
} vo_aov;

static double vmax(double a, double b) { return a < b ? b : a; } /* std::max(a, b) */
static double vmin(double a, double b) { return b < a ? b : a; } /* std::min(a, b) */

/* node_child: popcount rank (svo.cpp:21-39). Returns 0 absent, 1 node, 2 leaf. */
static int node_child(const vo_model* m, uint32_t node, unsigned oct, uint32_t* index) {
    const vo_node* n = &m->nodes[node];
    const unsigned bit = 1u << oct;
    if (!(n->valid & bit)) return 0;
    if (n->leaf & bit) {
        *index = n->attr_base + (uint32_t)__builtin_popcount((n->valid & n->leaf) & (bit - 1u));
        return 2;
    }
    *index = n->child_base + (uint32_t)__builtin_popcount((n->valid & ~n->leaf & 0xffu) & (bit - 1u));
    return 1;
}

typedef struct {
    double t_hit;
    int axis, path_len;
    uint8_t path[16];
    uint32_t attr, parent, fetches;
} vo_hit;

static double zero_plane(double plane, double o) { return plane > o ? INFINITY : -INFINITY; }

/* traverse_impl (traversal.cpp:115-245); returns 1 on a hit. */
static int traverse(const vo_model* m, const double o[3], const double d[3], const double h[3], vo_hit* out) {
    static const unsigned bitof[3] = {4u, 2u, 1u};
    double t0r[3], t1r[3], om[3];
    int zero[3];
    unsigned mirror = 0;
    for (int a = 0; a < 3; ++a) {
        const int mir = d[a] < 0.0;
        if (mir) mirror |= bitof[a];
        const double oa = mir ? -o[a] : o[a], da = mir ? -d[a] : d[a];
        om[a] = oa;
        zero[a] = d[a] == 0.0;
        if (da == 0.0) {
            t0r[a] = zero_plane(-h[a], oa);
            t1r[a] = zero_plane(h[a], oa);
        } else {
            t0r[a] = (-h[a] - oa) / da;
            t1r[a] = (h[a] - oa) / da;
        }
    }
    out->fetches = 0;
    {
        double te = t0r[0], tx = t1r[0];
        for (int a = 1; a < 3; ++a) te = vmax(te, t0r[a]), tx = vmin(tx, t1r[a]);
        if (te >= tx || tx < 0.0) return 0;
    }
    struct {
        uint32_t node;
        double t0[3], t1[3], c[3];
        unsigned cur;
    } st[16];
    uint8_t path[16] = {0};
    int sp = 0;
#define MID(f, a) (zero[a] ? zero_plane((f).c[a], om[a]) : 0.5 * ((f).t0[a] + (f).t1[a]))
    st[0].node = 0;
    for (int a = 0; a < 3; ++a) st[0].t0[a] = t0r[a], st[0].t1[a] = t1r[a], st[0].c[a] = 0.0;
    {
        double te = st[0].t0[0];
        if (st[0].t0[1] > te) te = st[0].t0[1];
        if (st[0].t0[2] > te) te = st[0].t0[2];
        st[0].cur = (MID(st[0], 0) < te ? 4u : 0u) | (MID(st[0], 1) < te ? 2u : 0u) | (MID(st[0], 2) < te ? 1u : 0u);
    }
    uint32_t fetches = 1;
    while (sp >= 0) {
        if (st[sp].cur == 8u) {
            --sp;
            continue;
        }
        const unsigned q = st[sp].cur;
        const int level = sp;
        double t0c[3], t1c[3], cc[3];
        for (int a = 0; a < 3; ++a) {
            const double tm = MID(st[sp], a);
            const double quarter = ldexp(h[a], -(level + 1));
            if (q & bitof[a]) {
                t0c[a] = tm, t1c[a] = st[sp].t1[a], cc[a] = st[sp].c[a] + quarter;
            } else {
                t0c[a] = st[sp].t0[a], t1c[a] = tm, cc[a] = st[sp].c[a] - quarter;
            }
        }
        { /* next_node */
            int ax = 0;
            double tx = t1c[0];
            if (t1c[1] < tx) ax = 1, tx = t1c[1];
            if (t1c[2] < tx) ax = 2;
            st[sp].cur = (q & bitof[ax]) ? 8u : (q | bitof[ax]);
        }
        int entry = 0;
        double te = t0c[0];
        if (t0c[1] > te) entry = 1, te = t0c[1];
        if (t0c[2] > te) entry = 2, te = t0c[2];
        const double tx = vmin(vmin(t1c[0], t1c[1]), t1c[2]);
        if (!(te < tx) || tx < 0.0) continue;
        const unsigned real = q ^ mirror;
        uint32_t idx = 0;
        const int kind = node_child(m, st[sp].node, real, &idx);
        if (kind == 0) continue;
        path[level] = (uint8_t)real;
        if (kind == 2) {
            out->t_hit = vmax(te, 0.0);
            out->axis = entry;
            out->path_len = level + 1;
            memcpy(out->path, path, sizeof(path));
            out->attr = idx;
            out->parent = st[sp].node;
            out->fetches = fetches;
            return 1;
        }
        if (level + 1 >= (int)m->depth || level + 1 >= 16) continue;
        ++sp;
        st[sp].node = idx;
        for (int a = 0; a < 3; ++a) st[sp].t0[a] = t0c[a], st[sp].t1[a] = t1c[a], st[sp].c[a] = cc[a];
        ++fetches;
        {
            double e = st[sp].t0[0];
            if (st[sp].t0[1] > e) e = st[sp].t0[1];
            if (st[sp].t0[2] > e) e = st[sp].t0[2];
            st[sp].cur = (MID(st[sp], 0) < e ? 4u : 0u) | (MID(st[sp], 1) < e ? 2u : 0u) | (MID(st[sp], 2) < e ? 1u : 0u);
        }
    }
#undef MID
    out->fetches = fetches;
    return 0;
}

typedef struct {
    int32_t id;
    int obj;
    double tc, tb;
} vo_cand;

static int cand_cmp_sorted(const void* x, const void* y) {
    const vo_cand* a = (const vo_cand*)x;
    const vo_cand* b = (const vo_cand*)y;
    if (a->tc != b->tc) return a->tc < b->tc ? -1 : 1;
    return (a->id > b->id) - (a->id < b->id);
}

static int cand_cmp_id(const void* x, const void* y) {
    const vo_cand* a = (const vo_cand*)x;
    const vo_cand* b = (const vo_cand*)y;
    return (a->id > b->id) - (a->id < b->id);
}

/*
 * Renders rows [row_begin, row_end) of the frame (no hit buffer): RGB8 into
 * rgb (3 bytes per pixel, rows relative to row_begin) and per-pixel AOVs.
 */
void vo_render(const vo_camera* cam, const vo_object* objs, int n_obj, const vo_model* models, int culling,
               int sorting, int row_begin, int row_end, uint8_t* rgb, vo_aov* aov) {
    const double tan_half = tan(cam->fov_deg * 3.14159265358979323846 / 360.0);
    const double aspect = (double)cam->width / cam->height;
    vo_cand* cand = (vo_cand*)malloc(sizeof(vo_cand) * (size_t)(n_obj > 0 ? n_obj : 1));
    double* sc = (double*)malloc(sizeof(double) * 4 * (size_t)(n_obj > 0 ? n_obj : 1));
    for (int i = 0; i < n_obj; ++i) { /* bounding spheres (scene.cpp:16-20) */
        const double* s = objs[i].s;
        sc[4 * i] = objs[i].t[0], sc[4 * i + 1] = objs[i].t[1], sc[4 * i + 2] = objs[i].t[2];
        sc[4 * i + 3] = 0.5 * sqrt(s[0] * s[0] + s[1] * s[1] + s[2] * s[2]);
    }
    for (int py = row_begin; py < row_end; ++py) {
        for (int px = 0; px < cam->width; ++px) {
            const double ndc_x = (px + 0.5) / cam->width * 2.0 - 1.0;
            const double ndc_y = 1.0 - (py + 0.5) / cam->height * 2.0;
            const double dc[3] = {ndc_x * tan_half * aspect, ndc_y * tan_half, -1.0};
            double w[3], d[3];
            for (int k = 0; k < 3; ++k) w[k] = cam->C[3 * k] * dc[0] + cam->C[3 * k + 1] * dc[1] + cam->C[3 * k + 2] * dc[2];
            const double len = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
            for (int k = 0; k < 3; ++k) d[k] = w[k] / len;
            const double* o = cam->pos;
            int nc = 0;
            for (int i = 0; i < n_obj; ++i) {
                const double l[3] = {sc[4 * i] - o[0], sc[4 * i + 1] - o[1], sc[4 * i + 2] - o[2]};
                const double tcen = l[0] * d[0] + l[1] * d[1] + l[2] * d[2];
                const double d2 = (l[0] * l[0] + l[1] * l[1] + l[2] * l[2]) - tcen * tcen;
                const double r = sc[4 * i + 3], r2 = r * r;
                const int hit = (culling || sorting) && !(d2 >= r2) && !(tcen + r < 0.0);
                if (culling && !hit) continue;
                vo_cand c = {objs[i].id, i, 0.0, 0.0};
                if (sorting) {
                    c.tc = tcen;
                    c.tb = hit ? vmax(tcen - sqrt(r2 - d2), 0.0) : 0.0;
                }
                cand[nc++] = c;
            }
            qsort(cand, (size_t)nc, sizeof(vo_cand), sorting ? cand_cmp_sorted : cand_cmp_id);
            int have = 0;
            double best_t = 0.0, best_n[3] = {0, 0, 0};
            int32_t best_id = -1;
            vo_hit bh;
            memset(&bh, 0, sizeof(bh));
            int best_obj = -1;
            uint32_t trav = 0, fetch = 0;
            for (int k = 0; k < nc; ++k) {
                if (have && best_t < cand[k].tb) continue; /* skip, do not break */
                const vo_object* ob = &objs[cand[k].obj];
                if (ob->model < 0) continue;
                double v[3], lo[3], ld[3], h[3];
                for (int a = 0; a < 3; ++a) v[a] = o[a] + -ob->t[a], h[a] = ob->s[a] * 0.5;
                for (int a = 0; a < 3; ++a) { /* R^T (o - t), R^T d */
                    lo[a] = ob->R[a] * v[0] + ob->R[3 + a] * v[1] + ob->R[6 + a] * v[2];
                    ld[a] = ob->R[a] * d[0] + ob->R[3 + a] * d[1] + ob->R[6 + a] * d[2];
                }
                ++trav;
                vo_hit hh;
                const int hit = traverse(&models[ob->model], lo, ld, h, &hh);
                fetch += hh.fetches;
                if (!hit) continue;
                if (!have || hh.t_hit < best_t || (hh.t_hit == best_t && ob->id < best_id)) {
                    have = 1;
                    best_t = hh.t_hit;
                    best_id = ob->id;
                    bh = hh;
                    best_obj = cand[k].obj;
                    double nl[3] = {0, 0, 0};
                    nl[hh.axis] = ld[hh.axis] > 0.0 ? -1.0 : 1.0;
                    for (int a = 0; a < 3; ++a)
                        best_n[a] = ob->R[3 * a] * nl[0] + ob->R[3 * a + 1] * nl[1] + ob->R[3 * a + 2] * nl[2];
                }
            }
            const size_t i = (size_t)(py - row_begin) * (size_t)cam->width + (size_t)px;
            uint8_t* pix = rgb + 3 * i;
            if (!have) {
                memcpy(pix, cam->background, 3);
            } else {
                const uint8_t* c = models[objs[best_obj].model].attrs + 4 * (size_t)bh.attr;
                const double facing = vmax(0.0, best_n[0] * -d[0] + best_n[1] * -d[1] + best_n[2] * -d[2]);
                const double f = 0.2 + 0.8 * facing;
                for (int k = 0; k < 3; ++k) pix[k] = (uint8_t)lround(c[k] * f);
            }
            vo_aov* a = &aov[i];
            memset(a, 0, sizeof(*a));
            a->object_id = have ? best_id : -1;
            a->t = have ? best_t : 0.0;
            a->kind = (uint8_t)(have ? (nc > 1 ? 2 : 1) : 0);
            a->traversals = trav;
            a->node_fetches = fetch;
            if (have) {
                a->node_index = bh.parent;
                a->attr_index = bh.attr;
                a->level = (uint8_t)bh.path_len;
                a->entry_axis = (uint8_t)bh.axis;
                for (int l = 0; l < bh.path_len; ++l) {
                    const unsigned oc = bh.path[l];
                    a->voxel[0] = (a->voxel[0] << 1) | ((oc >> 2) & 1u);
                    a->voxel[1] = (a->voxel[1] << 1) | ((oc >> 1) & 1u);
                    a->voxel[2] = (a->voxel[2] << 1) | (oc & 1u);
                }
            }
        }
    }
    free(cand);
    free(sc);
}
