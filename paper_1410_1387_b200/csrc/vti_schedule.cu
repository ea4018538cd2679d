// vti_schedule.cu -- host-side planning of the step launches (see vti_internal.h).
#include "vti_internal.h"

// ---- host-side planning (pure functions; exported for tests as vti_plan)
// Work items are (tile, z-chunk). Measured on B200: full z
// columns marching in lockstep keep the p apron re-reads in L2 and avoid the
// 2Rz-plane q priming of each chunk, and ~110 resident CTAs already saturate
// HBM (C2: 128 columns on 148 SMs beat 1024 chunks). The chunk count per
// launch minimises a wave cost, in units of one saturated plane-time: a round
// of a active CTAs costs the larger of its bandwidth time
//   zchunk * (1 + 8 Rz / (36 zchunk)) * a / min(a, SAT)   (q priming re-reads)
// and its latency time (zchunk + 2 Rz) * LAT (each item walks its stage loads
// in order; ~0.7 plane-times per dependent load, measured on C1 where 8 CTAs
// of 24 loads took 18.9 us). Small grids therefore get short chunks and many
// CTAs, large grids long columns.
static double sat_ctas(int ctas_per_sm)
{
    double sat = 110.0 * ctas_per_sm;
    if (const char *e = getenv("VTI_SAT")) sat = atof(e);
    return sat;
}

static double lat_planes()
{
    double lat = 0.7;
    if (const char *e = getenv("VTI_LAT")) lat = atof(e);
    return lat;
}

// HBM streaming efficiency falls when more than ~128 CTAs (per CTA-per-SM slot)
// stream at once: tools/stream_probe_bulk.cu moves the step's 7R+2W mix at 7.10
// TB/s with 110-128 CTAs but 6.90 TB/s with 148. eff(a) models that (0.97 at 148)
// for the fp32 kernels (C3 183 -> 190, C4 179 -> 191, C5 182 -> 187 Gpoints/s with
// a 128-CTA grid); the slower fp64 CTAs need the full grid to saturate HBM, so
// their plans keep it (measured: capping costs them 2-4 %).
static constexpr int CONC = 128;
static double conc_eff(long a, int ctas_per_sm)
{
    const double over = (double)a / ctas_per_sm - CONC;
    return over > 0 ? 1.0 - 0.0015 * over : 1.0;
}

struct Sched {
    int zchunk;   // planes per work item
    int cap;      // CTAs launched at most (<= slots)
};

static Sched plan_sched(int nz, int rz, int tiles, int slots, int ctas_per_sm, double sat, int tune_zchunk,
                        bool conc_model)
{
    if (tiles <= 0 || slots <= 0) return {nz, std::max(slots, 1)};
    sat = std::max(1.0, std::min(sat, (double)slots));
    const double lat = lat_planes();
    double best = 1e300;
    Sched out{tune_zchunk > 0 ? std::min(tune_zchunk, nz) : nz, slots};
    const int caps[2] = {slots, std::min(slots, CONC * ctas_per_sm)};
    for (int ci = 0; ci < (conc_model ? 2 : 1); ++ci) {
        const int cap = caps[ci];
        if (ci == 1 && cap == slots) break;
        for (int nzc = 1; nzc <= nz; ++nzc) {
            const int zc = (nz + nzc - 1) / nzc;
            if ((nz + zc - 1) / zc != nzc) continue;   // same chunking as a smaller nzc
            if (tune_zchunk > 0 && zc != std::min(tune_zchunk, nz)) continue;
            const long items = (long)tiles * nzc;
            const long full = items / cap, last = items % cap;
            const double prime = 1.0 + (8.0 * rz) / (36.0 * zc);
            const double lat_round = (zc + 2.0 * rz) * lat;
            auto round_cost = [&](long a) {
                const double eff = conc_model ? conc_eff(a, ctas_per_sm) : 1.0;
                return std::max(zc * prime * a / (std::min<double>(a, sat) * eff), lat_round);
            };
            double cost = (double)full * round_cost(cap);
            if (last) cost += round_cost(last);
            if (cost < best * (1.0 - 1e-3)) {
                best = cost;
                out = {zc, cap};
            }
        }
    }
    return out;
}

// nranks > 1: the edge launch covers every tile row that intersects the first
// or the last R_xy rows of the slab (the rows the neighbours receive), i.e.
// tile rows [0, e1) and [e2, nty); the interior launch covers [e1, e2).
static void plan_edge_rows(int nty, int r, int ty, int nyl, int &e1, int &e2)
{
    e1 = std::min(nty, (r + ty - 1) / ty);
    e2 = std::max(e1, std::min(nty, (nyl - r) / ty));
}

// CTA slots of a launch: resident CTAs, optionally capped (env VTI_MAXGRID, experiments)
int slots(const vti_s *h)
{
    static const int cap = getenv("VTI_MAXGRID") ? atoi(getenv("VTI_MAXGRID")) : 0;
    const int n = h->sms * h->ctas_per_sm;
    return cap > 0 ? std::min(n, cap) : n;
}

static Sched choose_sched(const vti_s *h, int tiles)
{
    return plan_sched(h->cfg.nz, h->RZ, tiles, slots(h), h->ctas_per_sm, sat_ctas(h->ctas_per_sm), h->tune_zchunk,
                      h->es == 4);
}

void edge_rows(const vti_s *h, int &e1, int &e2) { plan_edge_rows(h->nty, h->R, h->TY, h->nyl, e1, e2); }

// Default schedule: one launch over all tile rows (single slab), or an edge
// launch plus an interior launch (nranks > 1).
void choose_schedule(vti_s *h)
{
    int e1, e2;
    edge_rows(h, e1, e2);
    const int edge_rows = e1 + (h->nty - e2), inner_rows = e2 - e1;
    const Sched a = choose_sched(h, h->ntx * h->nty), e = choose_sched(h, h->ntx * edge_rows),
                i = choose_sched(h, h->ntx * inner_rows);
    h->zchunk = a.zchunk;
    h->cap = a.cap;
    h->zchunk_edge = e.zchunk;
    h->cap_edge = e.cap;
    h->zchunk_inner = i.zchunk;
    h->cap_inner = i.cap;
    h->nzc = (h->cfg.nz + h->zchunk - 1) / h->zchunk;
    const long items = (long)h->ntx * h->nty * h->nzc;
    h->grid = (int)std::min<long>(items, (long)h->cap);
}

int precision_bits(const vti_config *c) { return c->precision == 0 ? 32 : c->precision; }

vti_status check_cfg(const vti_config *c)
{
    if (!c) return VTI_E_PARAM;
    if (c->r_xy < 1 || c->r_z < 1 || c->r_xy > MAX_R || !(c->h > 0) || !(c->dt > 0) || c->damp_width < 0)
        return VTI_E_PARAM;
    if (precision_bits(c) != 32 && precision_bits(c) != 64) return VTI_E_PARAM;
    if (c->nx < 1 || c->ny < 1 || c->nz < 1) return VTI_E_GEOMETRY;
    if (c->nz < 2 * c->r_z + 1) return VTI_E_GEOMETRY;   // too few planes
    if (c->damp_width > 0 && (2 * c->damp_width >= c->nx || 2 * c->damp_width >= c->ny || 2 * c->damp_width >= c->nz))
        return VTI_E_GEOMETRY;
    if (c->nranks < 1 || c->rank < 0 || c->rank >= c->nranks) return VTI_E_PARAM;
    if (c->nranks > 1 && c->ny / c->nranks < c->r_xy) return VTI_E_GEOMETRY;   // slab thinner than the halo
    return VTI_OK;
}

extern "C" {

vti_status vti_slab(const vti_config *cfg, int32_t *y0, int32_t *ny_local)
{
    if (!cfg || !y0 || !ny_local || cfg->nranks < 1 || cfg->rank < 0 || cfg->rank >= cfg->nranks || cfg->ny < 1)
        return VTI_E_PARAM;
    const int base = cfg->ny / cfg->nranks, extra = cfg->ny % cfg->nranks;
    *ny_local = base + (cfg->rank < extra ? 1 : 0);
    *y0 = cfg->rank * base + std::min(cfg->rank, extra);
    return VTI_OK;
}

vti_status vti_plan(const vti_config *cfg, int32_t tile_y, int32_t sms, int32_t ctas_per_sm, vti_plan_info *out)
{
    if (!cfg || !out || tile_y < 1 || sms < 1 || ctas_per_sm < 1) return VTI_E_PARAM;
    vti_status st = check_cfg(cfg);
    if (st != VTI_OK) return st;
    vti_slab(cfg, &out->y0, &out->ny_local);
    out->ntx = (cfg->nx + TX - 1) / TX;
    out->nty = (out->ny_local + tile_y - 1) / tile_y;
    int e1, e2;
    plan_edge_rows(out->nty, cfg->r_xy, tile_y, out->ny_local, e1, e2);
    out->edge_lo = e1;
    out->edge_hi = e2;
    const int slots = sms * ctas_per_sm;
    const double sat = sat_ctas(ctas_per_sm);
    const bool f32 = precision_bits(cfg) == 32;
    const Sched a = plan_sched(cfg->nz, cfg->r_z, out->ntx * out->nty, slots, ctas_per_sm, sat, 0, f32);
    out->zchunk = a.zchunk;
    out->zchunk_edge =
        plan_sched(cfg->nz, cfg->r_z, out->ntx * (e1 + out->nty - e2), slots, ctas_per_sm, sat, 0, f32).zchunk;
    out->zchunk_inner = plan_sched(cfg->nz, cfg->r_z, out->ntx * (e2 - e1), slots, ctas_per_sm, sat, 0, f32).zchunk;
    const long items = (long)out->ntx * out->nty * ((cfg->nz + out->zchunk - 1) / out->zchunk);
    out->items = (int32_t)items;
    out->grid = (int32_t)std::min<long>(items, a.cap);
    return VTI_OK;
}

}  // extern "C"
