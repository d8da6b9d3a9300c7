// Host-side math of the engine (fp64, compiled with -ffp-contract=off so every
// product rounds as the reference's does, proj/CMakeLists.txt:16): spread tables,
// per-env wind factors, the fuel palette, and the synthetic-input generators.
#pragma once
#include <cstddef>
#include <cstdint>

namespace ebl {

struct Cfg6 {
  double p_base, alpha_w1, alpha_w2, alpha_s, alpha_gamma, p_continue;
};

double wrap_angle(double a);     // grid.cpp:37-42
double offset_angle(int k);      // grid.cpp:44-47
// kappa_wind for the 8 offsets (kernel.hpp:21-26); direction is wrapped first
// as WindField construction does (grid.cpp:57-60).
void kappa_wind8(double speed, double direction, const Cfg6& c, double kw[8]);
// SpreadTables<double> (engine.hpp:79-110) of n cells; OpenMP over cells.
void build_tables(size_t n, const double* speed, const double* dir, const double* veg,
                  const double* den, const double* slope8, const Cfg6& c, double* pot,
                  double* gamma);
// Per-cell derivative factors of pot for the deterministic adjoint on general layers:
// F = (1+veg)(1+den), pb[k] = dpot/dp_base = F kw ks, V, Va[k] = V (cos(phi_k - dir) - 1), S[k].
void build_det_factors(size_t n, const double* speed, const double* dir, const double* veg,
                       const double* den, const double* slope8, const Cfg6& c, double* F,
                       double* pb, double* V, double* Va, double* S);
// SpreadTables<double> of terrain-form statics (slope_from_dem of the fp32 elevation, palette
// fuel, uniform wind per table): pot [n_tables][h*w][8], gamma [n_tables][h*w].  Table t uses
// grid t*grid_stride (stride 0: shared) and wind t*wind_stride.
void build_terrain_tables(int n_tables, int h, int w, const uint8_t* fuel, const float* elev,
                          size_t grid_stride, const double* class_veg, const double* class_den,
                          double cellsize, const double* wind_speed, const double* wind_dir,
                          int wind_stride, const Cfg6& c, double* pot, double* gamma);
// The config-free part of build_terrain_tables: S[g][cell][k] = atan(dz / dist) of every grid (0
// toward out-of-bounds or nodata neighbours), the value whose exp(alpha_s S) the table holds.
void build_terrain_slopes64(int n_grids, int h, int w, const float* elev, size_t grid_stride, double cellsize,
                            double* S);
// ceil(p_continue * 2^53): a Burning cell survives iff (word >> 11) < this.
uint64_t continue_threshold(double p_continue);

double clamp_fuel(double v);  // FuelField clamp to [-1, 1] (grid.cpp:75-76)

// Synthetic inputs.
void synth_terrain(uint64_t seed, uint32_t env_id0, int n_envs, int h, int w, double elev_max,
                   double wind_max, uint8_t* fuel_class, float* elevation, double* wind_speed,
                   double* wind_direction);
void worldcover_palette(int32_t* codes, double* veg, double* den);
int synth_ignitions(uint64_t seed, uint32_t env_id0, int n_envs, int h, int w,
                    const uint8_t* fuel_class, const double* class_veg, const double* class_den,
                    int count, uint8_t* states);

uint64_t rng_word(uint64_t seed, uint64_t step, uint64_t stream, uint64_t cell, uint64_t draw);
double rng_uniform(uint64_t seed, uint64_t step, uint64_t stream, uint64_t cell, uint64_t draw);
uint64_t rng_below(uint64_t seed, uint64_t step, uint64_t stream, uint64_t cell, uint64_t draw,
                   uint64_t n);

}  // namespace ebl
