// planner.cpp -- host-only refinement planner helpers of the C-ABI (include/dem.h).
// Pure functions of the paper's planning formulas: Eq. 1, Eq. 8,
// Eq. 9, Eq. 10; layer aggressiveness gamma(r, eta) = (r-1)/(r eta).
#include <cmath>

#include "../../include/dem.h"

extern "C" {

double dem_profile_diameter(double d_min, double d_max, double gamma, double depth)
{
    if (!(gamma > 0.0)) return d_min;
    const double z_max = (d_max - d_min) / gamma;
    return depth < z_max ? d_min + gamma * depth : d_max;
}

double dem_contact_network_length(double d_min, double d_max, double r, double eta, double h)
{
    if (!(d_max > d_min) || !(r > 1.0)) return h / d_max;           // uniform bed: n_d = h/d
    const double gamma = (r - 1.0) / (r * eta);
    const double z_max = (d_max - d_min) / gamma;
    const double layers = eta * std::log(d_max / d_min) / std::log(r);
    return h >= z_max ? layers + (h - z_max) / d_max : layers * h / z_max;   // h < z_max: truncated
}

int32_t dem_plan_iterations(double n_d, double eps)
{
    if (!(eps > 0.0) || !(n_d > 0.0)) return 1;
    const double v = std::ceil(0.1 * n_d / eps - 1e-9);
    return v < 1.0 ? 1 : (int32_t)v;
}

double dem_plan_timestep(double d, double eps, double rho, double sigma)
{
    const double a = 3.0 * sigma / (2.0 * rho * d);                   // a ~ sigma A / m
    return 0.5 * std::sqrt(eps * d / a);
}

}  // extern "C"
