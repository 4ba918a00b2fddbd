// mpfd_b200_run -- `mpfd run <config>` (tools/mpfd.cpp:23-26, runner.cpp:69-88)
// on the B200 path, through the C++ adapter (include/mpfd_b200.hpp).
//
// Reads the reference's `key = value` config (config.cpp:120-235, the keys
// of the hot path), runs init + advance on cuda:0 and writes the
// diagnostics CSV in the reference format (io.cpp:19-36, %.17g), so the two
// CSVs can be compared byte for byte.  Exit codes as the reference CLI:
// 0 completed, 1 configuration error, 2 diverged.
//
//   g++ -O2 -std=c++17 -Iinclude tools/mpfd_b200_run.cpp
//       -Lpaper_2505_20911_b200 -lmpfd_b200 -Wl,-rpath,$PWD/paper_2505_20911_b200
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>

#include "mpfd_b200.hpp"

namespace {

std::string trim(const std::string& s) {
    const auto b = s.find_first_not_of(" \t\r");
    if (b == std::string::npos) return "";
    return s.substr(b, s.find_last_not_of(" \t\r") - b + 1);
}

struct Cfg {
    std::string case_kind = "tgv", precision = "DP", emulation = "strict", split = "Blaisdell";
    std::string strategy = "default", output = "diagnostics.csv", ke = "plain";
    int n = 32, threads = 1, diag_interval = -1;
    double M = 0.5, Re = 800.0, Pr = 0.72, gamma = 1.4, dt = 0.005, t_end = 20.0;
    long n_iter = -1;
    bool viscous = true;
    std::map<std::string, std::string> custom;  // precision.custom.<name>
};

Cfg load(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw mpfd_b200::ConfigError("cannot open config file: " + path);
    Cfg c;
    bool saw_t = false;
    std::string line;
    int ln = 0;
    while (std::getline(in, line)) {
        ++ln;
        const auto h = line.find('#');
        if (h != std::string::npos) line = line.substr(0, h);
        line = trim(line);
        if (line.empty()) continue;
        const auto eq = line.find('=');
        if (eq == std::string::npos)
            throw mpfd_b200::ConfigError("line " + std::to_string(ln) + ": expected 'key = value'");
        const std::string k = trim(line.substr(0, eq)), v = trim(line.substr(eq + 1));
        if (k == "case") c.case_kind = v;
        else if (k == "n") c.n = std::stoi(v);
        else if (k == "M") c.M = std::stod(v);
        else if (k == "Re") c.Re = std::stod(v);
        else if (k == "Pr") c.Pr = std::stod(v);
        else if (k == "gamma") c.gamma = std::stod(v);
        else if (k == "viscous") c.viscous = (v == "true" || v == "1");
        else if (k == "dt") c.dt = std::stod(v);
        else if (k == "t_end") { c.t_end = std::stod(v); saw_t = true; }
        else if (k == "n_iterations") c.n_iter = std::lround(std::stod(v));
        else if (k == "precision") c.precision = v;
        else if (k == "emulation") c.emulation = v;
        else if (k == "split") c.split = v;
        else if (k == "strategy") c.strategy = v;
        else if (k == "ke_weighting") c.ke = v;
        else if (k == "diagnostics_interval") c.diag_interval = std::stoi(v);
        else if (k == "output") c.output = v;
        else if (k == "threads") c.threads = std::stoi(v);
        else if (k.rfind("precision.custom.", 0) == 0) c.custom[k.substr(17)] = v;
        else throw mpfd_b200::ConfigError("line " + std::to_string(ln) + ": unknown key '" + k + "'");
    }
    // finalize_sim (config.cpp:217-235)
    if (c.n_iter >= 0 && !saw_t) c.t_end = c.n_iter * c.dt;
    if (c.n_iter < 0) c.n_iter = std::lround(c.t_end / c.dt);
    if (c.diag_interval < 0) c.diag_interval = (int)std::max(1l, std::lround(0.5 / c.dt));
    return c;
}

void g17(std::string& out, double v) {
    char b[32];
    std::snprintf(b, sizeof b, "%.17g", v);
    out += b;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc != 3 || std::string(argv[1]) != "run") {
        std::cerr << "usage: mpfd_b200_run run <config>\n";
        return 1;
    }
    try {
        const Cfg c = load(argv[2]);
        mpfd_precision p = mpfd_b200::resolve_preset(c.precision.c_str());
        p.emulation = c.emulation == "storeround" ? MPFD_STOREROUND : MPFD_STRICT;
        std::vector<std::string> names;
        std::vector<const char*> np;
        std::vector<int> kinds;
        for (const auto& kv : c.custom) {
            names.push_back(kv.first);
            kinds.push_back(kv.second == "B16" ? MPFD_B16 : kv.second == "B32" ? MPFD_B32 : MPFD_B64);
        }
        for (const auto& s : names) np.push_back(s.c_str());
        p.n_overrides = (int)names.size();
        p.override_names = np.data();
        p.override_kinds = kinds.data();
        const mpfd_flow flow{c.M, c.Re, c.Pr, c.gamma, c.viscous ? 1 : 0};
        mpfd_b200::Solver s(c.n, p, c.strategy == "storesome" ? MPFD_STORESOME : MPFD_DEFAULT, flow,
                            mpfd_b200::split_preset(c.split.c_str()));
        if (c.case_kind == "tgv") s.init_tgv();
        else s.init_uniform();
        mpfd_step st = mpfd_b200::default_step(c.dt, c.n_iter, c.diag_interval);
        st.ke_weighting = c.ke == "density" ? MPFD_KE_DENSITY : MPFD_KE_PLAIN;
        st.threads = c.threads;
        const auto r = s.advance(st);
        std::string csv = "t,kinetic_energy,enstrophy,solenoidal_dissipation,ke_normalized,diverged\n";
        for (const auto& d : r.series) {
            g17(csv, d.t);
            csv += ',';
            g17(csv, d.kinetic_energy);
            csv += ',';
            g17(csv, d.enstrophy);
            csv += ',';
            g17(csv, d.eps_s);
            csv += ',';
            g17(csv, d.ke_normalized);
            csv += d.diverged ? ",1\n" : ",0\n";
        }
        std::ofstream(c.output, std::ios::binary) << csv;
        std::cout << "wrote " << c.output << " (" << r.series.size() << " samples)\n";
        if (r.diverged) {
            const auto& e = *r.divergence;
            std::cout << "DIVERGED at t = " << e.time << " (iteration " << e.iteration << ", substep "
                      << e.substep << "): " << e.what << " first at (" << e.i << "," << e.j << "," << e.k
                      << ")\n";
            return 2;
        }
        return 0;
    } catch (const mpfd_b200::ConfigError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 3;
    }
}
