// mpfd_b200_run -- the reference CLI's `run`, `compare` and `sweep` commands
// (tools/mpfd.cpp:23-52; runner.cpp:69-173) and `report` on the B200 path, through
// the C++ adapter (include/mpfd_b200.hpp).
//
// Reads the reference's `key = value` config (config.cpp:120-235, the keys
// of the hot path), runs init + advance on cuda:0 and writes the
// diagnostics CSV in the reference format (io.cpp:19-36, %.17g), so the two
// CSVs can be compared byte for byte.  `compare a.csv b.csv` is
// compare_series (tgv.cpp:177-197) with the reference's output format;
// `sweep <spec>` is run_sweep: DP reference plus each preset over the dt x M
// grid, mean |delta eps_S| matrix.  Exit codes as the reference CLI:
// 0 completed, 1 configuration or comparison error, 2 diverged.
//
//   g++ -O2 -std=c++17 -Iinclude tools/mpfd_b200_run.cpp
//       -Lpaper_2505_20911_b200 -lmpfd_b200 -Wl,-rpath,$PWD/paper_2505_20911_b200
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <map>
#include <stdexcept>
#include <vector>
#include <algorithm>
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
    // sweep spec (config.cpp:259-282)
    std::vector<double> sweep_dt, sweep_M;
    std::vector<std::string> sweep_presets;
    std::string sweep_output;
    bool saw_t_end = false;
    // report (config.cpp:190-205)
    int procs[3] = {4, 1, 1};  // SimConfig default (config.hpp:33)
    std::vector<double> snap_times;
    std::string snap_path = "snapshot.bin";
    double comm[4] = {-1, -1, -1, -1};  // comm.q_vector / rk_arrays / residuals / wk_arrays
};

std::vector<std::string> split_list(const std::string& key, const std::string& v, int ln) {
    std::vector<std::string> out;
    std::string item;
    std::istringstream in(v);
    while (std::getline(in, item, ',')) {
        item = trim(item);
        if (!item.empty()) out.push_back(item);
    }
    if (out.empty())
        throw mpfd_b200::ConfigError("line " + std::to_string(ln) + ": field '" + key +
                                     "' expects a comma-separated list");
    return out;
}

Cfg load(const std::string& path, bool sweep = false) {
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
        else if (sweep && k == "sweep.dt") { for (auto& x : split_list(k, v, ln)) c.sweep_dt.push_back(std::stod(x)); }
        else if (sweep && k == "sweep.M") { for (auto& x : split_list(k, v, ln)) c.sweep_M.push_back(std::stod(x)); }
        else if (sweep && k == "sweep.presets") {
            c.sweep_presets = split_list(k, v, ln);
            for (const auto& pr : c.sweep_presets) mpfd_b200::resolve_preset(pr.c_str());  // validate
        }
        else if (sweep && k == "sweep.output") c.sweep_output = v;
        else if (k == "procs") {
            const auto l = split_list(k, v, ln);
            if (l.size() != 3)
                throw mpfd_b200::ConfigError("line " + std::to_string(ln) + ": field 'procs': expected px,py,pz");
            for (int i = 0; i < 3; ++i) c.procs[i] = std::stoi(l[i]);
        }
        else if (k == "comm.q_vector") c.comm[0] = std::stod(v);
        else if (k == "comm.rk_arrays") c.comm[1] = std::stod(v);
        else if (k == "comm.residuals") c.comm[2] = std::stod(v);
        else if (k == "comm.wk_arrays") c.comm[3] = std::stod(v);
        else if (k == "snapshot_times") { for (auto& x : split_list(k, v, ln)) c.snap_times.push_back(std::stod(x)); }
        else if (k == "snapshot_path") c.snap_path = v;
        else throw mpfd_b200::ConfigError("line " + std::to_string(ln) + ": unknown key '" + k + "'");
    }
    if (sweep && c.sweep_presets.empty()) throw mpfd_b200::ConfigError("sweep spec: missing 'sweep.presets'");
    c.saw_t_end = saw_t;
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

struct Run {
    std::vector<mpfd_diag> series;
    bool diverged = false;
    mpfd_b200::AdvanceResult raw;
};

// the resolved PrecisionConfig of a config (preset + per-name overrides)
struct Prec {
    mpfd_precision p;
    std::vector<std::string> names;
    std::vector<const char*> np;
    std::vector<int> kinds;
    explicit Prec(const Cfg& c) {
        p = mpfd_b200::resolve_preset(c.precision.c_str());
        p.emulation = c.emulation == "storeround" ? MPFD_STOREROUND : MPFD_STRICT;
        for (const auto& kv : c.custom) {
            names.push_back(kv.first);
            kinds.push_back(kv.second == "B16" ? MPFD_B16 : kv.second == "B32" ? MPFD_B32 : MPFD_B64);
        }
        for (const auto& s : names) np.push_back(s.c_str());
        p.n_overrides = (int)names.size();
        p.override_names = np.data();
        p.override_kinds = kinds.data();
    }
};

// run_simulation (runner.cpp:11-48) on cuda:0
Run run_cfg(const Cfg& c) {
    const Prec pr(c);
    const mpfd_precision& p = pr.p;
    const mpfd_flow flow{c.M, c.Re, c.Pr, c.gamma, c.viscous ? 1 : 0};
    mpfd_b200::Solver s(c.n, p, c.strategy == "storesome" ? MPFD_STORESOME : MPFD_DEFAULT, flow,
                        mpfd_b200::split_preset(c.split.c_str()));
    if (c.case_kind == "tgv") s.init_tgv();
    else s.init_uniform();
    mpfd_step st = mpfd_b200::default_step(c.dt, c.n_iter, c.diag_interval);
    st.ke_weighting = c.ke == "density" ? MPFD_KE_DENSITY : MPFD_KE_PLAIN;
    st.threads = c.threads;
    if (!c.snap_times.empty()) s.set_snapshots(c.snap_times, c.snap_path.c_str());
    Run r;
    r.raw = s.advance(st);
    r.series = r.raw.series;
    r.diverged = r.raw.diverged;
    return r;
}

int cmd_run(const char* path) {
    const Cfg c = load(path);
    const Run run = run_cfg(c);
    const auto& r = run.raw;
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
}

// read_diagnostics_csv (io.cpp:46-67)
struct Rec {
    double t, ke, ens, eps, ken;
    int div;
};
std::vector<Rec> read_csv(const std::string& path) {
    std::ifstream f(path);
    if (!f) throw std::runtime_error("cannot open: " + path);
    std::string line;
    if (!std::getline(f, line)) throw std::runtime_error("empty CSV: " + path);
    if (line.rfind("t,kinetic_energy", 0) != 0) throw std::runtime_error("unexpected CSV header in " + path);
    std::vector<Rec> out;
    int ln = 1;
    while (std::getline(f, line)) {
        ++ln;
        if (line.empty()) continue;
        Rec r;
        if (std::sscanf(line.c_str(), "%lf,%lf,%lf,%lf,%lf,%d", &r.t, &r.ke, &r.ens, &r.eps, &r.ken, &r.div) != 6)
            throw std::runtime_error(path + ": malformed CSV row at line " + std::to_string(ln));
        out.push_back(r);
    }
    return out;
}

// pairwise_sum (reduce.cpp:14-22), leaf 32
double pairwise_sum(const double* v, size_t n) {
    if (n <= 32) {
        double s = 0.0;
        for (size_t i = 0; i < n; ++i) s += v[i];
        return s;
    }
    const size_t h = n / 2;
    return pairwise_sum(v, h) + pairwise_sum(v + h, n - h);
}

// compare_series (tgv.cpp:177-197): candidate vs reference eps_S
struct Cmp {
    std::vector<double> t, d;
    double mean = 0.0, max = 0.0;
};
Cmp compare(const std::vector<double>& ta, const std::vector<double>& ea, const std::vector<double>& tb,
            const std::vector<double>& eb) {
    if (ta.size() != tb.size())
        throw std::runtime_error("sample counts differ (" + std::to_string(ta.size()) + " vs " +
                                 std::to_string(tb.size()) + ")");
    Cmp c;
    for (size_t i = 0; i < ta.size(); ++i) {
        if (ta[i] != tb[i]) throw std::runtime_error("sample grids differ at index " + std::to_string(i));
        c.t.push_back(ta[i]);
        c.d.push_back(std::abs(ea[i] - eb[i]));
    }
    if (!c.d.empty()) {
        c.mean = pairwise_sum(c.d.data(), c.d.size()) / (double)c.d.size();
        for (double x : c.d) c.max = std::max(c.max, x);
    }
    return c;
}

int cmd_compare(const char* a, const char* b) {
    const auto A = read_csv(a), B = read_csv(b);
    std::vector<double> ta, ea, tb, eb;
    for (const auto& r : A) ta.push_back(r.t), ea.push_back(r.eps);
    for (const auto& r : B) tb.push_back(r.t), eb.push_back(r.eps);
    const Cmp c = compare(ta, ea, tb, eb);
    std::printf("t,abs_diff_eps_s\n");
    for (size_t i = 0; i < c.t.size(); ++i) std::printf("%.17g,%.17g\n", c.t[i], c.d[i]);
    std::printf("mean_abs_diff=%.17g\n", c.mean);
    std::printf("max_abs_diff=%.17g\n", c.max);
    return 0;
}

// run_sweep (runner.cpp:108-173)
int cmd_sweep(const char* path) {
    const Cfg spec = load(path, true);
    const std::vector<double> dts = spec.sweep_dt.empty() ? std::vector<double>{spec.dt} : spec.sweep_dt;
    const std::vector<double> machs = spec.sweep_M.empty() ? std::vector<double>{spec.M} : spec.sweep_M;
    std::string csv = "dt,M";
    for (const auto& p : spec.sweep_presets) csv += "," + p;
    csv += "\n";
    for (double dt : dts) {
        for (double mach : machs) {
            Cfg cell = spec;
            cell.dt = dt;
            cell.M = mach;
            cell.n_iter = std::lround(cell.t_end / dt);
            cell.diag_interval = (int)std::max(1l, std::lround(0.5 / dt));
            Cfg ref = cell;
            ref.precision = "DP";
            ref.custom.clear();
            std::cout << "sweep: DP reference at dt=" << dt << " M=" << mach << "\n";
            const Run rr = run_cfg(ref);
            char num[32];
            std::snprintf(num, sizeof num, "%.17g", dt);
            csv += num;
            std::snprintf(num, sizeof num, ",%.17g", mach);
            csv += num;
            for (const auto& preset : spec.sweep_presets) {
                Cfg cand = cell;
                cand.precision = preset;
                cand.custom.clear();
                std::cout << "sweep: " << preset << " at dt=" << dt << " M=" << mach << "\n";
                const Run cr = run_cfg(cand);
                if (cr.diverged || rr.diverged) {
                    csv += ",inf";
                    continue;
                }
                std::vector<double> ta, ea, tb, eb;
                for (const auto& d : cr.series) ta.push_back(d.t), ea.push_back(d.eps_s);
                for (const auto& d : rr.series) tb.push_back(d.t), eb.push_back(d.eps_s);
                std::snprintf(num, sizeof num, ",%.17g", compare(ta, ea, tb, eb).mean);
                csv += num;
            }
            csv += "\n";
        }
    }
    if (!spec.sweep_output.empty()) {
        std::ofstream f(spec.sweep_output, std::ios::binary);
        if (!f) throw std::runtime_error("cannot open for writing: " + spec.sweep_output);
        f << csv;
    }
    std::cout << csv;
    if (!spec.sweep_output.empty()) std::cout << "wrote " << spec.sweep_output << "\n";
    return 0;
}

// print_report (runner.cpp:90-106): the analytic memory census of
// make_solver_fields' set (physics.cpp:441-475, memory_report registry.cpp:24-39)
// and the modelled halo volume (comm_volume_report registry.cpp:41-66) with
// the exchange counts of config.cpp:9-17; no run
int cmd_report(const char* path) {
    const Cfg c = load(path);
    const Prec pr(c);
    struct F {
        const char* name;
        int cls;
    };
    std::vector<F> fields;
    static const char* qn[5] = {"rho", "rhou", "rhov", "rhow", "rhoE"};
    static const char* tn[5] = {"rk_rho", "rk_rhou", "rk_rhov", "rk_rhow", "rk_rhoE"};
    static const char* rn[5] = {"res_rho", "res_rhou", "res_rhov", "res_rhow", "res_rhoE"};
    static const char* wn[5] = {"u", "v", "w", "p", "T"};
    static const char* gn[12] = {"dudx", "dudy", "dudz", "dvdx", "dvdy", "dvdz",
                                 "dwdx", "dwdy", "dwdz", "dTdx", "dTdy", "dTdz"};
    for (auto n : qn) fields.push_back({n, 0});
    for (auto n : tn) fields.push_back({n, 1});
    for (auto n : rn) fields.push_back({n, 2});
    for (auto n : wn) fields.push_back({n, 3});
    if (c.strategy != "storesome")
        for (auto n : gn) fields.push_back({n, 3});
    const size_t ext = (size_t)c.n + 8, pts = ext * ext * ext;
    size_t cnt[5] = {0}, bytes[5] = {0}, total = 0, base = 0;
    std::vector<int> kinds;
    for (const auto& f : fields) {
        int k = 2;
        if (mpfd_b200_field_kind(&pr.p, f.cls, f.name, &k)) throw mpfd_b200::ConfigError(mpfd_b200_last_error());
        kinds.push_back(k);
        const size_t b = pts * (k == 0 ? 2 : k == 1 ? 4 : 8);
        ++cnt[f.cls];
        bytes[f.cls] += b;
        total += b;
        base += pts * 8;
    }
    static const char* names[5] = {"q_vector", "rk_arrays", "residuals", "wk_arrays", "diagnostics"};
    std::cout << "memory census (analytic, halos included):\n";
    for (int k = 0; k < 5; ++k) {
        if (cnt[k] == 0) continue;
        std::cout << "  " << names[k] << ": " << cnt[k] << " fields, " << bytes[k] << " bytes\n";
    }
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.4f", total == 0 ? 1.0 : (double)base / (double)total);
    std::cout << "  total: " << total << " bytes (all-B64 baseline " << base << " bytes, gain " << buf << "x)\n";
    // exchange counts (config.cpp:9-17) and the face model, depth 2
    const double counts[5] = {c.comm[0] >= 0 ? c.comm[0] : 3.0, c.comm[1] >= 0 ? c.comm[1] : 0.0,
                              c.comm[2] >= 0 ? c.comm[2] : 0.0,
                              c.comm[3] >= 0 ? c.comm[3] : (c.strategy != "storesome" ? 3.0 : 0.0), 0.0};
    const int px = c.procs[0], py = c.procs[1], pz = c.procs[2];
    double per[5] = {0}, tot = 0.0;
    for (size_t i = 0; i < fields.size(); ++i) {
        const int n = c.n;
        if (px < 1 || py < 1 || pz < 1) throw mpfd_b200::ConfigError("process grid dimensions must be >= 1");
        if (n % px != 0 || n % py != 0 || n % pz != 0)
            throw mpfd_b200::ConfigError("grid n=" + std::to_string(n) + " is not divisible by the process grid");
        const double lx = (double)n / px, ly = (double)n / py, lz = (double)n / pz;
        double faces = 0.0;
        if (px > 1) faces += ly * lz;
        if (py > 1) faces += lx * lz;
        if (pz > 1) faces += lx * ly;
        const int k = kinds[i];
        const double vol = 2.0 * 2 * faces * (k == 0 ? 2 : k == 1 ? 4 : 8) * counts[fields[i].cls];
        per[fields[i].cls] += vol;
        tot += vol;
    }
    std::cout << "modeled halo-exchange volume per process per iteration (procs " << px << "x" << py << "x" << pz
              << "):\n";
    for (int k = 0; k < 5; ++k) {
        if (per[k] == 0.0) continue;
        std::cout << "  " << names[k] << ": " << per[k] << " bytes\n";
    }
    std::cout << "  total: " << tot << " bytes\n";
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    const std::string cmd = argc > 1 ? argv[1] : "";
    try {
        if (cmd == "run" && argc == 3) return cmd_run(argv[2]);
        if (cmd == "compare" && argc == 4) return cmd_compare(argv[2], argv[3]);
        if (cmd == "sweep" && argc == 3) return cmd_sweep(argv[2]);
        if (cmd == "report" && argc == 3) return cmd_report(argv[2]);
        std::cerr << "usage:\n  mpfd_b200_run run <config>\n  mpfd_b200_run compare <a.csv> <b.csv>\n"
                     "  mpfd_b200_run sweep <spec>\n  mpfd_b200_run report <config>\n";
        return 1;
    } catch (const mpfd_b200::ConfigError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    } catch (const mpfd_b200::DeviceError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 3;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
