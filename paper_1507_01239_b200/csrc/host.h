// Host-side determinism and data plumbing of the trainer, restated from the
// reference semantics (bit-exact for every integer/index stream):
//   Rng              rng.cpp:11-77, rng.hpp:35-41 (xoshiro256** / splitmix64)
//   shuffles/shards  data.cpp:162-168, parallel.cpp:61-77, data.cpp:185-203
//   synthetic data   data.cpp:124-160, 170-183, 205-242
//   init             network.cpp:40-60
//   LR schedules     optimizer.cpp:159-208
//   checkpoints      network.cpp:291-369 (PARNNET1)
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace pnb {
namespace host {

// A double as the reference's error messages print it (operator<< with the
// default stream format: 6 significant digits, "1.5", "1e-07", "nan" / "-nan").
std::string fmt_num(double v);

// xoshiro256** advances its 256-bit state linearly over GF(2); a Jump holds
// the columns of T^n so n draws can be skipped in O(256) word operations.
struct Jump {
    uint64_t col[256][4];
};
Jump make_jump(uint64_t n);
Jump jump_square(const Jump& j);  // T^2n from T^n

class Rng {
public:
    explicit Rng(uint64_t seed);
    uint64_t next_u64();
    double uniform();
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    uint64_t uniform_index(uint64_t bound);
    double gaussian(double mean, double stddev);
    void jump(const Jump& j);
    // the full generator state, for callers that carry a reference Rng across
    // the C ABI (the xoshiro256** words and the polar-method spare, rng.hpp)
    void get_state(uint64_t s[4], double* spare, bool* has_spare) const {
        for (int i = 0; i < 4; ++i) s[i] = s_[i];
        *spare = spare_;
        *has_spare = has_spare_;
    }
    void set_state(const uint64_t s[4], double spare, bool has_spare) {
        for (int i = 0; i < 4; ++i) s_[i] = s[i];
        spare_ = spare;
        has_spare_ = has_spare;
    }
    template <typename T>
    void shuffle(std::vector<T>& v) {
        for (size_t i = v.size(); i > 1; --i) {
            const size_t j = static_cast<size_t>(uniform_index(i));
            T t = v[i - 1];
            v[i - 1] = v[j];
            v[j] = t;
        }
    }

private:
    uint64_t s_[4];
    double spare_ = 0.0;
    bool has_spare_ = false;
};

std::vector<uint64_t> shuffled_indices(uint64_t n, uint64_t seed);
// m shards of floor(n/m) row ids each, shard-major.
std::vector<uint64_t> partition_rows(uint64_t n, uint64_t m, uint64_t seed);
// floor(n/b) batches of b positions into the shard, batch-major.
std::vector<uint64_t> minibatch_rows(uint64_t n, uint64_t b, uint64_t seed);

struct HostData {
    std::vector<double> x;
    std::vector<int32_t> y;
    uint64_t n = 0, d = 0;
};
HostData generate_synthetic(uint64_t classes, uint64_t dim, uint64_t per_class, double sep, uint64_t seed);
// load_csv / save_csv (data.cpp:66-122): 'label,f1,...' rows, '#' comments and
// blank lines skipped, errors naming the 1-based line; parsed on all host threads
HostData load_csv(const std::string& path, uint64_t* classes);
void save_csv(const std::string& path, const HostData& d);
void split_cv(const HostData& all, double cv_fraction, uint64_t seed, HostData& train, HostData& cv);
void feature_stats(const HostData& d, std::vector<double>& mean, std::vector<double>& sd);
void standardize(HostData& d, const std::vector<double>& mean, const std::vector<double>& sd);

uint64_t param_count(const std::vector<uint64_t>& dims);
std::vector<double> init_random(const std::vector<uint64_t>& dims, Rng& rng);

struct Schedule {
    bool newbob = false;
    double lr_init = 0.32;
    double halve_threshold = 0.005;
    double stop_threshold = 0.001;
    bool halving = false;
    double newbob_lr = 0.32;
    double final_ratio = 0.01;
    uint64_t planned_epochs = 15;
};
Schedule make_schedule(bool newbob, double lr_init, uint64_t epochs);
double exponential_lr(const Schedule& s, double progress);
bool newbob_next(Schedule& s, double prev_acc, double acc, double* lr_out);
double scale_lr_for_workers(double lr_init, uint64_t workers);

void save_model(const std::string& path, const std::vector<uint64_t>& dims, int act, const std::vector<double>& p);
void load_model(const std::string& path, std::vector<uint64_t>& dims, int& act, std::vector<double>& p);

// NG low-rank initial basis: rank x dim, orthonormal rows. Rng(seed).gaussian
// drawn row-major, then modified Gram-Schmidt in fp64 (oracle/ng_lowrank.py).
std::vector<double> lowrank_basis(uint64_t dim, uint64_t rank, uint64_t seed);
uint64_t lowrank_seed(int layer, int side);

// fixed midpoint-tree mean (parallel.cpp:26-59) on host vectors
std::vector<double> allreduce_average(const std::vector<const double*>& contrib, uint64_t len);

}  // namespace host
}  // namespace pnb
