// Native next-chunk predictor: classification, swap history and pattern
// recognition of the reference's `specpipe.predictor`
// (/root/reference/pkg/src/specpipe/predictor.py), decision for decision.
//
//   classify            predictor.py:63-94   (incl. defect C3: a whole layer
//                                             larger than one chunk is not in
//                                             its own size set)
//   SwapHistory         predictor.py:128-162 (incremental stack / streaks)
//   outstanding_groups  predictor.py:165-183 (incremental groups)
//   _find_cycle         predictor.py:186-215 (longest suffix with a border,
//                                             memoised per history length)
//   recognize           predictor.py:218-249 (REPETITIVE > LIFO > FIFO)
//   predict_batches     predictor.py:252-297
//   Predictor           predictor.py:316-375 (decision_log)
//
// Batches are interned (sorted block tuple -> small int) so the cycle search
// compares integers.  Everything here is host control plane: no CUDA.
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "sppool.hpp"

namespace sppipe {

struct ValueErr : std::runtime_error { using std::runtime_error::runtime_error; };
struct UnknownBlockErr : std::runtime_error { using std::runtime_error::runtime_error; };
struct AmbiguousProfileErr : std::runtime_error { using std::runtime_error::runtime_error; };

enum TransferClass : int { TC_WEIGHTS = 0, TC_KV = 1, TC_SMALL = 2 };
enum PatternKind : int { PK_REPETITIVE = 0, PK_LIFO = 1, PK_FIFO = 2, PK_UNKNOWN = 3 };

struct PredConfig {
    uint64_t small_io_threshold = 8 * 1024;
    uint64_t swap_min = 128 * 1024;
    uint64_t chunk_bytes = 32ull * 1024 * 1024;
    int64_t warmup_matches = 2;
    int64_t history_cap = 128;
    uint64_t layer_param_bytes = 0;  // profile (0 = none configured)
    uint64_t kv_block_bytes = 0;
};

// Message sizes a transfer of `total` bytes splits into (predictor.py:63-71).
inline bool in_chunked_sizes(uint64_t size, uint64_t total, uint64_t chunk) {
    if (total <= chunk) return size == total;
    uint64_t tail = total % chunk;
    return size == chunk || (tail && size == tail);
}

inline TransferClass classify(uint64_t size, const PredConfig& c) {
    if (size < 1) throw ValueErr("transfer size must be positive");
    if (c.layer_param_bytes == c.kv_block_bytes)
        throw AmbiguousProfileErr("profile: layer and KV unit sizes are both " +
                                  std::to_string(c.layer_param_bytes) + " bytes");
    if (in_chunked_sizes(size, c.layer_param_bytes, c.chunk_bytes)) return TC_WEIGHTS;
    if (in_chunked_sizes(size, c.kv_block_bytes, c.chunk_bytes)) return TC_KV;
    return TC_SMALL;
}

struct Hypothesis {
    PatternKind kind = PK_UNKNOWN;
    int64_t confidence = 0;
    std::vector<int> cycle;  // interned batch ids
    int64_t phase = 0;
};

struct Decision {
    int event;  // 0 lock, 1 drop
    PatternKind pattern;
    int64_t confidence;
    int64_t after_batches;
};

struct Prediction {
    int64_t block;
    uint64_t iv;
    uint64_t leeway;
    int32_t batch;
};

class Predictor {
  public:
    explicit Predictor(const PredConfig& c) : cfg(c) {}

    PredConfig cfg;
    std::vector<Decision> decision_log;

    TransferClass classify_size(uint64_t size) const {
        if (cfg.layer_param_bytes == 0 && cfg.kv_block_bytes == 0) throw ValueErr("no model profile configured");
        return classify(size, cfg);
    }

    bool is_outstanding(int64_t b) const { return scripted_ ? script_out_.count(b) != 0 : out_pos_.count(b) != 0; }
    // outstanding blocks in swap-out order (== the reference's stack)
    const std::vector<int64_t>& outstanding_in_order() const { return stack_; }
    size_t in_batch_count() const { return in_batches_.size(); }

    // Event log of SwapHistory.events (predictor.py:128-150): kind 0 = swap
    // out (a = block), 1 = swap-in batch (a = index into the in-batches),
    // 2 = sync.
    struct Event {
        int32_t kind;
        int64_t a;
    };
    const std::vector<Event>& events() const { return events_; }

    // Scripted mode: a fixed prediction schedule handed out once, a fixed
    // outstanding set, observations ignored (the reference's scenario mock,
    // cli.py:241-259 _ScriptedPredictor).  `rounds` (optional, one entry per
    // prediction) hands entries of round r out on the r-th predict call.
    void script(std::vector<Prediction> preds, std::vector<int64_t> outstanding, std::vector<int> rounds = {}) {
        scripted_ = true;
        script_rounds_.clear();
        for (size_t k = 0; k < preds.size(); ++k) {
            const size_t r = k < rounds.size() ? (size_t)std::max(0, rounds[k]) : 0;
            if (script_rounds_.size() <= r) script_rounds_.resize(r + 1);
            script_rounds_[r].push_back(preds[k]);
        }
        script_out_ = std::unordered_set<int64_t>(outstanding.begin(), outstanding.end());
    }
    bool scripted() const { return scripted_; }
    std::vector<int64_t> outstanding_list() const {
        if (!scripted_) return stack_;
        std::vector<int64_t> v(script_out_.begin(), script_out_.end());
        std::sort(v.begin(), v.end());
        return v;
    }

    void observe_swap_out(int64_t block) {
        if (scripted_) return;
        if (is_outstanding(block))
            throw UnknownBlockErr("block " + std::to_string(block) + " is already swapped out");
        out_pos_.insert(block);
        stack_.push_back(block);
        open_.push_back(block);
        events_.push_back({0, block});
    }

    void observe_swap_in(const std::vector<int64_t>& blocks_in) {
        if (scripted_) return;
        std::vector<int64_t> batch(blocks_in);
        std::sort(batch.begin(), batch.end());
        batch.erase(std::unique(batch.begin(), batch.end()), batch.end());
        if (batch.empty()) throw ValueErr("swap-in batch must be non-empty");
        std::vector<int64_t> missing;
        for (int64_t b : batch)
            if (!is_outstanding(b)) missing.push_back(b);
        if (!missing.empty()) {
            std::string m = "swap-in names blocks never swapped out: [";
            for (size_t i = 0; i < missing.size(); ++i) m += (i ? ", " : "") + std::to_string(missing[i]);
            throw UnknownBlockErr(m + "]");
        }
        events_.push_back({1, (int64_t)in_batches_.size()});
        in_batches_.push_back(intern(batch));
        PUSet<int64_t> bs(batch.begin(), batch.end());
        for (int64_t b : batch) out_pos_.erase(b);
        // LIFO/FIFO streaks against the stack of all swap-outs (predictor.py:231-239)
        size_t k = batch.size(), n = stack_.size();
        auto set_eq = [&](size_t lo, size_t hi) {  // set(stack[lo:hi]) == batch
            if (hi - lo != bs.size()) return false;  // stack entries are distinct
            for (size_t i = lo; i < hi; ++i)
                if (!bs.count(stack_[i])) return false;
            return true;
        };
        size_t lo_l = n > k ? n - k : 0;
        lifo_ = set_eq(lo_l, n) ? lifo_ + 1 : 0;
        fifo_ = set_eq(0, std::min(k, n)) ? fifo_ + 1 : 0;
        std::vector<int64_t> ns;
        ns.reserve(n);
        for (int64_t b : stack_)
            if (!bs.count(b)) ns.push_back(b);
        stack_.swap(ns);
        // groups close at a swap-in (predictor.py:165-183)
        close_group();
        std::vector<std::vector<int64_t>> ng;
        for (auto& g : groups_) {
            std::vector<int64_t> g2;
            for (int64_t b : g)
                if (!bs.count(b)) g2.push_back(b);
            if (!g2.empty()) ng.push_back(std::move(g2));
        }
        groups_.swap(ng);
        Hypothesis h = recognize();
        if (h.kind != last_kind_) {
            decision_log.push_back({h.kind != PK_UNKNOWN ? 0 : 1, h.kind, h.confidence,
                                    (int64_t)in_batches_.size()});
            last_kind_ = h.kind;
        }
    }

    void observe_sync() {
        if (scripted_) return;
        events_.push_back({2, 0});
        close_group();
    }
    const std::vector<int64_t>& in_batch(size_t i) const { return batch_of(in_batches_.at(i)); }

    Hypothesis recognize() {
        int64_t n = (int64_t)in_batches_.size();
        if (memo_n_ != n) {
            memo_n_ = n;
            memo_found_ = find_cycle(memo_cycle_, memo_conf_, memo_phase_);
        }
        Hypothesis h;
        if (memo_found_) {
            h.kind = PK_REPETITIVE;
            h.confidence = memo_conf_;
            h.cycle = memo_cycle_;
            h.phase = memo_phase_;
        } else if (lifo_ >= cfg.warmup_matches) {
            h.kind = PK_LIFO;
            h.confidence = lifo_;
        } else if (fifo_ >= cfg.warmup_matches) {
            h.kind = PK_FIFO;
            h.confidence = fifo_;
        }
        return h;
    }

    // predictor.py:252-297 (stateful facade 365-370).  `outstanding`, when
    // given, replaces the history's outstanding set in the two places the
    // reference's free function takes it as a parameter (the REPETITIVE
    // subset test and the counter assignment).
    std::vector<Prediction> predict_batches(uint64_t current_iv, uint64_t leeway, int depth,
                                            const std::unordered_set<int64_t>* outstanding = nullptr) {
        std::vector<Prediction> out;
        if (scripted_) {
            if (script_next_ < script_rounds_.size()) out.swap(script_rounds_[script_next_++]);  // each round once
            return out;
        }
        auto is_out = [&](int64_t b) { return outstanding ? outstanding->count(b) != 0 : is_outstanding(b); };
        Hypothesis h = recognize();
        if (h.kind == PK_UNKNOWN) return out;
        std::vector<std::vector<int64_t>> batches;
        if (h.kind == PK_REPETITIVE) {
            for (int i = 0; i < depth; ++i) {
                const auto& nxt = batch_of(h.cycle[(size_t)((h.phase + i) % (int64_t)h.cycle.size())]);
                bool sub = true;
                for (int64_t b : nxt)
                    if (!is_out(b)) { sub = false; break; }
                if (!sub) break;
                batches.push_back(nxt);
            }
        } else {
            std::vector<std::vector<int64_t>> groups(groups_);
            if (!open_.empty()) groups.push_back(open_);
            if (h.kind == PK_LIFO) {
                for (int i = 0; i < depth && i < (int)groups.size(); ++i) {
                    std::vector<int64_t> g(groups[groups.size() - 1 - i]);
                    std::reverse(g.begin(), g.end());
                    batches.push_back(std::move(g));
                }
            } else {
                for (int i = 0; i < depth && i < (int)groups.size(); ++i) batches.push_back(groups[i]);
            }
        }
        // consecutive counters from current_iv + leeway (predictor.py:287-297)
        uint64_t iv = current_iv + leeway;
        for (size_t bi = 0; bi < batches.size(); ++bi) {
            std::vector<Prediction> preds;
            for (int64_t b : batches[bi]) {
                if (!is_out(b)) return out;
                preds.push_back({b, iv, leeway, (int32_t)bi});
                ++iv;
            }
            out.insert(out.end(), preds.begin(), preds.end());
        }
        return out;
    }

    const std::vector<int64_t>& batch_of(int id) const { return batch_by_id_[(size_t)id]; }

  private:
    struct VecHash {
        size_t operator()(const std::vector<int64_t>& v) const {
            uint64_t h = 1469598103934665603ull;
            for (int64_t x : v) { h ^= (uint64_t)x + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2); }
            return (size_t)h;
        }
    };

    int intern(const std::vector<int64_t>& sorted_batch) {
        auto it = ids_.find(sorted_batch);
        if (it != ids_.end()) return it->second;
        int id = (int)batch_by_id_.size();
        ids_.emplace(sorted_batch, id);
        batch_by_id_.push_back(sorted_batch);
        return id;
    }

    void close_group() {
        if (!open_.empty()) {
            groups_.push_back(std::move(open_));
            open_.clear();
        }
    }

    // Longest suffix (within the last history_cap) whose smallest period p
    // leaves a non-empty border (predictor.py:200-215).
    bool find_cycle(std::vector<int>& cycle, int64_t& conf, int64_t& phase) const {
        int64_t n = (int64_t)in_batches_.size();
        int64_t k0 = std::max<int64_t>(0, n - cfg.history_cap);
        std::vector<int64_t> fail;
        for (int64_t k = k0; k < n - 1; ++k) {
            const int* seq = in_batches_.data() + k;
            int64_t len = n - k;
            fail.assign((size_t)len, 0);
            int64_t q = 0;
            for (int64_t i = 1; i < len; ++i) {
                while (q && seq[i] != seq[q]) q = fail[(size_t)q - 1];
                if (seq[i] == seq[q]) ++q;
                fail[(size_t)i] = q;
            }
            int64_t p = len - fail[(size_t)len - 1];
            if (len >= p + 1) {
                cycle.assign(seq, seq + p);
                conf = len - p;
                phase = len % p;
                return true;
            }
        }
        return false;
    }

    std::vector<Event> events_;
    bool scripted_ = false;
    std::vector<std::vector<Prediction>> script_rounds_;
    size_t script_next_ = 0;
    std::unordered_set<int64_t> script_out_;
    PUSet<int64_t> out_pos_;  // pooled nodes: one insert per swap-out, one erase per swap-in
    std::vector<int64_t> stack_;
    std::vector<int64_t> open_;
    std::vector<std::vector<int64_t>> groups_;
    std::vector<int> in_batches_;
    std::unordered_map<std::vector<int64_t>, int, VecHash> ids_;
    std::vector<std::vector<int64_t>> batch_by_id_;
    int64_t lifo_ = 0, fifo_ = 0;
    PatternKind last_kind_ = PK_UNKNOWN;
    int64_t memo_n_ = -1;
    bool memo_found_ = false;
    std::vector<int> memo_cycle_;
    int64_t memo_conf_ = 0, memo_phase_ = 0;
};

}  // namespace sppipe
