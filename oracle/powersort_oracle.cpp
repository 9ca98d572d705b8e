// powersort_oracle.cpp -- TEST INFRASTRUCTURE ONLY (the parity checker).
//
// A single-threaded CPU restatement of the reference Multiway Powersort
// (arXiv 2209.06909, /root/reference/pkg/src/powersort/*.py).  Every function
// below cites the reference file:line it restates.  It is used by tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// ONLY; the product (paper_2209_06909_b200, libpowersort_b200.so) never links
// or calls it.
//
// Parity pin: tests/golden/*.json were produced by importing the Python
// reference itself (tests/golden/make_golden.py); tests/test_oracle_golden.py
// checks this restatement against every one of them, including the
// comparison / move counters and the on_merge trace.
//
// Elements are (key, int32 value) records compared by key only (the
// reference's SortConfig(key=itemgetter(0)) on (key, index) records).
// The reserved SENTINEL of statskit.py:33-46 is modelled by a per-slot flag in
// the merge buffer, with the uncounted short-circuits of statskit.py:63-67.

#include <stdint.h>
#include <string.h>
#include <stdexcept>
#include <vector>

extern "C" {

typedef struct {
    int64_t comparisons, merge_cost, buffer_cost, moves, max_stack_height,
        runs_detected, merges2, merges3, merges4, scan_reads, scan_writes;
} pso_stats;

}  // extern "C"

namespace {

enum { PSO_OK = 0, PSO_EINVAL = 1, PSO_EOVERFLOW = 5, PSO_EASSERT = 4 };

struct PsoError {
    int code;
};

// Variant ids, policy.py:49-69.
enum Variant {
    V_2WAY = 0,
    V_2WAY_COPY_SMALLER = 1,
    V_2WAY_NOSENTINEL = 2,
    V_4WAY = 3,
    V_4WAY_NOSENTINEL = 4,
};

struct TraceSink {
    int64_t* rows;  // rows of 7: width, b0..b4 (unused = -1), length
    int64_t cap;
    int64_t count;
    void push(const int64_t* begins, int w, int64_t end) {
        if (rows && count < cap) {
            int64_t* r = rows + 7 * count;
            r[0] = w;
            for (int i = 0; i < 5; ++i) r[1 + i] = -1;
            for (int i = 0; i < w; ++i) r[1 + i] = begins[i];
            r[1 + w] = end;
            r[6] = end - begins[0];
        }
        count++;
    }
};

// ---------------------------------------------------------------- power.py
// power.py:24-34
int64_t ceil_log(int64_t k, int64_t n) {
    if (k < 2 || n < 1) throw PsoError{PSO_EINVAL};
    int64_t m = 0;
    __int128 p = 1;
    while (p < n) {
        p *= k;
        m++;
    }
    return m;
}

// power.py:37-44
int64_t run_stack_capacity(int64_t k, int64_t n) { return (k - 1) * (ceil_log(k, n) + 1); }

// power.py:58-74: least p >= 1 with (A*k^p)//2n < (B*k^p)//2n, exact.
int node_power_any(int64_t k, int64_t n, int64_t b1, int64_t e1, int64_t b2, int64_t e2) {
    if (k < 2) throw PsoError{PSO_EINVAL};
    if (!(0 <= b1 && b1 < e1 && e1 == b2 && b2 < e2 && e2 <= n)) throw PsoError{PSO_EINVAL};
    unsigned __int128 A = (unsigned __int128)(b1 + e1);
    unsigned __int128 B = (unsigned __int128)(b2 + e2);
    unsigned __int128 two_n = (unsigned __int128)(2 * n);
    int p = 1;
    unsigned __int128 kp = (unsigned __int128)k;
    while ((A * kp) / two_n == (B * kp) / two_n) {
        p++;
        kp *= (unsigned __int128)k;
    }
    return p;
}

// ------------------------------------------------------------- statskit.py
template <class K>
struct Sorter {
    K* key;
    int32_t* val;
    int64_t n;
    // MergeBuffer (merges.py:43-60): records plus a SENTINEL flag per slot.
    std::vector<K> bk;
    std::vector<int32_t> bv;
    std::vector<uint8_t> bs;
    pso_stats st;
    int64_t comparisons = 0;  // CountingOrder.comparisons (statskit.py:49-72)

    // CountingOrder.le on two list elements (statskit.py:68-72).
    inline bool le_kk(const K& a, const K& b) {
        comparisons++;
        return a <= b;
    }
    // le(B[i], B[j]) with the SENTINEL short-circuits (statskit.py:63-67).
    inline bool le_bb(int64_t i, int64_t j) {
        if (bs[j]) return true;
        if (bs[i]) return false;
        comparisons++;
        return bk[i] <= bk[j];
    }
    // le(B[i], lst[j]) (copy-smaller forward loop, merges.py:163-167)
    inline bool le_bl(int64_t i, int64_t j) {
        comparisons++;
        return bk[i] <= key[j];
    }
    // le(lst[i], B[j]) (copy-smaller backward loop, merges.py:181-185)
    inline bool le_lb(int64_t i, int64_t j) {
        comparisons++;
        return key[i] <= bk[j];
    }
    inline void to_buf(int64_t slot, int64_t src) {
        bk[slot] = key[src];
        bv[slot] = val[src];
        bs[slot] = 0;
    }
    inline void sentinel(int64_t slot) { bs[slot] = 1; }
    inline void from_buf(int64_t dst, int64_t slot) {
        key[dst] = bk[slot];
        val[dst] = bv[slot];
    }

    // merges.py:63-72
    void check_regions(const int64_t* bounds, int nb, int64_t need) {
        if (bounds[0] < 0 || bounds[nb - 1] > n) throw PsoError{PSO_EINVAL};
        for (int i = 0; i + 1 < nb; ++i)
            if (bounds[i] >= bounds[i + 1]) throw PsoError{PSO_EINVAL};
        if ((int64_t)bk.size() < need) throw PsoError{PSO_EINVAL};
    }

    // ------------------------------------------------------------- runs.py
    // runs.py:23-47 -> returns end of the run starting at begin
    int64_t find_first_run(int64_t begin, int64_t end) {
        int64_t i = begin + 1;
        if (i == end) return i;
        if (le_kk(key[begin], key[i])) {
            i++;
            while (i < end && le_kk(key[i - 1], key[i])) i++;
            return i;
        }
        i++;
        while (i < end && !le_kk(key[i - 1], key[i])) i++;
        // lst[begin:i] = lst[begin:i][::-1]  (runs.py:45)
        for (int64_t a = begin, b = i - 1; a < b; ++a, --b) {
            K tk = key[a];
            key[a] = key[b];
            key[b] = tk;
            int32_t tv = val[a];
            val[a] = val[b];
            val[b] = tv;
        }
        st.moves += i - begin;  // runs.py:46
        return i;
    }

    // runs.py:50-68
    void insertion_sort(int64_t begin, int64_t end, int64_t sorted_prefix_len) {
        int64_t start = begin + sorted_prefix_len;
        if (sorted_prefix_len == 0) start = begin + 1;
        for (int64_t i = start; i < end; ++i) {
            K xk = key[i];
            int32_t xv = val[i];
            int64_t j = i - 1;
            while (j >= begin && !le_kk(key[j], xk)) {
                key[j + 1] = key[j];
                val[j + 1] = val[j];
                j--;
            }
            if (j + 1 != i) {
                key[j + 1] = xk;
                val[j + 1] = xv;
                st.moves += i - j;
            }
        }
    }

    // ----------------------------------------------------------- merges.py
    // merges.py:75-104
    void merge_2way_sentinel(int64_t l, int64_t m, int64_t r) {
        int64_t b[3] = {l, m, r};
        check_regions(b, 3, (r - l) + 2);
        int64_t nn = r - l, n1 = m - l;
        for (int64_t i = 0; i < n1; ++i) to_buf(i, l + i);
        sentinel(n1);
        for (int64_t i = 0; i < r - m; ++i) to_buf(n1 + 1 + i, m + i);
        sentinel(nn + 1);
        int64_t c1 = 0, c2 = n1 + 1;
        for (int64_t o = l; o < r; ++o) {
            if (le_bb(c1, c2)) {
                from_buf(o, c1);
                c1++;
            } else {
                from_buf(o, c2);
                c2++;
            }
        }
        st.merge_cost += nn;
        st.buffer_cost += nn;
        st.moves += 2 * nn;
        st.scan_reads += 2 * nn;
        st.scan_writes += 2 * nn + 2;
        st.merges2 += 1;
    }

    // merges.py:107-142
    void merge_2way_no_sentinel(int64_t l, int64_t m, int64_t r) {
        int64_t b[3] = {l, m, r};
        check_regions(b, 3, r - l);
        int64_t nn = r - l, n1 = m - l;
        for (int64_t i = 0; i < nn; ++i) to_buf(i, l + i);
        int64_t c1 = 0, e1 = n1, c2 = n1, e2 = nn, o = l;
        while (c1 < e1 && c2 < e2) {
            if (le_bb(c1, c2)) {
                from_buf(o, c1);
                c1++;
            } else {
                from_buf(o, c2);
                c2++;
            }
            o++;
        }
        while (c1 < e1) from_buf(o++, c1++);
        while (c2 < e2) from_buf(o++, c2++);
        st.merge_cost += nn;
        st.buffer_cost += nn;
        st.moves += 2 * nn;
        st.scan_reads += 2 * nn;
        st.scan_writes += 2 * nn;
        st.merges2 += 1;
    }

    // merges.py:145-201
    void merge_2way_copy_smaller(int64_t l, int64_t m, int64_t r) {
        int64_t n1 = m - l, n2 = r - m;
        int64_t b[3] = {l, m, r};
        check_regions(b, 3, n1 < n2 ? n1 : n2);
        int64_t nn = r - l;
        int64_t written = 0;
        if (n1 <= n2) {
            for (int64_t i = 0; i < n1; ++i) to_buf(i, l + i);
            int64_t c1 = 0, c2 = m, o = l;
            while (c1 < n1 && c2 < r) {
                if (le_bl(c1, c2)) {
                    from_buf(o, c1);
                    c1++;
                } else {
                    key[o] = key[c2];
                    val[o] = val[c2];
                    c2++;
                }
                o++;
            }
            while (c1 < n1) from_buf(o++, c1++);
            written = o - l;
        } else {
            for (int64_t i = 0; i < n2; ++i) to_buf(i, m + i);
            int64_t c1 = m - 1, c2 = n2 - 1, o = r - 1;
            while (c1 >= l && c2 >= 0) {
                if (le_lb(c1, c2)) {
                    from_buf(o, c2);
                    c2--;
                } else {
                    key[o] = key[c1];
                    val[o] = val[c1];
                    c1--;
                }
                o--;
            }
            while (c2 >= 0) from_buf(o--, c2--);
            written = r - 1 - o;
        }
        int64_t copied = n1 < n2 ? n1 : n2;
        st.merge_cost += nn;
        st.buffer_cost += copied;
        st.moves += copied + written;
        st.scan_reads += copied + written;
        st.scan_writes += copied + written;
        st.merges2 += 1;
    }

    // merges.py:204-275 (four runs) and merges.py:278-334 (three runs, y =
    // run 2's head).  Winner tree with x (runs 0/1), y (runs 2/3), root z.
    void merge_tournament_sentinel(const int64_t* g, int w) {
        // g: w+1 bounds
        check_regions(g, w + 1, (g[w] - g[0]) + w);
        int64_t l = g[0], r = g[w];
        int64_t nn = r - l;
        int64_t s[4] = {0, 0, 0, 0};
        int64_t at = 0;
        for (int i = 0; i < w; ++i) {
            s[i] = at;
            for (int64_t j = g[i]; j < g[i + 1]; ++j) to_buf(at++, j);
            sentinel(at++);
        }
        int64_t c0 = s[0], c1 = s[1], c2 = s[2], c3 = (w == 4) ? s[3] : 0;
        int64_t x, y, z;
        bool z_left;
        if (le_bb(c0, c1)) {
            x = c0++;
        } else {
            x = c1++;
        }
        if (w == 4) {
            if (le_bb(c2, c3)) {
                y = c2++;
            } else {
                y = c3++;
            }
        } else {
            y = c2++;
        }
        if (le_bb(x, y)) {
            z = x;
            z_left = true;
        } else {
            z = y;
            z_left = false;
        }
        from_buf(l, z);
        for (int64_t o = l + 1; o < r; ++o) {
            if (z_left) {
                if (le_bb(c0, c1)) {
                    x = c0++;
                } else {
                    x = c1++;
                }
            } else if (w == 4) {
                if (le_bb(c2, c3)) {
                    y = c2++;
                } else {
                    y = c3++;
                }
            } else {
                y = c2++;
            }
            if (le_bb(x, y)) {
                z = x;
                z_left = true;
            } else {
                z = y;
                z_left = false;
            }
            from_buf(o, z);
        }
        st.merge_cost += nn;
        st.buffer_cost += nn;
        st.moves += 2 * nn;
        st.scan_reads += 2 * nn;
        st.scan_writes += 2 * nn + w;
        if (w == 4)
            st.merges4 += 1;
        else
            st.merges3 += 1;
    }

    // merges.py:442-467 (_stage_2way)
    int64_t stage_2way(int64_t out, std::vector<int64_t>& cs, std::vector<int64_t>& es) {
        int64_t c0 = cs[0], e0 = es[0], c1 = cs[1], e1 = es[1];
        while (c0 < e0 && c1 < e1) {
            if (le_bb(c0, c1)) {
                from_buf(out, c0);
                c0++;
            } else {
                from_buf(out, c1);
                c1++;
            }
            out++;
        }
        while (c0 < e0) from_buf(out++, c0++);
        while (c1 < e1) from_buf(out++, c1++);
        return out;
    }

    // merges.py:470-545 (_stage_tournament)
    int64_t stage_tournament(int64_t out, std::vector<int64_t>& cs, std::vector<int64_t>& es) {
        bool four = cs.size() == 4;
        auto fetch_left = [&](int64_t& pos, int& run) {
            int64_t a = cs[0], b = cs[1];
            if (le_bb(a, b)) {
                cs[0] = a + 1;
                pos = a;
                run = 0;
            } else {
                cs[1] = b + 1;
                pos = b;
                run = 1;
            }
        };
        auto fetch_right = [&](int64_t& pos, int& run) {
            if (four) {
                int64_t a = cs[2], b = cs[3];
                if (le_bb(a, b)) {
                    cs[2] = a + 1;
                    pos = a;
                    run = 2;
                } else {
                    cs[3] = b + 1;
                    pos = b;
                    run = 3;
                }
            } else {
                int64_t a = cs[2];
                cs[2] = a + 1;
                pos = a;
                run = 2;
            }
        };
        int64_t x_pos, y_pos;
        int x_run, y_run;
        fetch_left(x_pos, x_run);
        fetch_right(y_pos, y_run);
        bool z_left = le_bb(x_pos, y_pos);
        for (;;) {
            int64_t safe = INT64_MAX;
            for (size_t i = 0; i < cs.size(); ++i) {
                int64_t d = es[i] - cs[i];
                if (d < safe) safe = d;
            }
            if (safe > 0) {
                for (int64_t it = 0; it < safe; ++it) {
                    if (z_left) {
                        from_buf(out++, x_pos);
                        fetch_left(x_pos, x_run);
                    } else {
                        from_buf(out++, y_pos);
                        fetch_right(y_pos, y_run);
                    }
                    z_left = le_bb(x_pos, y_pos);
                }
                continue;
            }
            if (z_left) {
                from_buf(out++, x_pos);
                cs[y_run] -= 1;
            } else {
                from_buf(out++, y_pos);
                cs[x_run] -= 1;
            }
            for (size_t i = 0; i < cs.size(); ++i)
                if (cs[i] == es[i]) return out;
            fetch_left(x_pos, x_run);
            fetch_right(y_pos, y_run);
            z_left = le_bb(x_pos, y_pos);
        }
    }

    // merges.py:337-439 (merge_{4,3}way_stages + _merge_stages)
    void merge_stages(const int64_t* g, int w) {
        check_regions(g, w + 1, (g[w] - g[0]) + 1);
        int64_t l = g[0], r = g[w];
        int64_t nn = r - l;
        for (int64_t i = 0; i < nn; ++i) to_buf(i, l + i);
        bk[nn] = bk[nn - 1];  // guard slot, never consulted
        bv[nn] = bv[nn - 1];
        bs[nn] = 0;
        std::vector<int64_t> cs, es;
        for (int i = 0; i < w; ++i) {
            cs.push_back(g[i] - l);
            es.push_back(g[i + 1] - l);
        }
        int64_t out = l;
        for (;;) {
            size_t i = 0;
            while (i < cs.size()) {
                if (cs[i] == es[i]) {
                    cs.erase(cs.begin() + i);
                    es.erase(es.begin() + i);
                } else {
                    i++;
                }
            }
            size_t width = cs.size();
            if (width == 0) break;
            if (width == 1) {
                for (int64_t c = cs[0]; c < es[0]; ++c) from_buf(out++, c);
                break;
            }
            if (width == 2) {
                out = stage_2way(out, cs, es);
                break;
            }
            out = stage_tournament(out, cs, es);
        }
        if (out != r) throw PsoError{PSO_EASSERT};
        st.merge_cost += nn;
        st.buffer_cost += nn;
        st.moves += 2 * nn + 1;
        st.scan_reads += 2 * nn;
        st.scan_writes += 2 * nn + 1;
        if (w == 4)
            st.merges4 += 1;
        else
            st.merges3 += 1;
    }
};

// ------------------------------------------------------------ policy.py
// RunStack, policy.py:94-129
struct RunStack {
    int64_t capacity, height = 0;
    std::vector<int64_t> begins, powers;
    explicit RunStack(int64_t cap) : capacity(cap), begins(cap + 1, 0), powers(cap + 1, 0) {}
    int64_t top_power() const { return powers[height]; }
    void push(int64_t begin, int64_t power) {
        if (!(power >= powers[height])) throw PsoError{PSO_EASSERT};
        if (height == capacity) throw PsoError{PSO_EOVERFLOW};
        height++;
        begins[height] = begin;
        powers[height] = power;
    }
    int64_t pop() { return begins[height--]; }
};

// _merge_one_group, policy.py:132-143
template <class DoMerge>
int64_t merge_one_group(RunStack& stack, int64_t run_begin, int64_t run_end, int k, DoMerge& do_merge) {
    int64_t group_power = stack.top_power();
    std::vector<int64_t> begins;
    begins.push_back(stack.pop());
    while (stack.top_power() == group_power) begins.push_back(stack.pop());
    if ((int64_t)begins.size() > k - 1) throw PsoError{PSO_EASSERT};
    std::vector<int64_t> b(begins.rbegin(), begins.rend());
    b.push_back(run_begin);
    do_merge(b.data(), (int)b.size(), run_end);
    return b[0];
}

// _merge_down, policy.py:146-175
template <class DoMerge>
void merge_down(RunStack& stack, int64_t run_begin, int64_t run_end, int k, bool strict, DoMerge& do_merge) {
    if (k == 4 && !strict) {
        int64_t n_runs = stack.height + 1;
        int64_t rem = n_runs % 3;
        if (rem == 0) {
            int64_t b2 = stack.pop();
            int64_t b1 = stack.pop();
            int64_t bb[3] = {b1, b2, run_begin};
            do_merge(bb, 3, run_end);
            run_begin = b1;
        } else if (rem == 2) {
            int64_t b1 = stack.pop();
            int64_t bb[2] = {b1, run_begin};
            do_merge(bb, 2, run_end);
            run_begin = b1;
        }
        if (stack.height % 3 != 0) throw PsoError{PSO_EASSERT};
        while (stack.height) {
            int64_t b3 = stack.pop();
            int64_t b2 = stack.pop();
            int64_t b1 = stack.pop();
            int64_t bb[4] = {b1, b2, b3, run_begin};
            do_merge(bb, 4, run_end);
            run_begin = b1;
        }
    } else {
        while (stack.height) {
            int64_t cnt = (k - 1) < stack.height ? (k - 1) : stack.height;
            std::vector<int64_t> b;
            for (int64_t i = 0; i < cnt; ++i) b.push_back(stack.pop());
            std::vector<int64_t> bb(b.rbegin(), b.rend());
            bb.push_back(run_begin);
            do_merge(bb.data(), (int)bb.size(), run_end);
            run_begin = bb[0];
        }
    }
}

// policy.py:178-194
int validated_k(int k, int variant, int64_t min_run_len) {
    if (k != 2 && k != 4) throw PsoError{PSO_EINVAL};
    int vk;
    switch (variant) {
        case V_2WAY:
        case V_2WAY_COPY_SMALLER:
        case V_2WAY_NOSENTINEL:
            vk = 2;
            break;
        case V_4WAY:
        case V_4WAY_NOSENTINEL:
            vk = 4;
            break;
        default:
            throw PsoError{PSO_EINVAL};
    }
    if (vk != k) throw PsoError{PSO_EINVAL};
    if (min_run_len < 1) throw PsoError{PSO_EINVAL};
    return vk;
}

// stable_sort_with, policy.py:201-262.  (The SENTINEL fallback of :211-214
// never fires for numeric inputs -- SURVEY Appendix A.10.)
template <class K>
void sort_impl(K* key, int32_t* val, int64_t n, int k, int variant, int64_t min_run_len, bool strict,
               pso_stats* out, int64_t* run_lengths, int64_t* nat_lengths, TraceSink& trace) {
    validated_k(k, variant, min_run_len);
    Sorter<K> s;
    memset(&s.st, 0, sizeof(s.st));
    s.key = key;
    s.val = val;
    s.n = n;
    if (n == 0) {
        *out = s.st;
        return;
    }
    s.bk.resize(n + k);
    s.bv.resize(n + k);
    s.bs.assign(n + k, 0);
    s.st.scan_reads += n;
    s.st.scan_writes += n;
    RunStack stack(run_stack_capacity(k, n));
    int64_t nruns = 0;

    auto do_merge = [&](const int64_t* begins, int w, int64_t end) {
        int64_t g[5];
        for (int i = 0; i < w; ++i) g[i] = begins[i];
        g[w] = end;
        if (w == 2) {
            if (variant == V_2WAY || variant == V_4WAY)
                s.merge_2way_sentinel(g[0], g[1], g[2]);
            else if (variant == V_2WAY_COPY_SMALLER)
                s.merge_2way_copy_smaller(g[0], g[1], g[2]);
            else
                s.merge_2way_no_sentinel(g[0], g[1], g[2]);
        } else {
            if (variant == V_4WAY)
                s.merge_tournament_sentinel(g, w);
            else
                s.merge_stages(g, w);
        }
        s.st.comparisons = s.comparisons;
        trace.push(begins, w, end);
    };

    auto next_run = [&](int64_t at, int64_t& rb, int64_t& re) {
        int64_t e = s.find_first_run(at, n);
        if (nat_lengths) nat_lengths[nruns] = e - at;
        if (e - at < min_run_len) {
            // extend_run, runs.py:71-82
            int64_t new_end = (at + min_run_len < n) ? at + min_run_len : n;
            s.insertion_sort(at, new_end, e - at);
            e = new_end;
        }
        s.st.runs_detected += 1;
        if (run_lengths) run_lengths[nruns] = e - at;
        nruns++;
        rb = at;
        re = e;
    };

    int64_t a_begin, a_end, b_begin, b_end;
    next_run(0, a_begin, a_end);
    while (a_end < n) {
        next_run(a_end, b_begin, b_end);
        int64_t power = node_power_any(k, n, a_begin, a_end, b_begin, b_end);
        while (stack.top_power() > power) a_begin = merge_one_group(stack, a_begin, a_end, k, do_merge);
        stack.push(a_begin, power);
        if (stack.height > s.st.max_stack_height) s.st.max_stack_height = stack.height;
        a_begin = b_begin;
        a_end = b_end;
    }
    merge_down(stack, a_begin, a_end, k, strict, do_merge);
    s.st.comparisons = s.comparisons;
    *out = s.st;
}

// The run chain of stable_sort_with alone (next_run, policy.py:241-248, with
// find_first_run runs.py:23-47 and extend_run runs.py:71-82), read-only: a
// step from `at` only reads positions >= at, and the reversal / insertion
// sort of a run only rewrites positions before the next step's start, so the
// chain of the unmodified input is the chain of the sort.  For inputs too big
// for the full oracle (cfg5, n = 2^31).
template <class K>
int64_t detect_impl(const K* key, int64_t n, int64_t min_run_len, int64_t* run_lengths, int64_t* nat_lengths,
                    int64_t cap) {
    int64_t r = 0;
    for (int64_t at = 0; at < n;) {
        int64_t i = at + 1;
        if (i < n) {
            if (key[at] <= key[i]) {
                i++;
                while (i < n && key[i - 1] <= key[i]) i++;
            } else {
                i++;
                while (i < n && !(key[i - 1] <= key[i])) i++;
            }
        }
        int64_t e = i;
        if (r < cap && nat_lengths) nat_lengths[r] = e - at;
        if (e - at < min_run_len) e = (at + min_run_len < n) ? at + min_run_len : n;
        if (r < cap && run_lengths) run_lengths[r] = e - at;
        r++;
        at = e;
    }
    return r;
}

}  // namespace

extern "C" {

// Run profile of the input (see detect_impl); returns the run count r (the
// arrays receive min(r, cap) entries) or -PSO_EINVAL.
int64_t pso_detect_runs(int dtype, const void* keys, int64_t n, int64_t min_run_len, int64_t* run_lengths,
                        int64_t* nat_lengths, int64_t cap) {
    if (n < 0 || min_run_len < 1) return -PSO_EINVAL;
    switch (dtype) {
        case 0: return detect_impl((const int32_t*)keys, n, min_run_len, run_lengths, nat_lengths, cap);
        case 1: return detect_impl((const int64_t*)keys, n, min_run_len, run_lengths, nat_lengths, cap);
        case 2: return detect_impl((const float*)keys, n, min_run_len, run_lengths, nat_lengths, cap);
        case 3: return detect_impl((const double*)keys, n, min_run_len, run_lengths, nat_lengths, cap);
        default: return -PSO_EINVAL;
    }
}

// dtype: 0 int32, 1 int64, 2 float32, 3 float64
int pso_sort(int dtype, void* keys, int32_t* vals, int64_t n, int k, int variant, int64_t min_run_len,
             int strict, pso_stats* st, int64_t* run_lengths, int64_t* nat_lengths, int64_t* trace_rows,
             int64_t trace_cap, int64_t* trace_count) {
    TraceSink t{trace_rows, trace_cap, 0};
    try {
        switch (dtype) {
            case 0:
                sort_impl((int32_t*)keys, vals, n, k, variant, min_run_len, strict != 0, st, run_lengths,
                          nat_lengths, t);
                break;
            case 1:
                sort_impl((int64_t*)keys, vals, n, k, variant, min_run_len, strict != 0, st, run_lengths,
                          nat_lengths, t);
                break;
            case 2:
                sort_impl((float*)keys, vals, n, k, variant, min_run_len, strict != 0, st, run_lengths,
                          nat_lengths, t);
                break;
            case 3:
                sort_impl((double*)keys, vals, n, k, variant, min_run_len, strict != 0, st, run_lengths,
                          nat_lengths, t);
                break;
            default:
                return PSO_EINVAL;
        }
    } catch (PsoError& e) {
        return e.code;
    } catch (std::bad_alloc&) {
        return 3;
    }
    if (trace_count) *trace_count = t.count;
    return PSO_OK;
}

// merge_cost_for_profile, policy.py:270-304
int pso_merge_cost_for_profile(const int64_t* lengths, int64_t r, int k, int strict, int64_t* cost,
                               int64_t* max_stack_height, int64_t* trace_rows, int64_t trace_cap,
                               int64_t* trace_count) {
    TraceSink t{trace_rows, trace_cap, 0};
    try {
        if (k != 2 && k != 4) throw PsoError{PSO_EINVAL};
        if (r < 1) throw PsoError{PSO_EINVAL};
        int64_t n = 0;
        for (int64_t i = 0; i < r; ++i) {
            if (lengths[i] < 1) throw PsoError{PSO_EINVAL};
            n += lengths[i];
        }
        int64_t c = 0, msh = 0;
        auto do_merge = [&](const int64_t* begins, int w, int64_t end) {
            c += end - begins[0];
            t.push(begins, w, end);
        };
        RunStack stack(run_stack_capacity(k, n));
        int64_t a_begin = 0, a_end = lengths[0];
        for (int64_t i = 1; i < r; ++i) {
            int64_t b_begin = a_end, b_end = a_end + lengths[i];
            int64_t power = node_power_any(k, n, a_begin, a_end, b_begin, b_end);
            while (stack.top_power() > power) a_begin = merge_one_group(stack, a_begin, a_end, k, do_merge);
            stack.push(a_begin, power);
            if (stack.height > msh) msh = stack.height;
            a_begin = b_begin;
            a_end = b_end;
        }
        merge_down(stack, a_begin, a_end, k, strict != 0, do_merge);
        *cost = c;
        if (max_stack_height) *max_stack_height = msh;
    } catch (PsoError& e) {
        return e.code;
    }
    if (trace_count) *trace_count = t.count;
    return PSO_OK;
}

// power.py:47-55 (node_power) and power.py:58 (_node_power_any, any k >= 2)
int pso_node_power(int k, int64_t n, int64_t b1, int64_t e1, int64_t b2, int64_t e2, int any_k) {
    try {
        if (!any_k && k != 2 && k != 3 && k != 4) return -PSO_EINVAL;
        return node_power_any(k, n, b1, e1, b2, e2);
    } catch (PsoError& e) {
        return -e.code;
    }
}

int64_t pso_run_stack_capacity(int64_t k, int64_t n) {
    try {
        return run_stack_capacity(k, n);
    } catch (PsoError& e) {
        return -e.code;
    }
}

}  // extern "C"
