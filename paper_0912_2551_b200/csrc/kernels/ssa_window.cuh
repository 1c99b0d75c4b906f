// ssa_window.cuh -- the WINDOW MONITOR: on-the-fly literal |= for formulas
// outside the streaming templates of reading R16 (arbitrary nesting, non-zero inner lower
// bounds, X under F/G/U), with memory bounded by the formula's
// windows instead of the trace (reading R27).
//
// Every subformula node is a stream that emits, in position order m = 0, 1, 2, ..., the
// pair (v, r) of its value at sigma^m and the FIRST prefix index r at which that value is
// definite in the three-valued semantics of a prefix (entries 0..n and the sojourn of
// entry n, the future unknown; R24).  Values and r compose exactly (Kleene logic):
//   atom / true / false at m: (bit, m);   NOT: (not v, r);
//   AND: false at the min r of its false operands, true at the max r of both;  OR dual;
//   X^I at m: tau_m in I ? the child's (v, r) at m+1 : (0, m);
//   phi1 U^I phi2 at m: the OR over the terms k with elapsed(m, k) in I of
//     (AND_{m<=j<k} phi1(j)) AND phi2(k) -- true at the min over true terms of
//     max(r2(k), max_j r1(j)); false at max(n0, max over terms of their zero time), n0 =
//     min(window close c, first prefix at which the AND is 0), c = the last k whose
//     elapsed is not beyond I (elapsed(m, c+1) = elapsed(m, c) + tau_c is beyond);
//   F^I phi = true U^I phi;  G^I phi = not F^I not phi.
// elapsed(m, k) = tau_m + ... + tau_{k-1} left to right, exactly the oracle's sum, kept per
// pending position.  A temporal node's pending positions all consume the child stream in
// lock step (child position j updates every pending m <= j), so the state per position is
// O(1) (elapsed, best true r, max zero r, the AND's state) and a position is final -- and
// leaves the window -- once no later child value can change (v, r): a true term with r <=
// j + 1 (later terms have r >= their position), the AND became 0, or the window closed.
// The root's r is the replica's event count, identical to the oracle's exact
// first decision index; the few events simulated until the root's r is known are not
// counted (like speculative replicas).
//
// Memory per replica slot: W ring entries (W a power of two, per launch) of
//   t_k, tau_k (8 + 8 B), one (v, r) queue per node (8 B), one 32-byte state per pending
//   position of each temporal node;
// a node only creates positions whose entry time is within the time the root can reach
// through it (its `tlim`, the formula's reach along the path; `plim` positions for
// root-level booleans), so the rings hold one window, not the trace.  A ring that would
// overflow ends the replica as an error.
//
// Generated before this header (codegen.cpp window_code): SMC_WIN_NODES, SMC_WIN_ROOT,
// SMC_WIN_PER_ENTRY, SMC_LIT_H, smc_lit_mask(x), and per node
//   template <> struct SmcWN<i> { kind, a, b, atom, par, lo, hi, lo_open, hi_open, hi_inf,
//                                 tlim, plim, oq, ost };
// The same struct serves the thread-owned literal kernel (one lane per slot) and the tile
// kernel (the TW lanes of a tile share a slot and split the pending positions).

enum { SMC_WK_ATOM = 0, SMC_WK_TRUE, SMC_WK_FALSE, SMC_WK_NOT, SMC_WK_AND, SMC_WK_OR, SMC_WK_X, SMC_WK_U,
       SMC_WK_F, SMC_WK_G };
#define SMC_WINF 0x7fffffff

struct SmcWSt {            // pending position of a temporal node: all but the elapsed time (32 B)
    int tb;                // min r over true terms (SMC_WINF: none); once final: the result r
    int zm;                // max zero time over the false terms (-1: none)
    int p1;                // U: max r over the phi1 values (all 1 so far)
    int pz;                // U: min r over the phi1 zeros (SMC_WINF: none)
    int fl;                // bit 0 final, bits 1-2 value, bit 3 unknown term, bits 4-5 AND state
    int pad[3];
};
// The elapsed time of a pending position lives in its own array (8 B per position: the
// step that only advances it -- every position before its window opens -- touches a quarter
// of a sector); a final position's elapsed is set to -1 (elapsed times are >= 0).

template <int I> struct SmcWN;

__device__ __forceinline__ smc_u64 smc_wpack(int v, int r) { return ((smc_u64)(unsigned)r << 2) | (smc_u64)v; }

struct SmcMon {
    char* S;                                   // this slot's rings
    int W, msk;                                // ring entries (power of two)
    int lane, nl;                              // this lane's index among the slot's nl lanes
    unsigned gm;                               // the slot's lanes
    int leader;
    int qh[SMC_WIN_NODES], qt[SMC_WIN_NODES];  // output queue: consumed by the parent / emitted
    int lo[SMC_WIN_NODES], hi[SMC_WIN_NODES];  // temporal: next position to emit / create; X: next
    bool stop[SMC_WIN_NODES];                  // no more positions will be created
    // F / G nodes: the head position's window [ka, kb) over the child stream, the next child
    // entry jc to consume, monotone deques (child indices) of the true entries (min r) and the
    // false entries (max r) in [ka, jc), unknown entries in [ka, jc)
    int ka[SMC_WIN_NODES], kb[SMC_WIN_NODES], jc[SMC_WIN_NODES];
    int dth[SMC_WIN_NODES], dtt[SMC_WIN_NODES], dzh[SMC_WIN_NODES], dzt[SMC_WIN_NODES], nunk[SMC_WIN_NODES];
    unsigned char hf[SMC_WIN_NODES];           // bit 0 head set, bit 1 ka found, bit 2 kb known, bit 3 elh valid
    double elh[SMC_WIN_NODES];                 // elapsed(head, jc - 1), exact, while bit 3 is set
    int ne;                                    // entries processed (positions 0 .. ne-1)
    int ntau;                                  // sojourns known (tau_0 .. tau_{ntau-1})
    bool pend;                                 // an entered entry not yet processed
    unsigned pmask;
    double pt;
    int last;                                  // index of the last entered entry
    int res, decided_at;
    bool err;

    __device__ __forceinline__ double* tt() const { return (double*)S; }
    __device__ __forceinline__ double* tau() const { return (double*)(S + (long long)8 * W); }
    // array of node I at offset `off` (bytes-per-entry units): W entries, or SMC_WIN_SE entries
    // in the small area for single-position nodes (their indices stay below 2)
    template <int I> __device__ __forceinline__ char* arr(long long off) const {
        if constexpr (SmcWN<I>::small) return S + (long long)W * SMC_WIN_PER_ENTRY + off * SMC_WIN_SE;
        else return S + off * W;
    }
    template <int I> __device__ __forceinline__ long long len() const { return SmcWN<I>::small ? SMC_WIN_SE : W; }
    template <int I> __device__ __forceinline__ smc_u64* q() const { return (smc_u64*)arr<I>(SmcWN<I>::oq); }
    template <int I> __device__ __forceinline__ SmcWSt* st() const { return (SmcWSt*)arr<I>(SmcWN<I>::ost); }
    template <int I> __device__ __forceinline__ double* elp() const { return (double*)arr<I>(SmcWN<I>::oel); }
    // F / G deques of (child index, r)
    template <int I> __device__ __forceinline__ int2* dqt() const { return (int2*)arr<I>(SmcWN<I>::odq); }
    template <int I> __device__ __forceinline__ int2* dqz() const { return (int2*)(arr<I>(SmcWN<I>::odq) + 8 * len<I>()); }
    __device__ __forceinline__ void sync() const { if (nl > 1) __syncwarp(gm); }

    __device__ __forceinline__ void bind(const SmcParams& Q, smc_u64 slot, unsigned mask, int lead) {
        W = (int)Q.lit_cap;
        msk = W - 1;
        S = (char*)Q.lit_t + slot * ((smc_u64)W * (smc_u64)SMC_WIN_PER_ENTRY + (smc_u64)SMC_WIN_SMALL);
        gm = mask;
        leader = lead;
        nl = __popc(mask);
        lane = (int)(threadIdx.x & 31u) - lead;
    }
    __device__ __forceinline__ void init() {
#pragma unroll
        for (int i = 0; i < SMC_WIN_NODES; ++i) {
            qh[i] = qt[i] = lo[i] = hi[i] = 0;
            stop[i] = false;
            ka[i] = kb[i] = jc[i] = dth[i] = dtt[i] = dzh[i] = dzt[i] = nunk[i] = 0;
            hf[i] = 0;
            elh[i] = 0.0;
        }
        ne = ntau = 0;
        pend = false;
        last = 0;
        res = -1;
        decided_at = -1;
        err = false;
    }

    template <int I> __device__ __forceinline__ static bool contains(double e) {
        using D = SmcWN<I>;
        const bool lo_ok = D::lo_open ? (e > D::lo) : (e >= D::lo);
        if (D::hi_inf) return lo_ok;
        return lo_ok && (D::hi_open ? (e < D::hi) : (e <= D::hi));
    }
    template <int I> __device__ __forceinline__ static bool beyond(double e) {
        using D = SmcWN<I>;
        if (D::hi_inf) return false;
        return D::hi_open ? (e >= D::hi) : (e > D::hi);
    }

    // ---------------------------------------------------------------- queues
    template <int I> __device__ __forceinline__ void emit(int v, int r) {
        if (qt[I] - qh[I] >= W) { err = true; return; }
        q<I>()[qt[I] & msk] = smc_wpack(v, r);            // every lane writes the same value
        ++qt[I];
    }
    template <int C> __device__ __forceinline__ void peek(int p, int& v, int& r) const {
        const smc_u64 e = q<C>()[p & msk];
        v = (int)(e & 3ull);
        r = (int)(e >> 2);
    }
    // node I will emit no more positions (stopped and drained into its queue)
    template <int I> __device__ __forceinline__ bool ended() const {
        using D = SmcWN<I>;
        if constexpr (D::kind == SMC_WK_ATOM || D::kind == SMC_WK_TRUE || D::kind == SMC_WK_FALSE) return stop[I];
        else if constexpr (D::kind == SMC_WK_X) return stop[I];
        else if constexpr (D::kind == SMC_WK_F || D::kind == SMC_WK_G) return stop[I];
        else if constexpr (D::kind == SMC_WK_U) return stop[I] && lo[I] == hi[I];
        else if constexpr (D::kind == SMC_WK_NOT) return ended<D::a>() && qh[D::a] == qt[D::a];
        else return (ended<D::a>() && qh[D::a] == qt[D::a]) || (ended<D::b>() && qh[D::b] == qt[D::b]);
    }
    // the parent of I consumes no more (it is done, or it is the root and the root is known)
    template <int I> __device__ __forceinline__ bool dead() const {
        using D = SmcWN<I>;
        if constexpr (D::par < 0) return qt[I] > 0;
        else return dead<D::par>() || ended<D::par>();
    }

    // ---------------------------------------------------------------- leaves
    template <int I> __device__ __forceinline__ void leaf(int k, double t, unsigned mk) {
        using D = SmcWN<I>;
        if constexpr (D::kind == SMC_WK_ATOM || D::kind == SMC_WK_TRUE || D::kind == SMC_WK_FALSE) {
            if (stop[I] || dead<I>()) return;
            if (k >= D::plim || !(t <= D::tlim)) { stop[I] = true; return; }
            const int v = D::kind == SMC_WK_ATOM ? (int)((mk >> D::atom) & 1u) : (D::kind == SMC_WK_TRUE ? 1 : 0);
            emit<I>(v, k);                                 // an atom's value is known at its entry
        }
    }
    template <int I> __device__ __forceinline__ void leaves(int k, double t, unsigned mk) {
        if constexpr (I < SMC_WIN_NODES) { leaf<I>(k, t, mk); leaves<I + 1>(k, t, mk); }
    }

    // ---------------------------------------------------------------- temporal nodes
    __device__ __forceinline__ static void tfinal(SmcWSt& s, int v, int r) {
        s.tb = r;
        s.fl = (s.fl & ~7) | 1 | (v << 1);
    }
    // the window of the position closed after term c (no later terms)
    __device__ __forceinline__ static void tclose(SmcWSt& s, int c) {
        const int pv = (s.fl >> 4) & 3;
        if (s.tb != SMC_WINF) tfinal(s, 1, s.tb);
        else if (s.fl & 8) tfinal(s, 2, SMC_WINF);
        else tfinal(s, 0, max(pv == 0 ? min(c, s.pz) : c, s.zm));
    }
    // position m consumes child position j (the term j and the AND's operand j); `el` is
    // elapsed(m, j - 1) on entry (0 for m == j); returns the new elapsed (< 0: final)
    template <int I> __device__ __forceinline__ double tstep(SmcWSt* ST, int m, int j, double el, double tj, int v1,
                                                             int r1, int v2, int r2, bool fresh) const {
        using D = SmcWN<I>;
        if (m < j) el = __dadd_rn(el, tj);                // elapsed(m, j), left to right
        const bool clo = m < j && beyond<I>(el);
        const bool term = !clo && contains<I>(el);
        if (!clo && !term && D::kind != SMC_WK_U && !fresh) return el;   // before the window: elapsed only
        SmcWSt s;
        if (fresh) { s.tb = SMC_WINF; s.zm = -1; s.p1 = -1; s.pz = SMC_WINF; s.fl = 1 << 4; }
        else s = ST[m & msk];
        if (clo) {
            tclose(s, j - 1);
        } else {
            int pv = (s.fl >> 4) & 3;
            if (term) {
                if (pv == 0 || v2 == 0) s.zm = max(s.zm, min(pv == 0 ? s.pz : SMC_WINF, v2 == 0 ? r2 : SMC_WINF));
                else if (pv == 1 && v2 == 1) s.tb = min(s.tb, max(s.p1, r2));
                else s.fl |= 8;                           // an unknown term (end of trace only)
            }
            if constexpr (D::kind == SMC_WK_U) {
                if (v1 == 0) { s.pz = min(s.pz, r1); pv = 0; }
                else if (v1 == 1) { if (pv == 1) s.p1 = max(s.p1, r1); }
                else if (pv == 1) pv = 2;
                s.fl = (s.fl & ~0x30) | (pv << 4);
            }
            if (s.tb != SMC_WINF && (s.tb <= j + 1 || pv == 0)) tfinal(s, 1, s.tb);
            else if (s.tb == SMC_WINF && !(s.fl & 8) && pv == 0 && s.pz <= j) tfinal(s, 0, max(s.pz, s.zm));
        }
        ST[m & msk] = s;
        return (s.fl & 1) ? -1.0 : el;
    }
    // the trace ended (or the child stream did) after child position jl: close or leave open
    template <int I> __device__ __forceinline__ void tend(SmcWSt& s, double el, int jl, bool fin, bool absorbed, int N) {
        if (fin && absorbed && jl == N) { tclose(s, N); return; }     // no further entries (R7)
        const double e2 = __dadd_rn(el, tau()[jl & msk]);
        if (beyond<I>(e2)) { tclose(s, jl); return; }
        if (!(fin && jl == N)) { err = true; return; }               // child ended inside the window
        const int pv = (s.fl >> 4) & 3;                              // the future term is unknown
        if (s.tb != SMC_WINF) tfinal(s, 1, s.tb);
        else if (pv == 0 && !(s.fl & 8)) tfinal(s, 0, max(s.pz, s.zm));
        else tfinal(s, 2, SMC_WINF);
    }
    template <int I> __device__ __forceinline__ void temit() {
        using D = SmcWN<I>;
        SmcWSt* ST = st<I>();
        const double* EL = elp<I>();
        while (lo[I] < hi[I]) {
            if (!(EL[lo[I] & msk] < 0.0)) break;
            const int f = ST[lo[I] & msk].fl;
            int v = (f >> 1) & 3;
            if (D::kind == SMC_WK_G && v != 2) v = 1 - v;   // G = not F not
            emit<I>(v, ST[lo[I] & msk].tb);
            ++lo[I];
        }
    }
    template <int I> __device__ __forceinline__ void temporal(bool fin, bool absorbed, int N) {
        using D = SmcWN<I>;
        constexpr int A = D::a;
        constexpr int B = D::kind == SMC_WK_U ? D::b : D::a;
        SmcWSt* ST = st<I>();
        for (;;) {
            const int j = qh[B];
            if (qh[B] >= qt[B] || (D::kind == SMC_WK_U && qh[A] >= qt[A])) break;
            int v1 = 1, r1 = -1, v2, r2;
            peek<B>(j, v2, r2);
            if constexpr (D::kind == SMC_WK_U) peek<A>(j, v1, r1);
            if constexpr (D::kind == SMC_WK_G) { if (v2 != 2) v2 = 1 - v2; }
            if (!stop[I]) {                                   // position j of this node
                if (j < D::plim && tt()[j & msk] <= D::tlim) {
                    if (hi[I] - lo[I] >= W) { err = true; return; }
                    hi[I] = j + 1;
                } else {
                    stop[I] = true;
                }
            }
            const double tj = j > 0 ? tau()[(j - 1) & msk] : 0.0;
            double* EL = elp<I>();
            for (int m = lo[I] + lane; m < hi[I]; m += nl) {
                const bool fresh = m == j;
                const double e0 = fresh ? 0.0 : EL[m & msk];
                if (e0 < 0.0) continue;                       // final, waiting to be emitted
                EL[m & msk] = tstep<I>(ST, m, j, e0, tj, v1, r1, v2, r2, fresh);
            }
            ++qh[B];
            if constexpr (D::kind == SMC_WK_U) ++qh[A];
            sync();
            temit<I>();
        }
        const bool cend = ended<B>() && qh[B] == qt[B] && (D::kind != SMC_WK_U || (ended<A>() && qh[A] == qt[A]));
        if (fin || cend) {                                    // no more child positions
            stop[I] = true;
            if (lo[I] < hi[I]) {
                const int jl = qh[B] - 1;
                double* EL = elp<I>();
                for (int m = lo[I] + lane; m < hi[I]; m += nl) {
                    const double e0 = EL[m & msk];
                    if (e0 < 0.0) continue;
                    SmcWSt s = ST[m & msk];
                    tend<I>(s, e0, jl, fin, absorbed, N);
                    ST[m & msk] = s;
                    EL[m & msk] = -1.0;
                }
                sync();
                temit<I>();
            }
        }
    }


    // ---------------------------------------------------------------- F and G (head windows)
    // F^I phi at m is the OR over the child entries k in the window [ka(m), kb(m)) (elapsed(m, k)
    // in I; elapsed is monotone in k); G = not F not.  Positions are evaluated in order, one at
    // a time (the head m = lo): the window's entries enter two monotone deques as the child
    // stream delivers them -- the min r over the true entries and the max r over the false
    // ones -- and leave them when the head advances (the windows of consecutive positions move
    // forward), so a position costs O(1) amortized instead of O(window).  The window bounds
    // compare elapsed(m, k) -- the left-to-right sum of the semantics -- with I: decided by the
    // entry-time difference t_k - t_m when that is farther from the bound than the rounding of
    // both sums can move it (|error| <= 4 (k + 2) u t_k, u = 2^-53), else by the exact sum.

    __device__ __forceinline__ double t_at(int k) const {   // entry time t_k (k <= ne, tau_{k-1} known)
        return k < ne ? tt()[k & msk] : __dadd_rn(tt()[(k - 1) & msk], tau()[(k - 1) & msk]);
    }
    __device__ __forceinline__ double el_exact(int m, int k) const {   // tau_m + ... + tau_{k-1}
        double e = 0.0;
        for (int i = m; i < k; ++i) e = (i == m) ? tau()[i & msk] : __dadd_rn(e, tau()[i & msk]);
        return e;
    }
    // sign of elapsed(m, k) - B: -1, 0, +1
    __device__ __forceinline__ int el_cmp(int m, int k, double B) const {
        if (k == m) return 0.0 < B ? -1 : (0.0 > B ? 1 : 0);
        const double tk = t_at(k);
        const double d = __dsub_rn(tk, tt()[m & msk]);
        const double dl = __dmul_rn(__dmul_rn((double)(k + 2), 4.4408920985006271e-16), __dmul_rn(tk, 1.0000010000000000));
        if (__dsub_rn(d, dl) > B) return 1;
        if (__dadd_rn(d, dl) < B) return -1;
        const double e = el_exact(m, k);
        return e < B ? -1 : (e > B ? 1 : 0);
    }
    // elapsed(m, k) against a bound: the head's exact running sum when k is the next entry of a
    // head started from scratch (bit 3), else the entry-time difference with its error bound
    template <int I> __device__ __forceinline__ int fg_cmp(int m, int k, double B) const {
        if ((hf[I] & 8) && k == jc[I]) {
            const double e = k == m ? 0.0 : __dadd_rn(elh[I], tau()[(k - 1) & msk]);
            return e < B ? -1 : (e > B ? 1 : 0);
        }
        return el_cmp(m, k, B);
    }
    template <int I> __device__ __forceinline__ bool fg_lo_ok(int m, int k) const {   // elapsed(m,k) >= / > lo
        using D = SmcWN<I>;
        const int c = fg_cmp<I>(m, k, D::lo);
        return D::lo_open ? c > 0 : c >= 0;
    }
    template <int I> __device__ __forceinline__ bool fg_beyond(int m, int k) const {
        using D = SmcWN<I>;
        if (D::hi_inf) return false;
        const int c = fg_cmp<I>(m, k, D::hi);
        return D::hi_open ? c >= 0 : c > 0;
    }
    template <int I> __device__ __forceinline__ void fg_val(int k, int& v, int& r) const {
        using D = SmcWN<I>;
        peek<D::a>(k, v, r);
        if (D::kind == SMC_WK_G && v != 2) v = 1 - v;      // G = not F not
    }
    template <int I> __device__ __forceinline__ void fg_push(int k) {
        using D = SmcWN<I>;
        int v, r;
        fg_val<I>(k, v, r);
        if (lo[I] + 1 >= D::plim) {                          // the node's last position: its window
            if (v == 1) {                                     // never moves, only the extremes matter
                int2* DT = dqt<I>();
                if (dtt[I] == dth[I]) { DT[dth[I] & msk] = make_int2(k, r); dtt[I] = dth[I] + 1; }
                else if (r < DT[dth[I] & msk].y) DT[dth[I] & msk] = make_int2(k, r);
            } else if (v == 0) {
                int2* DZ = dqz<I>();
                if (dzt[I] == dzh[I]) { DZ[dzh[I] & msk] = make_int2(k, r); dzt[I] = dzh[I] + 1; }
                else if (r > DZ[dzh[I] & msk].y) DZ[dzh[I] & msk] = make_int2(k, r);
            } else {
                ++nunk[I];
            }
            return;
        }
        if (v == 1) {
            int2* DT = dqt<I>();
            while (dtt[I] > dth[I] && DT[(dtt[I] - 1) & msk].y >= r) --dtt[I];
            DT[dtt[I] & msk] = make_int2(k, r);
            ++dtt[I];
        } else if (v == 0) {
            int2* DZ = dqz<I>();
            while (dzt[I] > dzh[I] && DZ[(dzt[I] - 1) & msk].y <= r) --dzt[I];
            DZ[dzt[I] & msk] = make_int2(k, r);
            ++dzt[I];
        } else {
            ++nunk[I];
        }
        if (dtt[I] - dth[I] > W || dzt[I] - dzh[I] > W) err = true;
    }
    // restart the head's window from scratch (rounding made a window bound move backwards)
    template <int I> __device__ __forceinline__ void fg_reset(int m) {
        ka[I] = kb[I] = 0;
        jc[I] = m;
        dth[I] = dtt[I] = dzh[I] = dzt[I] = nunk[I] = 0;
        hf[I] = 1 | 8;                                        // the running sum starts at the head
        elh[I] = 0.0;
    }
    template <int I> __device__ __forceinline__ void fgnode(bool fin, bool absorbed, int N) {
        using D = SmcWN<I>;
        constexpr int C = D::a;
        const bool cend = ended<C>();
        for (;;) {
            if (stop[I]) return;
            const int m = lo[I];
            if (!(hf[I] & 1)) {                               // a new head position
                if (m >= ne) return;                          // entry m not processed yet
                if (!(m < D::plim && tt()[m & msk] <= D::tlim)) { stop[I] = true; return; }
                fg_reset<I>(m);
            }
            // consume the child entries of the head's window
            bool open_end = false;
            for (;;) {
                const int k = jc[I];
                if (!(hf[I] & 4) && k > m) {                  // does the window end before entry k?
                    if (fin && k == N + 1) {
                        if (absorbed || fg_beyond<I>(m, k)) { kb[I] = k; hf[I] |= 4; }
                        else { open_end = true; break; }
                    } else if (k < ne || k - 1 < ntau) {
                        if (fg_beyond<I>(m, k)) { kb[I] = k; hf[I] |= 4; }
                    } else {
                        break;                                // t_k not known yet
                    }
                }
                if ((hf[I] & 4) && k >= kb[I]) break;        // window closed and consumed
                if (k >= qt[C]) {
                    if (cend || fin) {                        // the child stream ended inside the window
                        if (!(fin && k == N + 1)) { err = true; return; }
                    }
                    break;
                }
                if (!(hf[I] & 2) && fg_lo_ok<I>(m, k)) { ka[I] = k; hf[I] |= 2; }
                if (hf[I] & 2) fg_push<I>(k);
                if (hf[I] & 8) elh[I] = k == m ? 0.0 : __dadd_rn(elh[I], tau()[(k - 1) & msk]);
                ++jc[I];
                if (m + 1 >= D::plim) qh[C] = jc[I];         // the last position: the deques hold what it needs
            }
            // is the head's (v, r) final?
            const bool closed = (hf[I] & 4) && jc[I] >= kb[I];
            const int tb = dtt[I] > dth[I] ? dqt<I>()[dth[I] & msk].y : SMC_WINF;
            int v, r;
            if (tb != SMC_WINF && (tb <= jc[I] || closed || open_end)) { v = 1; r = tb; }
            else if (closed && nunk[I] == 0) {
                const int zr = dzt[I] > dzh[I] ? dqz<I>()[dzh[I] & msk].y : -1;
                v = 0;
                r = max(kb[I] - 1, zr);
            } else if (open_end || closed) { v = 2; r = SMC_WINF; }      // the end of the trace: unknown
            else return;
            emit<I>(D::kind == SMC_WK_G && v != 2 ? 1 - v : v, r);
            if (err) return;
            // advance the head to m + 1: drop the entries before its window
            const int m1 = m + 1;
            lo[I] = m1;
            qh[C] = min(m1, qt[C]);                           // the child ring keeps [head, ...)
            if (fin && m1 > N) { stop[I] = true; return; }
            if (m1 >= ne) { hf[I] = 0; return; }              // entry m + 1 not processed yet
            if (!(m1 < D::plim && tt()[m1 & msk] <= D::tlim)) { stop[I] = true; return; }
            if (jc[I] < m1) { fg_reset<I>(m1); continue; }
            // the new window's lower end: later or equal (else restart), entries before it leave
            int a = (hf[I] & 2) ? max(ka[I], m1) : jc[I];
            if (a > m1 && a - 1 < jc[I] && fg_lo_ok<I>(m1, a - 1)) { fg_reset<I>(m1); continue; }
            while (a < jc[I] && !fg_lo_ok<I>(m1, a)) ++a;
            if (jc[I] > m1 && fg_beyond<I>(m1, jc[I] - 1)) { fg_reset<I>(m1); continue; }
            {
                const int2* DT = dqt<I>();
                const int2* DZ = dqz<I>();
                while (dth[I] < dtt[I] && DT[dth[I] & msk].x < a) ++dth[I];
                while (dzh[I] < dzt[I] && DZ[dzh[I] & msk].x < a) ++dzh[I];
                if (nunk[I] > 0) {
                    for (int k = (hf[I] & 2) ? ka[I] : a; k < a; ++k) { int vv, rr; fg_val<I>(k, vv, rr); if (vv == 2) --nunk[I]; }
                }
            }
            if (a < jc[I]) { ka[I] = a; hf[I] |= 2; }
            else hf[I] &= ~2;
            hf[I] &= ~(4 | 8);                                // the window end is re-determined
        }
    }

    // ---------------------------------------------------------------- X, booleans
    template <int I> __device__ __forceinline__ void xnode(bool fin, bool absorbed, int N) {
        using D = SmcWN<I>;
        constexpr int A = D::a;
        while (!stop[I]) {
            const int m = lo[I];
            if (m >= ne) break;                               // entry m not processed yet
            if (m >= D::plim || !(tt()[m & msk] <= D::tlim)) { stop[I] = true; break; }
            int v = 0, r = m;
            if (fin && m == N) {                              // the last entry
                if (absorbed) { v = 0; r = N; }
                else if (contains<I>(tau()[m & msk])) { v = 2; r = SMC_WINF; }
            } else {
                if (m >= ntau) break;                         // tau_m not drawn yet
                if (contains<I>(tau()[m & msk])) {            // sigma^1 |= phi and delta(sigma, 0) in I
                    while (qh[A] < m + 1 && qh[A] < qt[A]) ++qh[A];
                    if (qh[A] == m + 1 && qh[A] < qt[A]) { peek<A>(m + 1, v, r); ++qh[A]; }
                    else if (ended<A>()) { err = true; return; }
                    else break;
                }
            }
            emit<I>(v, r);
            ++lo[I];
            if (fin && m == N) stop[I] = true;
        }
        if (fin) stop[I] = true;
    }
    template <int I> __device__ __forceinline__ void boolean() {
        using D = SmcWN<I>;
        constexpr int A = D::a;
        if constexpr (D::kind == SMC_WK_NOT) {
            while (qh[A] < qt[A]) {
                int v, r;
                peek<A>(qh[A], v, r);
                ++qh[A];
                emit<I>(v == 2 ? 2 : 1 - v, r);
            }
        } else {
            constexpr int B = D::b;
            while (qh[A] < qt[A] && qh[B] < qt[B]) {
                int va, ra, vb, rb;
                peek<A>(qh[A], va, ra);
                peek<B>(qh[B], vb, rb);
                ++qh[A];
                ++qh[B];
                if (D::kind == SMC_WK_OR) {                   // OR = not (not a and not b)
                    va = va == 2 ? 2 : 1 - va;
                    vb = vb == 2 ? 2 : 1 - vb;
                }
                int v, r;
                if (va == 0 && vb == 0) { v = 0; r = min(ra, rb); }
                else if (va == 0) { v = 0; r = ra; }
                else if (vb == 0) { v = 0; r = rb; }
                else if (va == 1 && vb == 1) { v = 1; r = max(ra, rb); }
                else { v = 2; r = SMC_WINF; }
                if (D::kind == SMC_WK_OR && v != 2) v = 1 - v;
                emit<I>(v, r);
            }
        }
    }

    template <int I> __device__ __forceinline__ void pump_node(bool fin, bool absorbed, int N) {
        using D = SmcWN<I>;
        if (err || dead<I>()) return;
        if constexpr (D::kind == SMC_WK_F || D::kind == SMC_WK_G) fgnode<I>(fin, absorbed, N);
        else if constexpr (D::kind == SMC_WK_U) temporal<I>(fin, absorbed, N);
        else if constexpr (D::kind == SMC_WK_X) xnode<I>(fin, absorbed, N);
        else if constexpr (D::kind == SMC_WK_NOT || D::kind == SMC_WK_AND || D::kind == SMC_WK_OR) boolean<I>();
    }
    template <int I> __device__ __forceinline__ void pump_from(bool fin, bool absorbed, int N) {
        if constexpr (I < SMC_WIN_NODES) { pump_node<I>(fin, absorbed, N); pump_from<I + 1>(fin, absorbed, N); }
    }
    // oldest ring index still needed (tau_{j-1} / t_j of the next child position of each
    // temporal node, tau_m / t_m of each X node's next position)
    template <int I> __device__ __forceinline__ int ring_lo(int lo_) const {
        if constexpr (I < SMC_WIN_NODES) {
            using D = SmcWN<I>;
            int l = lo_;
            if constexpr (D::kind == SMC_WK_F || D::kind == SMC_WK_G) {
                // the head's t and taus (a later head re-reads them), or only tau_{jc-1} when
                // the head is the node's last position (its running sum carries the rest)
                if (!stop[I] && !dead<I>()) l = min(l, (lo[I] + 1 < D::plim) ? lo[I] : max(lo[I], jc[I] - 1));
            } else if constexpr (D::kind == SMC_WK_U) {
                if (!(stop[I] && lo[I] == hi[I]) && !dead<I>()) l = min(l, qh[D::b] - 1);
            } else if constexpr (D::kind == SMC_WK_X) {
                if (!stop[I] && !dead<I>()) l = min(l, lo[I]);
            }
            return ring_lo<I + 1>(l);
        } else {
            return lo_;
        }
    }
    __device__ __forceinline__ void ring_put(double* a, int k, double v) {
        if (k - ring_lo<0>(k) >= W) { err = true; return; }
        a[k & msk] = v;                                   // every lane writes the same value
    }
    __device__ __forceinline__ void result() {
        if (err) { res = 2; return; }
        if (qt[SMC_WIN_ROOT] > 0) {
            int v, r;
            peek<SMC_WIN_ROOT>(0, v, r);
            if (v != 2) { res = v; decided_at = r; }
        }
    }
    // process the entered entry: leaves emit its position, every node consumes what it can
    __device__ __forceinline__ void process_pending() {
        if (!pend) return;
        pend = false;
        ring_put(tt(), last, pt);
        ne = last + 1;
        if (err) return;
        leaves<0>(last, pt, pmask);
    }

    // ---------------------------------------------------------------- monitor interface
    template <class XA> __device__ __forceinline__ void enter(smc_u32 k, double t, double tp, const XA& x) {
        (void)tp;
        if (res >= 0) return;
        pend = true;
        pmask = smc_lit_mask(x);
        pt = t;
        last = (int)k;
    }
    // the trace ends after entry N (prefix N, sojourn tau_N known unless absorbed)
    __device__ __forceinline__ void finish(int N, bool absorbed) {
        if (!err) pump_from<0>(true, absorbed, N);
        if (err) { res = 2; return; }
        int v = 2, r = N;
        if (qt[SMC_WIN_ROOT] > 0) peek<SMC_WIN_ROOT>(0, v, r);
        if (v == 2) { res = 0; decided_at = N; }          // unknown -> false at the root (R4)
        else { res = v; decided_at = r; }
    }
    __device__ __forceinline__ void advance(smc_u32 k, double tn, double tj) {
        if (res >= 0) return;
        process_pending();
        ring_put(tau(), (int)k, tj);
        ntau = (int)k + 1;
        if (!err) pump_from<0>(false, false, 0);
        result();
        if (res < 0 && tn > SMC_LIT_H) finish((int)k, false);   // the trace covers the horizon
    }
    __device__ __forceinline__ void absorb() {
        if (res >= 0) return;
        process_pending();
        if (!err) pump_from<0>(false, false, 0);
        result();
        if (res < 0) finish(last, true);
    }
    // the event cap reached at entry k (entered, not processed): the prefix up to entry k - 1
    // decides, else the replica is an error
    __device__ __forceinline__ int at_cap(long long k) {
        pend = false;
        if (!err) pump_from<0>(true, false, (int)k - 1);
        int v = 2, r = 0;
        if (!err && qt[SMC_WIN_ROOT] > 0) peek<SMC_WIN_ROOT>(0, v, r);
        if (v == 2) return 2;
        decided_at = r;
        return v;
    }
    __device__ __forceinline__ void timeout() {}
    __device__ __forceinline__ int verdict() const { return res; }
    __device__ __forceinline__ long long events(long long k) const { return decided_at >= 0 ? decided_at : k; }
};
