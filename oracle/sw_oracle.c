/*
 * oracle/sw_oracle.c -- CPU ORACLE for batched Smith-Waterman with affine
 * (Gotoh) gaps.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this code.  The
 * product path (paper_2208_12350_b200/, include/sw.h) never links, includes or
 * calls anything in oracle/, and this file includes nothing from the product:
 * it has its own alphabet tables, its own BLOSUM62 copy and its own scoring
 * struct.
 *
 * What it computes (plain definition, full int32 matrices, no blocking, no
 * fusion, no reordering):
 *
 *   PAPER.md:157-159 (sec. II-B1): H is (n+1) x (m+1); H_ij is the highest
 *     score of an alignment ending in the pair (a_i, b_j).
 *   H_ij = max over the diagonal + s(a_i, b_j), the
 *     vertical and horizontal gap directions, and 0 (local alignment).
 *   PAPER.md:507, 713-714 (Fig. data_exchange): the gap state E is extended
 *     with `extendGap` and opened from H with `startGap` -> affine (Gotoh)
 *     form; a gap of length k scores gap_open + (k-1)*gap_extend
 *     (reading R1).
 *   PAPER.md:165 + Fig. 2 caption: forward pass fills the
 *     matrix and keeps the highest score; the reverse pass recovers where the
 *     alignment starts ("until score zero is reached").
 *
 * Tie rules (the paper is silent; readings R5/R6, SURVEY.md
 * sec. 8(c) C-4/C-5):
 *   end   = lexicographically smallest (j, i) among cells with H = S
 *   start = run the same recurrence on reverse(q[0..q_end]) x
 *           reverse(r[0..r_end]); take the lexicographically smallest
 *           (j', i') with H' = S; q_start = q_end-(i'-1), r_start = r_end-(j'-1)
 *   S == 0 (or an empty sequence)  -> (0, -1, -1, -1, -1)
 *   invalid pair (bad symbol)      -> (-1, -1, -1, -1, -1)
 *
 * Pins (tests/test_oracle_*.py): brute-force enumeration of all local
 * alignments on tiny inputs, the paper's Fig. 2 example (score 7),
 * closed forms (identity, ungapped Kadane, longest common substring), global
 * re-scoring of the reported interval, symmetries, monotonicity, SPEC's
 * diagonal>up>left traceback.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define ORACLE_OK 0
#define ORACLE_BAD_PAIR 1
#define ORACLE_BAD_SCORING 2
#define ORACLE_NO_MEMORY 4
#define ORACLE_REVERSE_MISMATCH 99 /* pin P14 violated: max H' != S */

#define ORACLE_DNA 0
#define ORACLE_PROTEIN 1

typedef struct {
    int32_t alphabet;   /* ORACLE_DNA or ORACLE_PROTEIN                     */
    int32_t match;      /* DNA only                                          */
    int32_t mismatch;   /* DNA only                                          */
    int32_t gap_open;   /* score of the first residue of a gap (negative)    */
    int32_t gap_extend; /* score of each further residue (gap_open <= x <= 0) */
} oracle_scoring;

/* NCBI BLOSUM62, order ARNDCQEGHILKMFPSTWYVBZX* (
 * DESIGN.md reading R11).  Own copy: the product has a separate one. */
static const char PROT_ORDER[25] = "ARNDCQEGHILKMFPSTWYVBZX*";
static const int8_t BLOSUM62[24][24] = {
/*        A   R   N   D   C   Q   E   G   H   I   L   K   M   F   P   S   T   W   Y   V   B   Z   X   * */
/* A */ { 4, -1, -2, -2,  0, -1, -1,  0, -2, -1, -1, -1, -1, -2, -1,  1,  0, -3, -2,  0, -2, -1,  0, -4},
/* R */ {-1,  5,  0, -2, -3,  1,  0, -2,  0, -3, -2,  2, -1, -3, -2, -1, -1, -3, -2, -3, -1,  0, -1, -4},
/* N */ {-2,  0,  6,  1, -3,  0,  0,  0,  1, -3, -3,  0, -2, -3, -2,  1,  0, -4, -2, -3,  3,  0, -1, -4},
/* D */ {-2, -2,  1,  6, -3,  0,  2, -1, -1, -3, -4, -1, -3, -3, -1,  0, -1, -4, -3, -3,  4,  1, -1, -4},
/* C */ { 0, -3, -3, -3,  9, -3, -4, -3, -3, -1, -1, -3, -1, -2, -3, -1, -1, -2, -2, -1, -3, -3, -2, -4},
/* Q */ {-1,  1,  0,  0, -3,  5,  2, -2,  0, -3, -2,  1,  0, -3, -1,  0, -1, -2, -1, -2,  0,  3, -1, -4},
/* E */ {-1,  0,  0,  2, -4,  2,  5, -2,  0, -3, -3,  1, -2, -3, -1,  0, -1, -3, -2, -2,  1,  4, -1, -4},
/* G */ { 0, -2,  0, -1, -3, -2, -2,  6, -2, -4, -4, -2, -3, -3, -2,  0, -2, -2, -3, -3, -1, -2, -1, -4},
/* H */ {-2,  0,  1, -1, -3,  0,  0, -2,  8, -3, -3, -1, -2, -1, -2, -1, -2, -2,  2, -3,  0,  0, -1, -4},
/* I */ {-1, -3, -3, -3, -1, -3, -3, -4, -3,  4,  2, -3,  1,  0, -3, -2, -1, -3, -1,  3, -3, -3, -1, -4},
/* L */ {-1, -2, -3, -4, -1, -2, -3, -4, -3,  2,  4, -2,  2,  0, -3, -2, -1, -2, -1,  1, -4, -3, -1, -4},
/* K */ {-1,  2,  0, -1, -3,  1,  1, -2, -1, -3, -2,  5, -1, -3, -1,  0, -1, -3, -2, -2,  0,  1, -1, -4},
/* M */ {-1, -1, -2, -3, -1,  0, -2, -3, -2,  1,  2, -1,  5,  0, -2, -1, -1, -1, -1,  1, -3, -1, -1, -4},
/* F */ {-2, -3, -3, -3, -2, -3, -3, -3, -1,  0,  0, -3,  0,  6, -4, -2, -2,  1,  3, -1, -3, -3, -1, -4},
/* P */ {-1, -2, -2, -1, -3, -1, -1, -2, -2, -3, -3, -1, -2, -4,  7, -1, -1, -4, -3, -2, -2, -1, -2, -4},
/* S */ { 1, -1,  1,  0, -1,  0,  0,  0, -1, -2, -2,  0, -1, -2, -1,  4,  1, -3, -2, -2,  0,  0,  0, -4},
/* T */ { 0, -1,  0, -1, -1, -1, -1, -2, -2, -1, -1, -1, -1, -2, -1,  1,  5, -2, -2,  0, -1, -1,  0, -4},
/* W */ {-3, -3, -4, -4, -2, -2, -3, -2, -2, -3, -2, -3, -1,  1, -4, -3, -2, 11,  2, -3, -4, -3, -2, -4},
/* Y */ {-2, -2, -2, -3, -2, -1, -2, -3,  2, -1, -1, -2, -1,  3, -3, -2, -2,  2,  7, -1, -3, -2, -1, -4},
/* V */ { 0, -3, -3, -3, -1, -2, -2, -3, -3,  3,  1, -2,  1, -1, -2, -2,  0, -3, -1,  4, -3, -2, -1, -4},
/* B */ {-2, -1,  3,  4, -3,  0,  1, -1,  0, -3, -4,  0, -3, -3, -2,  0, -1, -4, -3, -3,  4,  1, -1, -4},
/* Z */ {-1,  0,  0,  1, -3,  3,  4, -2,  0, -3, -3,  1, -1, -3, -1,  0, -1, -3, -2, -2,  1,  4, -1, -4},
/* X */ { 0, -1, -1, -1, -2, -1, -1, -1, -1, -1, -1, -1, -1, -1, -2,  0,  0, -2, -1, -1, -1, -1, -1, -4},
/* * */ {-4, -4, -4, -4, -4, -4, -4, -4, -4, -4, -4, -4, -4, -4, -4, -4, -4, -4, -4, -4, -4, -4, -4,  1},
};

/* Symbol -> code, case-insensitive; -1 if not in the alphabet
 * (reading R10: DNA = ACGT only, protein = the 24 BLOSUM62 symbols). */
static int oracle_code(int32_t alphabet, uint8_t ch)
{
    if (ch >= 'a' && ch <= 'z') ch = (uint8_t)(ch - 'a' + 'A');
    if (alphabet == ORACLE_DNA) {
        switch (ch) {
        case 'A': return 0;
        case 'C': return 1;
        case 'G': return 2;
        case 'T': return 3;
        default: return -1;
        }
    }
    for (int k = 0; k < 24; ++k)
        if ((uint8_t)PROT_ORDER[k] == ch) return k;
    return -1;
}

/* s(a_i, b_j) of PAPER.md:161-162 */
static int32_t oracle_sigma(const oracle_scoring* sc, int a, int b)
{
    if (sc->alphabet == ORACLE_DNA) return a == b ? sc->match : sc->mismatch;
    return BLOSUM62[a][b];
}

int oracle_blosum62(int a, int b) { return BLOSUM62[a][b]; }

/* Preconditions (reading R3): o < 0, o <= e <= 0; DNA: match > 0,
 * mismatch < match; magnitudes bounded so int32 cannot overflow. */
int oracle_check_scoring(const oracle_scoring* sc)
{
    if (sc->alphabet != ORACLE_DNA && sc->alphabet != ORACLE_PROTEIN) return ORACLE_BAD_SCORING;
    if (!(sc->gap_open < 0)) return ORACLE_BAD_SCORING;
    if (!(sc->gap_open <= sc->gap_extend && sc->gap_extend <= 0)) return ORACLE_BAD_SCORING;
    if (sc->gap_open < -32768) return ORACLE_BAD_SCORING;
    if (sc->alphabet == ORACLE_DNA) {
        if (!(sc->match > 0) || !(sc->mismatch < sc->match)) return ORACLE_BAD_SCORING;
        if (sc->match > 32767 || sc->mismatch < -32768) return ORACLE_BAD_SCORING;
    }
    return ORACLE_OK;
}

#define NEG_INF (INT32_MIN / 4)
#define IDX(i, j) ((size_t)(i) * (size_t)(mcols) + (size_t)(j))

/*
 * C-2: fill full (n+1) x (m+1) matrices H, E, F for
 * query codes q (rows i) and reference codes r (columns j).
 *   H[i][0] = H[0][j] = 0, E[i][0] = -inf, F[0][j] = -inf
 *   E[i][j] = max(E[i][j-1] + e, H[i][j-1] + o)      horizontal gap
 *   F[i][j] = max(F[i-1][j] + e, H[i-1][j] + o)      vertical gap
 *   H[i][j] = max(0, H[i-1][j-1] + s(q_{i-1}, r_{j-1}), E[i][j], F[i][j])
 * H must have (n+1)*(m+1) entries; E and F too.
 */
static void oracle_fill(const int* q, int64_t n, const int* r, int64_t m,
                        const oracle_scoring* sc, int32_t* H, int32_t* E, int32_t* F)
{
    const int64_t mcols = m + 1;
    const int32_t o = sc->gap_open, e = sc->gap_extend;
    for (int64_t j = 0; j <= m; ++j) { H[IDX(0, j)] = 0; E[IDX(0, j)] = NEG_INF; F[IDX(0, j)] = NEG_INF; }
    for (int64_t i = 1; i <= n; ++i) {
        H[IDX(i, 0)] = 0; E[IDX(i, 0)] = NEG_INF; F[IDX(i, 0)] = NEG_INF;
        for (int64_t j = 1; j <= m; ++j) {
            int32_t ev = E[IDX(i, j - 1)] + e;
            int32_t eo = H[IDX(i, j - 1)] + o;
            int32_t Ev = ev > eo ? ev : eo;
            int32_t fv = F[IDX(i - 1, j)] + e;
            int32_t fo = H[IDX(i - 1, j)] + o;
            int32_t Fv = fv > fo ? fv : fo;
            int32_t h = 0;
            int32_t d = H[IDX(i - 1, j - 1)] + oracle_sigma(sc, q[i - 1], r[j - 1]);
            if (d > h) h = d;
            if (Ev > h) h = Ev;
            if (Fv > h) h = Fv;
            E[IDX(i, j)] = Ev;
            F[IDX(i, j)] = Fv;
            H[IDX(i, j)] = h;
        }
    }
}

/* C-3 / C-4: S = max H; the lexicographically smallest (j, i) holding S.
 * Returns S; *bi, *bj are 1-based matrix indices (0 if S == 0). */
static int32_t oracle_argmax(const int32_t* H, int64_t n, int64_t m, int64_t* bi, int64_t* bj)
{
    const int64_t mcols = m + 1;
    int32_t S = 0;
    for (int64_t i = 1; i <= n; ++i)
        for (int64_t j = 1; j <= m; ++j)
            if (H[IDX(i, j)] > S) S = H[IDX(i, j)];
    *bi = 0; *bj = 0;
    if (S == 0) return 0;
    for (int64_t j = 1; j <= m; ++j)          /* column-major scan: smallest j first */
        for (int64_t i = 1; i <= n; ++i)      /* then smallest i                      */
            if (H[IDX(i, j)] == S) { *bi = i; *bj = j; return S; }
    return S; /* unreachable */
}

/* Full-matrix H of one pair (for tests, e.g. the Fig. 2 matrix).  H_out must
 * hold (n+1)*(m+1) int32.  Returns an ORACLE_* status. */
int oracle_fill_H(const uint8_t* qs, int64_t n, const uint8_t* rs, int64_t m,
                  const oracle_scoring* sc, int32_t* H_out)
{
    if (oracle_check_scoring(sc)) return ORACLE_BAD_SCORING;
    if (n < 0 || m < 0) return ORACLE_BAD_PAIR;
    int* q = (int*)malloc(sizeof(int) * (size_t)(n + 1));
    int* r = (int*)malloc(sizeof(int) * (size_t)(m + 1));
    size_t cells = (size_t)(n + 1) * (size_t)(m + 1);
    int32_t* E = (int32_t*)malloc(sizeof(int32_t) * cells);
    int32_t* F = (int32_t*)malloc(sizeof(int32_t) * cells);
    int st = ORACLE_OK;
    if (!q || !r || !E || !F) { st = ORACLE_NO_MEMORY; goto done; }
    for (int64_t i = 0; i < n; ++i) if ((q[i] = oracle_code(sc->alphabet, qs[i])) < 0) { st = ORACLE_BAD_PAIR; goto done; }
    for (int64_t j = 0; j < m; ++j) if ((r[j] = oracle_code(sc->alphabet, rs[j])) < 0) { st = ORACLE_BAD_PAIR; goto done; }
    oracle_fill(q, n, r, m, sc, H_out, E, F);
done:
    free(q); free(r); free(E); free(F);
    return st;
}

/*
 * One pair: C-1 .. C-5.  out = {score, q_end, r_end, q_start, r_start}.
 * Returns ORACLE_OK, ORACLE_BAD_PAIR (out = all -1), ORACLE_NO_MEMORY or
 * ORACLE_REVERSE_MISMATCH (pin P14 broken -- must never happen).
 */
int oracle_align(const uint8_t* qs, int64_t n, const uint8_t* rs, int64_t m,
                 const oracle_scoring* sc, int32_t out[5])
{
    for (int k = 0; k < 5; ++k) out[k] = -1;
    if (oracle_check_scoring(sc)) return ORACLE_BAD_SCORING;
    if (n < 0 || m < 0) return ORACLE_BAD_PAIR;
    int* q = (int*)malloc(sizeof(int) * (size_t)(n + 1));
    int* r = (int*)malloc(sizeof(int) * (size_t)(m + 1));
    if (!q || !r) { free(q); free(r); return ORACLE_NO_MEMORY; }
    for (int64_t i = 0; i < n; ++i) if ((q[i] = oracle_code(sc->alphabet, qs[i])) < 0) { free(q); free(r); return ORACLE_BAD_PAIR; }
    for (int64_t j = 0; j < m; ++j) if ((r[j] = oracle_code(sc->alphabet, rs[j])) < 0) { free(q); free(r); return ORACLE_BAD_PAIR; }

    out[0] = 0; /* S = 0 convention (reading R7): coordinates stay -1 */
    if (n == 0 || m == 0) { free(q); free(r); return ORACLE_OK; }

    size_t cells = (size_t)(n + 1) * (size_t)(m + 1);
    int32_t* H = (int32_t*)malloc(sizeof(int32_t) * cells);
    int32_t* E = (int32_t*)malloc(sizeof(int32_t) * cells);
    int32_t* F = (int32_t*)malloc(sizeof(int32_t) * cells);
    int st = ORACLE_OK;
    if (!H || !E || !F) { st = ORACLE_NO_MEMORY; goto done; }

    /* forward pass ("iterating ... from top left to bottom right") */
    oracle_fill(q, n, r, m, sc, H, E, F);
    int64_t bi, bj;
    int32_t S = oracle_argmax(H, n, m, &bi, &bj);
    out[0] = S;
    if (S == 0) goto done;
    int64_t q_end = bi - 1, r_end = bj - 1;
    out[1] = (int32_t)q_end;
    out[2] = (int32_t)r_end;

    /* reverse pass (C-5): the same recurrence on the reversed prefixes */
    {
        int64_t n2 = q_end + 1, m2 = r_end + 1;
        int* q2 = (int*)malloc(sizeof(int) * (size_t)n2);
        int* r2 = (int*)malloc(sizeof(int) * (size_t)m2);
        if (!q2 || !r2) { free(q2); free(r2); st = ORACLE_NO_MEMORY; goto done; }
        for (int64_t i = 0; i < n2; ++i) q2[i] = q[q_end - i];
        for (int64_t j = 0; j < m2; ++j) r2[j] = r[r_end - j];
        /* the reversed rectangle is no larger than the forward one: reuse buffers */
        oracle_fill(q2, n2, r2, m2, sc, H, E, F);
        int64_t ri, rj;
        int32_t S2 = oracle_argmax(H, n2, m2, &ri, &rj);
        free(q2); free(r2);
        if (S2 != S) { st = ORACLE_REVERSE_MISMATCH; goto done; }
        out[3] = (int32_t)(q_end - (ri - 1));
        out[4] = (int32_t)(r_end - (rj - 1));
    }
done:
    free(q); free(r); free(H); free(E); free(F);
    if (st == ORACLE_NO_MEMORY || st == ORACLE_REVERSE_MISMATCH) for (int k = 0; k < 5; ++k) out[k] = -2;
    return st;
}

/* ------------------------------------------------------------- traceback */

/*
 * Alignment path of a pair (reading R20).
 * Given the pair's (S, q_end, r_end, q_start, r_start) from oracle_align with
 * S > 0, the path is an optimal GLOBAL affine alignment of the substrings
 * A = q[q_start..q_end] and B = r[r_start..r_end] (its score equals S: it is a
 * local alignment, so <= S, and the reported alignment is one, so >= S), taken
 * by the traceback of PAPER.md:153 / 165 ("tracing back from the highest
 * score") from the bottom-right cell.  Among all optimal alignments it is the
 * one whose op string, read from the end, is lexicographically greatest with
 * M > I > D -- SPEC.md:395/464's diagonal > up > left, where 'M' is an aligned
 * pair, 'I' a query residue against a gap (vertical, state F) and 'D' a
 * reference residue against a gap (horizontal, state E).  As a state machine:
 *   H state: diagonal optimal -> 'M'; else H == F -> F state; else E state.
 *   F state ('I', consuming query row i): go back to H if the gap opened here
 *     and the cell above prefers the diagonal (next op 'M'); else stay in F if
 *     the gap extends here or the cell above prefers F (next op 'I'); else H.
 *   E state ('D', consuming reference column j): back to H if the gap opened
 *     here and the cell to the left prefers the diagonal or F (next op 'M' or
 *     'I'); else stay in E (next op 'D').
 * Global recurrence (no 0 term; gap of length k scores o + (k-1) e, R1):
 *   H[0][0] = 0, H[i][0] = F[i][0] = o + (i-1) e, H[0][j] = E[0][j] = o + (j-1) e
 *   E[i][j] = max(E[i][j-1] + e, H[i][j-1] + o)
 *   F[i][j] = max(F[i-1][j] + e, H[i-1][j] + o)
 *   H[i][j] = max(H[i-1][j-1] + s(A_i, B_j), E[i][j], F[i][j])
 * ops (a + b bytes capacity) receives the ops from start to end; returns the
 * number of ops, 0 for S == 0, -1 for an invalid pair or scoring, -2 if the
 * global optimum differs from S (must never happen).
 */
#define ORACLE_NEG_INF (-(1 << 28))
int oracle_traceback(const uint8_t* qs, int64_t n, const uint8_t* rs, int64_t m, const oracle_scoring* sc,
                     const int32_t res[5], char* ops)
{
    if (oracle_check_scoring(sc)) return -1;
    const int32_t S = res[0];
    if (S < 0) return -1;
    if (S == 0) return 0;
    const int64_t q0 = res[3], q1 = res[1], r0 = res[4], r1 = res[2];
    if (q0 < 0 || r0 < 0 || q1 < q0 || r1 < r0 || q1 >= n || r1 >= m) return -1;
    const int64_t a = q1 - q0 + 1, b = r1 - r0 + 1;
    int* A = (int*)malloc(sizeof(int) * (size_t)a);
    int* B = (int*)malloc(sizeof(int) * (size_t)b);
    size_t cells = (size_t)(a + 1) * (size_t)(b + 1);
    int32_t* H = (int32_t*)malloc(sizeof(int32_t) * cells);
    int32_t* E = (int32_t*)malloc(sizeof(int32_t) * cells);
    int32_t* F = (int32_t*)malloc(sizeof(int32_t) * cells);
    char* rev = (char*)malloc((size_t)(a + b));
    int ret = -1;
    if (!A || !B || !H || !E || !F || !rev) goto done;
    for (int64_t i = 0; i < a; ++i) if ((A[i] = oracle_code(sc->alphabet, qs[q0 + i])) < 0) goto done;
    for (int64_t j = 0; j < b; ++j) if ((B[j] = oracle_code(sc->alphabet, rs[r0 + j])) < 0) goto done;
    {
        const int32_t o = sc->gap_open, e = sc->gap_extend;
#define AT(X, i, j) X[(size_t)(i) * (size_t)(b + 1) + (size_t)(j)]
        AT(H, 0, 0) = 0; AT(E, 0, 0) = ORACLE_NEG_INF; AT(F, 0, 0) = ORACLE_NEG_INF;
        for (int64_t j = 1; j <= b; ++j) {
            AT(H, 0, j) = o + (int32_t)(j - 1) * e; AT(E, 0, j) = AT(H, 0, j); AT(F, 0, j) = ORACLE_NEG_INF;
        }
        for (int64_t i = 1; i <= a; ++i) {
            AT(H, i, 0) = o + (int32_t)(i - 1) * e; AT(F, i, 0) = AT(H, i, 0); AT(E, i, 0) = ORACLE_NEG_INF;
            for (int64_t j = 1; j <= b; ++j) {
                int32_t ev = AT(E, i, j - 1) + e, eo = AT(H, i, j - 1) + o;
                int32_t fv = AT(F, i - 1, j) + e, fo = AT(H, i - 1, j) + o;
                AT(E, i, j) = ev > eo ? ev : eo;
                AT(F, i, j) = fv > fo ? fv : fo;
                int32_t d = AT(H, i - 1, j - 1) + oracle_sigma(sc, A[i - 1], B[j - 1]);
                int32_t h = d;
                if (AT(F, i, j) > h) h = AT(F, i, j);
                if (AT(E, i, j) > h) h = AT(E, i, j);
                AT(H, i, j) = h;
            }
        }
        if (AT(H, a, b) != S) { ret = -2; goto done; }
        /* preferred move out of H at (i, j): 0 diagonal, 1 F (vertical), 2 E (horizontal) */
#define h_pref(ii, jj) ((ii) > 0 && (jj) > 0 && AT(H, ii, jj) == AT(H, (ii) - 1, (jj) - 1) + oracle_sigma(sc, A[(ii) - 1], B[(jj) - 1]) ? 0 \
                        : ((ii) > 0 && AT(H, ii, jj) == AT(F, ii, jj)) ? 1 : 2)
        /* traceback from (a, b) in state H */
        int64_t i = a, j = b, k = 0;
        int state = 0; /* 0 = H, 1 = F (vertical), 2 = E (horizontal) */
        while (i > 0 || j > 0) {
            if (state == 0) {
                if (i > 0 && j > 0 && AT(H, i, j) == AT(H, i - 1, j - 1) + oracle_sigma(sc, A[i - 1], B[j - 1])) {
                    rev[k++] = 'M'; --i; --j;
                } else if (i > 0 && AT(H, i, j) == AT(F, i, j)) {
                    state = 1;
                } else {
                    state = 2;
                }
            } else if (state == 1) {
                rev[k++] = 'I';
                const int open = AT(F, i, j) == AT(H, i - 1, j) + o;
                const int ext = AT(F, i, j) == AT(F, i - 1, j) + e;
                const int up = h_pref(i - 1, j);
                if (open && up == 0) state = 0;
                else if (ext || (open && up == 1)) state = 1;
                else state = 0;
                --i;
            } else {
                rev[k++] = 'D';
                const int open = AT(E, i, j) == AT(H, i, j - 1) + o;
                const int left = h_pref(i, j - 1);
                state = (open && left != 2) ? 0 : 2;
                --j;
            }
        }
#undef h_pref
#undef AT
        for (int64_t t = 0; t < k; ++t) ops[t] = rev[k - 1 - t];
        ret = (int)k;
    }
done:
    free(A); free(B); free(H); free(E); free(F); free(rev);
    return ret;
}

/* ------------------------------------------------------------------ batch */

typedef struct {
    const uint8_t* queries; const int64_t* q_off;
    const uint8_t* refs;    const int64_t* r_off;
    const oracle_scoring* sc;
    int32_t *score, *q_end, *r_end, *q_start, *r_start;
    const int64_t* order;   /* longest first */
    int64_t n_pairs;
    int64_t next;           /* shared work counter */
    pthread_mutex_t lock;
    int worst_status;
} oracle_job;

static int cmp_cost_desc(const void* a, const void* b)
{
    const int64_t* x = (const int64_t*)a; const int64_t* y = (const int64_t*)b;
    if (x[0] != y[0]) return x[0] < y[0] ? 1 : -1;  /* cost descending */
    return x[1] < y[1] ? -1 : (x[1] > y[1]);          /* index ascending */
}

static void* oracle_worker(void* arg)
{
    oracle_job* job = (oracle_job*)arg;
    for (;;) {
        pthread_mutex_lock(&job->lock);
        int64_t k = job->next++;
        pthread_mutex_unlock(&job->lock);
        if (k >= job->n_pairs) break;
        int64_t p = job->order[k];
        int64_t n = job->q_off[p + 1] - job->q_off[p];
        int64_t m = job->r_off[p + 1] - job->r_off[p];
        int32_t out[5];
        int st = oracle_align(job->queries + job->q_off[p], n, job->refs + job->r_off[p], m, job->sc, out);
        job->score[p] = out[0]; job->q_end[p] = out[1]; job->r_end[p] = out[2];
        job->q_start[p] = out[3]; job->r_start[p] = out[4];
        if (st == ORACLE_NO_MEMORY || st == ORACLE_REVERSE_MISMATCH) {
            pthread_mutex_lock(&job->lock);
            if (st > job->worst_status) job->worst_status = st;
            pthread_mutex_unlock(&job->lock);
        }
    }
    return NULL;
}

/*
 * Batch over CSR arrays (host memory): pair p is queries[q_off[p]..q_off[p+1])
 * vs refs[r_off[p]..r_off[p+1]).  Pairs run longest-first on n_threads POSIX
 * threads.  Per-pair errors are encoded in the outputs (all -1); the return
 * value is ORACLE_OK, ORACLE_BAD_SCORING, ORACLE_NO_MEMORY or
 * ORACLE_REVERSE_MISMATCH.
 */
int oracle_align_batch(const uint8_t* queries, const int64_t* q_off,
                       const uint8_t* refs, const int64_t* r_off, int64_t n_pairs,
                       const oracle_scoring* sc,
                       int32_t* score, int32_t* q_end, int32_t* r_end,
                       int32_t* q_start, int32_t* r_start, int n_threads)
{
    if (oracle_check_scoring(sc)) return ORACLE_BAD_SCORING;
    if (n_pairs <= 0) return ORACLE_OK;
    if (n_threads < 1) n_threads = 1;
    int64_t* keyed = (int64_t*)malloc(sizeof(int64_t) * 2 * (size_t)n_pairs);
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)n_pairs);
    if (!keyed || !order) { free(keyed); free(order); return ORACLE_NO_MEMORY; }
    for (int64_t p = 0; p < n_pairs; ++p) {
        int64_t n = q_off[p + 1] - q_off[p], m = r_off[p + 1] - r_off[p];
        keyed[2 * p] = (n > 0 && m > 0) ? n * m : 0;
        keyed[2 * p + 1] = p;
    }
    qsort(keyed, (size_t)n_pairs, 2 * sizeof(int64_t), cmp_cost_desc);
    for (int64_t k = 0; k < n_pairs; ++k) order[k] = keyed[2 * k + 1];
    free(keyed);

    oracle_job job;
    job.queries = queries; job.q_off = q_off; job.refs = refs; job.r_off = r_off;
    job.sc = sc; job.score = score; job.q_end = q_end; job.r_end = r_end;
    job.q_start = q_start; job.r_start = r_start; job.order = order;
    job.n_pairs = n_pairs; job.next = 0; job.worst_status = ORACLE_OK;
    pthread_mutex_init(&job.lock, NULL);
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n_threads);
    int started = 0;
    for (int t = 0; t < n_threads; ++t)
        if (pthread_create(&th[t], NULL, oracle_worker, &job) == 0) ++started;
    if (started == 0) oracle_worker(&job);
    for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
    free(th);
    pthread_mutex_destroy(&job.lock);
    free(order);
    return job.worst_status;
}
