// occ_v2_kernel.cuh -- body of the fused TMEM-resident step kernel (included
// once, by occ_v2.cu).  Design and fragment bookkeeping: occ_v2.cuh.
//
// Index permutations used below (legal because a contraction index, and the
// row/column order of an MMA output, may be permuted as long as both operands
// and the consumer of the result agree):
//  * phase 1, P^T = Q^T A^T (K = tile columns): k-index t <-> column 2t and
//    t+4 <-> 2t+1 of an 8-column k-step, so a lane's B-operand pair is one
//    8-byte shared load;
//  * the cell layout (phases 1/3/5): lane (g,t) owns rows {t, t+4} x columns
//    {2g, 2g+1} of the 8 x 16 cell, so phase-3 K (rows) is the identity map,
//    phase-3/5 column n <-> 2n (n < 8), 2(n-8)+1 (n >= 8), phase-5 N (rows)
//    n <-> n/2 + 4 (n & 1), and phase-5 stores are 8-byte pairs.
#pragma once

template <int R, bool MBF>
__global__ void __launch_bounds__(NT, 1) occ_v2_kernel(const __grid_constant__ Params2 p) {
  constexpr int RP = K<R>::RP, MT = K<R>::MT, KS5 = K<R>::KS5, NP = K<R>::NP;
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t mbar[2 * MAX_STAGES];   // full[], empty[]
  __shared__ unsigned tmem_base_sh;

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, t = lane & 3;
  const Tile T = tile_of(p);
  const bool active = T.rb < p.nr && T.th > 0 && T.tw > 0;
  unsigned nb = 0;
  auto gbar = [&]() { nb++; grid_barrier_spread(p.barl, nb); };
#ifdef OCC_TRACE
  // Instrumented build (libocc_trace.so, tools/trace.py): per-CTA phase stamps
  // and timing experiments.  The product build compiles all of it out: its
  // instructions would occupy the instruction cache the hot path needs.
  constexpr bool kTrace = true;
  const bool stamp = blockIdx.x == 0 && tid == 0;
  auto tr = [&](int k) {   // per-CTA phase trace (occ_read_trace)
    if (tid == 0) {
      p.trace[blockIdx.x * (2 * kTrStamps) + k] = clock64();
      p.trace[blockIdx.x * (2 * kTrStamps) + kTrStamps + k] = gtimer();
    }
  };
  auto trw = [&](int k) {   // stamp from lane 0 of the calling warp
    if (lane == 0) {
      p.trace[blockIdx.x * (2 * kTrStamps) + k] = clock64();
      p.trace[blockIdx.x * (2 * kTrStamps) + kTrStamps + k] = gtimer();
    }
  };
#else
  constexpr bool kTrace = false;
  constexpr bool stamp = false;
  auto tr = [](int) {};
  auto trw = [](int) {};
#endif
  if (stamp) p.stats->t_ns[0] = gtimer();
  tr(0);

  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  {   // the staging ring starts zeroed: rows a partial last stage does not copy and the row padding are
      // read (multiplied by zero factors), so they must hold finite values, never stale NaN bit patterns
    uint4* z = reinterpret_cast<uint4*>(sm + p.off_stm);
    const int nz = (p.off_qs - p.off_stm) / 16;
    for (int x = tid; x < nz; x += NT) z[x] = make_uint4(0u, 0u, 0u, 0u);
  }
  if (tid == 0) {
    for (int s = 0; s < MAX_STAGES; s++) {
      mbar_init(&mbar[s], 1);                      // full: the producer's expect_tx arrival
      mbar_init(&mbar[MAX_STAGES + s], NCW);       // empty: one arrival per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tbase = tmem_base_sh;
  // programmatic dependent launch: everything above touched only shared and
  // tensor memory; global memory (inputs, workspace barrier words) waits for
  // the previous grid in the stream to complete (a no-op without PDL)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // TMEM: warp w reaches lanes 32 (w % 4) ..; the warps sharing a lane quadrant split its 512 columns
  const unsigned taddr_w = tbase + ((unsigned)((w & 3) * 32) << 16) + (unsigned)((w >> 2) * (512 / (NW / 4)));
  // TMEM slot of a cell: column-group major, so one column group's cells are contiguous
  auto cell_slot = [&](int rblk, int cg) { return (cg / NCW) * T.nrblk + rblk; };
  auto consumer_sync = [&]() { asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32) : "memory"); };

  // ============================================================== phase 1
  unsigned char* stM = sm + p.off_stm;
  float* stE = reinterpret_cast<float*>(sm + p.off_ste);  // e, then A = M + e
  float* qs = reinterpret_cast<float*>(sm + p.off_qs);    // [W][RP] Q_prev slice (r > 16)
  float* red = reinterpret_cast<float*>(sm + p.off_red);  // [NCW][nrblk][8][RP] per-warp P partials
  const int nst = active ? T.nrblk : 0;
  const size_t esz = MBF ? 2 : 4;
  uint64_t* full = mbar;
  uint64_t* empty = mbar + MAX_STAGES;
  const int sw = p.sw;
  // one stage = SR rows of M and e: the expect_tx arrival (lane 0), then one
  // bulk copy per row and matrix, issued by 2 SR lanes of the producer warp in
  // one instruction (a single issuing thread caps a CTA at ~40 GB/s of 2 KB copies)
  const unsigned long long pol_ef = l2_evict_first();
  // stores: evict-first by default; OCC_V2_DEBUG bit 1024: the normal policy (experiment)
  const unsigned long long pol_st = (p.debug & 1024) ? l2_evict_normal() : pol_ef;
  auto issue = [&](int s) {
    const int slot = s % p.ns;
    const int r0 = s * SR, nrow = min(SR, T.th - r0);
    const unsigned rbM = (unsigned)(T.tw * esz), rbE = (unsigned)(T.tw * 4);
    if (lane == 0) mbar_expect_tx(&full[slot], (unsigned)nrow * (rbM + (p.err_in ? rbE : 0u)));
    __syncwarp();
    const int i = lane >> 1;
    if (i < nrow) {
      const size_t gi = (size_t)(T.row0 + r0 + i);
      if ((lane & 1) == 0)
        bulk_g2s_hint(stM + ((size_t)(slot * SR + i) * sw) * 4,
                      reinterpret_cast<const char*>(p.M) + (gi * p.ldm + T.col0) * esz, rbM, &full[slot], pol_ef);
      else if (p.err_in)
        bulk_g2s_hint(stE + (size_t)(slot * SR + i) * sw, p.err_in + gi * p.lde_in + T.col0, rbE, &full[slot], pol_ef);
    }
  };
  // Q_prev^T fragments (A operand, 3-term split) of this warp's k-steps
  constexpr bool QREG = (R <= 16);
  constexpr int KREG = QREG ? (R <= 8 ? 8 : 4) : 1;
  const int nk = T.tw / 8;
  unsigned qf[KREG][MT][8];
  auto qfrag = [&](const float* src, int ld, int c, int mt, unsigned (&f)[8]) {
    const int k0 = 16 * mt + g;
    const float* r0 = src + (size_t)(c + 2 * t) * ld;
    const float* r1 = r0 + ld;
    const float v0 = (k0 < R) ? r0[k0] : 0.f;
    const float v1 = (k0 + 8 < R) ? r0[k0 + 8] : 0.f;
    const float v2 = (k0 < R) ? r1[k0] : 0.f;
    const float v3 = (k0 + 8 < R) ? r1[k0 + 8] : 0.f;
    split3(v0, f[0], f[4]); split3(v1, f[1], f[5]); split3(v2, f[2], f[6]); split3(v3, f[3], f[7]);
  };
  unsigned long long wait_ns = 0;
  if (w == NW - 1) {
    // ---------------- producer
    if (active) {   // the whole producer warp (copies issued by 2 SR lanes)
      for (int s = 0; s < nst; s++) {
        const int slot = s % p.ns;
        if (s >= p.ns) mbar_wait(&empty[slot], (unsigned)(((s / p.ns) - 1) & 1));
        issue(s);
      }
    }
  } else {
    // ---------------- consumers
    if (active) {
      if constexpr (QREG) {
#pragma unroll
        for (int j = 0; j < KREG; j++) {
          const int kk = w + NCW * j;
#pragma unroll
          for (int mt = 0; mt < MT; mt++) {
            if (kk < nk) qfrag(p.Qprev + (size_t)T.col0 * R, R, 8 * kk, mt, qf[j][mt]);
            else for (int q = 0; q < 8; q++) qf[j][mt][q] = 0u;
          }
        }
      } else {
        for (int x = tid; x < T.tw * RP; x += NCW * 32) {
          const int c = x / RP, k = x % RP;
          qs[x] = (k < R) ? __ldcg(p.Qprev + (size_t)(T.col0 + c) * R + k) : 0.f;
        }
        consumer_sync();
      }
    }
    if (stamp) p.stats->t_ns[7] = gtimer();
    // One stage = SR rows.  Per lane, everything that does not change from stage
    // to stage is computed once: the staging offsets of its k-step B operands
    // (row g, columns 8 kk + 2t; a k-step past the tile reads column 2t, finite
    // data times the zero Q fragment, so the loop has no per-k-step branch) and
    // of its TMEM cells (rows t, t+4, columns 16 cg + 2g).  Rows past a partial
    // last stage are not masked: they hold finite staging data (the ring starts
    // zeroed) and only ever meet zero P rows or bounds-checked stores.  The
    // slot / parity counters replace a division per stage.
    auto consume = [&](auto he) {
      constexpr bool HASE = decltype(he)::value;
      constexpr int MS = MBF ? 2 : 1;   // M staging: element units per float of the row stride
      int offB[KREG];   // column of the k-step B operand (row g)
#pragma unroll
      for (int j = 0; j < KREG; j++) {
        const int kk = w + NCW * j;
        offB[j] = (kk < nk ? 8 * kk : 0) + 2 * t;
      }
      const int ncw = T.ncg > w ? (T.ncg - w + NCW - 1) / NCW : 0;   // TMEM column groups of this warp
      const int colC = 16 * w + 2 * g;                                // its first cell's column
      int slot = 0;
      unsigned par = 0;
      for (int s = 0; s < nst; s++) {
        const unsigned long long tw0 = stamp ? gtimer() : 0;
        mbar_wait(&full[slot], par);
        if (stamp) wait_ns += gtimer() - tw0;
        if (kTrace && (p.debug & 1)) {   // streaming-floor experiment: consume the slot without computing
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[slot]);
          if (++slot == p.ns) { slot = 0; par ^= 1u; }
          continue;
        }
        const unsigned char* sMb = stM + (size_t)slot * SR * sw * 4;
        const float* sEb = stE + (size_t)slot * SR * sw;
        // A[i][j..j+1] = M + e (FADD2); M rows are sw floats = MS sw elements apart
        auto A2 = [&](int i, int j) -> float2 {
          float2 a;
          if (MBF) a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(
                       reinterpret_cast<const __nv_bfloat16*>(sMb) + (i * MS * sw + j)));
          else a = *reinterpret_cast<const float2*>(reinterpret_cast<const float*>(sMb) + (i * sw + j));
          if (HASE) a = add2(a, *reinterpret_cast<const float2*>(sEb + (i * sw + j)));
          return a;
        };
        // (a) P^T[k][rows] = Q_prev^T[k][cols] A^T[cols][rows]; warps split the column k-steps,
        //     one accumulator chain per k-step (independent MMA chains)
        float acc[KREG][MT][4];
#pragma unroll
        for (int j = 0; j < KREG; j++)
#pragma unroll
          for (int mt = 0; mt < MT; mt++) acc[j][mt][0] = acc[j][mt][1] = acc[j][mt][2] = acc[j][mt][3] = 0.f;
        if constexpr (QREG) {
          unsigned bh[KREG][2], bl[KREG][2];
#pragma unroll
          for (int j = 0; j < KREG; j++) {
            const float2 b = A2(g, offB[j]);
            split3(b.x, bh[j][0], bl[j][0]);
            split3(b.y, bh[j][1], bl[j][1]);
          }
#pragma unroll
          for (int mt = 0; mt < MT; mt++)
#pragma unroll
            for (int j = 0; j < KREG; j++) {   // the KREG chains interleave
              const unsigned ah[4] = {qf[j][mt][0], qf[j][mt][1], qf[j][mt][2], qf[j][mt][3]};
              mma_tf32(acc[j][mt], ah, bl[j][0], bl[j][1]);
            }
#pragma unroll
          for (int mt = 0; mt < MT; mt++)
#pragma unroll
            for (int j = 0; j < KREG; j++) {
              const unsigned al[4] = {qf[j][mt][4], qf[j][mt][5], qf[j][mt][6], qf[j][mt][7]};
              mma_tf32(acc[j][mt], al, bh[j][0], bh[j][1]);
            }
#pragma unroll
          for (int mt = 0; mt < MT; mt++)
#pragma unroll
            for (int j = 0; j < KREG; j++) {
              const unsigned ah[4] = {qf[j][mt][0], qf[j][mt][1], qf[j][mt][2], qf[j][mt][3]};
              mma_tf32(acc[j][mt], ah, bh[j][0], bh[j][1]);
            }
        } else {
          for (int kk = w; kk < nk; kk += NCW) {
            const float2 b = A2(g, 8 * kk + 2 * t);
            unsigned bh0, bl0, bh1, bl1;
            split3(b.x, bh0, bl0);
            split3(b.y, bh1, bl1);
#pragma unroll
            for (int mt = 0; mt < MT; mt++) {
              unsigned f[8];
              qfrag(qs, RP, 8 * kk, mt, f);
              const unsigned ah[4] = {f[0], f[1], f[2], f[3]}, al[4] = {f[4], f[5], f[6], f[7]};
              mma3(acc[0][mt], ah, al, bh0, bh1, bl0, bl1);
            }
          }
        }
        // (b) TMEM: the cells of row block s in this warp's column groups
        for (int jj = 0; jj < ncw; jj++) {
          const int cs = jj * T.nrblk + s;   // cell_slot(s, w + NCW jj)
          if (cs >= TMEM_CELLS) break;       // (cs grows with jj)
          const int c = colC + 16 * NCW * jj;
          const float2 x0 = A2(t, c), x1 = A2(t + 4, c);
          tmem_st4(taddr_w + (unsigned)(cs * 4), x0.x, x1.x, x0.y, x1.y);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);   // this warp is done with the slot
        // this warp's partial P^T for rows 8s..8s+7 -> its own slot (reduced once after the loop)
        // D[k][row]: c0 = (k=16mt+g, row=2t), c1 = (g, 2t+1), c2 = (g+8, 2t), c3 = (g+8, 2t+1)
        float* rw = red + ((size_t)w * nst + s) * SR * RP;
#pragma unroll
        for (int mt = 0; mt < MT; mt++) {
          float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
          for (int j = 0; j < KREG; j++) { a0 += acc[j][mt][0]; a1 += acc[j][mt][1]; a2 += acc[j][mt][2]; a3 += acc[j][mt][3]; }
          const int k0 = 16 * mt + g;
          rw[(2 * t) * RP + k0] = a0;
          rw[(2 * t + 1) * RP + k0] = a1;
          if (k0 + 8 < RP) {
            rw[(2 * t) * RP + k0 + 8] = a2;
            rw[(2 * t + 1) * RP + k0 + 8] = a3;
          }
        }
        if (++slot == p.ns) { slot = 0; par ^= 1u; }
      }
    };
    if (p.err_in) consume(std::true_type{});
    else consume(std::false_type{});
    consumer_sync();
    // P_part rows of this tile: sum of the NCW warp partials (fixed order)
    for (int x = tid; x < T.th * R; x += NCW * 32) {
      const int i = x / R, k = x % R;
      const float* rr = red + (size_t)i * RP + k;   // row i = stage i/8, row-in-stage i%8
      float v0 = 0.f, v1 = 0.f;
#pragma unroll
      for (int ww = 0; ww < NCW; ww++) {
        const float q = rr[(size_t)ww * nst * SR * RP];
        if (ww & 1) v1 += q; else v0 += q;
      }
      p.P_part[((size_t)T.cb * p.n + T.row0 + i) * R + k] = v0 + v1;
    }
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  if (stamp) p.stats->t_ns[8] = wait_ns;
  tr(1);
  gbar();
  tr(2);
  if (stamp) p.stats->t_ns[1] = gtimer();

  // ============================================================== phase 2
  // P_band (sum of the band's nc column-tile partials); then, concurrently,
  //   compute warps:  Q~_part = A_tile^T P_band   (tensor cores, A from TMEM)
  //   warp NW-1:      the band's Gram partial P_band^T P_band (fp64, cb == 0)
  // Q = A^T P_hat = (A^T P) Li^T with P_hat = P Li^T, Li = D^-1/2 L^-1 (reading
  // C20), so the product with A needs no orthonormalised factor and leaves the
  // critical path; Li is applied to the reduced Q~ in phase 3.
  const int H8 = T.nrblk * 8;
  float* ps = reinterpret_cast<float*>(sm + p.off_ps);   // [H8][RP] P_band, later P_hat
  float* ps2 = ps + (size_t)((p.H + 7) / 8 * 8) * RP;   // [H8][RP]
  double* gscr = reinterpret_cast<double*>(sm + p.off_gs);
  OrthW& o = *reinterpret_cast<OrthW*>(sm + p.off_orth);
  uint4* pa = reinterpret_cast<uint4*>(sm + p.off_pa);   // [nrblk][MT][32][2] (hi, lo)
  uint4* pb = reinterpret_cast<uint4*>(sm + p.off_pb);   // [nrblk][KS5][32]   (h0, h1, l0, l1)
  float* qsm = reinterpret_cast<float*>(sm + p.off_qsm);   // phase 3: the reduced Q~ slice
  if (tid == 0) o.prog = 0;   // ldl_warp publish protocol (phase 3; every CTA, active or not)
  if (active) {
    for (int x = tid; x < H8 * RP; x += NT) {
      const int i = x / RP, k = x % RP;
      float v = 0.f;
      if (i < T.th && k < R) {   // the nc partials live in L2: 8 independent loads in flight (fixed order)
        const float* src = p.P_part + ((size_t)T.row0 + i) * R + k;
        for (int c0 = 0; c0 < p.nc; c0 += 8) {
          float u[8];
#pragma unroll
          for (int j = 0; j < 8; j++) u[j] = (c0 + j < p.nc) ? __ldcg(src + (size_t)(c0 + j) * p.n * R) : 0.f;
#pragma unroll
          for (int j = 0; j < 8; j++) v += u[j];
        }
      }
      ps[x] = v;
    }
    __syncthreads();
    build_pa<R>(ps, T.nrblk, pa);
    __syncthreads();
    if (w == NW - 1) {
      if (T.cb == 0) band_gram_warp<R>(ps, T.th, p.G_band + (size_t)T.rb * NP);
      trw(14);
    } else {
      q_part_from_tmem<R, MBF>(p, T, pa, taddr_w);
    }
  }
  tr(3);
  gbar();
  tr(4);
  if (stamp) p.stats->t_ns[2] = gtimer();

  // ============================================================== phase 3
  // Warp groups (occ_v2_la.cuh): group A reduces G = sum of the nr band
  // partials and hands it to warp NW-1 (named barrier 3: A arrives, NW-1
  // waits), which factors it with the degenerate-column test and forms
  // Li = D^-1/2 L^-1, kappa and amp (LDL^T, then the inverse), publishing
  // o.prog = R + 2 (or -1: degenerate).  (A single Gauss-Jordan chain on the
  // augmented [G | I] was tried: its longer straight-line code, fetched cold,
  // made it slower, 4.6 vs 3.8 us from G to Li.)  Meanwhile all compute warps
  // reduce this CTA's column slice of Q~ over the nr row bands.  Then P_hat =
  // P Li^T and Q = Q~ Li^T in one parallel pass (reading C20; the fused Q's
  // rounding is amplified by amp = ||S Li^T||, ~sqrt(r) for a warm-started P).
  // A degenerate column, a forced or needed CholQR2 pass (kappa > kappa_thr),
  // or amp > amp_thr take the general path (cold_orth_q) before phase 5.
  const int2 qs_cols = active ? q_slice(T, p.nr) : make_int2(0, 0);
  const int nqc = qs_cols.y - qs_cols.x;
  const bool force2 = p.force_two_pass != 0;
  bool deg;
  if (w == NW - 1) {
    asm volatile("bar.sync 3, %0;" ::"r"((NWA + 1) * 32) : "memory");
    if (p.check_finite && blockIdx.x == 0 && lane < R && !isfinite(o.gdiag[lane])) atomicOr(&g_nonfinite_v2, 1u);
    deg = ldl_warp_unrolled<R>(o, p.tau * p.tau, true) != 0;
    trw(8);
    if (!deg) {
      inverse_warp_unrolled<R>(o);
      trw(15);
    }
  } else {
    if (in_group_a(w)) {
      reduce_partials<R>(p.G_band, p.nr, o, gscr, group_a_index(), NWA * 32, SyncGroupA());
      asm volatile("bar.arrive 3, %0;" ::"r"((NWA + 1) * 32) : "memory");
      tr(6);
      if (stamp) p.stats->t_ns[9] = gtimer();
    }
    if (active) {   // all compute warps (group B waits here for A's G reduce)
      strided_sum<float>(p.Q_part + (size_t)(T.col0 + qs_cols.x) * R, (size_t)p.m * R, p.nr, nqc * R,
                         reinterpret_cast<float*>(gscr), [&](int e, float v) { qsm[e] = v; }, tid, NCW * 32,
                         SyncCompute());   // (scratch first written after a compute-group barrier: A is done with it)
      tr(7);
    }
    deg = !wait_prog(o, R + 2);
  }
  if (stamp) p.stats->t_ns[10] = gtimer();
  tr(5);
  // uniform over the grid (every CTA factors the same G); warp NW-1 published
  // kappa / amp before R + 2 (and read its own values)
  bool fused = !deg && !force2 && !(o.kappa > p.kappa_thr) && !(o.amp > p.amp_thr);
  float* phat = ps2;
  if (fused) {
    if (w < NCW && active)
      apply_li<R>(ps, H8, T.th, qsm, nqc, o, ps2, p.Qout + (size_t)(T.col0 + qs_cols.x) * R, tid, NCW * 32);
  } else {
    __syncthreads();
    nb = cold_orth_q<R, MBF>(p, T, o, ps, ps2, gscr, pa, taddr_w, nb, active, deg);
    phat = ps;
  }
  if (p.wire_bf16 && w < NCW && active) {
    // OCC_WIRE_BF16 (reading C7): the factors that leave the GPU are bf16, so
    // the reconstruction and e_new use the rounded values (this CTA's P_hat
    // rows and the Q slice it wrote; the slices are read by others after B3)
    SyncCompute()();
    auto rb = [](float x) { return __bfloat162float(__float2bfloat16_rn(x)); };
    for (int x = tid; x < H8 * R; x += NCW * 32) phat[(x / R) * RP + x % R] = rb(phat[(x / R) * RP + x % R]);
    float* qs_out = p.Qout + (size_t)(T.col0 + qs_cols.x) * R;
    for (int x = tid; x < nqc * R; x += NCW * 32) qs_out[x] = rb(qs_out[x]);
  }
  tr(12);
  {   // (the fused / general decision is final here: phase 3 already knows kappa and amp)
    if (w < NCW) {
      // ---------------------------------------------------------- tables, B3 (compute warps)
      SyncCompute()();   // P_hat rows of every compute thread are written
      if (active) {
        if (T.cb == 0)
          for (int x = tid; x < T.th * R; x += NCW * 32)
            p.Pout[((size_t)T.row0 + x / R) * R + x % R] = phat[(x / R) * RP + x % R];
        for (int x = tid; x < T.nrblk * KS5 * 32; x += NCW * 32) {  // phase-5 B operand: P_hat^T, N = rows n/2 + 4(n&1)
          const int ln = x % 32, ks = (x / 32) % KS5, rblk = x / (32 * KS5);
          const int gg = ln >> 2, tt = ln & 3;
          const int r = 8 * rblk + (gg >> 1) + 4 * (gg & 1), k = 8 * ks + tt;
          uint4 v;
          unsigned h0, l0, h1, l1;
          split3((k < R) ? phat[r * RP + k] : 0.f, h0, l0);
          split3((k + 4 < R) ? phat[r * RP + k + 4] : 0.f, h1, l1);
          v.x = h0; v.y = h1; v.z = l0; v.w = l1;
          pb[x] = v;
        }
      }
      tr(13);
      if (stamp) p.stats->t_ns[4] = gtimer();
      tr(9);
      // occ_link: this CTA's P_hat rows and Q slice are final; warp NW-1 pushes them
      if (p.push.P) asm volatile("bar.arrive 5, %0;" ::"r"((NCW + 1) * 32) : "memory");
      nb++;
      grid_barrier_spread(p.barl, nb, SyncCompute());
      tr(10);
      if (stamp) p.stats->t_ns[5] = gtimer();

      // the next step's grid may start launching (its CTAs wait for this grid's
      // completion in griddepcontrol.wait before touching global memory)
      asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
      // ---------------------------------------------------------- phase 5 (compute warps)
      // The A operand Q (M = columns 2g | 2g+1, K = rank) of a column group is
      // used by exactly one lane: it is loaded straight from L2 (no staging, no
      // CTA barrier), the next column group's values while this one computes.
      tr(16);
      auto phase5 = [&](auto hr, auto he) {
        constexpr bool HASR = decltype(hr)::value, HASE = decltype(he)::value;
        auto load_q = [&](int cg, float (&qv)[KS5][4]) {
          const int cl = 16 * cg + 2 * g;
          const bool okA = cg < T.ncg && cl < T.tw, okB = cg < T.ncg && cl + 1 < T.tw;
          const float* qa_ = p.Qout + (size_t)(T.col0 + cl) * R;
#pragma unroll
          for (int ks = 0; ks < KS5; ks++) {
            const int k0 = 8 * ks + t;
            qv[ks][0] = (okA && k0 < R) ? __ldcg(qa_ + k0) : 0.f;
            qv[ks][1] = (okB && k0 < R) ? __ldcg(qa_ + R + k0) : 0.f;
            qv[ks][2] = (okA && k0 + 4 < R) ? __ldcg(qa_ + k0 + 4) : 0.f;
            qv[ks][3] = (okB && k0 + 4 < R) ? __ldcg(qa_ + R + k0 + 4) : 0.f;
          }
        };
        // cells with all 8 rows and both columns of the lane inside store through
        // row pointers (advanced by 32 rows per group of four cells): no per-cell
        // index arithmetic beyond one bounds test
        using RT = typename std::conditional<MBF, __nv_bfloat16, float>::type;
        float qnext[KS5][4];
        load_q(w, qnext);
        for (int cg = w; cg < T.ncg; cg += NCW) {
          unsigned qh[KS5][4], ql[KS5][4];
#pragma unroll
          for (int ks = 0; ks < KS5; ks++)
#pragma unroll
            for (int q = 0; q < 4; q++) split3(qnext[ks][q], qh[ks][q], ql[ks][q]);
          load_q(cg + NCW, qnext);
          const int c = 16 * cg + 2 * g;
          const bool colin = c + 1 < T.tw;
          RT* rp = HASR ? reinterpret_cast<RT*>(p.recon) + ((size_t)(T.row0 + t) * p.ldr + (T.col0 + c)) : nullptr;
          float* ep = HASE ? p.err_out + ((size_t)(T.row0 + t) * p.lde_out + (T.col0 + c)) : nullptr;
          const size_t r4 = 4 * (size_t)p.ldr, e4 = 4 * (size_t)p.lde_out;
          for (int rb0 = 0; rb0 < T.nrblk; rb0 += 4) {
            float v16[16];
            const int cs0 = cell_slot(rb0, cg);
            if (cs0 + 4 <= TMEM_CELLS) tmem_ld16(taddr_w + (unsigned)(cs0 * 4), v16);
            else cells4_slow<MBF>(p, T, taddr_w, rb0, cg, cs0, g, t, v16);
            const bool first = kTrace && cg == w && rb0 == 0;
            if (first) tr(17);
            float mr4[4][4];   // four cells, four independent MMA chains
#pragma unroll
            for (int jj = 0; jj < 4; jj++) mr4[jj][0] = mr4[jj][1] = mr4[jj][2] = mr4[jj][3] = 0.f;
#pragma unroll
            for (int ks = 0; ks < KS5; ks++)
#pragma unroll
              for (int jj = 0; jj < 4; jj++) {
                const int rblk = min(rb0 + jj, T.nrblk - 1);
                const uint4 b = pb[(rblk * KS5 + ks) * 32 + lane];
                mma3(mr4[jj], qh[ks], ql[ks], b.x, b.y, b.z, b.w);
              }
            if (kTrace && first) {
              if (mr4[0][0] == 1.2345e-30f) p.stats->grid = -2;   // keep the MMA results live before the stamp
              tr(18);
            }
            if (MBF) {
#pragma unroll
              for (int jj = 0; jj < 4; jj++)
#pragma unroll
                for (int q = 0; q < 4; q++) mr4[jj][q] = __bfloat162float(__float2bfloat16_rn(mr4[jj][q]));
            }
            // mr/v: 0 = (row t, col 2g), 1 = (t+4, 2g), 2 = (t, 2g+1), 3 = (t+4, 2g+1)
#pragma unroll
            for (int jj = 0; jj < 4; jj++) {
              const int rblk = rb0 + jj;
              if (rblk >= T.nrblk) break;
              const float* mr = mr4[jj];
              const float* v = v16 + 4 * jj;
              if (colin && 8 * rblk + 8 <= T.th) {   // the cell's 8 rows and both columns inside: pair stores
                const size_t ro = (size_t)(8 * jj) * p.ldr, eo = (size_t)(8 * jj) * p.lde_out;
                if (HASR) {
                  if (MBF) {
                    const __nv_bfloat162 b0 = __floats2bfloat162_rn(mr[0], mr[2]), b1 = __floats2bfloat162_rn(mr[1], mr[3]);
                    st_b32_hint(rp + ro, *reinterpret_cast<const unsigned*>(&b0), pol_st);
                    st_b32_hint(rp + ro + r4, *reinterpret_cast<const unsigned*>(&b1), pol_st);
                  } else {
                    st_f2_hint(reinterpret_cast<float*>(rp + ro), make_float2(mr[0], mr[2]), pol_st);
                    st_f2_hint(reinterpret_cast<float*>(rp + ro + r4), make_float2(mr[1], mr[3]), pol_st);
                  }
                }
                if (HASE) {
                  st_f2_hint(ep + eo, sub2(make_float2(v[0], v[2]), make_float2(mr[0], mr[2])), pol_st);
                  st_f2_hint(ep + eo + e4, sub2(make_float2(v[1], v[3]), make_float2(mr[1], mr[3])), pol_st);
                }
              } else {
                store_cell_edge<MBF>(p, T, 8 * rblk + t, c, make_float4(mr[0], mr[1], mr[2], mr[3]),
                                     make_float4(v[0], v[1], v[2], v[3]));
              }
            }
            if (HASR) rp += 32 * (size_t)p.ldr;
            if (HASE) ep += 32 * (size_t)p.lde_out;
            if (first) tr(19);
          }
          if (cg == w) tr(20);
        }
      };
      if (active) {
        if (p.recon) {
          if (p.err_out) phase5(std::true_type{}, std::true_type{});
          else phase5(std::true_type{}, std::false_type{});
        } else if (p.err_out) {
          phase5(std::false_type{}, std::true_type{});
        }
      }
      if (stamp) p.stats->t_ns[6] = gtimer();
      tr(11);
    } else if (p.push.P) {
      // occ_link sender (include/occ.h): while the compute warps run phase 5, the
      // producer warp copies this CTA's final P_hat rows (column band 0) and Q
      // slice into slot seq % 2 of the peer's mailbox over NVLink, after the
      // peer's receiver has acknowledged the slot's previous use (seq - 2)
      asm volatile("bar.sync 5, %0;" ::"r"((NCW + 1) * 32) : "memory");
      if (lane == 0 && p.push.seq > 2) link_wait_geq(p.push.ack, p.push.seq - 2);
      __syncwarp();
      if (active) {
        auto copy = [&](const float* src, float* dst, int count) {   // count % 4 == 0, 16-byte aligned
          const float4* s4 = reinterpret_cast<const float4*>(src);
          float4* d4 = reinterpret_cast<float4*>(dst);
          for (int x = lane; x < count / 4; x += 32) d4[x] = __ldcg(s4 + x);
        };
        if (T.cb == 0) copy(p.Pout + (size_t)T.row0 * R, p.push.P + (size_t)T.row0 * R, T.th * R);
        copy(p.Qout + (size_t)(T.col0 + qs_cols.x) * R, p.push.Q + (size_t)(T.col0 + qs_cols.x) * R, nqc * R);
      }
      __syncwarp();
      if (lane == 0) link_cta_done(p.push.ctr, p.push.flag, p.push.seq);
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && tid == 0) {
    int cnt = 0;
    if (deg)
      for (int j = 0; j < R; j++) cnt += o.rep[j];
    p.stats->fallback_columns = cnt;
    p.stats->second_pass = (p.force_two_pass || o.kappa > p.kappa_thr) ? 1 : 0;
    p.stats->kappa_est = o.kappa;
    p.stats->q_amp = deg ? -1.0 : o.amp;
    p.stats->q_fused = fused ? 1 : 0;
  }

  // ============================================================== teardown
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
  if (tid == 0) {
    const unsigned old = atomicAdd(p.bar + 1, 1u);
    if (old == gridDim.x - 1) {   // last CTA out: reset the barrier words for the next launch
      for (int j = 0; j < kBarLines; j++) atomicExch(p.barl + j * 32, 0u);
      atomicExch(p.bar, 0u);
      atomicExch(p.bar + 1, 0u);
    }
  }
  if (blockIdx.x == 0 && tid == 0) {
    p.stats->path = 3;
    p.stats->grid = gridDim.x;
  }
}
